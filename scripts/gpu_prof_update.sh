# ncu of the update kernels: the full update's segmented sums (iterations 0-3) and the steady-state count pass
bash scripts/profile_kernel.sh segsum_v4 r02_c3_segsum c3 auto 1
python scripts/ncu_summary.py gpurun_out/prof_r02_c3_segsum.ncu-rep
bash scripts/profile_kernel.sh count_labels_kernel r02_c3_count c3 auto 8
python scripts/ncu_summary.py gpurun_out/prof_r02_c3_count.ncu-rep
bash scripts/profile_kernel.sh relayout_rows_bf16 r02_c3_relayout c3 auto 0
python scripts/ncu_summary.py gpurun_out/prof_r02_c3_relayout.ncu-rep
