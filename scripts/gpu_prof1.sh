# ncu evidence at HEAD: c3 screen kernel (full set), c5 screen kernel, deltatc at c4, launch lists
mkdir -p gpurun_out
bash scripts/launches.sh c3 auto r02_c3_fp8s | tail -25
bash scripts/profile_kernel.sh "assign_screen_bf16_kernel" r02_c3_screen c3 auto 4
bash scripts/profile_kernel.sh "assign_delta_tc_kernel" r02_c4_deltatc c4 deltatc 3
python scripts/ncu_summary.py gpurun_out/prof_r02_c3_screen.ncu-rep
python scripts/ncu_summary.py gpurun_out/prof_r02_c4_deltatc.ncu-rep
