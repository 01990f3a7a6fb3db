# round-end style check + c1/c2 lines + ncu of the c2 assignment kernel
bash scripts/gpu_final2.sh
bash scripts/profile_kernel.sh "assign_rowcst" c2final c2 auto 4
python scripts/ncu_summary.py gpurun_out/prof_c2final.ncu-rep > gpurun_out/prof_c2final_summary.txt 2>&1
ncu -i gpurun_out/prof_c2final.ncu-rep --page raw --csv > gpurun_out/prof_c2final_raw.csv 2>/dev/null
cat gpurun_out/prof_c2final_summary.txt
