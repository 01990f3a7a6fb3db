bash scripts/profile_kernel.sh screen_exact_kernel r02_c3_sexact c3 auto 3
python scripts/ncu_summary.py gpurun_out/prof_r02_c3_sexact.ncu-rep
ncu -i gpurun_out/prof_r02_c3_sexact.ncu-rep --page raw --csv > gpurun_out/sexact_raw.csv
ncu -i gpurun_out/prof_r02_c3_sexact.ncu-rep --page source --csv --print-source sass > gpurun_out/sexact_src.csv
