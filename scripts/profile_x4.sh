# ncu --set full of the c3 and c5 screen kernels (one launch each after warm-up)
bash scripts/profile_kernel.sh assign_screen_bf16_kernel r02_c3_screen_x4 c3 auto 4
bash scripts/profile_kernel.sh assign_screen_bf16_kernel r02_c5_screen_x4 c5 auto 4
ls -la gpurun_out/prof_r02_c*_x4.ncu-rep
