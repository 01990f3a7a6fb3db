# the multi-rank protocol over NCCL with one rank (PCB_FORCE_MULTI=1) + the distributed GPU tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_nccl1.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/nccl1_test.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/nccl1_test.log
