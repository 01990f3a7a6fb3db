set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 400 python bench.py > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
tail -5 gpurun_out/gputest.log
tail -1 gpurun_out/bench_c3.log
tail -1 gpurun_out/bench_ref.log
