timeout 1200 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_steady_state.py tests/test_gpu_registry.py tests/test_gpu_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python scripts/shard_probe.py
