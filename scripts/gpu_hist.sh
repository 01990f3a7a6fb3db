timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_parity.py tests/test_gpu_registry.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python scripts/hist_probe.py
