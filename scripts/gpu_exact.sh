timeout 900 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_registry.py tests/test_gpu_tc.py -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/launches_cold.sh c3 > gpurun_out/cold.txt; grep -E "exact_tiled|tc3xtf32|gather_split" gpurun_out/cold.txt | head -8
bash scripts/launches_steady.sh c3 | grep -E "exact_tiled|exact_merge"
