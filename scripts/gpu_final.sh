# round-end style check: GPU tests, smoke, default bench (c3 with e2e + CPU baseline), reference arm
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_test.log
tail -3 gpurun_out/final_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1; tail -1 gpurun_out/final_bench.log > gpurun_out/final_bench.json
timeout 400 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; tail -1 gpurun_out/final_ref.log > gpurun_out/final_ref.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/final_bench.json")); r = d["roofline"]; e = d["e2e"]
print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 4), "kernel", round(r["kernel_ms"], 4), "frac", round(r["frac"], 3),
      "e2e", round(e["value"], 1), "default", round(e["default_contract"]["value"], 1), "first", round(e["default_contract"]["first_call_wall_s"], 3),
      "launches", d["gpu_launches"], "clocks", d["clocks"])
x = json.load(open("gpurun_out/final_ref.json")); print("reference", x["value"], x["cpu_baseline"]["sample"])
PY
