# resolver workload at steady state (c3 and one 8-rank shard's rows): list sizes per iteration
mkdir -p gpurun_out
timeout 600 python scripts/probe_counts.py > gpurun_out/counts_c3.log 2>&1; tail -4 gpurun_out/counts_c3.log
timeout 600 python scripts/probe_counts.py 1250000 > gpurun_out/counts_shard8.log 2>&1; tail -4 gpurun_out/counts_shard8.log
