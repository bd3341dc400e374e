# one JSON line per config (20 steps, full-key comparison included) -> gpurun_out/cfg_table.jsonl
mkdir -p gpurun_out; : > gpurun_out/cfg_table.jsonl
for c in 2 3 4 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/cfg_table.jsonl; done
echo done
