# Round-2 tail evidence: the new parity cases, the cfg table (rebuild with its own warm-up)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "run_boundaries or refine" > gpurun_out/par_tail.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/par_tail.log
: > gpurun_out/cfg_table.jsonl
for c in 2 3 4 5; do timeout 600 python bench.py --config $c --steps 60 --warmup 3 --no-e2e --no-cpu-baseline 2>> gpurun_out/cfg_table.err | tail -1 >> gpurun_out/cfg_table.jsonl; done
echo done
