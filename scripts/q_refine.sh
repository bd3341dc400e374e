mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "refine or prefix or config or cfg or tie or run or sort or lsd or shard" > gpurun_out/par.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/par.log
for c in 5 4 3; do timeout 600 python bench.py --config $c --steps 60 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['ms_per_step'],4), d['stages_ms'])"; done
