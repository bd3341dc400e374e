# Round-2 evidence: GPU tests, the default bench line, one line per config, the cfg5 launch list.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
: > gpurun_out/cfg_table.jsonl
for c in 2 3 4 5; do timeout 600 python bench.py --config $c --steps 60 --warmup 3 --no-e2e --no-cpu-baseline 2>> gpurun_out/cfg_table.err | tail -1 >> gpurun_out/cfg_table.jsonl; done
CFG=5 bash scripts/launches.sh > /dev/null
python scripts/launch_summary.py gpurun_out/launches_cfg5.csv > gpurun_out/launches_cfg5_summary.txt
head -12 gpurun_out/launches_cfg5_summary.txt
echo done
