mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "${K:-sort or build_configs or full_size or refine}" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/q_pytest.log
for c in ${CFGS:-5 2}; do
timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild --config $c > gpurun_out/q_bench$c.json 2> gpurun_out/q_bench$c.err; echo "bench rc $?"
python - $c <<'PY'
import json,sys
c=sys.argv[1]
d = json.loads(open(f"gpurun_out/q_bench{c}.json").read().strip().splitlines()[-1])
print("cfg",c,"ms", round(d["ms_per_step"], 4), "a5", d["stages_ms"]["a5_sort"], "frac", round(d["roofline"]["frac"], 3), "kms", round(d["roofline"]["kernel_ms_per_step"],4))
PY
done
