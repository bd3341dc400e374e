# quick GPU iteration: refine/build parity subset + a short cfg5 bench line (stages)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "${K:-refine or build_configs or sort_modes or full_size or contention}" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild --config ${CFG:-5} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("ms", round(d["ms_per_step"], 4), "stages", d["stages_ms"], "frac", round(d["roofline"]["frac"], 3),
      "path", round(d["path_roofline"]["actual_frac_of_peak"], 3), "B/key", round(d["path_roofline"]["actual_bytes_per_key"], 1))
PY
