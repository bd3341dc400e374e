q() { timeout 60 python bench.py --config ${CFG:-5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1','ms',round(d['ms_per_step'],3),'ws_ms',round(r['kernel_ms_per_step'],3),'frac',round(r['frac'],3), d['stages_ms'])"; }
timeout 100 python -m pytest tests -m gpu -x -q -k "sort or build or refine" 2>&1 | tail -1
q "cfg5"
CFG=3 q "cfg3"
CFG=4 q "cfg4"
