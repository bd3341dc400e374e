q() { timeout 60 python bench.py --config ${CFG:-5} --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1','ms',round(d['ms_per_step'],3), d['stages_ms']['a5_sort'])"; }
for c in 3 5; do CFG=$c q "cfg$c events"; CKS_NO_KERNEL_EVENTS=1 CFG=$c q "cfg$c no-events"; done
