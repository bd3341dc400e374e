q() { timeout 60 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1','pass_ms',round(d['roofline']['avg_launch_ms'],4),'total',d['stages_ms']['total'])"; }
for d in 0 1 2 3; do CKS_LSD_DEBUG=$d q "ws debug $d"; done
