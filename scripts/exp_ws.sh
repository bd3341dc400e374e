q() { timeout 60 python bench.py --config ${CFG:-5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1','pass_ms',round(d['roofline']['avg_launch_ms'] or 0,4),'total',d['stages_ms']['total'], d['stages_ms'])"; }
timeout 100 python -m pytest tests -m gpu -x -q -k "sort or build" 2>&1 | tail -1
CKS_REFINE=2 timeout 100 python -m pytest tests -m gpu -x -q -k "sort or build" 2>&1 | tail -1
for r in 0 2; do CKS_REFINE=$r q "refine $r"; done
for c in 3 4; do CFG=$c q "cfg $c"; done
