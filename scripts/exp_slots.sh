q() { timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1','pass_ms',round(d['roofline']['avg_launch_ms'],4),'total',d['stages_ms']['total'])"; }
timeout 300 python -m pytest tests -m gpu -x -q -k "sort or build_configs" 2>&1 | tail -1
for it in 8 16; do for sl in 4 5 6 8; do CKS_LSD_ITEMS=$it CKS_LSD_SLOTS=$sl q "lsd items $it slots $sl"; done; done
for dbg in 1 2; do CKS_LSD_DEBUG=$dbg CKS_LSD_ITEMS=8 CKS_LSD_SLOTS=8 q "lsd items 8 slots 8 debug $dbg"; done
