q() { timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1','pass_ms',round(d['roofline']['avg_launch_ms'],4),'total',d['stages_ms']['total'])"; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for it in ${ITS:-16}; do for sl in ${SLS:-4 5}; do CKS_LSD_ITEMS=$it CKS_LSD_SLOTS=$sl q "lsd items $it slots $sl"; done; done
