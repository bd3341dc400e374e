mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for it in ${ITEMS:-8 16}; do for sl in ${SLOTS:-3 4}; do for ch in ${CHUNK:-16}; do
  CKS_SORT_ALGO=1 CKS_LSD_ITEMS=$it CKS_LSD_SLOTS=$sl CKS_LSD_CHUNK=$ch timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lsd items',$it,'slots',$sl,'chunk',$ch,'ms/step',round(d['ms_per_step'],3),'pass_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],3), d['stages_ms'])"
done; done; done
