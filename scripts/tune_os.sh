# quick onesweep tuning sweep (prints a5 per-pass time for each setting)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for ps in ${PERSIST:-1 0}; do for it in ${ITEMS:-8 16}; do for sl in ${SLOTS:-3 4}; do
  CKS_OS_PERSIST=$ps CKS_OS_RANK=0 CKS_OS_ITEMS=$it CKS_OS_SLOTS=$sl timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('persist',$ps,'items',$it,'slots',$sl,'ms/step',round(d['ms_per_step'],3),'pass_ms',round(d['roofline']['avg_launch_ms'],4),'frac',round(d['roofline']['frac'],3))"
done; done; done
