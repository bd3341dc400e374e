# timing experiments on the onesweep pass (results are NOT correct with debug bits set)
for rk in 0 1; do for it in 8 16; do for dbg in 0 3; do
  CKS_OS_RANK=$rk CKS_OS_PERSIST=${PS:-0} CKS_OS_DEBUG=$dbg CKS_OS_ITEMS=$it CKS_OS_SLOTS=4 timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('rank $rk items $it debug',$dbg,'pass_ms',round(d['roofline']['avg_launch_ms'],4))"
done; done; done
