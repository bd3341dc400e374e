# timing experiments on the LSD downsweep (results are NOT correct with debug bits set)
# debug bits: 1 = identity scatter (ranking still done), 2 = skip ranking (+identity), 4 = match_any ranking
for it in ${ITS:-8 16}; do for dbg in ${DBGS:-0 1 2 4}; do
  CKS_SORT_ALGO=1 CKS_LSD_DEBUG=$dbg CKS_LSD_ITEMS=$it CKS_LSD_SLOTS=${SL:-4} timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | \
   python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('items $it debug',$dbg,'pass_ms',round(d['roofline']['avg_launch_ms'],4), d['stages_ms'])"
done; done
