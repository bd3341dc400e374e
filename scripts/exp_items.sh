# experiments build: LSD tile shape 4096 (16 ranker + 8 writer warps, 1 CTA/SM) vs 2048 (8 + 4, 2 CTAs/SM)
CKS_EXPERIMENTS=1 python -c "from paper_2009_11543_b200 import _build; _build.build(force=True)" || exit 1
for it in 16 8; do
  for c in ${CFGS:-5 2}; do
    CKS_LSD_ITEMS=$it python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('items $it cfg$c', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['stages_ms']['a5_sort'])"
  done
done
