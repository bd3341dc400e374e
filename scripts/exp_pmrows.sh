# experiments build: P_M planes below round 0 row-major (CKS_PM_ROWS) and the widest run a CTA
# sorts (CKS_REF_CTA_WORDS), on cfg4 / cfg3. The knobs live in scripts/pmrows.patch (measured,
# not kept: DESIGN.md Sec. 6.2); apply it with `git apply scripts/pmrows.patch` first.
CKS_EXPERIMENTS=1 python -c "from paper_2009_11543_b200 import _build; _build.build(force=True)" || exit 1
for c in ${CFGS:-4 3}; do
  for pr in 0 1; do
    for cw in ${CWS:-8}; do
      CKS_PM_ROWS=$pr CKS_REF_CTA_WORDS=$cw python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('cfg$c pm_rows $pr cta_words $cw', round(d['ms_per_step'],4), 'compress', s['a3_compress'], 'sort', s['a5_sort'], 'a7', s['a7_packed_D'])"
    done
  done
done
python -c "from paper_2009_11543_b200 import _build; _build.build(force=True)"
