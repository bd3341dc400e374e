q() { timeout 60 python bench.py --config ${CFG:-5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1','ms',round(d['ms_per_step'],3),'T',d['config']['round0_bits'],'passes',d['config']['lsd_passes'],'refined',d['config']['refined_keys'], d['stages_ms']['a5_sort'], d['stages_ms']['a7_packed_D'])"; }
T1=$(timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)
T2=$(CKS_ROUND0_BITS=24 timeout 300 python -m pytest tests -m gpu -x -q -k "refine or build or modes" 2>&1 | tail -1)
T3=$(CKS_ROUND0_BITS=48 timeout 300 python -m pytest tests -m gpu -x -q -k "refine or build or modes" 2>&1 | tail -1)
for c in 2 3 4 5; do CFG=$c q "cfg$c auto"; done
echo "TESTS auto: $T1"; echo "TESTS T24: $T2"; echo "TESTS T48: $T3"
