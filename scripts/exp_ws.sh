q() { timeout 60 python bench.py --config ${CFG:-5} --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1','ms',round(d['ms_per_step'],3),'T',d['config']['round0_bits'],'passes',d['config']['lsd_passes'], d['stages_ms']['a5_sort'])"; }
T1=$(timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)
T2=$(CKS_ROUND0_BITS=16 timeout 300 python -m pytest tests -m gpu -x -q -k "refine or build or modes" 2>&1 | tail -1)
for c in 3 4 5; do CFG=$c q "cfg$c"; done
CKS_REFINE_LOG=1 python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key 2>&1 | grep refine | tail -3
echo "TESTS: $T1"; echo "TESTS T16: $T2"
