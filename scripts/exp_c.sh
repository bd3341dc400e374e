T1=$(timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2)
for c in ${CFGS:-3 4 5}; do timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg',$c,'ms',round(d['ms_per_step'],3), d['stages_ms'])"; done
echo "TESTS: $T1"
