for c in 5 2; do python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['stages_ms']['a5_sort'])"; done
