mkdir -p gpurun_out
for c in 0 14 21 28 42 56; do
  CKS_LSD_CHUNK=$c timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild --config 5 > gpurun_out/sw_$c.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sw_$c.json').read().strip().splitlines()[-1]); print('chunk', $c, round(d['ms_per_step'],4))"
done
