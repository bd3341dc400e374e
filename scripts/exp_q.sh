q() { timeout 120 python bench.py --config $1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2 cfg',$1,'ms',round(d['ms_per_step'],3),'T',d['config']['round0_bits'],'passes',d['config']['lsd_passes'],'sort',d['stages_ms']['a5_sort'])"; }
for c in ${CFGS:-5}; do q $c now; done
CFG=5 bash scripts/launches.sh > /dev/null
python scripts/launch_summary.py gpurun_out/launches_cfg5.csv | head -12
