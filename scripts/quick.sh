mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step',round(d['ms_per_step'],3),'Gkeys/s',round(d['value']/1e9,3),'pass_ms',round(d['roofline']['avg_launch_ms'],4),'path_frac8',round(d['path_roofline']['frac_of_8tbs'],3), d['stages_ms'])"
