CKS_REFINE=2 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for c in 3 4 5; do CFG=$c; CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
CKS_REFINE=2 $CMD > gpurun_out/plain_l.log 2>&1 && CKS_REFINE=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ref_cfg$c.csv $CMD > /dev/null 2>&1; done
