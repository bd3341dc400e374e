# usage: CFG=5 bash scripts/launches.sh  -> gpurun_out/launches_cfg$CFG.csv
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-5} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild"
$CMD > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg${CFG:-5}.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo done $?
