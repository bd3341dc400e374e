mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_misc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_occupancy|k_adjacent|k_bulk" -s 8 -c 4 -o gpurun_out/prof_misc $CMD > gpurun_out/ncu_misc.log 2>&1
echo done
