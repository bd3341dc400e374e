mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep" -s 40 -c 1 -o gpurun_out/prof_os $CMD > gpurun_out/ncu3.log 2>&1
echo done
