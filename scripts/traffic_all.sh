# ncu --set full of one dominant-kernel launch (k_downsweep_ws) per config -> gpurun_out/prof_ds_cfg<c>.ncu-rep
# plus the summary lines (dram bytes, time) in gpurun_out/traffic_cfg<c>.txt
mkdir -p gpurun_out
for c in ${CFGS:-2 3 4 5}; do
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_downsweep_ws -s ${S:-12} -c 1 \
      -o gpurun_out/prof_ds_cfg$c $CMD > gpurun_out/ncu_ds_cfg$c.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_ds_cfg$c.ncu-rep 0 > gpurun_out/traffic_cfg$c.txt 2>&1
  echo "cfg$c rc $?"; head -4 gpurun_out/traffic_cfg$c.txt
done
