mkdir -p gpurun_out
export CKS_SORT_ALGO=1 CKS_LSD_ITEMS=${IT:-8} CKS_LSD_SLOTS=${SL:-4}
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_lsd.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 70 -c 48 --csv --log-file gpurun_out/launches_lsd.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_downsweep|k_upsweep|k_chunk_scan" -s 15 -c 3 -o gpurun_out/prof_lsd_${TAG:-x} $CMD > gpurun_out/ncu_lsd.log 2>&1
echo done
