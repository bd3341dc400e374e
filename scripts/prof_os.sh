mkdir -p gpurun_out
export CKS_OS_PERSIST=${PS:-0} CKS_OS_DEBUG=${DBG:-0} CKS_OS_ITEMS=${IT:-8} CKS_OS_SLOTS=4
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_os.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_onesweep" -s 40 -c 1 -o gpurun_out/prof_os_${TAG:-x} $CMD > gpurun_out/ncu_os.log 2>&1
echo done
