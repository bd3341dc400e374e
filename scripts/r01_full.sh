# Round-1 GPU evidence: gpu tests, one bench line, launch list (ncu time only), one full capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -1 gpurun_out/bench.json
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K:-k_downsweep_ws}" -s ${S:-12} -c 1 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc $?"
echo done
