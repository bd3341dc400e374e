# usage: [CFG=5] K=<kernel regex> S=<skip> C=<count> TAG=name bash scripts/prof_k.sh
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG:-5} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild"
$CMD > gpurun_out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-20} -c ${C:-1} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_k.log 2>&1
echo done
