# usage: K=<kernel regex> S=<skip> C=<count> TAG=name bash scripts/prof_one.sh
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-3} -c ${C:-1} -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_one.log 2>&1
echo done
