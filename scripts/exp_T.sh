for t in 24 32; do
  echo "T=$t"; CKS_ROUND0_BITS=$t timeout 120 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
  CKS_ROUND0_BITS=$t CFG=5 bash scripts/launches.sh > /dev/null; python scripts/launch_summary.py gpurun_out/launches_cfg5.csv | head -12
  CKS_REFINE_LOG=1 CKS_ROUND0_BITS=$t python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-full-key --no-rebuild 2>&1 | grep refine | tail -3
done
