q() { timeout 60 python bench.py --config ${CFG:-5} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1','compress',d['stages_ms']['a3_compress'],'packed',d['stages_ms']['a7_packed_D'])"; }
for c in 3 4 5; do for v in 0 1 2 3; do CKS_COMPRESS_V=$v CFG=$c q "cfg$c v$v"; done; done
