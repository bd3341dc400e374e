"""SHA-256 and |V| / |D+| of each generated key column (BASELINE.md asks to record them)."""
import hashlib
import sys
sys.path.insert(0, '/root/repo')
import cksgen
import oracle
for c in (1, 2, 3, 4, 5):
    k = cksgen.config(c)
    h = hashlib.sha256(k.tobytes()).hexdigest()
    v = oracle.popcount(oracle.variant_bitmap(k))
    dp = oracle.popcount(oracle.byteocc_superset(k))
    print(f"cfg{c} n={k.shape[0]} B={k.shape[1]} |V|={v} |D+|={dp} sha256={h}", flush=True)
    del k
