"""NEXT-4 on the GPU: the sharded first build (paper_2009_11543_b200/shard.py) with the libcks
kernels, G ranks run as threads on cuda:0 (each with its own stream and context; no kernel
waits on another rank), slices concatenated and compared with the oracle's single build bit
for bit: permutation, D_i, exact D, P_D and the bulk-loaded tree."""
import numpy as np
import pytest

import cksgen
from shard_oracle_ops import check_slices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2009_11543_b200 import shard  # noqa: E402


def run(keys, sizes, **kw):
    cut = np.cumsum([0] + list(sizes))
    shards = [torch.from_numpy(np.ascontiguousarray(keys[a:b])).cuda() for a, b in zip(cut[:-1], cut[1:])]
    return shard.ThreadComm.run(len(sizes), lambda comm, k: shard.build_sharded(k, comm, **kw), shards)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("G", [1, 2, 4])
def test_sharded_configs(cfg, G):
    n = 120_001 if cfg > 1 else None
    keys = cksgen.config(cfg, n=n)
    N = keys.shape[0]
    sizes = [N // G] * (G - 1) + [N - (N // G) * (G - 1)]
    outs = run(keys, sizes)
    check_slices(keys, outs)
    loads = [o["perm"].numel() for o in outs]
    assert max(loads) <= 1.5 * N / G + 64                  # regular sampling keeps the slices balanced


@pytest.mark.parametrize("sizes", [[0, 5000, 1], [4999, 0, 0, 2], [1, 1, 1]])
def test_sharded_ragged_and_empty_shards(sizes):
    keys = cksgen.config(5, n=sum(sizes))
    check_slices(keys, run(keys, sizes, samples_per_rank=8))


def test_sharded_duplicates_and_equal_keys():
    rng = np.random.default_rng(5)
    dup = np.repeat(rng.integers(0, 256, (30, 24), dtype=np.uint8), 400, axis=0)[rng.permutation(12000)]
    check_slices(dup, run(dup, [7000, 5000]))
    eq = np.repeat(np.array([[1, 2, 3, 4, 5, 6, 7, 8]], np.uint8), 9000, axis=0)
    check_slices(eq, run(eq, [3000, 3000, 3000]))


def test_sharded_fanout_fill():
    keys = cksgen.config(3, n=50_000)
    check_slices(keys, run(keys, [20_000, 30_000], fanout=14, fill=0.9), fanout=14, fill=0.9)
