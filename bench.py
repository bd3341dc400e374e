"""Benchmark of the compressed key sort hot path on B200 (BASELINE.json metric:
"compressed-key-sort keys/s and achieved HBM GB/s vs roofline (1 B200)").

One step = one fused first build (cks_build): a1 superset mask -> a3 compress ->
a4 histograms -> a5 LSD passes -> a6 adjacency (exact D) -> a7 repack -> a8 bulk load
(fanout 64), over one synthetic key column already resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU) as the sharded build (NEXT-4, DESIGN.md
Sec. 7): every rank holds a full-size shard and the ranks build ONE index over the union with
one all-to-all exchange; weak scaling, value = all keys / max-over-ranks time. `--replicas`
runs independent per-rank builds instead. Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compressed-key-sort keys/s and achieved HBM GB/s vs roofline (1 B200)"
UNIT = "keys/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy r+w)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def formula_bytes(B: int, m: int):
    """SURVEY 8(d) roofline bytes per key of mask + compress + k radix passes, for a full-width
    LSD sort on the superset width m: B (a1) + (B + W) (a3) + k*2*(W+4) - 4 (a5) + W (a6),
    W = 4*ceil(m/32), k = ceil(m/8). The build sorts by distinguishing prefixes (NEXT-1) and
    moves fewer bytes than this; the formula is the contract's yardstick."""
    W = 4 * ((m + 31) // 32)
    k = (m + 7) // 8
    return {"a1_mask": B, "a3_compress": B + W, "a5_passes": (k * 2 * (W + 4) - 4) if k else 0, "a6_adjacent": W}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if args.backend == "nccl" else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)                 # NCCL binds this rank's device from here on
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def traffic_from_profiles(cfg_name: str):
    """ncu --set full dram__bytes_read+write of one profiled launch of the dominant kernel
    (profiles/ncu_traffic.json), with that launch's algorithmic bytes for comparison."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        e = d.get(cfg_name)
        if e:
            return float(e["dram_bytes_per_launch"]), e.get("source"), e.get("algorithmic_bytes_per_launch")
    return None, None, None


# ------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference): the oracle as it stands, all host cores

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_stages(keys, threads: int) -> dict:
    """The oracle's first build by stage (SURVEY 8(d) oracle timing): (i) exact D = full-key
    sort + adjacency, (ii) compress, (iii) compressed sort; plus the bulk load. cpu_s / wall =
    the parallelism it achieved (its compress is a single-threaded bit loop)."""
    import oracle
    c0 = os.times()
    t0 = time.perf_counter()
    perm = oracle.sort_keys(keys, threads=threads)
    dbit, mask = oracle.adjacent_dbits(keys, perm)
    t1 = time.perf_counter()
    planes = oracle.compress(keys, mask)
    t2 = time.perf_counter()
    oracle.sort_packed(planes, threads=threads)
    t3 = time.perf_counter()
    oracle.bulkload(perm, dbit, keys, 64, 1.0)
    t4 = time.perf_counter()
    c1 = os.times()
    cpu = (c1.user - c0.user) + (c1.system - c0.system)
    return {"exact_D_s": round(t1 - t0, 3), "compress_s": round(t2 - t1, 3), "compressed_sort_s": round(t3 - t2, 3),
            "bulkload_s": round(t4 - t3, 3), "total_s": round(t4 - t0, 3), "cpu_s": round(cpu, 3),
            "effective_cores": round(cpu / (t4 - t0), 2) if t4 > t0 else None}


def cpu_baseline(cfg: int, cfg_name: str, sample_n: int):
    import oracle
    threads = oracle.threads_default()
    import cksgen
    keys = cksgen.config(cfg, n=sample_n)
    st = oracle_stages(keys, threads)                       # all cores: __gnu_parallel::sort
    dt_total = st["total_s"]
    one_n = max(1, sample_n // 8)                           # one core (std::sort) on an eighth
    st1 = oracle_stages(keys[:one_n], 1)
    return {"value": sample_n / dt_total, "unit": UNIT, "cores": threads, "kind": "oracle",
            "cores_note": f"{threads} threads available to the parallel sort; the oracle's bit-loop compress is "
                          f"single-threaded, so the run averaged {st['effective_cores']} busy cores (cpu_s / wall)",
            "sample": f"first {sample_n:,} keys of {cfg_name} (same generator), oracle first build "
                      f"(parallel full-key sort + adjacency + bit-loop compress + packed sort) + bulk load, "
                      f"{dt_total:.1f} s", "seconds": round(dt_total, 3),
            "cores_affinity": len(os.sched_getaffinity(0)), "cpu_model": cpu_model(), "stages": st,
            "rebuild_keys_per_s": sample_n / (st["compress_s"] + st["compressed_sort_s"] + st["bulkload_s"]),
            "one_core": {"sample": f"first {one_n:,} keys", "stages": st1,
                         "value": one_n / st1["total_s"] if st1["total_s"] else None}}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle timed on the host cores, on a bounded sample per step."""
    import cksgen
    import oracle
    if rank != 0:
        return
    c = cksgen.CONFIGS[args.config]
    threads = oracle.threads_default()
    sample = args.ref_sample
    keys = cksgen.config(args.config, n=sample)

    def step():
        ref = oracle.first_build(keys, threads=threads)
        oracle.bulkload(ref["perm"], ref["dbit"], keys, 64, 1.0)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = sample / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": c["name"], "n": c["n"], "key_bytes": c["B"], "fanout": 64,
                       "sample_per_step": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"first {sample:,} keys of {c['name']} per step (bounded sample)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------

def run_sharded(args, world, rank, local):
    """--sharded (NEXT-4): every rank holds a full-size shard of the config (rank r: generator
    seed + r; rank 0's shard is the single-GPU workload) and the ranks build ONE index over the
    union (shard.build_sharded: occupancy all-gather, splitters, one all-to-all of (P, row id),
    boundary pairs, OR of D, rank-0 bulk load). Weak scaling: n keys per GPU."""
    import numpy as np
    import torch

    import cksgen
    from paper_2009_11543_b200 import cks, shard

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    c = cksgen.CONFIGS[args.config]
    n, B = c["n"], c["B"]
    host = torch.empty((n, B), dtype=torch.uint8, pin_memory=True)
    cksgen.config(args.config, seed=c["seed"] + rank, out=host.numpy())
    keys = host.to(device)
    comm = shard.TorchComm() if world > 1 else shard.ThreadComm.group(1)[0]
    stream = torch.cuda.current_stream(device)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        out = shard.build_sharded(keys, comm)
    torch.cuda.synchronize(device)
    k_ms = k_bytes = 0.0
    launches0 = cks.launches()
    barrier(world)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    every = max(1, args.steps // 10)                        # sampled kernel events, as run_single
    for i in range(args.steps):
        sample = (i + 1) % every == 0
        if sample:
            cks.set_timing(True)
        out = shard.build_sharded(keys, comm)
        if sample:
            kms, kby, _ = cks.kernel_stats()
            k_ms += kms
            k_bytes += kby
            cks.set_timing(False)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    clk = clocks.stop()
    barrier(world)
    gpu_launches = cks.launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_max = max_over_ranks(ms, world, device)
    peak, peak_src = measured_peaks()
    achieved = (k_bytes / (k_ms * 1e-3) / 1e9) if k_ms > 0 else None
    slice_max = max_over_ranks(float(out["perm"].numel()), world, device)
    # e2e through the same public call: every step copies this rank's shard in from pinned host
    # memory and its slice of the permutation back out (host wall clock, max over ranks)
    e2e = None
    if not args.no_e2e:
        steps_e = max(1, args.e2e_steps)
        perm_h = torch.empty(n + n // 2 + 1024, dtype=torch.int32, pin_memory=True)
        barrier(world)
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(steps_e):
            keys.copy_(host, non_blocking=True)
            o = shard.build_sharded(keys, comm)
            k = int(o["perm"].numel())
            perm_h[:k].copy_(o["perm"], non_blocking=True)
            torch.cuda.synchronize(device)
            d2h = k * 4 + B
        dt = max_over_ranks((time.perf_counter() - t0) / steps_e, world, device)
        e2e = {"value": n * world / dt, "unit": UNIT, "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": d2h,
               "ms_per_step": dt * 1e3, "steps": steps_e,
               "timing": "host wall clock per step (H2D of the rank's shard, sharded build, D2H of its slice), "
                         "max over ranks; byte counts are rank 0's"}
    if rank == 0:
        line = {"metric": METRIC, "value": n * world / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": c["name"], "n_per_rank": n, "n_total": n * world, "key_bytes": B,
                           "fanout": 64, "sort_bits": int(out["sort_bits"]), "d_bits": int(out["popcount"]),
                           "parallelism": f"sharded: range partition over {world} rank(s), one all-to-all",
                           "largest_slice": int(slice_max), "l2": "inputs larger than L2, no flush"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": (achieved / peak) if (achieved and peak) else None, "traffic": None,
                             "kernel": "k_downsweep_ws (warp-specialised LSD digit pass)", "peak_source": peak_src},
                "cpu_baseline": None, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--cpu-sample", type=int, default=12_000_000)
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-full-key", action="store_true", help="skip the full-key comparison (NEXT-2)")
    ap.add_argument("--no-rebuild", action="store_true", help="skip the rebuild timing (prior mask = D)")
    ap.add_argument("--full-key-steps", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="NEXT-4: one global build over all ranks' shards (range partition + all-to-all) "
                         "instead of one independent build per rank (the default when N > 1)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent per-rank builds (no exchange) instead of the sharded build")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3                                     # contract: W >= 3

    world, rank, local = dist_setup(args)
    if world > 1 and not args.replicas:
        args.sharded = True
    if args.sharded and args.impl == "ours":
        run_sharded(args, world, rank, local)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import numpy as np
    import torch

    import cksgen
    from paper_2009_11543_b200 import cks

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    c = cksgen.CONFIGS[args.config]
    n, B = c["n"], c["B"]

    # synthetic key column: generated on the host (seeded), copied once to HBM (untimed)
    host = torch.empty((n, B), dtype=torch.uint8, pin_memory=True)
    keys_h = host.numpy()
    cksgen.config(args.config, out=keys_h)
    keys = host.to(device, non_blocking=False)

    builder = cks.Builder(n, B, device, fanout=64, fill=1.0)
    stream = torch.cuda.current_stream(device)
    clocks = ClockSampler(local)                 # started before warm-up so it samples under load
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        builder(keys)
    torch.cuda.synchronize(device)
    m, d, passes = int(builder.out.sort_bits), int(builder.out.popcount), int(builder.out.passes)
    rounds, refined = int(builder.out.rounds), int(builder.out.refined_keys)
    round0_bits = int(builder.out.round0_bits)

    # ---- timed region: K fused builds, inputs resident in HBM (keys > 126 MB L2 for cfg2-5)
    stage_acc = None
    k_ms = k_bytes = 0.0
    k_count = 0
    launches0 = cks.launches()
    barrier(world)
    torch.cuda.synchronize(device)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    # every `every`-th build records the library's stage and dominant-kernel events
    # (cks_ctx_set_timing) and they are read right after it (a host wait); the other builds run
    # back to back without events, as a user's builds do -- event records between the digit
    # pass's launches break their programmatic dependent launch
    every = max(1, args.steps // 10)
    sampled = 0
    pbytes = []
    for i in range(args.steps):
        sample = (i + 1) % every == 0
        if sample:
            cks.set_timing(True)
        builder(keys)
        if sample:
            pbytes.append(cks.path_bytes())
            st = cks.stage_ms()                              # events on the library's stream
            stage_acc = st if stage_acc is None else [a + b for a, b in zip(stage_acc, st)]
            kms, kby, kc = cks.kernel_stats()                # the dominant kernel's own events
            k_ms += kms
            k_bytes += kby
            k_count += kc
            sampled += 1
            cks.set_timing(False)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    clk = clocks.stop()
    barrier(world)
    gpu_launches = cks.launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_max = max_over_ranks(ms, world, device)
    stages = [s / sampled for s in stage_acc]
    names = ["a1_mask", "a3_compress", "a4_sort_setup", "a5_sort", "a6_exact_D", "a7_packed_D", "a8_bulkload",
             "total"]
    stages_ms = dict(zip(names, [round(s, 4) for s in stages]))

    # ---- roofline of the dominant kernel: the warp-specialised LSD downsweep (one launch per
    # digit pass), algorithmic bytes = every stream of the pass read once and written once
    peak, peak_src = measured_peaks()
    achieved = (k_bytes / (k_ms * 1e-3) / 1e9) if k_ms > 0 else None
    traffic, traffic_src, traffic_alg = traffic_from_profiles(c["name"])
    fbytes = formula_bytes(B, m)
    path_bytes = sum(fbytes.values()) * n
    core_ms = sum(stages[i] for i in range(0, 5))            # mask .. exact D (no packed-D, no tree)
    path_gbs = path_bytes / (core_ms * 1e-3) / 1e9
    # the work actually run: algorithmic bytes of every kernel of a build (cks_ctx_path_bytes)
    actual_bytes = statistics.median(pbytes) if pbytes else None
    total_ms = stages[7]

    # ---- rebuild: the same column rebuilt with the previous exact D as the sort
    # mask (no superset pass; m = |D|) -- SURVEY 8(d)'s rebuild roofline column
    rebuild = None
    if not args.no_rebuild:
        rb = cks.Builder(n, B, device, fanout=64, fill=1.0)
        dmask = builder.mask.copy()
        rb(keys, prior_mask=dmask)                          # (default: checked against the rows)
        torch.cuda.synchronize(device)
        vs = max(1, min(args.steps, 10))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(vs):
            rb(keys, prior_mask=dmask)
        e1.record(stream)
        torch.cuda.synchronize(device)
        vms = max_over_ranks(e0.elapsed_time(e1) / vs, world, device)
        cks.set_verify(cks.VERIFY_OFF)                       # the paper's rebuild: no order check
        rb(keys, prior_mask=dmask)                          # (warm-up of this mode, untimed)
        torch.cuda.synchronize(device)
        rs = max(1, min(args.steps, 20))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(rs):
            rb(keys, prior_mask=dmask)
        e1.record(stream)
        torch.cuda.synchronize(device)
        rms = max_over_ranks(e0.elapsed_time(e1) / rs, world, device)
        cks.set_verify(cks.VERIFY_PRIOR)
        assert np.array_equal(rb.mask, dmask)
        assert torch.equal(rb.perm, builder.perm) and torch.equal(rb.dbit, builder.dbit)   # same column
        rebuild = {"ms_per_step": rms, "verified_ms_per_step": vms,
                   "note": "ms_per_step: the paper's rebuild (P:405-411), order check off; verified: with the "
                           "default check of a prior mask (cks_ctx_set_verify: the new keys' D+ inside the mask "
                           "proves the order, else the row-gather order check)",
                   "value": n * world / (rms * 1e-3), "unit": UNIT, "sort_bits": int(rb.out.sort_bits),
                   "steps": rs, "formula_bytes_per_key": sum(formula_bytes(B, int(rb.out.sort_bits)).values()) - B}
        del rb

    # ---- e2e: same call with HOST buffers (H2D keys + D2H perm inside the timed region)
    e2e = None
    if not args.no_e2e:
        perm_h = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        perm_h2 = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        steps_e = max(1, args.e2e_steps)
        cks.build_host_batch([keys_h, keys_h], perms=[perm_h, perm_h2], device=local)     # warm
        torch.cuda.synchronize(device)
        barrier(world)
        t0 = time.perf_counter()
        # every step copies its column to the device and its permutation back; the public
        # batch call overlaps step i's build with step i+1's copy and step i-1's result
        rs = cks.build_host_batch([keys_h] * steps_e, perms=[perm_h if i % 2 == 0 else perm_h2
                                                              for i in range(steps_e)], device=local)
        dt = (time.perf_counter() - t0) / steps_e
        dt = max_over_ranks(dt, world, device)
        r = rs[-1]
        e2e = {"value": n * world / dt, "unit": UNIT, "h2d_bytes_per_step": n * B,
               "d2h_bytes_per_step": n * 4 + B, "ms_per_step": dt * 1e3, "steps": steps_e,
               "timing": "host wall clock around cks_build_host_batch over all steps (it synchronises), "
                         "max over ranks"}
        assert np.array_equal(r["mask"], builder.mask)
        assert np.array_equal(r["perm"], builder.perm[:n].cpu().numpy().view(np.uint32))   # the device build's
        # the bound: this box's pinned host->device copy rate for the same bytes (plain copies,
        # no build), so e2e can be read against the link rather than the kernels
        kd = torch.empty((n, B), dtype=torch.uint8, device=device)
        kt = torch.from_numpy(keys_h)
        kd.copy_(kt, non_blocking=True)
        torch.cuda.synchronize(device)
        t1 = time.perf_counter()
        for _ in range(3):
            kd.copy_(kt, non_blocking=True)
        torch.cuda.synchronize(device)
        h2d = n * B * 3 / (time.perf_counter() - t1)
        del kd
        e2e.update({"h2d_copy_gbs": h2d / 1e9, "frac_of_h2d_copy": (n * B / dt) / h2d,
                    "bound": "PCIe host->device copy of the keys (h2d_copy_gbs: plain pinned copies of the "
                             "same bytes on this box)"})

    # ---- NEXT-2: the same pipeline on the FULL key (M = all 8B bits, one LSD sort over them),
    # the GPU analog of the paper's full-key build, and the paper's Table 2/6 statistics
    paper_stats = None
    if not args.no_full_key:
        rid_bits = max(1, (n - 1).bit_length())
        full_sort_key = 8 * ((B + 7) // 8) + 8                         # Table 2: key words + 8 B record id
        comp_sort_key = 8 * ((d + rid_bits + 63) // 64)
        paper_stats = {"full_key_bits": 8 * B, "d_bits": d, "compression_ratio": (8 * B / d) if d else None,
                       "record_id_bits": rid_bits, "full_sort_key_bytes": full_sort_key,
                       "compressed_sort_key_bytes": comp_sort_key,
                       "sort_key_ratio": full_sort_key / comp_sort_key if comp_sort_key else None,
                       "definitions": "P:523-526 (Table 2), P:559-563; total ratio as Table 6 (P:689-706)"}
        allbits = np.full(B, 0xFF, np.uint8)
        fs = max(1, min(args.steps, args.full_key_steps))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        cks.set_verify(cks.VERIFY_OFF)                 # (all key bits: a superset by definition)

        def timed_build(bld, prior, mode):
            cks.set_sort_mode(mode)
            bld(keys, prior_mask=prior)
            torch.cuda.synchronize(device)
            e0.record(stream)
            for _ in range(fs):
                bld(keys, prior_mask=prior)
            e1.record(stream)
            torch.cuda.synchronize(device)
            return e0.elapsed_time(e1) / fs, int(bld.out.passes)
        full = cks.Builder(n, B, device, fanout=64, fill=1.0)
        comp = cks.Builder(n, B, device, fanout=64, fill=1.0)
        # Table 6 compares the SAME sort on full and on compressed keys: both legs
        # run each sort mode; the full-key leg sorts M = every key bit, the compressed one
        # M = the D-bitmap the index maintains (the paper's extract + sort + build)
        dmask = builder.mask.copy()
        f_single, fp_single = timed_build(full, allbits, cks.SORT_SINGLE)
        c_single, cp_single = timed_build(comp, dmask, cks.SORT_SINGLE)
        f_prefix, fp_prefix = timed_build(full, allbits, cks.SORT_PREFIX)
        c_prefix, cp_prefix = timed_build(comp, dmask, cks.SORT_PREFIX)
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
        cks.set_verify(cks.VERIFY_PRIOR)
        assert np.array_equal(full.mask, builder.mask) and np.array_equal(comp.mask, builder.mask)
        paper_stats.update({
            "single_sort": {"full_key_ms": f_single, "full_key_passes": fp_single, "compressed_ms": c_single,
                            "compressed_passes": cp_single, "total_ratio": f_single / c_single},
            "by_prefixes": {"full_key_ms": f_prefix, "full_key_passes": fp_prefix, "compressed_ms": c_prefix,
                            "compressed_passes": cp_prefix, "total_ratio": f_prefix / c_prefix},
            "first_build_ms": ms,
            "total_ratio_note": "Table 6 (P:689-706): the same sort, then the bulk load, on full keys (prior "
                                "mask = every key bit) and on compressed keys (prior mask = the exact D-bitmap, "
                                "the paper's extract + sort + build), per sort mode; steps per leg: %d" % fs})
        del full, comp
        # NEXT-3: the paper's 256-byte-node index tree (pk = 32, fill 0.9), three ways:
        #   rows   cks_paper_tree: every partial-key bit from the key row (C(b), random row reads)
        #   ds     cks_paper_tree_ds: A from the sorted P_D, B from the reference key, C(b) rows only
        #          for variant bits outside D
        #   fused  cks_build with ptree_nodes: the bits partial keys need outside the sort mask ride
        #          through the sort as one more plane (C(a)); reported as the build's extra time
        ps = cks.paper_tree_shape(n, 0.9)
        nodes = torch.empty((int(ps.total_nodes), cks.PTREE_NODE_BYTES), dtype=torch.uint8, device=device)

        def timed(fn):
            fn()
            torch.cuda.synchronize(device)
            e0.record(stream)
            for _ in range(fs):
                fn()
            e1.record(stream)
            torch.cuda.synchronize(device)
            return e0.elapsed_time(e1) / fs
        pms = timed(lambda: cks.paper_tree(keys, builder.perm[:n], builder.dbit[:n], 32, 0.9, out=nodes))
        dsb = cks.Builder(n, B, device, fanout=64, fill=1.0, ds_metadata=True)
        dsb(keys)
        pk_planes = dsb.packed()
        dms = timed(lambda: cks.paper_tree_ds(keys, n, B, dsb.perm[:n], dsb.dbit[:n], pk_planes, pk_planes.stride(0),
                                              dsb.mask, dsb.variant, dsb.ref_key, 32, 0.9, out=nodes))
        same_ds = bool(torch.equal(nodes, cks.paper_tree(keys, dsb.perm[:n], dsb.dbit[:n], 32, 0.9)))
        del dsb, pk_planes
        fused = {}
        for name, src in (("auto", cks.PTREE_AUTO), ("decode", cks.PTREE_DECODE), ("rows", cks.PTREE_ROWS),
                          ("ds", cks.PTREE_DS), ("carry", cks.PTREE_CARRY)):
            fb = cks.Builder(n, B, device, fanout=64, fill=1.0, paper_tree_pk=32, paper_tree_fill=0.9,
                             paper_tree_source=src)
            try:
                fms = timed(lambda: fb(keys))
            except cks.CksError as e:                   # DECODE needs P_D+ kept sorted (the carried path)
                if e.code != cks.CKS_EINVAL:
                    raise
                fused[name] = {"applicable": False, "reason": str(e)}
                del fb
                continue
            fused[name] = {"build_with_tree_ms": fms, "tree_extra_ms": fms - ms,
                           "equals_rows_tree": bool(torch.equal(fb.ptree[:fb.ptree_nodes], nodes))}
            del fb
        paper_stats.update({"paper_tree_ms": pms, "paper_tree_ds_ms": dms, "fused_build_with_tree": fused,
                            "paper_tree_nodes": int(ps.total_nodes),
                            "paper_tree_height": int(ps.height), "ds_tree_equals_rows_tree": same_ds,
                            "paper_tree_note": "NEXT-3: 256-B nodes, leaf 12/14, inner 8/9 entries (fill 0.9), pk 32; "
                                               "paper_tree_ms: bits from the key rows (C(b)); paper_tree_ds_ms: A "
                                               "from P_D + B + C(b) where needed; fused into the build: decode (A "
                                               "alone: every byte decoded from its D+ bits, the default), rows, ds, "
                                               "carry (C(a), the needed variant bits carried through the sort), "
                                               "P:484-496"})
        del nodes

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, c["name"], min(args.cpu_sample, n))

    if rank == 0:
        line = {
            "metric": METRIC, "value": n * world / (ms_max * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": c["name"], "n": n, "key_bytes": B, "fanout": 64, "fill": 1.0,
                       "superset": "byteocc D+", "sort_bits": m, "d_bits": d, "lsd_passes": passes,
                       "refine_rounds": rounds, "refined_keys": refined, "round0_bits": round0_bits,
                       "sort": "by distinguishing prefixes (NEXT-1)" if rounds else "single LSD sort",
                       "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": f"inputs larger than L2 (keys {n * B / 1e6:.0f} MB vs 126 MB), no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "k_downsweep_ws (warp-specialised LSD digit pass)", "peak_source": peak_src,
                         "launches_per_step": k_count / sampled if sampled else None,
                         "kernel_ms_per_step": k_ms / sampled if sampled else None,
                         "sampled_steps": sampled,
                         "sampling": "the kernel's CUDA events (and the stage events) are recorded in every "
                                     "(steps/10)-th build of the timed region and read right after it; value and "
                                     "ms_per_step are CUDA events around all the timed builds",
                         "algorithmic_bytes_per_launch": (k_bytes / k_count) if k_count else None,
                         "traffic_source": traffic_src, "traffic_launch_algorithmic_bytes": traffic_alg},
            "path_roofline": {
                "actual_bytes_per_key": actual_bytes / n if actual_bytes else None,
                "actual_gbs": actual_bytes / (total_ms * 1e-3) / 1e9 if actual_bytes else None,
                "actual_frac_of_peak": actual_bytes / (total_ms * 1e-3) / 1e9 / peak if actual_bytes else None,
                "actual_note": "sum of the algorithmic bytes of every kernel one build launched "
                               "(cks_ctx_path_bytes; DESIGN.md Sec. 6) / the whole build's time (a1..a8)",
                "effective_formula": "SURVEY 8(d): mask + compress + k full-width LSD passes + adjacency; the "
                                     "build sorts by distinguishing prefixes and moves fewer bytes, so this is an "
                                     "effective speed-up over a full-width sort, not a roofline fraction",
                "formula_bytes_per_key": fbytes, "mask_to_exact_D_ms": core_ms,
                "effective_gbs": path_gbs, "effective_frac_of_peak": path_gbs / peak,
                "effective_frac_of_8tbs": path_gbs / 8000.0},
            "stages_ms": stages_ms,
            "paper_stats": paper_stats, "rebuild": rebuild,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
