#!/usr/bin/env python
"""Benchmark of the cuckoo-filter hot path (BASELINE.json configs[1]).

One STEP = the reference's throughput protocol (swarcuckoo/bench.py:149-197)
over one batch on a 2^28-slot f=16 b=16 table:
    insert n = floor(0.95 * 2^28) keys into the empty table (0 -> 95% load)
    lookup+  the same n keys
    lookup-  n disjoint negative keys
    delete   the n keys (table back to empty, so steps chain without a clear)
Keys are the reference's gen_keys streams (Philox; positives in [0,2^32),
negatives in [2^32,2^64)), generated once and resident in HBM before timing.
`value` = 4n ops / device time per step, in billion ops/s, max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): weak scaling, 2^28 slots per GPU;
each rank owns one hash shard and generates n keys, which are routed to their
owning GPU with NCCL all-to-all (paper_2603_15486_b200/sharded.py).

`--impl reference` times the reference algorithm on the host CPU cores (the
C restatement in oracle/, the reference itself being a numba package that
does not ship to the GPU box) on the same 2^28-slot table, a bounded 1/16
sample of each op's keys per step (CpuArm).
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "insert/lookup/delete billion ops/s at 95% load; fraction of HBM roofline"
UNIT = "B ops/s"
KEY_SPLIT = 1 << 32


def gen_keys(n: int, seed: int, negative: bool = False) -> np.ndarray:
    """The reference's key streams (swarcuckoo/bench.py:101-106)."""
    rng = np.random.Generator(np.random.Philox(key=[seed, int(negative)]))
    if negative:
        return rng.integers(KEY_SPLIT, 1 << 64, size=n, dtype=np.uint64)
    return rng.integers(0, KEY_SPLIT, size=n, dtype=np.uint64)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# CPU reference arm (oracle/ = C restatement of swarcuckoo's kernels)
# --------------------------------------------------------------------------

CPU_SAMPLE = 16  # the CPU arm times 1/16 of each op's keys per step


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


class CpuArm:
    """configs[1] on the host cores with the reference algorithm (oracle/ C port).

    Table: the full 2^log2-slot f=16 b=16 xor/bfs filter.  Setup (untimed,
    once): insert all but the last 1/CPU_SAMPLE of the n positive keys with
    the reference's workers>1 mode (filter.py:422-438; oracle
    ck_insert_batch_mt).  Step (a bounded sample of the step protocol on that
    same table): insert the held-back sample (load ~89 % -> 95 %), lookup+ of
    it, lookup- of as many negatives, delete it again (back to ~89 %); inserts
    and deletes in `threads` concurrent workers, lookups on `threads` threads
    (filter.py:458-469).  value = 4 * sample / step time."""

    def __init__(self, log2_slots: int, pos: np.ndarray, neg: np.ndarray, threads: int):
        import oracle

        oracle.build()
        self.threads = threads
        self.log2 = log2_slots
        cfg = oracle.make_cfg(1 << (log2_slots - 4), 16, 16, "xor", "bfs", 500, 0)
        self.n = len(pos)
        self.s = self.n // CPU_SAMPLE
        self.filt = oracle.OracleFilter(cfg)
        t0 = time.perf_counter()
        ok = self.filt.insert_batch_mt(pos[: self.n - self.s], threads)
        self.setup_s = time.perf_counter() - t0
        assert ok.all()
        self.p, self.q = pos[self.n - self.s:], neg[: self.s]

    def step(self) -> dict:
        f, s, th = self.filt, self.s, self.threads
        t0 = time.perf_counter()
        ok = f.insert_batch_mt(self.p, th)
        t1 = time.perf_counter()
        hp = f.query_batch(self.p, threads=th)
        t2 = time.perf_counter()
        hn = f.query_batch(self.q, threads=th)
        t3 = time.perf_counter()
        d = f.delete_batch_mt(self.p, th)
        t4 = time.perf_counter()
        assert ok.all() and hp.all() and d.all()
        total = t4 - t0
        return {"seconds": total, "value": 4 * s / total / 1e9, "fpr": float(hn.mean()),
                "per_op_Mops": {"insert": s / (t1 - t0) / 1e6, "lookup+": s / (t2 - t1) / 1e6,
                                "lookup-": s / (t3 - t2) / 1e6, "delete": s / (t4 - t3) / 1e6}}

    def describe(self) -> str:
        return (f"oracle/ C port of the reference kernels on {cpu_model()} x{self.threads} threads; the full "
                f"2^{self.log2}-slot table prefilled to {100 * (self.n - self.s) / (1 << self.log2):.1f} % "
                f"load (untimed, {self.setup_s:.1f} s); per step 1/{CPU_SAMPLE} of each op's keys "
                f"({self.s} keys): insert (to 95 %), lookup+, lookup-, delete, inserts/deletes in the "
                f"reference's concurrent workers mode, lookups on all threads")


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def per_gpu_log2(args, world: int) -> int:
    """Slots per GPU: configs[1]'s 2^28 per GPU (weak scaling), or with
    --strong configs[3]'s 2^31 in total over the N GPUs."""
    return args.strong_log2_total - (world.bit_length() - 1) if args.strong else args.log2_slots


def workload_config(log2: int, world: int, eviction: str, strong: bool = False) -> dict:
    n = int(0.95 * (1 << log2))
    wl = ("configs[3]: 2^31 slots total, hash-sharded over the GPUs, f=16 b=16 xor, insert 0->95% then "
          "lookup+/-, delete" if strong else
          "configs[1]: 2^28 slots/GPU f=16 b=16 xor, insert 0->95% then lookup+/-, delete")
    return {"workload": wl,
            "slots_per_gpu": 1 << log2, "keys_per_op_per_gpu": n, "fingerprint_bits": 16,
            "bucket_slots": 16, "policy": "xor", "eviction": eviction,
            "parallelism": f"hash-sharded x{world}" if world > 1 else "single GPU",
            "l2": f"inputs > L2 ({8 * int(0.95 * (1 << log2)) >> 20} MiB key arrays, {(1 << log2) * 2 >> 20} MiB "
                  "table vs 126 MB L2); no flush"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = host_threads()
    log2 = per_gpu_log2(args, args.gpus)
    n = int(0.95 * (1 << log2))
    pos, neg = gen_keys(n, 0), gen_keys(n, 0, negative=True)
    arm = CpuArm(log2, pos, neg, threads)
    for _ in range(args.warmup):
        arm.step()
    runs = [arm.step() for _ in range(args.steps)]
    secs = [r["seconds"] for r in runs]
    value = 4 * arm.s * len(runs) / sum(secs) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / len(secs),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (reference gen_keys Philox streams)",
        "config": workload_config(log2, args.gpus, args.eviction, args.strong),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": arm.describe(),
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_op_Mops": {k: round(v, 2) for k, v in runs[-1]["per_op_Mops"].items()},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

def alg_bytes(op: str, S: int, p2: float) -> float:
    """Algorithmic bytes per op (BASELINE.md §2 / SURVEY.md §8(d))."""
    if op == "lookup-":
        return 8 + 1 + 2 * S
    if op == "lookup+":
        return 9 + S * (1 + p2)
    # insert / delete: key + result + bucket read(s) + one dirty-sector write-back
    return 9 + S * (1 + p2) + 32


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # BENCH_BACKEND=gloo (developer check of the multi-rank path on a box with
    # fewer GPUs than ranks: ranks share the devices, gloo moves the data)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2603_15486_b200 import CuckooFilter, FilterConfig, _lib
    from paper_2603_15486_b200.sharded import ShardedCuckooFilter

    log2 = per_gpu_log2(args, world)
    f, b = 16, 16
    m_local = (1 << log2) // b
    n = int(0.95 * (1 << log2))  # keys per rank per op
    S = 32 * ((b * f // 8 + 31) // 32)
    cfg = FilterConfig(bucket_count=m_local * world, fingerprint_bits=f, bucket_slots=b,
                       policy="xor", eviction=args.eviction, seed=0)

    pos_h = gen_keys(n, rank)
    neg_h = gen_keys(n, rank, negative=True)
    pos = torch.from_numpy(pos_h.view(np.int64)).to(dev)
    neg = torch.from_numpy(neg_h.view(np.int64)).to(dev)
    if world > 1:
        filt = ShardedCuckooFilter(cfg, device=dev)
    else:
        filt = CuckooFilter(cfg, device=dev)

    stream = torch.cuda.current_stream(dev)
    ops = ("insert", "lookup+", "lookup-", "delete")

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        filt.insert_batch(pos)
        if ev:
            ev[1].record(stream)
        filt.query_batch(pos)
        if ev:
            ev[2].record(stream)
        filt.query_batch(neg)
        if ev:
            ev[3].record(stream)
        filt.delete_batch(pos)
        if ev:
            ev[4].record(stream)

    for _ in range(args.warmup):
        step()
    barrier()
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    launches0 = _lib.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        for k in range(args.steps):
            step(events[k])
        barrier()
    launches = _lib.kernel_launches() - launches0
    per_op = {o: 0.0 for o in ops}
    for evs in events:
        for j, o in enumerate(ops):
            per_op[o] += evs[j].elapsed_time(evs[j + 1])
    total_ms = sum(per_op.values())
    ms_step = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = 4 * n * world / (ms_step * 1e-3) / 1e9

    # ---- verification pass (untimed): parity properties at full size ----
    barrier()
    res = filt.insert_batch(pos)
    n_failed = res.n_failed
    q_alt_ins = res.n_alt / n if hasattr(res, "n_alt") else None
    hits = filt.query_batch(pos)
    no_fn = bool(hits.all())
    p2_pos = filt.last_counters()["n_alt"] / n
    fpr = float(filt.query_batch(neg).float().mean())
    d = filt.delete_batch(pos)
    p2_del = filt.last_counters()["n_alt"] / n
    all_deleted = bool(d.all())
    occ_end = len(filt)
    verify = {"insert_failures": int(n_failed), "no_false_negatives": no_fn, "fpr": fpr,
              "all_deleted": all_deleted, "occupancy_after_delete": int(occ_end)}

    peaks = measured_peaks()
    p2 = {"insert": q_alt_ins or 0.0, "lookup+": p2_pos, "lookup-": 1.0, "delete": p2_del}
    op_stats = {}
    for o in ops:
        t_s = per_op[o] / args.steps * 1e-3
        gops = n / t_s / 1e9
        bpo = alg_bytes(o, S, p2[o])
        op_stats[o] = {"G_ops_s": round(gops, 3), "ms": round(per_op[o] / args.steps, 4),
                       "bytes_per_op": round(bpo, 2), "p2": round(p2[o], 4),
                       "achieved_GBs": round(gops * bpo, 1), "frac": round(gops * bpo / peaks["hbm_gbs"], 4)}
    # The dominant op is a fixed pipeline of kernels on one stream (region schedule:
    # bin -> split -> probe on i1, bin -> split -> probe on i2, + evict / bit expansion);
    # its CUDA-event time above is the launch duration the roofline is taken over.
    dom = max(ops, key=lambda o: per_op[o])
    traffic, kernels = None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and log2 == 28:  # (the capture is of the 2^28-slot configuration)
        tj = json.loads(tf.read_text())
        traffic = tj.get(dom)
        kernels = [k[0] for k in tj.get(dom + "_kernels", [])]
    roofline = {"bound": "hbm", "achieved": op_stats[dom]["achieved_GBs"], "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": op_stats[dom]["frac"], "traffic": traffic,
                "kernel": f"{dom} ({'+'.join(kernels) if kernels else 'op pipeline'})",
                "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write summed over the op's kernels)",
                "peak_source": peaks["source"],
                "random_sector_ceiling": "~48 G random 32B sectors/s at 512 MiB (profiles/r01_probe_ceiling.txt)"}

    # ---- end to end through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        pos_p = torch.from_numpy(pos_h.view(np.int64)).pin_memory()
        neg_p = torch.from_numpy(neg_h.view(np.int64)).pin_memory()
        del pos, neg
        torch.cuda.empty_cache()

        debug = bool(os.environ.get("BENCH_DEBUG"))

        def e2e_step():
            t = [time.perf_counter()]
            r = filt.insert_batch(pos_p)
            ok_h = r.ok  # D2H of the per-key results
            t.append(time.perf_counter())
            q1 = filt.query_batch(pos_p)
            t.append(time.perf_counter())
            q2 = filt.query_batch(neg_p)
            t.append(time.perf_counter())
            dd = filt.delete_batch(pos_p)
            t.append(time.perf_counter())
            if debug:
                print("e2e ms per op:", [round(1e3 * (b - a), 1) for a, b in zip(t, t[1:])], file=sys.stderr)
            return ok_h, q1, q2, dd

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        ksteps = max(1, min(args.steps, args.e2e_steps))
        out = None
        for _ in range(ksteps):
            out = None  # release the previous step's host answers (their pinned blocks are reused)
            out = e2e_step()
        barrier()
        dt = (time.perf_counter() - t0) / ksteps
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        assert bool(out[1].all())
        e2e = {"value": 4 * n * world / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * 8 * n,
               "d2h_bytes_per_step": 4 * n, "ms_per_step": 1e3 * dt,
               "path": "CuckooFilter.*_batch(pinned host torch tensors) -> host results"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arm = CpuArm(log2, pos_h, neg_h, host_threads())
        r = arm.step()
        cpu = {"value": r["value"], "unit": UNIT, "cores": arm.threads, "kind": "port", "sample": arm.describe(),
               "cpu": cpu_model(), "step_s": round(r["seconds"], 3),
               "per_op_Mops": {k: round(v, 2) for k, v in r["per_op_Mops"].items()}}
        del arm

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "u64",
            "data": "synthetic (reference gen_keys Philox streams, seed = rank)",
            "config": workload_config(log2, world, args.eviction, args.strong),
            "roofline": roofline, "ops": op_stats, "verify": verify,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--log2-slots", type=int, default=28)
    ap.add_argument("--strong", action="store_true",
                    help="configs[3]: fixed 2^31 slots in total over the N GPUs (strong scaling)")
    ap.add_argument("--strong-log2-total", type=int, default=31)
    ap.add_argument("--eviction", choices=["dfs", "bfs"], default="bfs")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
