"""BASELINE configs[2] and [4] on one B200 via the reference-compatible harness.

configs[2]: load-factor sweep 50-98 % (2^28 slots, f=16, b=16), tail-quarter
insert throughput and BFS / DFS eviction-chain percentiles (the reference's
run_eviction_study protocol, bench.py:239-273).
configs[4]: FPR vs fingerprint size (8 / 16 / 32 bits, b=16, 95 % load,
10^8 disjoint negatives at 2^26 slots) against the analytic model.

    python tools/config_sweeps.py  -> profiles/r01s2_eviction_study.csv, profiles/r01s2_fpr_sweep.csv
"""
import sys
sys.path.insert(0, ".")
from paper_2603_15486_b200.bench_harness import RunSpec, emit_report, run_eviction_study, run_fpr_sweep

spec = RunSpec(bucket_count=(1 << 28) // 16, fingerprint_bits=16, bucket_slots=16, policy="xor", eviction="bfs")
alphas = [0.5, 0.6, 0.7, 0.8, 0.85, 0.9, 0.93, 0.95, 0.96, 0.97, 0.98]
run_eviction_study(spec, load_factors=[0.5], strategies=("bfs",))  # warm-up (context, first launches)
ev = run_eviction_study(spec, load_factors=alphas, strategies=("bfs", "dfs"))
emit_report(ev, "csv", "profiles/r01s2_eviction_study.csv")
for r in ev:
    print(f"{r.eviction} alpha={r.load_factor:.2f} tail {r.throughput / 1e9:6.2f} G/s  p90/p95/p99 "
          f"{r.eviction_p90}/{r.eviction_p95}/{r.eviction_p99}  failures {r.insert_failures}")
fp = []
for f in (8, 16, 32):
    s = RunSpec(bucket_count=1, fingerprint_bits=f, bucket_slots=16, policy="xor", eviction="bfs",
                load_factor=0.95)
    fp += run_fpr_sweep(s, memory_bytes=[(1 << 26) * f // 8], negative_queries=100_000_000)
emit_report(fp, "csv", "profiles/r01s2_fpr_sweep.csv")
for r in fp:
    print(f"f={r.fingerprint_bits} empirical {r.empirical_fpr:.3e} analytic {r.analytic_fpr:.3e} "
          f"({r.throughput / 1e9:.1f} G negative queries/s)")
