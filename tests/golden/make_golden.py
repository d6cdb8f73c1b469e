"""Generate tests/golden/golden_v1.npz by running the REFERENCE implementation.

Run in the build container (the reference is not present on the GPU box):

    cd /tmp && PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python /root/repo/tests/golden/make_golden.py

Everything stored here is an output of ``swarcuckoo`` itself
(/root/reference/pkg/src/swarcuckoo) or of the ``xxhash`` package the
reference pins its hash to (pkg/tests/test_placement.py:38-53).  The CPU
oracle (oracle/ckf_oracle.c) and the CUDA path are both checked against these
vectors; nothing in this file is computed by code from this repository.
"""

from __future__ import annotations

import json
import struct
import sys
from pathlib import Path

import numpy as np
import xxhash

import swarcuckoo
from swarcuckoo import CuckooFilter, FilterConfig, derive_placement, wordops
from swarcuckoo.bench import gen_keys

OUT = Path(__file__).resolve().parent / "golden_v1.npz"

# (name, bucket_count, f, b, policy, eviction, max_evictions, seed, load)
SCENARIOS = [
    ("x16b16_dfs", 256, 16, 16, "xor", "dfs", 500, 11, 0.97),
    ("x16b16_bfs", 256, 16, 16, "xor", "bfs", 500, 11, 0.97),
    ("o16b16_dfs", 192, 16, 16, "offset", "dfs", 500, 11, 0.97),
    ("o16b16_bfs", 192, 16, 16, "offset", "bfs", 500, 11, 0.97),
    ("x16b4_dfs", 1024, 16, 4, "xor", "dfs", 500, 0, 0.95),
    ("x16b4_bfs", 1024, 16, 4, "xor", "bfs", 500, 0, 0.95),
    ("x8b16_bfs", 256, 8, 16, "xor", "bfs", 500, 3, 0.96),
    ("x8b8_dfs", 512, 8, 8, "xor", "dfs", 500, 3, 0.95),
    ("x32b2_dfs", 1024, 32, 2, "xor", "dfs", 200, 5, 0.93),
    ("x32b16_bfs", 128, 32, 16, "xor", "bfs", 500, 5, 0.97),
    ("o32b4_bfs", 300, 32, 4, "offset", "bfs", 300, 5, 0.95),
    ("x16b12_bfs", 256, 16, 12, "xor", "bfs", 500, 7, 0.96),
    ("o16b12_dfs", 333, 16, 12, "offset", "dfs", 500, 7, 0.96),
    ("o8b24_bfs", 100, 8, 24, "offset", "bfs", 500, 9, 0.97),
    # overfilled: failures must be reported with the dropped payload
    ("x16b4_over_dfs", 256, 16, 4, "xor", "dfs", 60, 2, 1.05),
    ("x16b4_over_bfs", 256, 16, 4, "xor", "bfs", 60, 2, 1.05),
    ("o16b16_over_bfs", 96, 16, 16, "offset", "bfs", 80, 2, 1.03),
    # small m edge cases
    ("x16b16_m1", 1, 16, 16, "xor", "dfs", 20, 1, 1.2),
    ("o16b4_m2", 2, 16, 4, "offset", "bfs", 20, 1, 1.2),
]

PLACEMENTS = [
    (1 << 16, 16, 16, "xor", 0), (1 << 18, 16, 4, "xor", 0), (3000, 16, 16, "offset", 0),
    (1 << 12, 8, 16, "xor", 7), (1 << 12, 32, 16, "xor", 7), (3000, 32, 16, "offset", 7),
    (1 << 24, 16, 16, "xor", 0), (1000, 8, 8, "offset", 99), (2, 16, 4, "offset", 5),
    (1 << 20, 16, 16, "offset", 1), ((1 << 30) + 3, 16, 16, "offset", 3),
]


def main() -> None:
    rng = np.random.default_rng(20260317)
    out: dict[str, np.ndarray] = {}
    manifest: dict[str, object] = {"reference_version": swarcuckoo.__version__,
                                   "xxhash": xxhash.VERSION, "scenarios": [], "placements": []}

    # ---- xxh64 pinned to the xxhash package (pkg/tests/test_placement.py:48-53) ----
    keys = np.concatenate([
        np.array([0, 1, 2, 42, 0xFFFFFFFFFFFFFFFF, 1 << 63, 0xDEADBEEF], dtype=np.uint64),
        rng.integers(0, 1 << 64, size=2000, dtype=np.uint64, endpoint=False),
    ])
    seeds = np.array([0, 1, 42, 0xDEADBEEF, 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    hk, hs, hh = [], [], []
    for s in seeds:
        for k in keys:
            hk.append(k)
            hs.append(s)
            hh.append(xxhash.xxh64_intdigest(struct.pack("<Q", int(k)), seed=int(s)))
    out["hash_keys"] = np.array(hk, dtype=np.uint64)
    out["hash_seeds"] = np.array(hs, dtype=np.uint64)
    out["hash_out"] = np.array(hh, dtype=np.uint64)

    # ---- derive_placement (placement.py:219-232) ----
    for j, (m, f, b, pol, seed) in enumerate(PLACEMENTS):
        cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol, seed=seed)
        pk = rng.integers(0, 1 << 64, size=1500, dtype=np.uint64)
        trip = np.array([tuple(derive_placement(int(k), cfg)) for k in pk], dtype=np.uint64)
        out[f"place{j}_keys"] = pk
        out[f"place{j}_fii"] = trip
        manifest["placements"].append({"id": j, "m": m, "f": f, "b": b, "policy": pol, "seed": seed})

    # ---- SWAR (wordops.py) ----
    for f in (8, 16, 32):
        w = rng.integers(0, 1 << 64, size=2000, dtype=np.uint64)
        tpw = 64 // f
        for i in range(0, len(w), 2):  # plant zero lanes
            w[i] = np.uint64(wordops.replace_tag(int(w[i]), int(rng.integers(0, tpw)), 0, f))
        out[f"swar{f}_words"] = w
        out[f"swar{f}_zmask"] = np.array([wordops.zero_mask(int(x), f) for x in w], dtype=np.uint64)
        tags = rng.integers(0, 1 << f, size=200, dtype=np.uint64)
        out[f"swar{f}_tags"] = tags
        out[f"swar{f}_bcast"] = np.array([wordops.broadcast_tag(int(t), f) for t in tags],
                                         dtype=np.uint64)

    # ---- whole-filter scenarios through the reference CuckooFilter (workers=1) ----
    for (name, m, f, b, pol, ev, max_ev, seed, load) in SCENARIOS:
        cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol,
                           eviction=ev, max_evictions=max_ev, seed=seed)
        n = int(load * cfg.total_slots)
        ins = gen_keys(n, seed)
        neg = gen_keys(4 * n + 16, seed, negative=True)
        filt = CuckooFilter(cfg)
        res = filt.insert_batch(ins)
        out[f"{name}_keys"] = ins
        out[f"{name}_ok"] = res.ok.astype(np.uint8)
        out[f"{name}_ev"] = res.evictions
        out[f"{name}_lost"] = res.lost_fingerprints
        out[f"{name}_words_ins"] = filt.words.copy()
        occ_ins = filt.occupancy
        out[f"{name}_qpos"] = filt.query_batch(ins).astype(np.uint8)
        out[f"{name}_neg"] = neg
        out[f"{name}_qneg"] = filt.query_batch(neg).astype(np.uint8)
        dels = np.concatenate([ins[::3], neg[:64]])
        out[f"{name}_dkeys"] = dels
        out[f"{name}_dres"] = filt.delete_batch(dels).astype(np.uint8)
        out[f"{name}_words_del"] = filt.words.copy()
        out[f"{name}_qafter"] = filt.query_batch(ins).astype(np.uint8)
        out[f"{name}_blobhdr"] = np.frombuffer(filt.to_bytes()[:44], dtype=np.uint8)
        manifest["scenarios"].append({
            "name": name, "m": m, "f": f, "b": b, "policy": pol, "eviction": ev,
            "max_evictions": max_ev, "seed": seed, "load": load, "n": n,
            "occ_after_insert": occ_ins, "occ_after_delete": filt.occupancy,
            "n_failed": res.n_failed,
        })
        print(f"{name}: n={n} failed={res.n_failed} max_ev={int(res.evictions.max())}",
              file=sys.stderr)

    out["manifest"] = np.frombuffer(json.dumps(manifest).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)", file=sys.stderr)


if __name__ == "__main__":
    main()
