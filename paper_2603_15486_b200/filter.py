"""``CuckooFilter`` -- the drop-in facade over the sm_100a kernels.

Same public API as the reference ``swarcuckoo.filter.CuckooFilter``
(/root/reference/pkg/src/swarcuckoo/filter.py:115-574): batch
``insert_batch / query_batch / delete_batch``, scalar ``insert / query /
delete``, ``occupancy / load_factor / len / in``, ``clear``, ``stored_tags``,
``collect_eviction_stats`` and CKGF ``to_bytes / from_bytes / save / load``.

What differs is where the state lives and who runs the loops:

* the word table is a torch ``int64`` tensor of ``m * wpb`` words in HBM
  (reinterpreted as uint64 by the kernels), 256-byte aligned so every
  f=16/b=16 bucket is one 32-byte sector;
* every batch call is ONE C-ABI call (``libckf.so``) enqueued on the current
  CUDA stream -- no per-key Python, no CPU fallback;
* occupancy is a device counter updated by the kernels (the paper's
  hierarchical count) instead of per-worker dict shards;
* keys may be numpy arrays / sequences (results come back as numpy, exactly
  like the reference) or torch tensors (results stay torch, on the device).

``workers`` is accepted for compatibility and ignored: the GPU runs one
thread per key.  ``deterministic=True`` selects the single-device-thread
parity mode, bit-identical to the reference ``workers=1`` batch loop
(filter.py:416-421).
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from .config import Eviction, FilterConfig, MASK64, Policy
from .errors import PhaseError

_MAGIC = b"CKGF"
_VERSION = 1
# magic, version, f, b, m, policy, occupancy, seed (filter.py:38-42)
_HEADER = struct.Struct("<4sIIIQIQQ")

_OP_NAMES = {_lib.OP_QUERY: "query", _lib.OP_INSERT: "insert", _lib.OP_DELETE: "delete"}

_REC_DTYPE = np.dtype([("index", "<u8"), ("lost", "<u8"), ("evictions", "<u4"), ("ok", "<u4")])
assert _REC_DTYPE.itemsize == _lib.RECORD_BYTES


class InsertResult(NamedTuple):
    """Outcome of one insert (filter.py:45-58)."""

    ok: bool
    evictions: int
    lost_fingerprint: Optional[int] = None

    def __bool__(self) -> bool:
        return self.ok


@dataclass
class EvictionStats:
    """Per-insert eviction-round counts with percentile readout (filter.py:61-92)."""

    samples: np.ndarray
    failures: int = 0

    def percentile(self, p: float) -> int:
        if len(self.samples) == 0:
            return 0
        return int(np.percentile(self.samples, p, method="inverted_cdf"))

    @property
    def p90(self) -> int:
        return self.percentile(90)

    @property
    def p95(self) -> int:
        return self.percentile(95)

    @property
    def p99(self) -> int:
        return self.percentile(99)

    @property
    def mean(self) -> float:
        return float(self.samples.mean()) if len(self.samples) else 0.0

    @property
    def max(self) -> int:
        return int(self.samples.max()) if len(self.samples) else 0


class BatchInsertResult:
    """Index-aligned per-key insert outcomes (filter.py:95-112).

    The kernels write a dense ``ok`` byte per key plus sparse records for
    the keys that went through the eviction pass; ``evictions`` and
    ``lost_fingerprints`` are rebuilt from those records on first access
    (directly placed keys have 0 evictions and nothing lost).  Arrays are numpy
    when the keys were host data and torch device tensors when they were a
    CUDA tensor.
    """

    def __init__(self, n: int, ok_dev: torch.Tensor, records: torch.Tensor, counters: torch.Tensor,
                 kind: str):
        self._n = n
        self._ok_dev = ok_dev
        self._rec = records
        self._ctr = counters
        self._kind = kind
        self._numpy = kind == "numpy"
        self._ok = None
        self._ev = None
        self._lost = None
        self._nrec = None

    @classmethod
    def from_parts(cls, n: int, ok_host: torch.Tensor, parts) -> "BatchInsertResult":
        """Result of a chunked host pipeline: host ok + per-chunk records."""
        self = cls.__new__(cls)
        self._n = n
        self._ok_dev = None
        self._ok = ok_host
        self._parts = parts
        self._kind = "cpu"
        self._numpy = False
        self._ev = self._lost = None
        self._nrec = None
        return self

    # -- device-side summaries (one tiny D2H each) --
    def _counts(self):
        if getattr(self, "_parts", None) is not None and self._nrec is None:
            c = torch.stack([ctr for _, _, ctr in self._parts]).cpu()
            self._nok_cached = int(c[:, 0].sum())
            self._nrec = int(c[:, 1].sum())
            self._nalt = int(c[:, 3].sum())
            self._part_nrec = c[:, 1].tolist()
            return self._nok_cached, self._nrec
        if self._nrec is None:
            c = self._ctr.cpu()
            self._nok_cached = int(c[0])
            self._nrec = int(c[1])
            self._nalt = int(c[3])
        return self._nok_cached, self._nrec

    @property
    def n_alt(self) -> int:
        """Keys whose primary bucket was full (they probed the alternate)."""
        self._counts()
        return self._nalt

    @property
    def n_ok(self) -> int:
        return self._counts()[0]

    @property
    def n_failed(self) -> int:
        return self._n - self.n_ok

    def records(self) -> np.ndarray:
        """The sparse (index, lost, evictions, ok) records, host structured array."""
        nrec = self._counts()[1]
        if getattr(self, "_parts", None) is not None:
            out = []
            for (lo, rec, _), cnt in zip(self._parts, self._part_nrec):
                r = rec[: cnt * _lib.RECORD_BYTES].cpu().numpy().view(_REC_DTYPE).copy()
                r["index"] += lo
                out.append(r)
            return np.concatenate(out) if out else np.zeros(0, dtype=_REC_DTYPE)
        raw = self._rec[: nrec * _lib.RECORD_BYTES].cpu().numpy()
        return raw.view(_REC_DTYPE)

    @property
    def ok(self):
        if self._ok is None:
            self._ok = CuckooFilter._answer(self._ok_dev.view(torch.bool), self._kind)
        return self._ok

    def _expand(self):
        rec = self.records()
        ev = np.zeros(self._n, dtype=np.int64)
        lost = np.zeros(self._n, dtype=np.uint64)
        if len(rec):
            idx = rec["index"].astype(np.int64)
            ev[idx] = rec["evictions"]
            lost[idx] = rec["lost"]
        if self._numpy:
            self._ev, self._lost = ev, lost
        else:
            dev = self._ok_dev.device if self._kind == "cuda" else "cpu"
            self._ev = torch.from_numpy(ev).to(dev)
            self._lost = torch.from_numpy(lost).to(dev)

    @property
    def evictions(self):
        if self._ev is None:
            self._expand()
        return self._ev

    @property
    def lost_fingerprints(self):
        if self._lost is None:
            self._expand()
        return self._lost

    def eviction_stats(self) -> EvictionStats:
        ev = self.evictions
        ev = ev.cpu().numpy() if isinstance(ev, torch.Tensor) else ev.copy()
        return EvictionStats(ev, failures=self.n_failed)


def _default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("CuckooFilter needs a CUDA device (B200); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


class CuckooFilter:
    """GPU cuckoo filter with packed SWAR buckets and lock-free CAS updates.

    >>> filt = CuckooFilter(FilterConfig(bucket_count=1 << 10))
    >>> filt.insert(42).ok, 42 in filt, filt.delete(42)
    (True, True, True)
    """

    def __init__(self, cfg: FilterConfig, *, debug_phase: bool = False, device=None,
                 deterministic: bool = False, tiled: Optional[bool] = None):
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else _default_device()
        if self.device.type != "cuda":
            raise RuntimeError("CuckooFilter runs on CUDA devices only")
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self._params = cfg.ckf_params()
        self._deterministic = deterministic
        # None: library heuristic; True: region schedule whenever its plan applies; False: direct kernels
        self._tiled_flags = {None: 0, True: _lib.FORCE_TILED, False: _lib.FORCE_DIRECT}[tiled]
        self._ws = {}  # grow-only region-schedule scratch, one per CUDA stream
        self.last_schedule = None  # (schedule name, region runs) of the last batch call
        self._pipe = None  # streams + chunk buffers of the host pipeline
        with torch.cuda.device(self.device):
            self.words_device = torch.zeros(cfg.total_words, dtype=torch.int64, device=self.device)
            # [0] occupancy (kernels add/subtract), [1..4] scratch counters for scalar ops
            self._occ = torch.zeros(1, dtype=torch.int64, device=self.device)
            self._ctrs = {}  # per-CUDA-stream device counters of query / delete / mixed batches
        self._debug = debug_phase
        self._mut_depth = 0
        self._read_depth = 0

    # ---- bookkeeping ----

    @property
    def occupancy(self) -> int:
        """Stored-item count: successful inserts minus successful deletes."""
        return int(self._occ.item())

    @property
    def load_factor(self) -> float:
        return self.occupancy / self.cfg.total_slots

    def __len__(self) -> int:
        return self.occupancy

    def __contains__(self, key: int) -> bool:
        return self.query(key)

    def __repr__(self) -> str:
        c = self.cfg
        return (f"CuckooFilter(f={c.fingerprint_bits}, b={c.bucket_slots}, m={c.bucket_count}, "
                f"policy={c.policy.value}, eviction={c.eviction.value}, occupancy={self.occupancy}, "
                f"device={self.device})")

    @property
    def words(self) -> np.ndarray:
        """Host snapshot of the word table as uint64 (the reference attribute).

        A copy: mutate the table through ``filt.words = array`` (written back
        to HBM whole) or ``words_device``."""
        return self.words_device.cpu().numpy().view(np.uint64)

    @words.setter
    def words(self, value) -> None:
        arr = np.ascontiguousarray(value, dtype=np.uint64).reshape(-1)
        if arr.size != self.words_device.numel():
            raise ValueError(f"word array has {arr.size} words, expected {self.words_device.numel()}")
        self.words_device.copy_(torch.from_numpy(arr.view(np.int64)))

    @property
    def _ctr(self) -> torch.Tensor:
        """This CUDA stream's counters (batches on other streams never share them)."""
        s = self._stream()
        c = self._ctrs.get(s)
        if c is None:
            c = self._ctrs[s] = torch.zeros(4, dtype=torch.int64, device=self.device)
        return c

    def clear(self) -> None:
        self.words_device.zero_()
        self._occ.zero_()

    def stored_tags(self) -> np.ndarray:
        """(m, b) uint64 snapshot of every lane, 0 = empty (filter.py:194-208)."""
        c = self.cfg
        f, tpw = c.fingerprint_bits, c.tags_per_word
        w = self.words_device.view(c.bucket_count, c.words_per_bucket)
        lanes = torch.empty((c.bucket_count, c.bucket_slots), dtype=torch.int64, device=self.device)
        mask = (1 << f) - 1
        for slot in range(c.bucket_slots):
            lanes[:, slot] = torch.bitwise_and(w[:, slot // tpw] >> (f * (slot % tpw)), mask)
        return lanes.cpu().numpy().view(np.uint64)

    # ---- phase assertions (debug mode only; filter.py:212-226) ----

    def _enter_mutate(self) -> None:
        if self._read_depth:
            raise PhaseError("mutation started while queries are in flight")
        self._mut_depth += 1

    def _exit_mutate(self) -> None:
        self._mut_depth -= 1

    def _enter_read(self) -> None:
        if self._mut_depth:
            raise PhaseError("query started while mutations are in flight")
        self._read_depth += 1

    def _exit_read(self) -> None:
        self._read_depth -= 1

    # ---- plumbing ----

    def _stream(self) -> int:
        """Raw handle of this device's current CUDA stream (the cheap accessor:
        host time before the first launch is idle GPU time in a timed call)."""
        return torch._C._cuda_getCurrentRawStream(self._dev_index)

    def _as_keys(self, keys):
        """Contiguous device int64 view of the keys + where answers should go:
        "numpy" (host arrays / sequences, like the reference), "cpu" (a host
        torch tensor; pinned memory gives an async DMA) or "cuda" (stay on device)."""
        if isinstance(keys, torch.Tensor):
            if keys.dim() != 1:
                raise ValueError("keys must be one-dimensional")
            if keys.dtype == torch.uint64:
                keys = keys.view(torch.int64)
            elif keys.dtype != torch.int64:
                keys = keys.to(torch.int64)
            if keys.device.type == "cpu":
                return keys.contiguous().to(self.device, non_blocking=True), "cpu"
            if keys.device != self.device:
                return keys.to(self.device, non_blocking=True).contiguous(), "cuda"
            return keys.contiguous(), "cuda"
        arr = np.ascontiguousarray(keys, dtype=np.uint64)
        if arr.ndim != 1:
            raise ValueError("keys must be one-dimensional")
        t = torch.from_numpy(arr.view(np.int64))
        return t.to(self.device), "numpy"

    @staticmethod
    def _answer(dev_bool: torch.Tensor, kind: str):
        if kind == "cuda":
            return dev_bool
        if kind == "cpu":
            host = torch.empty(dev_bool.shape, dtype=torch.bool, pin_memory=True)
            host.copy_(dev_bool, non_blocking=True)
            torch.cuda.current_stream(dev_bool.device).synchronize()
            return host
        return dev_bool.cpu().numpy()

    def _flags(self, deterministic: Optional[bool]) -> int:
        det = self._deterministic if deterministic is None else deterministic
        return (_lib.MODE_SEQUENTIAL if det else _lib.MODE_CONCURRENT) | self._tiled_flags

    def _workspace(self, p, n: int, op: int, flags: int):
        """(pointer, bytes) of region-schedule scratch on the current stream, or
        (None, 0).  One grow-only buffer per stream: batches on different
        streams never share bins or result bitmaps, and a buffer is only freed
        after the work queued on its stream."""
        need = int(_lib.lib().ckf_workspace_bytes(ctypes.byref(p), n, op, flags))
        if need == 0:
            return None, 0
        s = self._stream()
        ws = self._ws.get(s)
        if ws is None or ws.numel() < need:
            if ws is not None:
                ws.record_stream(torch.cuda.current_stream(self.device))
            ws = self._ws[s] = None
            ws = self._ws[s] = torch.empty(need, dtype=torch.uint8, device=self.device)
        return ws.data_ptr(), ws.numel()

    def schedule(self, n: int, op: str = "insert", deterministic: Optional[bool] = None):
        """(schedule, runs) a batch of n device keys would run: "region" (binned,
        shared-memory probe; `runs` back-to-back region runs), "direct" or
        "sequential"."""
        code = {"query": _lib.OP_QUERY, "insert": _lib.OP_INSERT, "delete": _lib.OP_DELETE}[op]
        flags = self._flags(deterministic) if code != _lib.OP_QUERY else self._tiled_flags
        return self._schedule_of(self._params, n, code, flags, 0, *self._workspace(self._params, n, code, flags))

    @staticmethod
    def _schedule_of(p, n: int, op: int, flags: int, kptr: int, ws, wsb):
        runs = ctypes.c_uint64(0)
        sc = _lib.lib().ckf_schedule(ctypes.byref(p), n, op, flags, kptr, ws, wsb, ctypes.byref(runs))
        _lib.check(min(sc, 0))
        return _lib.SCHED_NAMES[sc], int(runs.value)

    def _params_for(self, worker: int):
        if worker == 0:
            return self._params
        p = _lib.Params.from_buffer_copy(self._params)
        p.worker = worker & MASK64
        return p

    # ---- scalar operations ----

    def insert(self, key: int, worker: int = 0) -> InsertResult:
        """Store one key; evict residents if both buckets are full (filter.py:230-240)."""
        if self._debug:
            self._enter_mutate()
        try:
            res = self._insert(np.array([key & MASK64], dtype=np.uint64), worker, None)
            ev = int(res.evictions[0])
            if bool(res.ok[0]):
                return InsertResult(True, ev)
            return InsertResult(False, ev, int(res.lost_fingerprints[0]))
        finally:
            if self._debug:
                self._exit_mutate()

    def query(self, key: int) -> bool:
        if self._debug:
            self._enter_read()
        try:
            return bool(self._query(np.array([key & MASK64], dtype=np.uint64))[0])
        finally:
            if self._debug:
                self._exit_read()

    def delete(self, key: int, worker: int = 0) -> bool:
        """Clear one lane matching the key's fingerprint (filter.py:252-264)."""
        if self._debug:
            self._enter_mutate()
        try:
            return bool(self._delete(np.array([key & MASK64], dtype=np.uint64), None)[0])
        finally:
            if self._debug:
                self._exit_mutate()

    # ---- batch operations ----

    def insert_batch(self, keys, workers: int = 1, *, deterministic: Optional[bool] = None,
                     hashed: bool = False) -> BatchInsertResult:
        """Insert every key; results are index-aligned with the input (filter.py:401-442).

        ``hashed=True``: the values are xxh64(key, seed) already (multi-GPU router)."""
        if self._debug:
            self._enter_mutate()
        try:
            return self._insert(keys, 0, deterministic, hashed)
        finally:
            if self._debug:
                self._exit_mutate()

    def query_batch(self, keys, workers: int = 1, *, hashed: bool = False):
        """Boolean membership per key (filter.py:444-473)."""
        if self._debug:
            self._enter_read()
        try:
            return self._query(keys, hashed)
        finally:
            if self._debug:
                self._exit_read()

    def delete_batch(self, keys, workers: int = 1, *, deterministic: Optional[bool] = None,
                     hashed: bool = False):
        """Delete each key once; True where a matching lane was cleared (filter.py:475-502)."""
        if self._debug:
            self._enter_mutate()
        try:
            return self._delete(keys, deterministic, hashed)
        finally:
            if self._debug:
                self._exit_mutate()

    def mixed_batch(self, ops, keys, *, hashed: bool = False):
        """Mixed lookup / insert / delete batch (BASELINE configs[4]) in ONE launch.

        ``ops[i]`` in {0: lookup, 1: insert, 2: delete} (``OP_QUERY`` /
        ``OP_INSERT`` / ``OP_DELETE``).  Returns per key: hit / stored /
        deleted.  An extension past the reference's phase contract
        (filter.py:9-15): all ops run concurrently, lookups with coherent
        loads, so a lookup's answer is exact for keys whose membership the
        batch does not change."""
        if self._debug:
            self._enter_mutate()
        try:
            k, kind = self._as_keys(keys)
            if isinstance(ops, torch.Tensor):
                o = ops.to(self.device, torch.uint8).contiguous()
            else:
                o = torch.from_numpy(np.ascontiguousarray(ops, dtype=np.uint8)).to(self.device)
            n = k.numel()
            if o.numel() != n:
                raise ValueError("ops and keys differ in length")
            with torch.cuda.device(self.device):
                out = torch.empty(n, dtype=torch.uint8, device=self.device)
                rec = torch.empty(max(n, 1) * _lib.RECORD_BYTES, dtype=torch.uint8, device=self.device)
                _lib.check(_lib.lib().ckf_mixed(
                    ctypes.byref(self._params), self.words_device.data_ptr(), o.data_ptr(), k.data_ptr(), n,
                    out.data_ptr(), rec.data_ptr(), n, self._ctr.data_ptr(), self._occ.data_ptr(),
                    _lib.INPUT_HASHED if hashed else 0, self._stream()))
            self.last_schedule = ("direct", 0)
            return self._answer(out.view(torch.bool), kind)
        finally:
            if self._debug:
                self._exit_mutate()

    # ---- one C-ABI launch on device buffers (current stream) ----

    def _launch(self, op: int, k: torch.Tensor, out: torch.Tensor, flags: int, p=None,
                rec: Optional[torch.Tensor] = None, ctr: Optional[torch.Tensor] = None) -> None:
        n = k.numel()
        p = self._params if p is None else p
        L = _lib.lib()
        ws, wsb = self._workspace(p, n, op, flags)
        # an NVTX range per batch call (nsys / ncu --nvtx), named op[n]; the
        # schedule is looked up after the launches (host time before them is
        # GPU idle time)
        with torch.cuda.nvtx.range(f"ckf.{_OP_NAMES[op]}[{n}]"):
            self._call(op, p, k, n, out, flags, rec, ctr, ws, wsb)
        self.last_schedule = self._schedule_of(p, n, op, flags, k.data_ptr(), ws, wsb)

    def _call(self, op, p, k, n, out, flags, rec, ctr, ws, wsb) -> None:
        L = _lib.lib()
        if op == _lib.OP_INSERT:
            _lib.check(L.ckf_insert(
                ctypes.byref(p), self.words_device.data_ptr(), k.data_ptr(), n, out.data_ptr(),
                None, None, rec.data_ptr(), n, ctr.data_ptr(), self._occ.data_ptr(), ws, wsb,
                flags, self._stream()))
        elif op == _lib.OP_QUERY:
            _lib.check(L.ckf_query(
                ctypes.byref(p), self.words_device.data_ptr(), k.data_ptr(), n, out.data_ptr(),
                self._ctr.data_ptr(), ws, wsb, flags, self._stream()))
        else:
            _lib.check(L.ckf_delete(
                ctypes.byref(p), self.words_device.data_ptr(), k.data_ptr(), n, out.data_ptr(),
                self._ctr.data_ptr(), self._occ.data_ptr(), ws, wsb, flags, self._stream()))

    # Host-resident batches larger than this stream through the GPU in chunks:
    # chunk i+1 is copied in while chunk i is processed and chunk i-1's answers
    # are copied out (PCIe is the bound for host data: ~55 GB/s each way).
    HOST_CHUNK = 1 << 25
    # The last chunk is cut short: once its keys are in, the H2D link idles
    # until the call returns (its kernels + its answers' D2H), so a small
    # tail keeps that bubble to ~0.2 ms instead of a whole chunk's compute.
    HOST_TAIL = 1 << 22

    def _chunk_bounds(self, n: int) -> list:
        body = max(n - self.HOST_TAIL, 0)
        cuts = list(range(0, body, self.HOST_CHUNK)) + [body, n]
        return [(lo, hi) for lo, hi in zip(cuts, cuts[1:]) if hi > lo]

    def _host_pipeline(self, op: int, keys: torch.Tensor, flags: int, p=None):
        """Chunked H2D -> kernel -> D2H with copy/compute overlap for CPU keys.
        Returns (host bool answers, [(offset, rec, ctr)] for insert)."""
        n = keys.numel()
        C = self.HOST_CHUNK
        dev = self.device
        comp = torch.cuda.current_stream(dev)
        if self._pipe is None:
            self._pipe = {
                "in": torch.cuda.Stream(dev), "out": torch.cuda.Stream(dev),
                "keys": [torch.empty(C, dtype=torch.int64, device=dev) for _ in range(2)],
                "res": [torch.empty(C, dtype=torch.uint8, device=dev) for _ in range(2)],
            }
        P = self._pipe
        ans = torch.empty(n, dtype=torch.bool, pin_memory=True)
        parts = []
        free_in, free_out = [None, None], [None, None]
        for ci, (lo, hi) in enumerate(self._chunk_bounds(n)):
            b = ci & 1
            m = hi - lo
            with torch.cuda.stream(P["in"]):
                if free_in[b] is not None:
                    P["in"].wait_event(free_in[b])
                P["keys"][b][:m].copy_(keys[lo:hi], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(P["in"])
            comp.wait_event(e_in)
            if free_out[b] is not None:
                comp.wait_event(free_out[b])
            rec = ctr = None
            if op == _lib.OP_INSERT:
                rec = torch.empty(m * _lib.RECORD_BYTES, dtype=torch.uint8, device=dev)
                ctr = torch.empty(4, dtype=torch.int64, device=dev)
                parts.append((lo, rec, ctr))
            self._launch(op, P["keys"][b][:m], P["res"][b][:m], flags, p, rec, ctr)
            e_c = torch.cuda.Event()
            e_c.record(comp)
            free_in[b] = e_c
            with torch.cuda.stream(P["out"]):
                P["out"].wait_event(e_c)
                ans[lo:hi].copy_(P["res"][b][:m].view(torch.bool), non_blocking=True)
                e_o = torch.cuda.Event()
                e_o.record(P["out"])
                free_out[b] = e_o
        P["out"].synchronize()
        return ans, parts

    def _insert(self, keys, worker: int, deterministic: Optional[bool], hashed: bool = False) -> BatchInsertResult:
        p = self._params_for(worker)
        flags = self._flags(deterministic) | (_lib.INPUT_HASHED if hashed else 0)
        if self._chunkable(keys):
            with torch.cuda.device(self.device):
                ans, parts = self._host_pipeline(_lib.OP_INSERT, self._cpu_keys(keys), flags, p)
            return BatchInsertResult.from_parts(keys.numel(), ans, parts)
        k, kind = self._as_keys(keys)
        n = k.numel()
        with torch.cuda.device(self.device):
            ok = torch.empty(n, dtype=torch.uint8, device=self.device)
            rec = torch.empty(max(n, 1) * _lib.RECORD_BYTES, dtype=torch.uint8, device=self.device)
            ctr = torch.empty(4, dtype=torch.int64, device=self.device)
            self._launch(_lib.OP_INSERT, k, ok, flags, p, rec, ctr)
        return BatchInsertResult(n, ok, rec, ctr, kind)

    def _query(self, keys, hashed: bool = False):
        flags = self._tiled_flags | (_lib.INPUT_HASHED if hashed else 0)
        if self._chunkable(keys):
            with torch.cuda.device(self.device):
                return self._host_pipeline(_lib.OP_QUERY, self._cpu_keys(keys), flags)[0]
        k, kind = self._as_keys(keys)
        with torch.cuda.device(self.device):
            out = torch.empty(k.numel(), dtype=torch.uint8, device=self.device)
            self._launch(_lib.OP_QUERY, k, out, flags)
        return self._answer(out.view(torch.bool), kind)

    def _delete(self, keys, deterministic: Optional[bool], hashed: bool = False):
        flags = self._flags(deterministic) | (_lib.INPUT_HASHED if hashed else 0)
        if self._chunkable(keys) and not (flags & _lib.MODE_SEQUENTIAL):
            with torch.cuda.device(self.device):
                return self._host_pipeline(_lib.OP_DELETE, self._cpu_keys(keys), flags)[0]
        k, kind = self._as_keys(keys)
        with torch.cuda.device(self.device):
            out = torch.empty(k.numel(), dtype=torch.uint8, device=self.device)
            self._launch(_lib.OP_DELETE, k, out, flags)
        return self._answer(out.view(torch.bool), kind)

    def _chunkable(self, keys) -> bool:
        """Large host torch tensors take the overlapped chunked pipeline."""
        return (isinstance(keys, torch.Tensor) and keys.device.type == "cpu" and keys.dim() == 1
                and keys.numel() > self.HOST_CHUNK and not self._deterministic)

    @staticmethod
    def _cpu_keys(keys: torch.Tensor) -> torch.Tensor:
        if keys.dtype == torch.uint64:
            keys = keys.view(torch.int64)
        elif keys.dtype != torch.int64:
            keys = keys.to(torch.int64)
        return keys.contiguous()

    def last_counters(self) -> dict:
        """Device counters of the last query / delete batch (one small D2H)."""
        c = self._ctr.cpu().tolist()
        return {"n_ok": c[0], "n_alt": c[3]}

    def collect_eviction_stats(self, keys, prefill_fraction: float = 0.75, workers: int = 1) -> EvictionStats:
        """Insert all keys, sampling eviction counts past the prefill (filter.py:504-519)."""
        if not 0.0 <= prefill_fraction < 1.0:
            raise ValueError("prefill_fraction must be in [0, 1)")
        k, _ = self._as_keys(keys)
        cut = int(k.numel() * prefill_fraction)
        if cut:
            self.insert_batch(k[:cut], workers=workers)
        tail = self.insert_batch(k[cut:], workers=workers)
        return tail.eviction_stats()

    # ---- CKGF serialization (filter.py:523-574) ----

    def to_bytes(self) -> bytes:
        c = self.cfg
        header = _HEADER.pack(_MAGIC, _VERSION, c.fingerprint_bits, c.bucket_slots, c.bucket_count,
                              0 if c.policy is Policy.XOR else 1, self.occupancy, c.seed)
        return header + self.words.astype("<u8", copy=False).tobytes()

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_bytes())

    @classmethod
    def from_bytes(cls, data: bytes, *, eviction=Eviction.DFS, max_evictions: int = 500,
                   device=None) -> "CuckooFilter":
        if len(data) < _HEADER.size:
            raise ValueError("truncated filter dump: header incomplete")
        magic, version, f, b, m, pol, occupancy, seed = _HEADER.unpack_from(data)
        if magic != _MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {_MAGIC!r}")
        if version != _VERSION:
            raise ValueError(f"unsupported dump version {version}")
        if pol not in (0, 1):
            raise ValueError(f"unknown policy code {pol}")
        cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b,
                           policy=Policy.XOR if pol == 0 else Policy.OFFSET,
                           eviction=eviction, max_evictions=max_evictions, seed=seed)
        body = memoryview(data)[_HEADER.size:]
        if len(body) != cfg.total_words * 8:
            raise ValueError(f"word array is {len(body)} bytes, expected {cfg.total_words * 8}")
        filt = cls(cfg, device=device)
        host = torch.from_numpy(np.frombuffer(body, dtype="<u8").view(np.int64).copy())
        filt.words_device.copy_(host)
        filt._occ.fill_(occupancy)
        return filt

    @classmethod
    def load(cls, path, **kwargs) -> "CuckooFilter":
        with open(path, "rb") as fh:
            return cls.from_bytes(fh.read(), **kwargs)
