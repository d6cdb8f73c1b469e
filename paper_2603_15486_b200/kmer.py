"""FASTA k-mer ingestion on the GPU (reference: swarcuckoo/kmer.py:1-138).

Same API and semantics as the reference module: ``pack_kmer``,
``stream_kmers`` and ``kmer_bench``.  Each k-mer (k <= 31) packs into one
64-bit key, two bits per base (A=0, C=1, G=2, T=3, either case), leftmost base
most significant; windows containing any other character (N, ...) are
skipped and windows never span FASTA records; k-mers are raw-strand, in
sequence order, duplicates kept (kmer.py:1-9).

What runs where: the host parses the FASTA structure (headers, blank lines,
the "sequence before the first header" error) into one byte buffer -- each
record's sequence lines concatenated, one separator byte between records --
and the window packing runs on the device (``ckf_kmers`` in include/ckf.h:
a count pass, a scan and an emit pass over 1024-base chunks).
``stream_kmers`` is the reference's lazy iterator of ints (the device packs
the whole source at the first ``next``); ``kmer_array`` returns the same
stream as one numpy uint64 array and ``stream_kmers(..., as_tensor=True)`` as
the device tensor ``insert_batch`` takes.
"""

from __future__ import annotations

from dataclasses import replace
from typing import Iterable, Optional

import numpy as np
import torch

from . import _lib
from .bench_harness import BenchReport, RunSpec, _report, _Timer
from .errors import FastaError
from .filter import CuckooFilter

_BASE_CODES = {"A": 0, "C": 1, "G": 2, "T": 3}
_BASE_CODES.update({b.lower(): c for b, c in _BASE_CODES.items()})
_SEPARATOR = b"\n"  # any byte outside ACGTacgt ends every window


def pack_kmer(bases: str) -> Optional[int]:
    """Pack a length-k base string into an integer, or None if ambiguous (kmer.py:28-45)."""
    if not 1 <= len(bases) <= 31:
        raise ValueError(f"k must be in [1, 31], got {len(bases)}")
    value = 0
    for ch in bases:
        code = _BASE_CODES.get(ch)
        if code is None:
            return None
        value = (value << 2) | code
    return value


def _lines(source) -> Iterable[str]:
    if isinstance(source, (str, bytes)) or hasattr(source, "__fspath__"):
        with open(source, "r") as fh:
            yield from fh
    else:
        yield from source


def sequence_buffer(source) -> bytes:
    """FASTA structure -> the device input of ``ckf_kmers``.

    Mirrors the reference's line loop (kmer.py:48-74): blank lines are
    skipped, a ``>`` line starts a record (windows never span records), lines
    are stripped, and sequence data before the first header raises
    ``FastaError`` with its 1-based line number."""
    parts = []
    saw_header = False
    for line_number, line in enumerate(_lines(source), 1):
        stripped = line.strip()
        if not stripped:
            continue
        if stripped.startswith(">"):
            saw_header = True
            parts.append(_SEPARATOR)
            continue
        if not saw_header:
            raise FastaError(line_number, "sequence data before the first '>' header")
        parts.append(stripped.encode("latin-1", "replace"))
    return b"".join(parts)


def kmers_from_buffer(buf, k: int, device=None) -> torch.Tensor:
    """Device k-mers (int64 view of uint64) of a ``sequence_buffer`` result."""
    if not 1 <= k <= 31:
        raise ValueError(f"k must be in [1, 31], got {k}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    L = _lib.lib()
    host = np.frombuffer(buf, dtype=np.uint8) if isinstance(buf, (bytes, bytearray)) else np.asarray(buf, np.uint8)
    n = len(host)
    with torch.cuda.device(dev):
        seq = torch.from_numpy(host.copy()).to(dev) if n else torch.empty(0, dtype=torch.uint8, device=dev)
        cap = max(n - k + 1, 1)
        out = torch.empty(cap, dtype=torch.int64, device=dev)
        n_out = torch.zeros(1, dtype=torch.int64, device=dev)
        wsb = int(L.ckf_kmer_workspace_bytes(n))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(L.ckf_kmers(seq.data_ptr() if n else None, n, k, out.data_ptr(), n_out.data_ptr(),
                               ws.data_ptr(), wsb, stream))
        return out[: int(n_out.item())]


def kmer_array(source, k: int, device=None) -> np.ndarray:
    """The packed stream of ``stream_kmers`` as one numpy uint64 array."""
    if not 1 <= k <= 31:
        raise ValueError(f"k must be in [1, 31], got {k}")
    return kmers_from_buffer(sequence_buffer(source), k, device).cpu().numpy().view(np.uint64)


def _iter_kmers(source, k: int, device):
    yield from (int(v) for v in kmer_array(source, k, device))


def stream_kmers(source, k: int, *, as_tensor: bool = False, device=None):
    """Yield every valid k-mer window of a FASTA source, packed (kmer.py:77-95).

    ``source`` is a path or an iterable of lines.  Like the reference, a lazy
    iterator: k and the FASTA structure are checked when iteration starts.
    ``as_tensor=True`` (extension) returns the whole stream at once as the
    device int64 tensor that ``CuckooFilter.insert_batch`` takes."""
    if as_tensor:
        if not 1 <= k <= 31:
            raise ValueError(f"k must be in [1, 31], got {k}")
        return kmers_from_buffer(sequence_buffer(source), k, device)
    return _iter_kmers(source, k, device)


def kmer_bench(path, k: int, spec: RunSpec) -> list[BenchReport]:
    """Insert, positive-query and delete throughput over a FASTA's k-mers (kmer.py:98-138).

    The k-mers are extracted on the device once; each phase is then timed as
    one whole batch with CUDA events (insert all, query all -- every one must
    hit -- delete all).  One report per phase; ``n_keys`` is the window count."""
    keys = stream_kmers(path, k, as_tensor=True)
    n = int(keys.numel())
    cfg = spec.config()
    filt = CuckooFilter(cfg)
    reports = []
    for op in ("insert", "query_pos", "delete"):
        phase = replace(spec, op=op)
        if op == "insert":
            with _Timer() as t:
                res = filt.insert_batch(keys, workers=spec.workers)
            dt = t.seconds
            reports.append(_report(phase, cfg, n, dt, n / dt if dt > 0 else float("inf"), None, res.n_failed,
                                   res.eviction_stats(), load_factor=filt.load_factor, repetitions=1))
        elif op == "query_pos":
            with _Timer() as t:
                filt.query_batch(keys, workers=spec.workers)
            dt = t.seconds
            reports.append(_report(phase, cfg, n, dt, n / dt if dt > 0 else float("inf"), None, 0, None,
                                   load_factor=filt.load_factor, repetitions=1))
        else:
            alpha = filt.load_factor
            with _Timer() as t:
                filt.delete_batch(keys, workers=spec.workers)
            dt = t.seconds
            reports.append(_report(phase, cfg, n, dt, n / dt if dt > 0 else float("inf"), None, 0, None,
                                   load_factor=alpha, repetitions=1))
    return reports
