"""Host-resident batches: overlap host<->device copies, host planning and
device evaluation.

``evaluate_host(submit, X_host, out_host, chunks)`` splits a pinned host
batch (B, n, n) into chunks and software-pipelines them:

  upload stream    H2D of chunk c+1 (double-buffered device input)
  compute stream   pre-planner graph and (speculatively, graphs.py) Horner
                   graph of each chunk; the host plans chunk c while its
                   Horner chain runs
  download stream  D2H of chunk c's result into ``out_host`` (words, B, n, n)

PCIe is full duplex and the copies run on the copy engines, so for a
multi-chunk batch only the first upload and the last download are exposed.
``submit(x_dev, slot)`` returns an object with ``finish() -> report``
(engine.submit_mixed_exp / submit_mixed_general, or ``eager(fn)`` for any
one-shot evaluator).  Reports are returned in chunk order.
"""

from __future__ import annotations

import time
from typing import Callable, List


def _torch():
    import torch
    return torch


def mixed_exp(m: int, ctx, **kw) -> Callable:
    """submit callable for ps_mixed_exp (fix_params=True)."""
    from .engine import submit_mixed_exp
    return lambda x, slot: submit_mixed_exp(x, m, ctx, slot=slot, **kw)


def mixed_general(series, ctx, **kw) -> Callable:
    """submit callable for ps_mixed_general."""
    from .engine import submit_mixed_general
    return lambda x, slot: submit_mixed_general(x, series, ctx, slot=slot, **kw)


def eager(fn: Callable) -> Callable:
    """submit callable running a one-shot evaluator at submit time."""
    from .engine import PendingEvaluation

    def sub(x, slot):
        rep = fn(x)
        return PendingEvaluation(lambda: rep)
    return sub


_STATE = {}


def _state(torch, dev):
    """Copy streams and double-buffered device inputs, reused across calls
    (creating streams/allocations per call costs ~0.4 ms of host time)."""
    st = _STATE.get(dev)
    if st is None:
        st = {"up": torch.cuda.Stream(), "down": torch.cuda.Stream(), "bufs": {}}
        _STATE[dev] = st
    return st


def split_sizes(B: int, chunks) -> List[int]:
    """Chunk sizes: an explicit list, or ``chunks`` parts tapered so the last
    chunk (whose download is exposed) is the smallest."""
    if not isinstance(chunks, int):
        sizes = [int(x) for x in chunks]
        if sum(sizes) != B or min(sizes) < 1:
            raise ValueError("chunk sizes must be positive and sum to the batch")
        return sizes
    k = max(1, min(int(chunks), B))
    if k == 1:
        return [B]
    last = max(1, B // (2 * k - 1))            # the last chunk is about half the others
    rest = B - last
    sizes = [(rest * (i + 1)) // (k - 1) - (rest * i) // (k - 1) for i in range(k - 1)]
    return sizes + [last]


def evaluate_host(submit: Callable, X_host, out_host, chunks=3, trace=None, streams: int = 1) -> List[object]:
    """``chunks``: a count (tapered split, see split_sizes) or explicit sizes.
    ``streams``: 1 runs the chunks one after another on the caller's stream;
    2 alternates them over two compute streams (slot c % 2 on stream c % 2),
    so chunk c+1's kernels fill the tails and gaps of chunk c's (a small
    chunk alone leaves SMs idle in every kernel's last wave).
    ``trace``: optional list; timing events (label, event) are appended
    (diagnostics, tools/e2e_chunks.py)."""
    torch = _torch()

    def mark(label, stream):
        if trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            trace.append((label, e, time.perf_counter()))
    B = X_host.shape[0]
    sizes = split_sizes(B, chunks)
    chunks = len(sizes)
    bounds = [0]
    for z in sizes:
        bounds.append(bounds[-1] + z)
    caller = torch.cuda.current_stream()
    st = _state(torch, caller.device)
    up, down = st["up"], st["down"]
    if streams > 1:
        comps = st.get("comps")
        if comps is None:
            comps = st["comps"] = [torch.cuda.Stream(), torch.cuda.Stream()]
        for cs in comps:
            cs.wait_stream(caller)
    else:
        comps = [caller, caller]
    up.wait_stream(caller)
    down.wait_stream(caller)
    dev_in = [None] * chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    pend = [None] * chunks
    reps = []

    def upload(c):
        # one device input buffer per chunk position (cached across calls), so
        # every upload is enqueued up front and never waits for a consumer
        lo, hi = bounds[c], bounds[c + 1]
        with torch.cuda.stream(up):
            shape = (hi - lo,) + tuple(X_host.shape[1:])
            buf = st["bufs"].get((c, shape))
            if buf is None:
                buf = torch.empty(shape, dtype=torch.float64, device=caller.device)
                st["bufs"][(c, shape)] = buf
            dev_in[c] = buf
            mark(f"up{c}<", up)
            buf.copy_(X_host[lo:hi], non_blocking=True)
            mark(f"up{c}>", up)
            ev_in[c].record(up)

    def start(c):
        comp = comps[c % 2]
        with torch.cuda.stream(comp):
            comp.wait_event(ev_in[c])
            mark(f"pre{c}<", comp)
            pend[c] = submit(dev_in[c], c % 2)
            mark(f"pre{c}>", comp)

    for c in range(chunks):
        upload(c)
    start(0)
    if streams > 1 and chunks > 1:
        start(1)
    for c in range(chunks):
        # submit() already enqueued chunk c's Horner chain speculatively
        # (graphs.py), so finishing c before starting the next chunk leaves
        # no GPU gap and chunk c's download can begin as soon as its chain
        # ends.
        comp = comps[c % 2]
        with torch.cuda.stream(comp):
            mark(f"post{c}<", comp)
            rep = pend[c].finish()
            mark(f"post{c}>", comp)
            done = torch.cuda.Event()
            done.record(comp)
        pend[c] = None
        if streams > 1:
            if c + 2 < chunks:
                start(c + 2)
        elif c + 1 < chunks:
            start(c + 1)
        lo, hi = bounds[c], bounds[c + 1]
        res = rep.result.data
        with torch.cuda.stream(down):
            down.wait_event(done)
            mark(f"down{c}<", down)
            for w in range(res.shape[0]):    # contiguous pinned destination per word
                out_host[w, lo:hi].copy_(res[w], non_blocking=True)
            res.record_stream(down)
            mark(f"down{c}>", down)
        reps.append(rep)
    for cs in set(comps):
        if cs is not caller:
            caller.wait_stream(cs)
    caller.wait_stream(down)
    caller.wait_stream(up)
    return reps
