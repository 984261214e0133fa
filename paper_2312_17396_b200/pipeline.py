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
from typing import Callable, List, Optional


def _torch():
    import torch
    return torch


def mixed_exp(m: int, ctx, **kw) -> Callable:
    """submit callable for ps_mixed_exp (fix_params=True)."""
    from .engine import submit_mixed_exp

    def sub(x, slot, static_result=False):
        return submit_mixed_exp(x, m, ctx, slot=slot, static_result=static_result, **kw)
    return sub


def mixed_general(series, ctx, **kw) -> Callable:
    """submit callable for ps_mixed_general."""
    from .engine import submit_mixed_general

    def sub(x, slot, static_result=False):
        return submit_mixed_general(x, series, ctx, slot=slot, static_result=static_result, **kw)
    return sub


def eager(fn: Callable) -> Callable:
    """submit callable running a one-shot evaluator at submit time."""
    from .engine import PendingEvaluation

    def sub(x, slot, static_result=False):
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


def evaluate_host(submit: Callable, X_host, out_host, chunks=3, trace=None, streams: int = 1,
                  ahead=None, window: Optional[int] = None) -> List[object]:
    """``chunks``: a count (tapered split, see split_sizes) or explicit sizes.

    ``streams=1``: chunks run one after another on the caller's stream, the
    next chunk submitted when the previous one is planned.
    ``streams=2``: every chunk is submitted up front (its own graph slot,
    chunk c on compute stream c % 2, the Horner chain replayed
    speculatively, graphs.py), so the GPU never waits for the host planner;
    the host then plans the chunks in order and each chunk's result is
    downloaded straight from its slot's buffer once final.  Reports of this
    mode reference those slot buffers: their ``result`` is valid until the
    next call with the same shapes (``out_host`` holds the copy).
    ``ahead`` (default: streams > 1) selects the submit-everything-up-front
    mode independently of the stream count.
    ``window`` (ahead mode): at most this many chunks in flight, each in
    graph slot ``c % window`` with its own device input buffer; chunk
    c + window is uploaded and submitted once chunk c is planned, its
    upload waiting on the GPU for chunk c's input copy and its evaluation
    for chunk c's download.  A long host stream (many batches) then runs
    through a bounded set of slots with the copies of one batch overlapping
    the evaluation of the next; a report's ``result`` is then valid only
    until chunk c + window is submitted (``out_host`` holds every result).
    Default: every chunk in flight.
    ``trace``: optional list; timing events (label, event, host time) are
    appended (diagnostics, tools/e2e_chunks.py)."""
    import gc
    gc_was = gc.isenabled()
    gc.disable()    # a gen-2 collection (~30 ms) would idle the GPU waiting on the host planner
    try:
        return _evaluate_host(submit, X_host, out_host, chunks, trace, streams, ahead, window)
    finally:
        if gc_was:
            gc.enable()


def _evaluate_host(submit, X_host, out_host, chunks, trace, streams, ahead, window):
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
    if ahead is None:
        ahead = streams > 1
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
    W = chunks if (window is None or not ahead) else max(1, min(int(window), chunks))
    dev_in = [None] * chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    consumed = [None] * chunks        # after chunk c's pre graph took its input
    downed = [None] * chunks          # after chunk c's result left the device
    pend = [None] * chunks
    reps = []

    def upload(c):
        # one device input buffer per chunk position (cached across calls), so
        # every upload is enqueued up front and never waits for a consumer
        # (with a window: per slot, after the previous chunk of the slot took it)
        lo, hi = bounds[c], bounds[c + 1]
        with torch.cuda.stream(up):
            if c >= W:
                up.wait_event(consumed[c - W])
            shape = (hi - lo,) + tuple(X_host.shape[1:])
            buf = st["bufs"].get((c % W, shape))
            if buf is None:
                buf = torch.empty(shape, dtype=torch.float64, device=caller.device)
                st["bufs"][(c % W, shape)] = buf
            dev_in[c] = buf
            mark(f"up{c}<", up)
            buf.copy_(X_host[lo:hi], non_blocking=True)
            mark(f"up{c}>", up)
            ev_in[c].record(up)

    def start(c):
        comp = comps[c % 2]
        with torch.cuda.stream(comp):
            comp.wait_event(ev_in[c])
            if c >= W:
                comp.wait_event(downed[c - W])     # the slot's result buffer is free
            mark(f"pre{c}<", comp)
            if ahead:
                pend[c] = submit(dev_in[c], c % W, static_result=True)
            else:
                pend[c] = submit(dev_in[c], c % 2)
            consumed[c] = torch.cuda.Event()
            consumed[c].record(comp)
            mark(f"pre{c}>", comp)

    for c in range(W):
        upload(c)
    if ahead:
        for c in range(W):
            start(c)
    else:
        start(0)
    for c in range(chunks):
        comp = comps[c % 2]
        with torch.cuda.stream(comp):
            mark(f"post{c}<", comp)
            rep = pend[c].finish()
            mark(f"post{c}>", comp)
            done = pend[c].done_event
            if done is None:
                done = torch.cuda.Event()
                done.record(comp)
        pend[c] = None
        if not ahead and c + 1 < chunks:
            # submitted after chunk c's planning: its speculative Horner
            # chain follows chunk c's without a GPU gap
            start(c + 1)
        lo, hi = bounds[c], bounds[c + 1]
        res = rep.result.data
        with torch.cuda.stream(down):
            down.wait_event(done)
            mark(f"down{c}<", down)
            for w in range(res.shape[0]):    # contiguous pinned destination per word
                out_host[w, lo:hi].copy_(res[w], non_blocking=True)
            res.record_stream(down)
            downed[c] = torch.cuda.Event()
            downed[c].record(down)
            mark(f"down{c}>", down)
        reps.append(rep)
        if ahead and c + W < chunks:
            upload(c + W)
            start(c + W)
    for cs in set(comps):
        if cs is not caller:
            caller.wait_stream(cs)
    caller.wait_stream(down)
    caller.wait_stream(up)
    return reps


def evaluate_stream(fn: Callable, X_host: List, out_host: List, results_of: Optional[Callable] = None,
                    keep_reports: bool = True) -> List[object]:
    """A stream of host-resident inputs through any one-shot evaluator
    ``fn(x_dev) -> report`` (e.g. ``lambda x: ps_mixed_general(cos_argument(x,
    ctx), series, ctx)`` for one large matrix per step), software-pipelined:

      upload stream    H2D of input t+1 (two device input slots)
      caller stream    fn(input t)
      download stream  D2H of result t into ``out_host[t]`` (pinned), while
                       input t+1 is evaluated

    ``results_of(report) -> [device tensors]`` (default: ``report.result.data``)
    names the tensors copied into the matching ``out_host[t]`` list entries.
    Inputs are pinned host tensors of one shape; returns the reports
    (``keep_reports=False``: none are kept, so each step's device result is
    released as soon as its download is done -- a long stream then runs in
    constant device memory)."""
    torch = _torch()
    caller = torch.cuda.current_stream()
    st = _state(torch, caller.device)
    up, down = st["up"], st["down"]
    up.wait_stream(caller)
    down.wait_stream(caller)
    results_of = results_of or (lambda rep: [rep.result.data])
    T = len(X_host)
    shape = tuple(X_host[0].shape)
    slots = st["bufs"].get(("stream", shape))
    if slots is None:
        slots = st["bufs"][("stream", shape)] = [torch.empty(shape, dtype=torch.float64, device=caller.device)
                                                 for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(T)]
    consumed = [None] * T

    def upload(t):
        with torch.cuda.stream(up):
            if t >= 2:
                up.wait_event(consumed[t - 2])       # the slot's previous input was taken
            slots[t % 2].copy_(X_host[t], non_blocking=True)
            ev_in[t].record(up)

    reps = []
    upload(0)
    for t in range(T):
        if t + 1 < T:
            upload(t + 1)
        caller.wait_event(ev_in[t])
        rep = fn(slots[t % 2])
        consumed[t] = torch.cuda.Event()
        consumed[t].record(caller)
        with torch.cuda.stream(down):
            down.wait_event(consumed[t])
            for dst, src in zip(out_host[t], results_of(rep)):
                dst.copy_(src, non_blocking=True)
                src.record_stream(down)
        if keep_reports:
            reps.append(rep)
        del rep
    caller.wait_stream(down)
    caller.wait_stream(up)
    return reps
