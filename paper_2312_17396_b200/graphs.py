"""CUDA-graph execution of the batched PS pipeline.

An evaluation has exactly one host synchronisation (the planner needs the
block norms, engine.py:467-472).  The device work on either side of it is
captured once per problem shape into two CUDA graphs and replayed:

  pre graph   X -> working format, digit-plane splits, power chain,
              fused block assembly + column norms, norms -> pinned host buffer
  (host)      certified batched planner (planner.plan_digits_batch)
  post graph  Horner chain for this plan structure (one graph per distinct
              (level formats, members) grouping; cfg2's 64 matrices share one)

The Horner graph depends on the plan only through its structure (the level
scalings are computed on the device from the norms), so the graph of the
previous evaluation's structure is replayed speculatively right after the
pre graph and the host plans while it runs; if the new plan's structure
differs, the right graph is replayed after it (same stream, overwriting
the speculative result).  Results are identical either way.

Buffers live in the graphs' private memory pool and are reused across
replays; inputs are always copied into the graph's static input buffer
(stream-ordered at submit, so the caller may reuse its tensor afterwards and
the post graph, which can re-read X^1 = the static input when a plan keeps
extra dd levels, never sees a later upload), and the result is cloned out, so
every call returns independent tensors.  Any capture failure turns
the graph path off for that shape (eager execution, same kernels).
"""

from __future__ import annotations

import collections
import os
from typing import Dict, Optional, Tuple

import numpy as np

from .precision import FP64, MatBatch

_ENABLED = os.environ.get("MPPS_GRAPHS", "1") != "0"
_SPECULATE = os.environ.get("MPPS_SPECULATE", "1") != "0"
_CACHE: "collections.OrderedDict[tuple, _ShapeGraphs]" = collections.OrderedDict()   # least recently used first
_FAILED = set()
# Every cached shape keeps its intermediates (powers, digit planes, blocks) in a private pool --
# ~1 GB at cfg2, ~20 GB at cfg5 -- so the cache is bounded by bytes: before a new shape is
# captured, least recently used shapes are dropped until the recorded pools fit the budget
# (MPPS_GRAPH_CACHE_GB; default: half of the device memory).
_BUDGET = None


def enabled() -> bool:
    return _ENABLED


def set_enabled(flag: bool) -> None:
    global _ENABLED
    _ENABLED = bool(flag)


def _torch():
    import torch
    return torch


def cache_budget() -> int:
    global _BUDGET
    if _BUDGET is None:
        env = os.environ.get("MPPS_GRAPH_CACHE_GB")
        if env:
            _BUDGET = int(float(env) * (1 << 30))
        else:
            _BUDGET = _torch().cuda.get_device_properties(_torch().cuda.current_device()).total_memory // 2
    return _BUDGET


def set_cache_budget(nbytes: Optional[int]) -> None:
    """Bytes of graph pools kept across shapes (None: the default)."""
    global _BUDGET
    _BUDGET = None if nbytes is None else int(nbytes)


def cache_info() -> dict:
    return {"shapes": len(_CACHE), "bytes": sum(g.bytes for g in _CACHE.values()), "budget": cache_budget()}


def clear() -> None:
    """Drop every cached graph and its pool (after the device is idle)."""
    if _CACHE:
        _torch().cuda.synchronize()
        _CACHE.clear()


def _make_room(keep: tuple) -> None:
    """Drop least recently used shapes while the recorded pools exceed the
    budget.  Evaluations in flight hold their graphs through ``Pending.g``;
    the device is drained first so no replay still reads a released pool."""
    budget = cache_budget()
    drained = False
    while len(_CACHE) > 1 and sum(g.bytes for g in _CACHE.values()) > budget:
        key = next(k for k in _CACHE if k != keep)
        if not drained:
            _torch().cuda.synchronize()
            drained = True
        del _CACHE[key]


class _ShapeGraphs:
    def __init__(self):
        self.bytes = 0            # device memory reserved while this entry was captured (its private pool + warm-up)
        self.pool = None
        self.x_in = None
        self.pre = None
        self.prep = None
        self.norms_pin = None
        self.post: Dict[tuple, tuple] = {}
        self.pre_launches = 0
        self.last_post = None     # structure of the previous evaluation (speculation)


_LAST_LAUNCHES = 0
_SPEC_STATS = {"hit": 0, "miss": 0}


def set_speculation(flag: bool) -> None:
    global _SPECULATE
    _SPECULATE = bool(flag)


def speculation_stats() -> dict:
    """Speculative Horner replays that matched / missed the plan."""
    return dict(_SPEC_STATS)


def last_launches() -> int:
    """Kernels of libmpps_b200.so executed by the last graphed evaluation
    (counted when the graphs were captured)."""
    return _LAST_LAUNCHES


class PlanError(Exception):
    """The host planner raised inside finish(); ``orig`` is its exception."""

    def __init__(self, orig):
        super().__init__(str(orig))
        self.orig = orig


class Pending:
    """A submitted evaluation: the pre graph is enqueued and the norms are
    on their way to pinned memory (``ready`` is recorded after the copy)."""

    __slots__ = ("g", "ready", "timer", "spec", "spec_done", "done")

    def __init__(self, g, ready, timer, spec=None, spec_done=None):
        self.g, self.ready, self.timer, self.spec = g, ready, timer, spec
        self.spec_done = spec_done    # event after the speculative Horner chain
        self.done = None              # event after the result is final (set by finish)


def submit(key: tuple, Xsrc, build_pre, timer, slot: int = 0) -> Optional[Pending]:
    """Enqueue the pre-planner graph of one evaluation (capturing it on first
    use).  ``slot`` selects an independent set of static buffers, so two
    evaluations of the same shape can be in flight (pre of chunk c+1 runs on
    the GPU while the host plans chunk c).  Returns None when graphs are off
    for this key (the caller runs eagerly)."""
    torch = _torch()
    key = key + (("slot", slot),)
    if not _ENABLED or key in _FAILED:
        return None
    g = _CACHE.get(key)
    try:
        if g is None:
            _make_room(key)
            mem0 = torch.cuda.memory_reserved()
            g = _ShapeGraphs()
            g.pool = torch.cuda.graph_pool_handle()
            g.x_in = torch.empty(Xsrc.shape, dtype=torch.float64, device="cuda")
            g.x_in.copy_(Xsrc, non_blocking=True)
            # warm-up (kernel attributes, handles, lazy module state) then capture
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                build_pre(g.x_in, capture=False)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            g.pre = torch.cuda.CUDAGraph()
            from . import _lib
            l0 = _lib.total_launches()
            with torch.cuda.graph(g.pre, pool=g.pool):
                g.prep = build_pre(g.x_in, capture=True)
                # the norms reach the host through a kernel's stores into pinned memory, not a
                # memcpy node: a device-to-host copy queues behind a running result download of
                # the host stream (pipeline.evaluate_host) and the planner would wait for it
                g.norms_pin = torch.empty(g.prep.norms_dev.shape, dtype=torch.float64, pin_memory=True)
                _lib.handle_for().store_host(g.prep.norms_dev.contiguous(), g.norms_pin)
            g.pre_launches = _lib.total_launches() - l0
            g.bytes = max(0, torch.cuda.memory_reserved() - mem0)
            _CACHE[key] = g
        else:
            _CACHE.move_to_end(key)
        g.x_in.copy_(Xsrc, non_blocking=True)
        timer.start("power_formation")
        g.pre.replay()
        ready = torch.cuda.Event()
        ready.record()
        timer.stop()
        spec = g.last_post if _SPECULATE else None
        spec_done = None
        if spec is not None:
            g.post[spec][0].replay()      # speculative Horner chain (checked in finish)
            spec_done = torch.cuda.Event()
            spec_done.record()
        return Pending(g, ready, timer, spec, spec_done)
    except Exception as exc:  # pragma: no cover - capture problems fall back to eager
        _FAILED.add(key)
        _CACHE.pop(key, None)
        import warnings
        warnings.warn(f"CUDA graph path disabled for this shape: {exc!r}")
        return None


def finish(p: Pending, run_post, clone: bool = True):
    """Wait for the submitted evaluation's norms (its event only, not the
    whole stream), plan on the host, enqueue the Horner graph for the plan
    structure and return (prep, norms numpy, result MatBatch, info).
    ``clone=False`` returns the graph's static result buffer itself (valid
    until this slot is submitted again; pipeline.evaluate_host downloads it
    directly) and sets ``p.done``, the event after which it is final."""
    torch = _torch()
    g, timer = p.g, p.timer
    timer.start("norm_estimation")
    p.ready.synchronize()
    norms = g.norms_pin.numpy().copy()
    timer.stop()
    g.prep.norms = norms
    try:
        post_key, post_fn, info = run_post(g.prep, norms)
    except Exception as exc:
        # the planner rejected the norms (a non-finite input: engine.py:467-472 raises the same
        # way in the reference): the caller's error, not a capture problem -- the graphs stay
        raise PlanError(exc) from exc
    entry = g.post.get(post_key)
    if entry is None:
        mem0 = torch.cuda.memory_reserved()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            post_fn(g.prep)                 # warm-up (new kernel instantiations)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        from . import _lib
        l0 = _lib.total_launches()
        with torch.cuda.graph(graph, pool=g.pool):
            res = post_fn(g.prep)
        entry = (graph, res, post_fn, _lib.total_launches() - l0)  # post_fn keeps its index tensors alive
        g.post[post_key] = entry
        g.bytes += max(0, torch.cuda.memory_reserved() - mem0)
    graph, res, _, post_launches = entry
    global _LAST_LAUNCHES
    _LAST_LAUNCHES = g.pre_launches + post_launches
    timer.start("mixed_horner")
    if p.spec is not None and p.spec == post_key:
        _SPEC_STATS["hit"] += 1
        p.done = p.spec_done
    else:
        if p.spec is not None:
            _SPEC_STATS["miss"] += 1
            _LAST_LAUNCHES += g.post[p.spec][3]   # the speculative chain ran too
        graph.replay()
        p.done = torch.cuda.Event()
        p.done.record()
    g.last_post = post_key
    out = MatBatch(res.data.clone(), res.fmt) if clone else MatBatch(res.data, res.fmt)
    if clone:
        # the caller's tensor is final only after the copy out of the static buffer: a consumer on
        # another stream (pipeline.evaluate_host's download) waited for the event recorded after the
        # Horner replay and could read the clone before it was written (tools/fuzz_pipeline.py)
        p.done = torch.cuda.Event()
        p.done.record()
    timer.stop()
    return g.prep, norms, out, info


def run(key: tuple, Xsrc, build_pre, run_post, timer):
    """Execute one evaluation through cached graphs: submit + finish.

    key       hashable problem shape (batch, n, series, digits, engine, ...)
    Xsrc      torch fp64 (B, n, n) tensor (device or pinned host)
    build_pre(Xstatic) -> _Prepared   eager pre-planner pipeline (captured)
    run_post(prep, norms) -> (post_key, post_fn, info)
              post_fn(prep) launches the Horner chain and returns the result
    Returns (prep, norms numpy, result MatBatch, info) or None when graphs
    are off for this key (caller runs eagerly)."""
    p = submit(key, Xsrc, build_pre, timer)
    if p is None:
        return None
    try:
        return finish(p, run_post)
    except PlanError as pe:
        raise pe.orig
    except Exception as exc:  # pragma: no cover - capture problems fall back to eager
        _FAILED.add(key + (("slot", 0),))
        import warnings
        warnings.warn(f"CUDA graph path disabled for this shape: {exc!r}")
        return None
