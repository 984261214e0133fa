"""ctypes binding of the C-ABI in include/mpps_b200.h.

The shared library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_2312_17396_b200.build``) at
``paper_2312_17396_b200/_lib/libmpps_b200.so``.  There is no fallback: if the
library is missing or a call fails, the error is raised with the library's
own message.
"""

from __future__ import annotations

import ctypes

import numpy as np
import os
import threading
from typing import Optional

from .precision import DimensionError, MatBatch, UnsupportedPrecisionError

LIB_PATH = os.environ.get("MPPS_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libmpps_b200.so")

MPPS_OK, MPPS_EINVAL, MPPS_EFMT, MPPS_ECUDA = 0, 1, 2, 3

EXPORTED = (
    "mpps_version", "mpps_create", "mpps_destroy", "mpps_set_stream",
    "mpps_last_error", "mpps_launch_count", "mpps_convert", "mpps_gemm",
    "mpps_axpy", "mpps_powers", "mpps_slice_into", "mpps_assemble_blocks", "mpps_assemble_blocks_hc", "mpps_assemble_hc_supported", "mpps_assemble_blocks_hc_n", "mpps_assemble_hc_n_supported", "mpps_one_norm", "mpps_one_norm_complex", "mpps_level_exps", "mpps_store_host",
    "mpps_horner_step", "mpps_horner_scalar_top", "mpps_probe_fma",
    "mpps_assemble_blocks_dist", "mpps_colmax", "mpps_slice", "mpps_gemm_sliced",
    "mpps_horner_step_sliced", "mpps_oz_slices_for", "mpps_oz_slices_for_bits", "mpps_oz_max_k_8bit", "mpps_oz_max_k", "mpps_probe_i8mma", "mpps_debug_oz_trace",
    "mpps_debug_oz_flags", "mpps_debug_probe_i8mma_n", "mpps_probe_ingest",
    "mpps_small_ps_supported", "mpps_small_ps_prepare", "mpps_small_ps_horner", "mpps_slice_ex", "mpps_small_ps_eval",
)


class CSlices(ctypes.Structure):
    _fields_ = [
        ("digits", ctypes.c_void_p),
        ("exps", ctypes.c_void_p),
        ("nslices", ctypes.c_int),
        ("batch", ctypes.c_int),
        ("rpad", ctypes.c_int),
        ("kpad", ctypes.c_int),
        ("digit_bits", ctypes.c_int),
    ]


class Slices:
    """Digit planes of one operand for the tensor-core path (torch buffers):
    digits int8 (S, batch, rpad, kpad), exps int32 (batch, rpad)."""

    __slots__ = ("digits", "exps", "S", "rows", "k", "db")

    def __init__(self, S: int, batch: int, rows: int, k: int, device, db: int = 7):
        import torch
        rpad = -(-rows // 128) * 128
        kpad = -(-k // 32) * 32
        self.digits = torch.empty((S, batch, rpad, kpad), dtype=torch.int8, device=device)
        self.exps = torch.empty((batch, rpad), dtype=torch.int32, device=device)
        self.S, self.rows, self.k, self.db = S, rows, k, db

    def c(self) -> CSlices:
        d = self.digits
        return CSlices(d.data_ptr(), self.exps.data_ptr(), d.shape[0], d.shape[1], d.shape[2], d.shape[3], self.db)


class CMat(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p),
        ("plane_stride", ctypes.c_longlong),
        ("batch_stride", ctypes.c_longlong),
        ("rows", ctypes.c_int),
        ("cols", ctypes.c_int),
        ("ld", ctypes.c_int),
        ("batch", ctypes.c_int),
        ("fmt", ctypes.c_int),
    ]


class MppsError(RuntimeError):
    pass


class MppsCudaError(MppsError):
    pass


_lib = None
_lib_lock = threading.Lock()


def load_library(path: Optional[str] = None):
    """Load (once) and declare the C-ABI.  Raises if the .so is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise ImportError(
                f"B200 kernel library not built: {p} is missing. Run "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(no CPU fallback exists by design).")
        lib = ctypes.CDLL(p)
        P = ctypes.POINTER
        vp, ip = ctypes.c_void_p, ctypes.c_int
        mp = P(CMat)
        lib.mpps_version.restype = ip
        lib.mpps_create.argtypes = [ip, vp, P(vp)]
        lib.mpps_destroy.argtypes = [vp]
        lib.mpps_set_stream.argtypes = [vp, vp]
        lib.mpps_last_error.argtypes = [vp]
        lib.mpps_last_error.restype = ctypes.c_char_p
        lib.mpps_launch_count.argtypes = [vp]
        lib.mpps_launch_count.restype = ctypes.c_longlong
        lib.mpps_convert.argtypes = [vp, mp, mp, vp, ip, vp]
        lib.mpps_gemm.argtypes = [vp, mp, mp, mp, vp, ip]
        lib.mpps_axpy.argtypes = [vp, P(ctypes.c_double), mp, mp, mp]
        lib.mpps_powers.argtypes = [vp, mp, ip]
        lib.mpps_assemble_blocks.argtypes = [vp, mp, ip, ip, vp, mp, vp]
        lib.mpps_assemble_blocks_hc.argtypes = [vp, mp, ip, ip, P(ctypes.c_double), mp, vp, ip]
        lib.mpps_assemble_hc_supported.argtypes = [ip, ip, ip]
        lib.mpps_assemble_blocks_hc_n.argtypes = [vp, mp, ip, ip, P(ctypes.c_double), mp, ip, vp]
        lib.mpps_assemble_hc_n_supported.argtypes = [ip, ip, ip, ip]
        lib.mpps_one_norm.argtypes = [vp, mp, vp]
        lib.mpps_one_norm_complex.argtypes = [vp, mp, ip, vp, ip]
        lib.mpps_level_exps.argtypes = [vp, vp, ip, ip, ctypes.c_ulonglong, vp, vp]
        lib.mpps_store_host.argtypes = [vp, vp, vp, ctypes.c_longlong]
        lib.mpps_horner_step.argtypes = [vp, mp, mp, mp, mp, vp, ip, vp, vp, vp]
        lib.mpps_horner_scalar_top.argtypes = [vp, P(ctypes.c_double), ip, mp, mp, mp, vp, ip, vp]
        lib.mpps_probe_fma.argtypes = [vp, ip, ip, ip, vp]
        lib.mpps_assemble_blocks_dist.argtypes = [vp, mp, ip, ip, vp, mp, vp, ip, ip]
        lib.mpps_colmax.argtypes = [vp, vp, ip, ip, ip, vp]
        sp = P(CSlices)
        lib.mpps_slice.argtypes = [vp, mp, ip, sp, vp, ip]
        lib.mpps_slice_into.argtypes = [vp, mp, sp, ip, vp, ip]
        lib.mpps_slice_ex.argtypes = [vp, mp, ip, sp, vp, ip, ip]
        lib.mpps_gemm_sliced.argtypes = [vp, sp, sp, ip, ip, ip, ip, mp, vp, ip]
        lib.mpps_horner_step_sliced.argtypes = [vp, sp, sp, ip, mp, mp, vp, ip, vp, vp, vp]
        lib.mpps_oz_slices_for.argtypes = [ip]
        lib.mpps_oz_slices_for_bits.argtypes = [ip, ip]
        lib.mpps_oz_max_k_8bit.argtypes = []
        lib.mpps_oz_max_k.argtypes = [ip, ip]
        lib.mpps_probe_i8mma.argtypes = [vp, ip, ip, vp]
        lib.mpps_debug_oz_trace.argtypes = [vp]
        lib.mpps_debug_oz_trace.restype = None
        lib.mpps_debug_oz_flags.argtypes = [ip]
        lib.mpps_debug_oz_flags.restype = None
        lib.mpps_debug_probe_i8mma_n.argtypes = [vp, ip, ip, ip, vp]
        lib.mpps_probe_ingest.argtypes = [vp, ip, ip, vp, ctypes.c_longlong]
        lib.mpps_small_ps_supported.argtypes = [ip, ip, ip]
        lib.mpps_small_ps_prepare.argtypes = [vp, mp, ip, ip, P(ctypes.c_double), vp, vp, vp]
        lib.mpps_small_ps_horner.argtypes = [vp, vp, vp, vp, ip, ip, ctypes.c_double, mp]
        lib.mpps_small_ps_eval.argtypes = [vp, mp, ip, ip, vp, ip, ctypes.c_double, ip, ip, vp, vp, vp, vp, vp, vp, mp]
        for name in EXPORTED:
            getattr(lib, name).restype = getattr(lib, name).restype or ip
        if path is None:
            _lib = lib
        return lib


def cmat(m: MatBatch) -> CMat:
    d = m.data
    st = d.stride()
    return CMat(d.data_ptr(), st[0], st[1], m.rows, m.cols, st[2], m.batch, m.fmt)


def cmat_array(ms):
    arr = (CMat * len(ms))()
    for i, m in enumerate(ms):
        arr[i] = cmat(m)
    return arr


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Handle:
    """One C handle per (device, stream).  Not thread-safe (like the ABI)."""

    def __init__(self, device: int, stream_ptr: int):
        self.lib = load_library()
        h = ctypes.c_void_p()
        rc = self.lib.mpps_create(device, ctypes.c_void_p(stream_ptr), ctypes.byref(h))
        if rc != MPPS_OK:
            raise MppsCudaError(f"mpps_create failed on device {device} (rc={rc})")
        self.h = h
        self.device = device
        self.stream_ptr = stream_ptr
        self._pins = {}           # pinned host buffers of host_array, by size
        # optional per-launch CUDA-event probe (bench.py): key -> [(start, end)]
        self.probe = None

    def _ev(self, key):
        if self.probe is None:
            return None
        import torch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self.probe.setdefault(key, []).append((a, b))
        return b

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.mpps_destroy(self.h)
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(self.lib.mpps_launch_count(self.h))

    def _check(self, rc: int, what: str):
        if rc == MPPS_OK:
            return
        msg = self.lib.mpps_last_error(self.h).decode(errors="replace")
        if rc == MPPS_EINVAL:
            shape_words = ("mat_mul", "mat_axpy", "shape", "operands must be", "batch mismatch",
                           "must match", "must share")
            if any(w in msg for w in shape_words):
                raise DimensionError(f"{what}: {msg}")
            raise ValueError(f"{what}: {msg}")
        if rc == MPPS_EFMT:
            raise UnsupportedPrecisionError(f"{what}: {msg}")
        raise MppsCudaError(f"{what}: {msg}")

    # --- operator seam -------------------------------------------------
    def convert(self, src: MatBatch, dst: MatBatch, sel=None, exp=None):
        c_src, c_dst = cmat(src), cmat(dst)
        nsel = 0 if sel is None else sel.numel()
        self._check(self.lib.mpps_convert(self.h, ctypes.byref(c_src), ctypes.byref(c_dst),
                                          _ptr(sel), nsel, _ptr(exp)), "convert")

    def gemm(self, A: MatBatch, B: MatBatch, C: MatBatch, sel=None):
        a, b, c = cmat(A), cmat(B), cmat(C)
        nsel = 0 if sel is None else sel.numel()
        end = self._ev(("gemm", A.fmt, C.fmt, A.rows, B.cols, A.cols, nsel or C.batch, 0, 0))
        self._check(self.lib.mpps_gemm(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                       _ptr(sel), nsel), "mat_mul")
        if end is not None:
            end.record()

    def axpy(self, alpha_words, A: MatBatch, B: MatBatch, C: MatBatch):
        al = (ctypes.c_double * 4)(*[float(x) for x in alpha_words])
        a, b, c = cmat(A), cmat(B), cmat(C)
        self._check(self.lib.mpps_axpy(self.h, al, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
                    "mat_axpy")

    def powers(self, powers):
        arr = cmat_array(powers)
        self._check(self.lib.mpps_powers(self.h, arr, len(powers)), "powers")

    def assemble_blocks(self, powers, m: int, coeff_dev, blocks, norms_dev):
        parr, barr = cmat_array(powers), cmat_array(blocks)
        self._check(self.lib.mpps_assemble_blocks(self.h, parr, len(powers), m, coeff_dev.data_ptr(),
                                                  barr, norms_dev.data_ptr()), "assemble_blocks")

    def assemble_hc_supported(self, fmt: int, s: int, m: int) -> bool:
        return bool(self.lib.mpps_assemble_hc_supported(fmt, s, m))

    def assemble_blocks_hc(self, powers, m: int, coeff_words, blocks, norms_dev, skip_top: bool = False):
        """Block assembly with host coefficient words ((m+1, 4) float64) in
        the kernel parameters; skip_top leaves B_r = b_m I unstored."""
        parr = cmat_array(powers)
        barr = cmat_array(blocks)
        cw = np.ascontiguousarray(coeff_words, dtype=np.float64)
        self._check(self.lib.mpps_assemble_blocks_hc(self.h, parr, len(powers), m,
                                                     cw.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), barr,
                                                     norms_dev.data_ptr(), 1 if skip_top else 0),
                    "assemble_blocks")

    def assemble_hc_n_supported(self, block_fmt: int, s: int, m: int, nblocks: int) -> bool:
        return bool(self.lib.mpps_assemble_hc_n_supported(block_fmt, s, m, nblocks))

    def assemble_blocks_hc_n(self, powers, m: int, coeff_words, blocks, norms_dev=None):
        """Blocks B_0..B_{len(blocks)-1} at the blocks' format (fp64 from the
        high words of dd powers, or dd); norms_dev (B, len(blocks)+1) or None."""
        parr = cmat_array(powers)
        barr = cmat_array(blocks)
        cw = np.ascontiguousarray(coeff_words, dtype=np.float64)
        self._check(self.lib.mpps_assemble_blocks_hc_n(self.h, parr, len(powers), m,
                                                       cw.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), barr,
                                                       len(blocks), None if norms_dev is None else norms_dev.data_ptr()),
                    "assemble_blocks")

    def assemble_blocks_dist(self, powers, m: int, coeff_dev, blocks, colsums_dev, row0: int, col0: int):
        parr, barr = cmat_array(powers), cmat_array(blocks)
        self._check(self.lib.mpps_assemble_blocks_dist(self.h, parr, len(powers), m, coeff_dev.data_ptr(),
                                                       barr, colsums_dev.data_ptr(), row0, col0),
                    "assemble_blocks_dist")

    def colmax(self, colsums_dev, nvec: int, cols: int, batch: int, out_dev):
        self._check(self.lib.mpps_colmax(self.h, colsums_dev.data_ptr(), nvec, cols, batch, out_dev.data_ptr()),
                    "colmax")

    # --- tensor-core path -------------------------------------------
    def slices_for(self, fmt: int, db: int = 7) -> int:
        return int(self.lib.mpps_oz_slices_for_bits(fmt, db))

    def max_k_8bit(self) -> int:
        return int(self.lib.mpps_oz_max_k_8bit())

    def max_k(self, fmt: int, db: int) -> int:
        """Largest exact K for fmt's full plane count at db-bit digits."""
        return int(self.lib.mpps_oz_max_k(int(fmt), int(db)))

    def slice(self, src: MatBatch, side: int, S: int, sel=None, db: int = 7) -> "Slices":
        """side 0: split rows (left operand); side 1: split columns (right);
        db: digit bits (7 or 8)."""
        rows, k = (src.rows, src.cols) if side == 0 else (src.cols, src.rows)
        out = Slices(S, src.batch, rows, k, src.device, db)
        c_src, c_out = cmat(src), out.c()
        nsel = 0 if sel is None else sel.numel()
        self._check(self.lib.mpps_slice(self.h, ctypes.byref(c_src), side, ctypes.byref(c_out), _ptr(sel), nsel),
                    "slice")
        return out

    def slice_ex(self, src: MatBatch, side: int, out: "Slices", mode: int, sel=None):
        """mode 1: only out.exps (row / column scales); mode 2: split with
        the scales already in out.exps (include/mpps_b200.h)."""
        c_src, c_out = cmat(src), out.c()
        nsel = 0 if sel is None else sel.numel()
        self._check(self.lib.mpps_slice_ex(self.h, ctypes.byref(c_src), side, ctypes.byref(c_out), _ptr(sel), nsel,
                                           int(mode)), "slice_ex")

    def slice_into(self, src: MatBatch, out: "Slices", row0: int, sel=None):
        """Column split of src into slice rows [row0, row0 + src.cols) of out."""
        c_src, c_out = cmat(src), out.c()
        nsel = 0 if sel is None else sel.numel()
        self._check(self.lib.mpps_slice_into(self.h, ctypes.byref(c_src), ctypes.byref(c_out), int(row0), _ptr(sel),
                                             nsel), "slice_into")

    def gemm_sliced(self, A: "Slices", B: "Slices", S: int, C: MatBatch, sel=None):
        a, b, c = A.c(), B.c(), cmat(C)
        nsel = 0 if sel is None else sel.numel()
        # the probe key and the launch both take N from C: B may hold more
        # column slices than this product uses (the power chain's [X | X^2]
        # operand feeds the N = n launch of X^2 and the N = 2n paired ones)
        end = self._ev(("gemm_tc", C.fmt, C.fmt, A.rows, C.cols, A.k, nsel or C.batch, S, A.db))
        self._check(self.lib.mpps_gemm_sliced(self.h, ctypes.byref(a), ctypes.byref(b), S, A.rows, C.cols, A.k,
                                              ctypes.byref(c), _ptr(sel), nsel), "mat_mul(tc)")
        if end is not None:
            end.record()

    def horner_step_sliced(self, Y: "Slices", phi: "Slices", S: int, Bprev, out, sel=None, exp_y=None,
                           exp_in=None, exp_out=None, fmt_in: int = 31):
        y, p, b, o = Y.c(), phi.c(), cmat(Bprev), cmat(out)
        nsel = 0 if sel is None else sel.numel()
        end = self._ev(("horner_tc", fmt_in, out.fmt, Y.rows, phi.rows, Y.k, nsel or out.batch, S, Y.db))
        self._check(self.lib.mpps_horner_step_sliced(self.h, ctypes.byref(y), ctypes.byref(p), S, ctypes.byref(b),
                                                     ctypes.byref(o), _ptr(sel), nsel, _ptr(exp_y), _ptr(exp_in),
                                                     _ptr(exp_out)), "horner_step(tc)")
        if end is not None:
            end.record()

    def one_norm_complex(self, A: MatBatch, nc: int, norms_dev, stride: int = 1):
        """Complex one_norm of the 2nc x 2nc real embeddings in A into
        norms_dev[b * stride] (norms_dev: a float64 device tensor view whose
        first element receives batch member 0)."""
        a = cmat(A)
        self._check(self.lib.mpps_one_norm_complex(self.h, ctypes.byref(a), int(nc), norms_dev.data_ptr(), int(stride)),
                    "one_norm_complex")

    def level_exps(self, norms_dev, r: int, fp32_mask: int, exps_dev, exp_y_dev):
        """norms_dev (B, r+2) float64 -> exps_dev (r+2, B), exp_y_dev (B,) int32."""
        self._check(self.lib.mpps_level_exps(self.h, norms_dev.data_ptr(), int(norms_dev.shape[0]), int(r),
                                             int(fp32_mask), exps_dev.data_ptr(), exp_y_dev.data_ptr()),
                    "level_exps")

    def store_host(self, src_dev, dst_pinned):
        """float64 device tensor -> pinned host tensor of the same size, stored by a kernel (no copy
        engine: a memcpy would queue behind a running result download)."""
        if not dst_pinned.is_pinned() or dst_pinned.numel() != src_dev.numel() or not src_dev.is_contiguous():
            raise ValueError("store_host: pinned destination of the source's size, contiguous source")
        self._check(self.lib.mpps_store_host(self.h, src_dev.data_ptr(), dst_pinned.data_ptr(), src_dev.numel()),
                    "store_host")

    def host_array(self, src_dev) -> "np.ndarray":
        """A small float64 device tensor as a numpy array: stored into pinned memory by a kernel
        (store_host), then one stream synchronisation -- the planner's norms never wait for the
        device-to-host copy engine."""
        import torch
        src = src_dev.contiguous()
        pin = self._pins.get(src.numel())
        if pin is None:
            pin = self._pins[src.numel()] = torch.empty(src.numel(), dtype=torch.float64, pin_memory=True)
        self.store_host(src, pin)
        torch.cuda.current_stream(src.device).synchronize()
        return pin.numpy().reshape(tuple(src.shape)).copy()

    def one_norm(self, A: MatBatch, norms_dev):
        a = cmat(A)
        self._check(self.lib.mpps_one_norm(self.h, ctypes.byref(a), norms_dev.data_ptr()), "one_norm")

    def horner_step(self, Y, phi, Bprev, out, sel=None, exp_y=None, exp_in=None, exp_out=None):
        y, p, b, o = cmat(Y), cmat(phi), cmat(Bprev), cmat(out)
        nsel = 0 if sel is None else sel.numel()
        end = self._ev(("horner", Y.fmt, out.fmt, Y.rows, Y.rows, Y.rows, nsel or out.batch, 0, 0))
        self._check(self.lib.mpps_horner_step(self.h, ctypes.byref(y), ctypes.byref(p), ctypes.byref(b),
                                              ctypes.byref(o), _ptr(sel), nsel, _ptr(exp_y), _ptr(exp_in),
                                              _ptr(exp_out)), "horner_step")
        if end is not None:
            end.record()

    def horner_scalar_top(self, bm_words, fmt_top: int, Y, Bprev, out, sel=None, exp_out=None):
        bm = (ctypes.c_double * 4)(*[float(x) for x in bm_words])
        y, b, o = cmat(Y), cmat(Bprev), cmat(out)
        nsel = 0 if sel is None else sel.numel()
        self._check(self.lib.mpps_horner_scalar_top(self.h, bm, fmt_top, ctypes.byref(y), ctypes.byref(b),
                                                    ctypes.byref(o), _ptr(sel), nsel, _ptr(exp_out)),
                    "horner_scalar_top")


    # --- K5: small matrices ------------------------------------------
    def small_ps_supported(self, n: int, m: int, fmt: int) -> bool:
        return bool(self.lib.mpps_small_ps_supported(int(n), int(m), int(fmt)))

    def small_ps_prepare(self, X: MatBatch, m: int, s: int, coeff, blocks, Y, norms):
        """X fp64 (1, B, n, n); coeff (m+1,) float64 host; blocks / Y / norms
        device float64 tensors (see include/mpps_b200.h)."""
        c = np.ascontiguousarray(coeff, dtype=np.float64)
        x = cmat(X)
        self._check(self.lib.mpps_small_ps_prepare(self.h, ctypes.byref(x), int(m), int(s),
                                                   c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                   blocks.data_ptr(), Y.data_ptr(), norms.data_ptr()), "small_ps")

    def small_ps_horner(self, Y, blocks, level_fmt: np.ndarray, m: int, s: int, bm: float, out: MatBatch):
        """level_fmt: host (B, r+1) int8 numpy array (0 fp32, 1 fp64)."""
        o = cmat(out)
        f = np.ascontiguousarray(level_fmt, dtype=np.int8)
        self._check(self.lib.mpps_small_ps_horner(self.h, Y.data_ptr(), blocks.data_ptr(), f.ctypes.data,
                                                  int(m), int(s), float(bm), ctypes.byref(o)), "small_ps")

    def small_ps_eval(self, X: MatBatch, m: int, s: int, coeff: np.ndarray, d: int, delta: float,
                      apply_switch: bool, fixed: bool, blocks, Y, norms_dev, out: MatBatch):
        """One call: prepare, host norms, certified digit rule, Horner.
        Returns (norms (B, r+2), digits (B, r), nu (B,), planned): planned is
        False when the certified rule declined (the caller plans exactly and
        runs small_ps_horner)."""
        B, r = X.batch, m // s
        norms = np.empty((B, r + 2), dtype=np.float64)
        digits = np.empty((B, max(r, 1)), dtype=np.int32)
        nu = np.empty(B, dtype=np.int32)
        x, o = cmat(X), cmat(out)
        rc = self.lib.mpps_small_ps_eval(self.h, ctypes.byref(x), int(m), int(s), coeff.ctypes.data, int(d),
                                         float(delta), int(bool(apply_switch)), int(bool(fixed)), blocks.data_ptr(),
                                         Y.data_ptr(), norms_dev.data_ptr(), norms.ctypes.data, digits.ctypes.data,
                                         nu.ctypes.data, ctypes.byref(o))
        if rc == 4:
            return norms, None, None, False
        self._check(rc, "small_ps")
        return norms, digits[:, :r], nu, True

    def probe_ingest(self, blocks: int, iters: int, src):
        self._check(self.lib.mpps_probe_ingest(self.h, blocks, iters, src.data_ptr(), src.numel() * src.element_size()),
                    "probe_ingest")

    def probe_i8mma(self, blocks: int, iters: int, scratch):
        self._check(self.lib.mpps_probe_i8mma(self.h, blocks, iters, scratch.data_ptr()), "probe_i8mma")

    def probe_fma(self, fmt: int, blocks: int, iters: int, scratch):
        self._check(self.lib.mpps_probe_fma(self.h, fmt, blocks, iters, scratch.data_ptr()), "probe_fma")


_handles = {}
_cuda_ok = False


def handle_for(device=None) -> Handle:
    """The handle bound to torch's current stream on ``device``."""
    import torch
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise MppsCudaError("no CUDA device: the B200 path has no CPU fallback")
        _cuda_ok = True
    dev = torch.cuda.current_device() if device is None else (
        device.index if hasattr(device, "index") and device.index is not None else int(device)
        if not hasattr(device, "type") else torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (dev, stream, threading.get_ident())
    h = _handles.get(key)
    if h is None:
        h = Handle(dev, stream)
        _handles[key] = h
    return h


def total_launches() -> int:
    return sum(h.launches for h in _handles.values())
