"""TEST INFRASTRUCTURE ONLY: a ctypes stand-in for the parts of gmpy2 the
reference package uses, so the UNMODIFIED reference (/root/reference/pkg)
can be imported and run in the build container (gmpy2 itself is not
installed and there is no network).

Every arithmetic operation calls the same MPFR 4.2.1 / MPC 1.3.1 functions
gmpy2 wraps (round-to-nearest), on the same precisions, so results are
bit-identical to the real gmpy2 for the reference's call sites
(SURVEY.md 8c lists them).  Semantics reproduced:

* ``mpfr(x[, prec])`` -- prec omitted -> the global context precision (53);
* ``context(precision=p, allow_complex=True)`` methods round at p; ops on
  ``mpc`` operands return ``mpc`` (MPC_RNDNN), ``abs(mpc)`` returns the
  modulus as ``mpfr``; ``div(mpz, mpz)`` is the correctly rounded quotient;
* Python operators on ``mpfr`` use the global context (53 bits);
  comparisons are exact.

Used only by oracle/make_golden.py and the reference-validation script;
never imported by the product or by tests that run on the GPU box.
"""

from __future__ import annotations

import ctypes
import math
from fractions import Fraction

_mpfr = ctypes.CDLL("libmpfr.so.6")
_mpc = ctypes.CDLL("libmpc.so.3")


class _FR(ctypes.Structure):
    _fields_ = [("prec", ctypes.c_long), ("sign", ctypes.c_int),
                ("exp", ctypes.c_long), ("d", ctypes.c_void_p)]


class _C(ctypes.Structure):
    _fields_ = [("re", _FR), ("im", _FR)]


_P = ctypes.POINTER
_fr = _P(_FR)
_c = _P(_C)
for name, args, res in [
    ("mpfr_init2", [_fr, ctypes.c_long], None), ("mpfr_clear", [_fr], None),
    ("mpfr_set", [_fr, _fr, ctypes.c_int], ctypes.c_int),
    ("mpfr_set_d", [_fr, ctypes.c_double, ctypes.c_int], ctypes.c_int),
    ("mpfr_set_str", [_fr, ctypes.c_char_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    ("mpfr_get_d", [_fr, ctypes.c_int], ctypes.c_double),
    ("mpfr_get_str", [ctypes.c_char_p, _P(ctypes.c_long), ctypes.c_int, ctypes.c_size_t, _fr, ctypes.c_int],
     ctypes.c_void_p),
    ("mpfr_free_str", [ctypes.c_void_p], None),
    ("mpfr_cmp", [_fr, _fr], ctypes.c_int),
    ("mpfr_nan_p", [_fr], ctypes.c_int), ("mpfr_inf_p", [_fr], ctypes.c_int),
    ("mpfr_zero_p", [_fr], ctypes.c_int), ("mpfr_sgn", [_fr], ctypes.c_int),
    ("mpfr_get_prec", [_fr], ctypes.c_long),
    ("mpfr_ceil", [_fr, _fr], ctypes.c_int),
    ("mpfr_div_2si", [_fr, _fr, ctypes.c_long, ctypes.c_int], ctypes.c_int),
    ("mpfr_rootn_ui", [_fr, _fr, ctypes.c_ulong, ctypes.c_int], ctypes.c_int),
    ("mpfr_const_pi", [_fr, ctypes.c_int], ctypes.c_int),
]:
    f = getattr(_mpfr, name)
    f.argtypes = args
    f.restype = res
for name in ("mpfr_add", "mpfr_sub", "mpfr_mul", "mpfr_div"):
    f = getattr(_mpfr, name)
    f.argtypes = [_fr, _fr, _fr, ctypes.c_int]
    f.restype = ctypes.c_int
for name in ("mpfr_abs", "mpfr_neg", "mpfr_log10", "mpfr_exp10", "mpfr_exp", "mpfr_log", "mpfr_log2",
             "mpfr_cos", "mpfr_sin", "mpfr_sqrt"):
    f = getattr(_mpfr, name)
    f.argtypes = [_fr, _fr, ctypes.c_int]
    f.restype = ctypes.c_int
for name, args in [("mpc_init2", [_c, ctypes.c_long]), ("mpc_clear", [_c])]:
    getattr(_mpc, name).argtypes = args
    getattr(_mpc, name).restype = None
for name in ("mpc_add", "mpc_sub", "mpc_mul", "mpc_div"):
    getattr(_mpc, name).argtypes = [_c, _c, _c, ctypes.c_int]
    getattr(_mpc, name).restype = ctypes.c_int
_mpc.mpc_set.argtypes = [_c, _c, ctypes.c_int]
_mpc.mpc_set_fr_fr.argtypes = [_c, _fr, _fr, ctypes.c_int]
_mpc.mpc_abs.argtypes = [_fr, _c, ctypes.c_int]
_mpc.mpc_neg.argtypes = [_c, _c, ctypes.c_int]
for f in (_mpc.mpc_set, _mpc.mpc_set_fr_fr, _mpc.mpc_abs, _mpc.mpc_neg):
    f.restype = ctypes.c_int

RNDN = 0
_DEFAULT_PREC = 53


class mpz(int):
    """gmpy2.mpz stand-in (a Python int)."""


# ------------------------------------------------------------------ mpfr
class mpfr:
    __slots__ = ("_s", "__weakref__")

    def __new__(cls, x=0, precision=0, context=None):
        # gmpy2: precision 0 -> context precision (53); 1 -> keep an mpfr's own
        if precision == 1 and isinstance(x, mpfr):
            return x
        prec = precision if precision > 1 else _DEFAULT_PREC
        self = object.__new__(cls)
        self._s = _FR()
        _mpfr.mpfr_init2(ctypes.byref(self._s), prec)
        _set_real(self._s, x)
        return self

    @classmethod
    def _raw(cls, prec):
        self = object.__new__(cls)
        self._s = _FR()
        _mpfr.mpfr_init2(ctypes.byref(self._s), prec)
        return self

    def __del__(self):
        try:
            _mpfr.mpfr_clear(ctypes.byref(self._s))
        except Exception:
            pass

    @property
    def precision(self):
        return _mpfr.mpfr_get_prec(ctypes.byref(self._s))

    @property
    def real(self):
        return self

    @property
    def imag(self):
        return mpfr(0, self.precision)

    def __float__(self):
        return _mpfr.mpfr_get_d(ctypes.byref(self._s), RNDN)

    def __int__(self):
        if _mpfr.mpfr_nan_p(ctypes.byref(self._s)) or _mpfr.mpfr_inf_p(ctypes.byref(self._s)):
            raise ValueError("cannot convert non-finite mpfr to int")
        return int(self._fraction())

    def _fraction(self) -> Fraction:
        if _mpfr.mpfr_zero_p(ctypes.byref(self._s)):
            return Fraction(0)
        ds, e, _ = self.digits(16, 0)
        neg = ds.startswith("-")
        ds = ds.lstrip("-")
        v = Fraction(int(ds, 16), 16 ** len(ds)) * Fraction(16) ** e
        return -v if neg else v

    def as_integer_ratio(self):
        f = self._fraction()
        return f.numerator, f.denominator

    def digits(self, base=10, prec=0):
        e = ctypes.c_long()
        p = _mpfr.mpfr_get_str(None, ctypes.byref(e), base, prec, ctypes.byref(self._s), RNDN)
        s = ctypes.string_at(p).decode()
        _mpfr.mpfr_free_str(p)
        return s, e.value, self.precision

    def is_nan(self):
        return bool(_mpfr.mpfr_nan_p(ctypes.byref(self._s)))

    # exact comparisons
    def _cmp(self, other):
        o = _as_mpfr_exact(other)
        if o is None:
            return NotImplemented
        if self.is_nan() or o.is_nan():
            return None
        return _mpfr.mpfr_cmp(ctypes.byref(self._s), ctypes.byref(o._s))

    def __eq__(self, other):
        if isinstance(other, mpc):
            return other == self
        c = self._cmp(other)
        return NotImplemented if c is NotImplemented else (c == 0 if c is not None else False)

    def __ne__(self, other):
        r = self.__eq__(other)
        return r if r is NotImplemented else not r

    def __lt__(self, other):
        c = self._cmp(other)
        return c if c is NotImplemented else (c is not None and c < 0)

    def __le__(self, other):
        c = self._cmp(other)
        return c if c is NotImplemented else (c is not None and c <= 0)

    def __gt__(self, other):
        c = self._cmp(other)
        return c if c is NotImplemented else (c is not None and c > 0)

    def __ge__(self, other):
        c = self._cmp(other)
        return c if c is NotImplemented else (c is not None and c >= 0)

    def __hash__(self):
        return hash(float(self))

    def __bool__(self):
        return not _mpfr.mpfr_zero_p(ctypes.byref(self._s))

    # arithmetic at the global context (53 bits)
    def _bin(self, other, fn, swap=False):
        if isinstance(other, mpc):
            return NotImplemented
        o = _as_mpfr_exact(other)
        if o is None:
            return NotImplemented
        a, b = (o, self) if swap else (self, o)
        r = mpfr._raw(_DEFAULT_PREC)
        fn(ctypes.byref(r._s), ctypes.byref(a._s), ctypes.byref(b._s), RNDN)
        return r

    def __add__(self, o): return self._bin(o, _mpfr.mpfr_add)
    def __radd__(self, o): return self._bin(o, _mpfr.mpfr_add, True)
    def __sub__(self, o): return self._bin(o, _mpfr.mpfr_sub)
    def __rsub__(self, o): return self._bin(o, _mpfr.mpfr_sub, True)
    def __mul__(self, o): return self._bin(o, _mpfr.mpfr_mul)
    def __rmul__(self, o): return self._bin(o, _mpfr.mpfr_mul, True)
    def __truediv__(self, o): return self._bin(o, _mpfr.mpfr_div)
    def __rtruediv__(self, o): return self._bin(o, _mpfr.mpfr_div, True)

    def __neg__(self):
        r = mpfr._raw(self.precision)
        _mpfr.mpfr_neg(ctypes.byref(r._s), ctypes.byref(self._s), RNDN)
        return r

    def __abs__(self):
        r = mpfr._raw(self.precision)
        _mpfr.mpfr_abs(ctypes.byref(r._s), ctypes.byref(self._s), RNDN)
        return r

    def __repr__(self):
        return f"mpfr('{self.digits(10, 0)[0]}e{self.digits(10, 0)[1]}',{self.precision})"

    def __str__(self):
        return repr(float(self))

    def __format__(self, spec):
        return format(float(self), spec)


def _set_real(s: _FR, x):
    """Set an initialised MPFR struct from a Python/gmpy2 value (RN)."""
    if isinstance(x, mpfr):
        _mpfr.mpfr_set(ctypes.byref(s), ctypes.byref(x._s), RNDN)
    elif isinstance(x, bool):
        _mpfr.mpfr_set_d(ctypes.byref(s), float(x), RNDN)
    elif isinstance(x, int):
        _mpfr.mpfr_set_str(ctypes.byref(s), str(int(x)).encode(), 10, RNDN)
    elif isinstance(x, float):
        _mpfr.mpfr_set_d(ctypes.byref(s), x, RNDN)
    elif isinstance(x, str):
        t = x.strip().lower()
        if t in ("inf", "+inf"):
            t = "@inf@"
        elif t == "-inf":
            t = "-@inf@"
        elif t == "nan":
            t = "@nan@"
        if _mpfr.mpfr_set_str(ctypes.byref(s), t.encode(), 10, RNDN) != 0 and "@" not in t:
            # mpfr_set_str returns 0 on success; a nonzero return means the
            # string was not fully parsed
            raise ValueError(f"invalid mpfr string {x!r}")
    elif isinstance(x, Fraction):
        num, den = _exact(x.numerator), _exact(x.denominator)
        _mpfr.mpfr_div(ctypes.byref(s), ctypes.byref(num._s), ctypes.byref(den._s), RNDN)
    else:
        raise TypeError(f"cannot convert {type(x).__name__} to mpfr")


def _exact(n: int) -> mpfr:
    r = mpfr._raw(max(2, abs(int(n)).bit_length() + 1))
    _mpfr.mpfr_set_str(ctypes.byref(r._s), str(int(n)).encode(), 10, RNDN)
    return r


def _as_mpfr_exact(x):
    """Exact mpfr for comparisons / mixed arithmetic, None if unsupported."""
    if isinstance(x, mpfr):
        return x
    if isinstance(x, bool):
        return _exact(int(x))
    if isinstance(x, int):
        return _exact(x)
    if isinstance(x, float):
        r = mpfr._raw(64)
        _mpfr.mpfr_set_d(ctypes.byref(r._s), x, RNDN)
        return r
    if isinstance(x, Fraction):
        return None
    return None


# ------------------------------------------------------------------- mpc
class mpc:
    __slots__ = ("_s", "__weakref__")

    def __new__(cls, re=0, im=None, precision=0, context=None):
        prec = precision or _DEFAULT_PREC
        self = object.__new__(cls)
        self._s = _C()
        _mpc.mpc_init2(ctypes.byref(self._s), prec)
        if im is None and isinstance(re, mpc):
            _mpc.mpc_set(ctypes.byref(self._s), ctypes.byref(re._s), RNDN)
            return self
        if im is None and isinstance(re, complex):
            re, im = re.real, re.imag
        _set_real(self._s.re, re if not isinstance(re, mpc) else re.real)
        _set_real(self._s.im, 0 if im is None else im)
        return self

    @classmethod
    def _raw(cls, prec):
        self = object.__new__(cls)
        self._s = _C()
        _mpc.mpc_init2(ctypes.byref(self._s), prec)
        return self

    def __del__(self):
        try:
            _mpc.mpc_clear(ctypes.byref(self._s))
        except Exception:
            pass

    @property
    def real(self):
        r = mpfr._raw(self._s.re.prec)
        _mpfr.mpfr_set(ctypes.byref(r._s), ctypes.byref(self._s.re), RNDN)
        return r

    @property
    def imag(self):
        r = mpfr._raw(self._s.im.prec)
        _mpfr.mpfr_set(ctypes.byref(r._s), ctypes.byref(self._s.im), RNDN)
        return r

    @property
    def precision(self):
        return (self._s.re.prec, self._s.im.prec)

    def __eq__(self, other):
        if isinstance(other, mpc):
            return (_mpfr.mpfr_cmp(ctypes.byref(self._s.re), ctypes.byref(other._s.re)) == 0 and
                    _mpfr.mpfr_cmp(ctypes.byref(self._s.im), ctypes.byref(other._s.im)) == 0)
        o = _as_mpfr_exact(other)
        if o is None:
            return NotImplemented
        return (_mpfr.mpfr_cmp(ctypes.byref(self._s.re), ctypes.byref(o._s)) == 0 and
                _mpfr.mpfr_zero_p(ctypes.byref(self._s.im)) != 0)

    def __ne__(self, other):
        r = self.__eq__(other)
        return r if r is NotImplemented else not r

    def __hash__(self):
        return hash((float(self.real), float(self.imag)))

    def __complex__(self):
        return complex(float(self.real), float(self.imag))

    def __repr__(self):
        return f"mpc({complex(self)!r})"


def _to_mpc(x, prec):
    if isinstance(x, mpc):
        return x
    return mpc(x, precision=max(prec, _prec_of(x)))


def _prec_of(x):
    if isinstance(x, mpfr):
        return x.precision
    if isinstance(x, int):
        return max(2, abs(int(x)).bit_length() + 1)
    return 64


# --------------------------------------------------------------- context
class context:
    def __init__(self, precision=53, allow_complex=False, **kw):
        self.precision = int(precision)
        self.allow_complex = allow_complex

    def _num(self, x):
        if isinstance(x, (mpfr, mpc)):
            return x
        if isinstance(x, (int, float)):
            return _as_mpfr_exact(x)
        if isinstance(x, Fraction):
            return mpfr(x, 256)
        raise TypeError(type(x))

    def _bin(self, a, b, rfn, cfn):
        a, b = self._num(a), self._num(b)
        if isinstance(a, mpc) or isinstance(b, mpc):
            a, b = _to_mpc(a, self.precision), _to_mpc(b, self.precision)
            r = mpc._raw(self.precision)
            cfn(ctypes.byref(r._s), ctypes.byref(a._s), ctypes.byref(b._s), RNDN)
            return r
        r = mpfr._raw(self.precision)
        rfn(ctypes.byref(r._s), ctypes.byref(a._s), ctypes.byref(b._s), RNDN)
        return r

    def add(self, a, b): return self._bin(a, b, _mpfr.mpfr_add, _mpc.mpc_add)
    def sub(self, a, b): return self._bin(a, b, _mpfr.mpfr_sub, _mpc.mpc_sub)
    def mul(self, a, b): return self._bin(a, b, _mpfr.mpfr_mul, _mpc.mpc_mul)

    def div(self, a, b):
        if isinstance(a, int) and isinstance(b, int) and not isinstance(a, bool):
            r = mpfr._raw(self.precision)
            ea, eb = _exact(a), _exact(b)   # keep the owners alive across the call
            _mpfr.mpfr_div(ctypes.byref(r._s), ctypes.byref(ea._s), ctypes.byref(eb._s), RNDN)
            return r
        return self._bin(a, b, _mpfr.mpfr_div, _mpc.mpc_div)

    def _un(self, a, fn):
        a = self._num(a)
        if isinstance(a, mpc):
            raise NotImplementedError("complex transcendental not needed by the reference hot path")
        r = mpfr._raw(self.precision)
        fn(ctypes.byref(r._s), ctypes.byref(a._s), RNDN)
        return r

    def abs(self, a):
        a = self._num(a)
        r = mpfr._raw(self.precision)
        if isinstance(a, mpc):
            _mpc.mpc_abs(ctypes.byref(r._s), ctypes.byref(a._s), RNDN)
        else:
            _mpfr.mpfr_abs(ctypes.byref(r._s), ctypes.byref(a._s), RNDN)
        return r

    def log10(self, a): return self._un(a, _mpfr.mpfr_log10)
    def exp10(self, a): return self._un(a, _mpfr.mpfr_exp10)
    def exp(self, a): return self._un(a, _mpfr.mpfr_exp)
    def log(self, a): return self._un(a, _mpfr.mpfr_log)
    def log2(self, a): return self._un(a, _mpfr.mpfr_log2)
    def cos(self, a): return self._un(a, _mpfr.mpfr_cos)
    def sin(self, a): return self._un(a, _mpfr.mpfr_sin)
    def sqrt(self, a): return self._un(a, _mpfr.mpfr_sqrt)

    def root(self, a, n):
        a = self._num(a)
        r = mpfr._raw(self.precision)
        _mpfr.mpfr_rootn_ui(ctypes.byref(r._s), ctypes.byref(a._s), int(n), RNDN)
        return r

    def div_2exp(self, a, n):
        a = self._num(a)
        if isinstance(a, mpc):
            r = mpc._raw(self.precision)
            _mpfr.mpfr_div_2si(ctypes.byref(r._s.re), ctypes.byref(a._s.re), int(n), RNDN)
            _mpfr.mpfr_div_2si(ctypes.byref(r._s.im), ctypes.byref(a._s.im), int(n), RNDN)
            return r
        r = mpfr._raw(self.precision)
        _mpfr.mpfr_div_2si(ctypes.byref(r._s), ctypes.byref(a._s), int(n), RNDN)
        return r

    def const_pi(self):
        r = mpfr._raw(self.precision)
        _mpfr.mpfr_const_pi(ctypes.byref(r._s), RNDN)
        return r


def is_nan(x):
    return isinstance(x, mpfr) and x.is_nan()


def is_infinite(x):
    return isinstance(x, mpfr) and bool(_mpfr.mpfr_inf_p(ctypes.byref(x._s)))


def ceil(x):
    x = x if isinstance(x, mpfr) else mpfr(x)
    r = mpfr._raw(x.precision)
    _mpfr.mpfr_ceil(ctypes.byref(r._s), ctypes.byref(x._s))
    return r


def get_context():
    return context(_DEFAULT_PREC)


version = lambda: "2.1.5-shim"  # noqa: E731
