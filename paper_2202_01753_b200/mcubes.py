"""Host-side mirror of the reference's public API (proj/include/mcubes/*.hpp).

Same names, fields, defaults and error behaviour as the C++ reference, so the
parity tests read like the reference's own tests.  Every sampling iteration,
grid adaptation and the weighted combination inside ``integrate`` run in the
sm_100a kernels behind ``libmcubes_b200.so`` (``include/mcubes_b200.h``); this
module only marshals arguments.

Reference map (paths under /root/reference/proj/include/mcubes/):

=========================  ===========================================
``RunConfig``/``setup``    driver.hpp:37-123
``weighted_estimate``      driver.hpp:146-169
``check_convergence``      driver.hpp:173-178
``integrate``              driver.hpp:215-258
``v_sample``               sampler.hpp:312-333
``v_sample_no_adjust``     sampler.hpp:339-349
``NonFiniteSample``        sampler.hpp:31-48
``Grid``                   grid.hpp:27-176
``BinAccumulator``         accumulators.hpp:18-56
``make_*``/``reference``   integrands.hpp:23-235
=========================  ===========================================
"""
from __future__ import annotations

import cmath
import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, List, NamedTuple, Optional, Sequence

import numpy as np

from . import _lib as L

# ----------------------------------------------------------------- errors


class NonFiniteSample(RuntimeError):
    """f(x)*J was not finite (sampler.hpp:31-48).  The GPU reports the first
    failure in serial (cube, sample) order, i.e. what the serial oracle throws."""

    def __init__(self, message: str, point: Sequence[float], value: float):
        super().__init__(message)
        self._point = list(point)
        self._value = value

    def point(self):
        return self._point

    def value(self):
        return self._value


class CudaError(RuntimeError):
    pass


def _raise(rc: int, ctx_ptr=None, dims: int = 0):
    if rc == L.MCB_OK:
        return
    lib = L.lib()
    msg = lib.mcb_last_error(ctx_ptr).decode() if ctx_ptr else "invalid argument"
    if rc == L.MCB_EINVAL:
        raise ValueError(msg)
    if rc == L.MCB_ENONFINITE:
        x = (C.c_double * max(dims, 1))()
        fx = C.c_double()
        lib.mcb_last_nonfinite(ctx_ptr, x, dims, C.byref(fx))
        raise NonFiniteSample(msg, [x[i] for i in range(dims)], fx.value)
    if rc == L.MCB_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


# ----------------------------------------------------------------- context


class Context:
    """A CUDA device + stream + scratch (mcb_ctx).  One host thread at a time."""

    def __init__(self, device: int = 0):
        self._lib = L.lib()
        p = C.c_void_p()
        rc = self._lib.mcb_ctx_create(device, C.byref(p))
        if rc != L.MCB_OK:
            raise CudaError(f"mcb_ctx_create(device={device}) failed with status {rc}: no usable CUDA device")
        self.ptr = p
        self.device = device

    def close(self):
        if getattr(self, "ptr", None):
            self._lib.mcb_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, cuda_stream: int):
        """Run on a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        _raise(self._lib.mcb_ctx_set_stream(self.ptr, C.c_void_p(cuda_stream)), self.ptr)

    def synchronize(self):
        _raise(self._lib.mcb_ctx_synchronize(self.ptr), self.ptr)

    @property
    def launches(self) -> int:
        """Kernels launched through this context (our own sm_100a kernels)."""
        return int(self._lib.mcb_ctx_launches(self.ptr))


_tls = threading.local()


def default_context(device: Optional[int] = None) -> Context:
    if device is None:
        device = getattr(_tls, "device", 0)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def set_device(device: int):
    _tls.device = device


# ----------------------------------------------------------------- integrands


@dataclass
class IntegrandSpec:
    """A ready-to-integrate built-in function (integrands.hpp:23-32).

    The callable lives on the device: ``id`` selects the kernel functor and
    ``params`` carries its state (e.g. the interpolation tables)."""

    name: str
    dims: int
    lower: List[float]
    upper: List[float]
    id: int
    params: Optional[np.ndarray] = None
    reference: Optional[float] = None

    def _c(self):
        params = _f64(self.params) if self.params is not None else np.zeros(0)
        s = L.mcb_integrand(self.id, len(params), _dptr(params) if len(params) else None)
        return s, params  # keep params alive


def _phase_factor(a: float) -> complex:
    return (cmath.exp(1j * a) - 1.0) / (1j * a)


def reference_value(family: int, d: int) -> float:
    """Exact integral of suite family over [0,1]^d (integrands.hpp:53-103)."""
    if d < 1:
        raise ValueError("reference_value: d must be >= 1")
    if family == 1:
        prod = 1.0 + 0j
        for i in range(1, d + 1):
            prod *= _phase_factor(float(i))
        return prod.real
    if family == 2:
        return math.pow(100.0 * math.atan(25.0), float(d))
    if family == 3:
        s = 0.0
        for mask in range(1 << d):
            denom, bits = 1.0, 0
            for i in range(d):
                if mask & (1 << i):
                    denom += float(i + 1)
                    bits += 1
            s += (-1.0 if bits % 2 else 1.0) / denom
        fact = 1.0
        for i in range(1, d + 1):
            fact *= float(i) * float(i)
        return s / fact
    if family == 4:
        return math.pow(math.sqrt(math.pi) / 25.0 * math.erf(12.5), float(d))
    if family == 5:
        return math.pow((1.0 - math.exp(-5.0)) / 5.0, float(d))
    if family == 6:
        prod = 1.0
        for i in range(1, d + 1):
            c = float(i) + 4.0
            u = min(1.0, (3.0 + float(i)) / 10.0)
            prod *= (math.exp(c * u) - 1.0) / c
        return prod
    raise ValueError(f"reference_value: unknown family {family}")


def make_suite_integrand(family: int, d: int) -> IntegrandSpec:
    """Genz-style family f1..f6 on [0,1]^d (integrands.hpp:107-176)."""
    if family < 1 or family > 6:
        raise ValueError("make_suite_integrand: family must be in 1..6")
    if d < 1:
        raise ValueError("make_suite_integrand: d must be >= 1")
    return IntegrandSpec(f"f{family}", d, [0.0] * d, [1.0] * d, family, None, reference_value(family, d))


def make_fA() -> IntegrandSpec:
    """sin(sum x) over (0,10)^6 (integrands.hpp:181-196)."""
    axis = (cmath.exp(10j) - 1.0) / 1j
    return IntegrandSpec("fA", 6, [0.0] * 6, [10.0] * 6, 7, None, (axis ** 6).imag)


def make_fB() -> IntegrandSpec:
    """Normalized 9D Gaussian on (-1,1)^9 (integrands.hpp:200-215)."""
    return IntegrandSpec("fB", 9, [-1.0] * 9, [1.0] * 9, 8, None,
                         math.pow(math.erf(1.0 / math.sqrt(2.0 * 0.01)), 9.0))


def make_integrand(name: str, dims: int) -> IntegrandSpec:
    """CLI-name lookup (integrands.hpp:221-235)."""
    if name in ("fA", "fB"):
        spec = make_fA() if name == "fA" else make_fB()
        if dims != 0 and dims != spec.dims:
            raise ValueError(f"{name} is fixed at {spec.dims} dimensions")
        return spec
    if len(name) == 2 and name[0] == "f" and name[1] in "123456":
        if dims == 0:
            raise ValueError(f"{name} requires an explicit dimension")
        return make_suite_integrand(int(name[1]), dims)
    raise ValueError(f'unknown integrand "{name}"')


def make_table_integrand(tables, lower, upper, name: str = "table") -> IntegrandSpec:
    """Stateful integrand with device-resident interpolation tables
    (BASELINE config 4; the paper's cosmology-style use case).

    f(x) = prod_j T_j(x_j), T_j piecewise linear on n uniform nodes over
    [lower_j, upper_j].  The exact integral is the product of trapezoid sums."""
    tables = np.asarray(tables, dtype=np.float64)
    d, n = tables.shape
    lower = [float(v) for v in lower]
    upper = [float(v) for v in upper]
    inv_h = [float(n - 1) / (upper[j] - lower[j]) for j in range(d)]
    params = np.concatenate([[float(n)], lower, inv_h, tables.reshape(-1)])
    ref = 1.0
    for j in range(d):
        h = (upper[j] - lower[j]) / (n - 1)
        ref *= h * (tables[j].sum() - 0.5 * (tables[j, 0] + tables[j, -1]))
    return IntegrandSpec(name, d, lower, upper, 9, params, ref)


_TEST_IDS = {"x0": 32, "const": 33, "x0sq_half": 34, "inf_if_x0_pos": 35, "inf": 36, "zero": 37,
             "inf_near_origin": 38}


def test_integrand(kind: str, dims: int, value: float = 0.0, lower=None, upper=None) -> IntegrandSpec:
    """The small functors of the reference's unit tests (test_oracle.cpp,
    test_sampler.cpp, test_driver.cpp): x0, const, x0sq_half, inf_if_x0_pos,
    inf, zero; plus inf_near_origin (+inf if every x_j < value) for the
    multi-rank failure path."""
    params = np.array([value]) if kind in ("const", "inf_near_origin") else None
    lower = [0.0] * dims if lower is None else list(lower)
    upper = [1.0] * dims if upper is None else list(upper)
    return IntegrandSpec(kind, dims, lower, upper, _TEST_IDS[kind], params, None)


# ----------------------------------------------------------------- accumulators


class BinAccumulator:
    """Per-axis, per-bin totals of (f*J)^2 (accumulators.hpp:18-56)."""

    def __init__(self, dims: int, n_bins: int, values=None, writes: int = 0):
        if values is None:
            if dims == 0:
                raise ValueError("BinAccumulator: dims must be >= 1")
            if n_bins == 0:
                raise ValueError("BinAccumulator: n_bins must be >= 1")
            values = np.zeros(dims * n_bins)
        values = _f64(values).reshape(-1)
        if values.size != dims * n_bins:
            raise ValueError("BinAccumulator: value matrix has wrong shape")
        self._dims, self._n_bins, self._values, self._writes = dims, n_bins, values, writes

    def deposit(self, axis: int, b: int, v: float):
        self._values[axis * self._n_bins + b] += v
        self._writes += 1

    def at(self, axis: int, b: int) -> float:
        return float(self._values[axis * self._n_bins + b])

    def axis_row(self, axis: int) -> np.ndarray:
        if axis >= self._dims:
            raise ValueError("BinAccumulator: axis out of range")
        return self._values[axis * self._n_bins:(axis + 1) * self._n_bins]

    @property
    def values(self) -> np.ndarray:
        return self._values

    def dims(self):
        return self._dims

    def n_bins(self):
        return self._n_bins

    def writes(self):
        return self._writes


# ----------------------------------------------------------------- grid


class Grid:
    """Per-axis importance grid (grid.hpp:19-176); right edges, d x n_bins."""

    def __init__(self, dims: int, n_bins: int, lower: Sequence[float], upper: Sequence[float],
                 _edges: Optional[np.ndarray] = None):
        lower, upper = [float(v) for v in lower], [float(v) for v in upper]
        if dims == 0:
            raise ValueError("Grid: dims must be >= 1")
        if n_bins < 2:
            raise ValueError("Grid: n_bins must be >= 2")
        if len(lower) != dims or len(upper) != dims:
            raise ValueError("Grid: bounds must have one entry per axis")
        self._dims, self._n_bins = dims, n_bins
        self._lower, self._upper = lower, upper
        if _edges is None:
            for j in range(dims):
                if not (lower[j] < upper[j]) or not math.isfinite(lower[j]) or not math.isfinite(upper[j]):
                    raise ValueError("Grid: requires finite lower < upper on every axis")
            e = np.zeros(dims * n_bins)
            lo, hi = _f64(lower), _f64(upper)
            _raise(L.lib().mcb_grid_uniform(dims, n_bins, _dptr(lo), _dptr(hi), _dptr(e)))
            self._edges = e
        else:
            e = _f64(_edges).reshape(-1).copy()
            for j in range(dims):
                if not (lower[j] < upper[j]):
                    raise ValueError("Grid: requires lower < upper on every axis")
                prev = lower[j]
                for v in e[j * n_bins:(j + 1) * n_bins]:
                    if not (v > prev):
                        raise ValueError("Grid: edges must increase strictly")
                    prev = v
                if e[(j + 1) * n_bins - 1] != upper[j]:
                    raise ValueError("Grid: last edge must equal the upper bound")
            self._edges = e

    @classmethod
    def from_edges(cls, dims, n_bins, lower, upper, edges):
        return cls(dims, n_bins, lower, upper, _edges=edges)

    def dims(self):
        return self._dims

    def n_bins(self):
        return self._n_bins

    def lower(self, axis: int) -> float:
        return self._lower[axis]

    def upper(self, axis: int) -> float:
        return self._upper[axis]

    def edges(self, axis: int) -> np.ndarray:
        return self._edges[axis * self._n_bins:(axis + 1) * self._n_bins]

    @property
    def raw_edges(self) -> np.ndarray:
        return self._edges

    @property
    def lowers(self):
        return list(self._lower)

    @property
    def uppers(self):
        return list(self._upper)

    def bin_index(self, u: float) -> int:
        nb = float(self._n_bins)
        z = u * nb
        if not (z > 0.0):
            return 0
        if z >= nb:
            return self._n_bins - 1
        return int(z)

    def transform(self, u: Sequence[float], want_bins: bool = False):
        """Host form of the bin map the sampling kernel applies (grid.hpp:204-224)."""
        nb = float(self._n_bins)
        x, bins, jac = [], [], 1.0
        for j in range(self._dims):
            z = u[j] * nb
            i = 0
            if z >= nb:
                i = self._n_bins - 1
            elif z > 0.0:
                i = int(z)
            row = self.edges(j)
            left = self._lower[j] if i == 0 else float(row[i - 1])
            width = float(row[i]) - left
            x.append(left + (z - float(i)) * width)
            jac *= nb * width
            bins.append(i)
        return (jac, x, bins) if want_bins else (jac, x)

    def _adjust(self, contrib: np.ndarray, alpha: float, symmetric: bool, ctx: Optional[Context]):
        ctx = ctx or default_context()
        out = np.zeros_like(self._edges)
        lo, hi = _f64(self._lower), _f64(self._upper)
        rc = L.lib().mcb_grid_adjust(ctx.ptr, self._dims, self._n_bins, _dptr(lo), _dptr(hi),
                                     _dptr(self._edges), _dptr(contrib), alpha, 1 if symmetric else 0, _dptr(out))
        _raise(rc, ctx.ptr)
        g = Grid.__new__(Grid)
        g._dims, g._n_bins, g._lower, g._upper, g._edges = self._dims, self._n_bins, list(self._lower), \
            list(self._upper), out
        return g

    def adjusted(self, contributions, alpha: float, ctx: Optional[Context] = None) -> "Grid":
        """One adaptation step on the GPU (grid.hpp:104-114)."""
        vals = contributions.values if isinstance(contributions, BinAccumulator) else _f64(contributions).reshape(-1)
        if isinstance(contributions, BinAccumulator) and (
                contributions.dims() != self._dims or contributions.n_bins() != self._n_bins):
            raise ValueError("Grid::adjusted: contribution shape mismatch")
        if vals.size != self._dims * self._n_bins:
            raise ValueError("Grid::adjusted: contribution shape mismatch")
        return self._adjust(_f64(vals), alpha, False, ctx)

    def adjusted_symmetric(self, axis0_contributions, alpha: float, ctx: Optional[Context] = None) -> "Grid":
        """Symmetric-integrand adaptation on the GPU (grid.hpp:122-146)."""
        row = _f64(axis0_contributions).reshape(-1)
        if row.size != self._n_bins:
            raise ValueError("Grid::adjusted_symmetric: contribution shape mismatch")
        full = np.zeros(self._dims * self._n_bins)
        full[:self._n_bins] = row
        return self._adjust(full, alpha, True, ctx)

    def write(self) -> str:
        """Plain-text form (grid.hpp:148-158)."""
        lines = [f"{self._dims} {self._n_bins}"]
        for j in range(self._dims):
            vals = [self._lower[j], self._upper[j]] + [float(v) for v in self.edges(j)]
            lines.append(" ".join(_g17(v) for v in vals))
        return "\n".join(lines) + "\n"

    @staticmethod
    def read(text: str) -> "Grid":
        """grid.hpp:161-174"""
        tok = text.split()
        try:
            dims, nb = int(tok[0]), int(tok[1])
        except (IndexError, ValueError):
            raise ValueError("Grid::read: malformed header")
        if dims == 0 or nb < 2:
            raise ValueError("Grid::read: malformed header")
        pos = 2
        lower, upper, edges = [], [], []
        for _ in range(dims):
            try:
                lower.append(float(tok[pos]))
                upper.append(float(tok[pos + 1]))
            except (IndexError, ValueError):
                raise ValueError("Grid::read: malformed axis bounds")
            pos += 2
            try:
                edges.extend(float(t) for t in tok[pos:pos + nb])
                if len(tok[pos:pos + nb]) != nb:
                    raise IndexError
            except (IndexError, ValueError):
                raise ValueError("Grid::read: malformed edge list")
            pos += nb
        return Grid.from_edges(dims, nb, lower, upper, np.array(edges))

    def __eq__(self, other):
        return (isinstance(other, Grid) and self._dims == other._dims and self._n_bins == other._n_bins
                and self._lower == other._lower and self._upper == other._upper
                and np.array_equal(self._edges, other._edges))


def _g17(v: float) -> str:
    s = "%.17g" % v
    return s


# ----------------------------------------------------------------- sampler


class BinUpdate(IntEnum):
    all_axes = 0
    axis0_only = 1


@dataclass
class SampleOutcome:
    raw_estimate: float
    raw_variance: float
    contributions: BinAccumulator


@dataclass
class EstimateVariance:
    raw_estimate: float
    raw_variance: float


RNG_CODES = {"compat": 0, "philox": 1, "philox_exact": 2}  # include/mcubes_b200.h mcb_rng


def rng_code(rng: str, bins: str = "") -> int:
    """mcb_rng for a (stream, bin precision) pair.  bins '' = the stream's
    default: exact for compat (the reference's ExactBins), r24 for philox
    ((f J)^2 rounded to 24 significant bits, then summed exactly)."""
    if rng == "compat":
        if bins not in ("", "exact"):
            raise ValueError("the compat stream sums exact bins (it is bitwise the reference)")
        return 0
    if rng == "philox":
        if bins not in ("", "r24", "exact"):
            raise ValueError("bins must be 'r24' or 'exact'")
        return 2 if bins == "exact" else 1
    raise ValueError(f"unknown rng {rng!r}: 'compat' or 'philox'")


def v_sample(f: IntegrandSpec, grid: Grid, m: int, s: int, p: int, seed: int, iteration: int,
             mode: BinUpdate = BinUpdate.all_axes, max_threads: int = 0, rng: str = "compat",
             ctx: Optional[Context] = None, bins: str = "") -> SampleOutcome:
    """One adjusting iteration on the GPU (sampler.hpp:312-333).  Output is
    bitwise identical for any ``s``/``max_threads`` (accepted, as in the
    reference).  ``writes()`` of the result is counted on the device."""
    ctx = ctx or default_context()
    fs, keep = f._c()
    lo, hi = _f64(grid.lowers), _f64(grid.uppers)
    est, var, writes = C.c_double(), C.c_double(), C.c_uint64()
    contrib = np.zeros(grid.dims() * grid.n_bins())
    rc = L.lib().mcb_v_sample_rng(ctx.ptr, C.byref(fs), rng_code(rng, bins), grid.dims(), grid.n_bins(), _dptr(lo),
                                  _dptr(hi), _dptr(grid.raw_edges), m, s, p, seed, iteration, int(mode),
                                  C.byref(est), C.byref(var), _dptr(contrib), C.byref(writes))
    _raise(rc, ctx.ptr, grid.dims())
    return SampleOutcome(est.value, var.value, BinAccumulator(grid.dims(), grid.n_bins(), contrib, writes.value))


def v_sample_no_adjust(f: IntegrandSpec, grid: Grid, m: int, s: int, p: int, seed: int, iteration: int,
                       max_threads: int = 0, rng: str = "compat", ctx: Optional[Context] = None) -> EstimateVariance:
    """Frozen-grid iteration on the GPU (sampler.hpp:339-349)."""
    ctx = ctx or default_context()
    fs, keep = f._c()
    lo, hi = _f64(grid.lowers), _f64(grid.uppers)
    est, var = C.c_double(), C.c_double()
    if rng == "philox":
        rc = L.lib().mcb_v_sample_rng(ctx.ptr, C.byref(fs), 1, grid.dims(), grid.n_bins(), _dptr(lo), _dptr(hi),
                                      _dptr(grid.raw_edges), m, s, p, seed, iteration, 2, C.byref(est),
                                      C.byref(var), None, None)
    else:
        rc = L.lib().mcb_v_sample_no_adjust(ctx.ptr, C.byref(fs), grid.dims(), grid.n_bins(), _dptr(lo),
                                            _dptr(hi), _dptr(grid.raw_edges), m, s, p, seed, iteration,
                                            C.byref(est), C.byref(var))
    _raise(rc, ctx.ptr, grid.dims())
    return EstimateVariance(est.value, var.value)


# ----------------------------------------------------------------- driver


class Variant(IntEnum):
    mcubes = 0
    mcubes1d = 1


def variant_name(v: Variant) -> str:
    return "mcubes" if v == Variant.mcubes else "mcubes1d"


def parse_variant(s: str) -> Optional[Variant]:
    return {"mcubes": Variant.mcubes, "mcubes1d": Variant.mcubes1d}.get(s)


@dataclass
class RunConfig:
    """driver.hpp:37-71, plus ``rng`` ('compat' = the reference stream, bitwise
    the reference; 'philox' = the north-star stream) and ``bins`` (the
    contribution precision: '' = the stream's default, 'exact' or 'r24'; see
    rng_code)."""

    dims: int = 0
    n_bins: int = 50
    maxcalls: int = 0
    itmax: int = 15
    ita: int = 10
    tau_rel: float = 1e-3
    alpha: float = 1.5
    chi2_dof_max: float = 1.5
    seed: int = 0
    variant: Variant = Variant.mcubes
    lower: List[float] = field(default_factory=list)
    upper: List[float] = field(default_factory=list)
    workers: int = 0
    rng: str = "compat"
    bins: str = ""

    def _c(self):
        # plain ctypes arrays (a numpy round trip costs ~10 us per integrate() call)
        lo = (C.c_double * len(self.lower))(*self.lower)
        hi = (C.c_double * len(self.upper))(*self.upper)
        c = L.mcb_config(self.dims, self.n_bins, self.maxcalls, self.itmax, self.ita, self.tau_rel, self.alpha,
                         self.chi2_dof_max, self.seed, int(self.variant), self.workers,
                         C.cast(lo, C.POINTER(C.c_double)) if len(self.lower) else None,
                         C.cast(hi, C.POINTER(C.c_double)) if len(self.upper) else None,
                         rng_code(self.rng, self.bins), 0)
        return c, (lo, hi)

    def validate(self):
        """Raises ValueError on the first broken invariant (driver.hpp:52-70)."""
        if self.dims < 1:
            raise ValueError("RunConfig: dims must be >= 1")
        if self.n_bins < 2:
            raise ValueError("RunConfig: n_bins must be >= 2")
        if self.dims >= 63 or self.maxcalls < (2 << self.dims):
            raise ValueError("RunConfig: maxcalls must be >= 2*2^dims")
        if not (self.tau_rel > 0.0) or not (self.tau_rel < 1.0):
            raise ValueError("RunConfig: tau_rel must lie in (0, 1)")
        if self.itmax < 1:
            raise ValueError("RunConfig: itmax must be >= 1")
        if self.ita > self.itmax:
            raise ValueError("RunConfig: ita must not exceed itmax")
        if not (self.alpha >= 0.0) or not math.isfinite(self.alpha):
            raise ValueError("RunConfig: alpha must be finite and >= 0")
        if not (self.chi2_dof_max > 0.0):
            raise ValueError("RunConfig: chi2_dof_max must be positive")
        if len(self.lower) != self.dims or len(self.upper) != self.dims:
            raise ValueError("RunConfig: bounds must have one entry per axis")
        for lo, hi in zip(self.lower, self.upper):
            if not math.isfinite(lo) or not math.isfinite(hi) or not (lo < hi):
                raise ValueError("RunConfig: requires finite lower < upper on every axis")


class SetupParams(NamedTuple):
    g: int
    m: int
    p: int
    s: int


def setup(cfg: RunConfig) -> SetupParams:
    """driver.hpp:114-123 (validates like the reference)."""
    cfg.validate()
    c, keep = cfg._c()
    g, m, p, s = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    _raise(L.lib().mcb_setup(C.byref(c), C.byref(g), C.byref(m), C.byref(p), C.byref(s)))
    return SetupParams(g.value, m.value, p.value, s.value)


def set_batch_size(m: int, workers: int) -> int:
    """driver.hpp:82-87"""
    s = C.c_uint64()
    rc = L.lib().mcb_set_batch_size(m, workers, C.byref(s))
    if rc != L.MCB_OK:
        raise ValueError("set_batch_size: m must be >= 1" if m == 0 else "set_batch_size: workers must be >= 1")
    return s.value


class IterationResult(NamedTuple):
    estimate: float
    variance: float
    index: int


class Combined(NamedTuple):
    estimate: float
    sigma: float
    chi2_dof: float


def weighted_estimate(history: Sequence[IterationResult]) -> Combined:
    """Inverse-variance combination (driver.hpp:146-169)."""
    if len(history) == 0:
        raise ValueError("weighted_estimate: history must be non-empty")
    for it in history:
        if not (it[1] >= 0.0):
            raise ValueError("weighted_estimate: negative variance")
    e = _f64([h[0] for h in history])
    v = _f64([h[1] for h in history])
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _raise(L.lib().mcb_weighted_estimate(len(e), _dptr(e), _dptr(v), C.byref(a), C.byref(b), C.byref(c)))
    return Combined(a.value, b.value, c.value)


def check_convergence(c: Combined, cfg: RunConfig) -> bool:
    """driver.hpp:173-178"""
    return bool(L.lib().mcb_check_convergence(c[0], c[1], c[2], cfg.tau_rel, cfg.chi2_dof_max))


@dataclass
class IntegrationResult:
    estimate: float = 0.0
    sigma: float = 0.0
    chi2_dof: float = 0.0
    iterations_used: int = 0
    converged: bool = False
    total_samples: int = 0
    bin_writes: int = 0
    params: SetupParams = SetupParams(0, 0, 0, 0)
    history: List[IterationResult] = field(default_factory=list)


@dataclass
class IterationView:
    iteration: int
    adjusting: bool
    result: IterationResult
    running: Combined
    grid: Grid
    bin_writes: int


def _result(r: "L.mcb_result", hist) -> IntegrationResult:
    h = [IterationResult(hist[i].estimate, hist[i].variance, hist[i].index) for i in range(r.iterations_used)]
    return IntegrationResult(r.estimate, r.sigma, r.chi2_dof, r.iterations_used, bool(r.converged),
                             r.total_samples, r.bin_writes, SetupParams(r.g, r.m, r.p, r.s), h)


@dataclass
class Checkpoint:
    """Resumable state of an integrate() run: the grid in
    force after the completed iterations and their results.  The stream is
    keyed by (seed, iteration), so resuming reproduces the uninterrupted run
    bit for bit.  Text form: the grid in grid.hpp:148-158's format, then one
    'index estimate variance' line per completed iteration (%.17g)."""
    grid: "Grid"
    history: List[IterationResult]

    def write(self) -> str:
        lines = [self.grid.write().rstrip("\n"), str(len(self.history))]
        lines += [f"{h.index} {_g17(h.estimate)} {_g17(h.variance)}" for h in self.history]
        return "\n".join(lines) + "\n"

    @staticmethod
    def read(text: str) -> "Checkpoint":
        rows = text.strip().split("\n")
        dims = int(rows[0].split()[0])
        grid = Grid.read("\n".join(rows[:1 + dims]))
        n = int(rows[1 + dims])
        hist = []
        for line in rows[2 + dims:2 + dims + n]:
            i, e, v = line.split()
            hist.append(IterationResult(float(e), float(v), int(i)))
        return Checkpoint(grid, hist)


def integrate(f: IntegrandSpec, cfg: RunConfig, observer: Optional[Callable[[IterationView], None]] = None,
              ctx: Optional[Context] = None, resume: Optional[Checkpoint] = None) -> IntegrationResult:
    """The full loop (driver.hpp:215-258) on the GPU.  Without an observer the
    whole schedule is enqueued with one synchronisation at the end.  With
    `resume`, the run continues after the checkpoint's iterations."""
    ctx = ctx or default_context()
    fs, keep = f._c()
    c, keep2 = cfg._c()
    res = L.mcb_result()
    hist = (L.mcb_iteration * max(cfg.itmax, 1))()
    cb = L.OBSERVER()
    errors = []
    if observer is not None:
        def _cb(vp, user):
            try:
                v = vp.contents
                n = cfg.dims * cfg.n_bins
                edges = np.ctypeslib.as_array(v.grid_edges, shape=(n,)).copy()
                g = Grid.from_edges(cfg.dims, cfg.n_bins, cfg.lower, cfg.upper, edges)
                observer(IterationView(v.iteration, bool(v.adjusting),
                                       IterationResult(v.result.estimate, v.result.variance, v.result.index),
                                       Combined(v.running_estimate, v.running_sigma, v.running_chi2_dof), g,
                                       v.bin_writes))
            except Exception as e:  # pragma: no cover - surfaced after the call
                errors.append(e)
        cb = L.OBSERVER(_cb)
    if resume is None:
        rc = L.lib().mcb_integrate(ctx.ptr, C.byref(fs), C.byref(c), C.byref(res), hist, cfg.itmax, cb, None)
    else:
        done = (L.mcb_iteration * max(len(resume.history), 1))()
        for i, h in enumerate(resume.history):
            done[i] = L.mcb_iteration(h.estimate, h.variance, h.index, 0)
        edges = np.ascontiguousarray(resume.grid.raw_edges, dtype=np.float64)
        rc = L.lib().mcb_integrate_resume(ctx.ptr, C.byref(fs), C.byref(c), _dptr(edges), done,
                                          len(resume.history), C.byref(res), hist, cfg.itmax, cb, None)
    _raise(rc, ctx.ptr, cfg.dims)
    if errors:
        raise errors[0]
    return _result(res, hist)


class Run:
    """A device-resident integrate() that is stepped one iteration at a time
    (the multi-GPU hook, see ``paper_2202_01753_b200.dist``)."""

    def __init__(self, f: IntegrandSpec, cfg: RunConfig, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.cfg = cfg
        self._lib = L.lib()
        fs, self._keep = f._c()
        c, self._keep2 = cfg._c()
        p = C.c_void_p()
        _raise(self._lib.mcb_run_create(self.ctx.ptr, C.byref(fs), C.byref(c), C.byref(p)), self.ctx.ptr, cfg.dims)
        self.ptr = p

    def close(self):
        if getattr(self, "ptr", None):
            self._lib.mcb_run_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def work_items(self) -> int:
        return int(self._lib.mcb_run_work_items(self.ptr))

    def exchange_words(self, it: int = 0) -> int:
        return int(self._lib.mcb_run_exchange_words(self.ptr, it))

    def set_exchange(self, device_ptr: int):
        _raise(self._lib.mcb_run_set_exchange(self.ptr, C.c_void_p(device_ptr)), self.ctx.ptr)

    def resume(self, cp: "Checkpoint") -> int:
        """Continue from a checkpoint (mcb_run_resume); returns the next iteration."""
        done = (L.mcb_iteration * max(len(cp.history), 1))()
        for i, h in enumerate(cp.history):
            done[i] = L.mcb_iteration(h.estimate, h.variance, h.index, 0)
        edges = np.ascontiguousarray(cp.grid.raw_edges, dtype=np.float64)
        nxt = C.c_uint32()
        _raise(self._lib.mcb_run_resume(self.ptr, _dptr(edges), done, len(cp.history), C.byref(nxt)), self.ctx.ptr)
        return nxt.value

    def failure_key(self):
        """(failed, key): whether the run stopped on a non-finite sample in any
        rank's slice, and this rank's first failing sample key t*p+k (2^64-1
        when none was in its slice)."""
        failed, key = C.c_int(0), C.c_uint64(0)
        _raise(self._lib.mcb_run_failure_key(self.ptr, C.byref(failed), C.byref(key)), self.ctx.ptr)
        return bool(failed.value), int(key.value)

    def set_peers(self, rank: int, npeers: int, bufs_odd, bufs_even, flags, counter: int):
        """Peer-memory exchange (mcb_run_set_peers): per-rank device pointers
        of the odd/even-iteration exchange buffers and flag arrays, and this
        rank's block counter.  npeers = 0 turns it off."""
        arr = lambda xs: (C.c_void_p * max(npeers, 1))(*[C.c_void_p(x) for x in xs])  # noqa: E731
        _raise(self._lib.mcb_run_set_peers(self.ptr, rank, npeers, arr(bufs_odd), arr(bufs_even), arr(flags),
                                           C.c_void_p(counter)), self.ctx.ptr)

    def set_failure_key(self, key: int):
        _raise(self._lib.mcb_run_set_failure_key(self.ptr, key), self.ctx.ptr)

    def set_progress(self, host_ptr: int):
        """Host-mapped progress flags (mcb_run_set_progress): pinned int32[itmax], zeroed."""
        _raise(self._lib.mcb_run_set_progress(self.ptr, C.c_void_p(host_ptr)), self.ctx.ptr)

    def sample(self, it: int, n0: int = 0, n1: int = (1 << 64) - 1):
        _raise(self._lib.mcb_run_sample(self.ptr, it, n0, n1), self.ctx.ptr, self.cfg.dims)

    def reduce(self, it: int):
        _raise(self._lib.mcb_run_reduce(self.ptr, it), self.ctx.ptr, self.cfg.dims)

    def finish(self, it: int):
        _raise(self._lib.mcb_run_finish(self.ptr, it), self.ctx.ptr, self.cfg.dims)

    # compact exchange (include/mcubes_b200.h): round this rank's slice,
    # all-gather, combine in rank order, epilogue
    def compact_len(self) -> int:
        """Doubles per rank in the compact exchange (d * n_bins + 6)."""
        return int(self._lib.mcb_run_compact_len(self.ptr))

    def round_local(self, it: int, device_ptr: int):
        _raise(self._lib.mcb_run_round_local(self.ptr, it, C.c_void_p(device_ptr)), self.ctx.ptr, self.cfg.dims)

    def combine(self, it: int, gathered_ptr: int, nranks: int):
        _raise(self._lib.mcb_run_combine(self.ptr, it, C.c_void_p(gathered_ptr), nranks), self.ctx.ptr,
               self.cfg.dims)

    def finish_rounded(self, it: int):
        _raise(self._lib.mcb_run_finish_rounded(self.ptr, it), self.ctx.ptr, self.cfg.dims)

    def step(self, it: int):
        """One whole iteration on this device (sample, reduce, finish)."""
        self.sample(it)
        self.reduce(it)
        self.finish(it)

    def set_grid(self, edges: np.ndarray):
        """Replace the device grid (stream-ordered H2D copy of dims*n_bins edges)."""
        _raise(self._lib.mcb_run_set_grid(self.ptr, _dptr(edges)), self.ctx.ptr)

    def grid_into(self, out: np.ndarray):
        """D2H copy of the current edges into ``out`` (synchronises)."""
        _raise(self._lib.mcb_run_grid(self.ptr, _dptr(out)), self.ctx.ptr)
        return out

    def grid(self) -> Grid:
        e = np.zeros(self.cfg.dims * self.cfg.n_bins)
        _raise(self._lib.mcb_run_grid(self.ptr, _dptr(e)), self.ctx.ptr)
        return Grid.from_edges(self.cfg.dims, self.cfg.n_bins, self.cfg.lower, self.cfg.upper, e)

    def result(self) -> IntegrationResult:
        res = L.mcb_result()
        hist = (L.mcb_iteration * max(self.cfg.itmax, 1))()
        _raise(self._lib.mcb_run_result(self.ptr, C.byref(res), hist, self.cfg.itmax), self.ctx.ptr, self.cfg.dims)
        return _result(res, hist)
