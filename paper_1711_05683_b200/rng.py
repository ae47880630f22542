"""Counter-addressed random numbers (reference rng.py:1-130).

A deviate is a pure function of (seed, stream, counter).  Two streams are
available to the device kernels:

* ``"reference"`` -- the reference's SplitMix64 construction
  ``mix64(base(seed, stream) + counter * GOLDEN)`` (rng.py:98-125), reproduced
  bit for bit in-kernel (csrc/hk_device.cuh: mix64/key_base/draw_bits);
* ``"philox"`` -- Philox4x32-10 keyed by base(seed, stream), counter =
  (global event index, draw block, tag): the production stream
  (SPEC.md:343 allows any counter-based bijection).  Not bit-compatible with
  the reference; statistically equivalent.

Bulk deviates are produced on the GPU (hk_rng_uniform / hk_rng_raw64).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np

from . import _lib

GOLDEN = 0x9E3779B97F4A7C15   # rng.py:33
STREAMS = {"sampling": 0, "phasespace": 1, "toys": 2, "integration": 3, "unweight": 4}  # cli.py:49-53
RNG_MODES = {"reference": _lib.HK_RNG_REFERENCE, "philox": _lib.HK_RNG_PHILOX}


@dataclass(frozen=True)
class RngKey:
    """(seed, stream, counter) address of a deviate (rng.py:45-62)."""

    seed: int
    stream: int = 0
    counter: int = 0

    def at(self, counter: int) -> "RngKey":
        return replace(self, counter=counter)

    def offset(self, delta: int) -> "RngKey":
        return replace(self, counter=self.counter + delta)


@dataclass(frozen=True)
class BoundedRegion:
    """Axis-aligned box (rng.py:65-95)."""

    bounds: tuple[tuple[float, float], ...]

    def __post_init__(self):
        if len(self.bounds) < 1:
            raise ValueError("region needs at least one dimension")
        for d, (lo, hi) in enumerate(self.bounds):
            if not lo < hi:
                raise ValueError(f"dimension {d}: lower {lo} must be < upper {hi}")

    @property
    def dim(self) -> int:
        return len(self.bounds)

    @property
    def lower(self) -> np.ndarray:
        return np.array([lo for lo, _ in self.bounds])

    @property
    def upper(self) -> np.ndarray:
        return np.array([hi for _, hi in self.bounds])

    def volume(self) -> float:
        return float(np.prod(self.upper - self.lower))

    @classmethod
    def cube(cls, lo: float, hi: float, dim: int) -> "BoundedRegion":
        return cls(tuple((lo, hi) for _ in range(dim)))


class CeilingError(ValueError):
    """The integrand exceeded the accept-reject ceiling at a concrete point."""


def rng_mode(name: str) -> int:
    try:
        return RNG_MODES[name]
    except KeyError:
        raise ValueError(f"unknown rng {name!r}; choose from {sorted(RNG_MODES)}") from None


def _device_counters(counters):
    t = _lib.torch()
    c = np.ascontiguousarray(np.asarray(counters, dtype=np.uint64).ravel())
    return t.from_numpy(c.view(np.int64)).to(_lib.device()), c.shape


def raw64(key: RngKey, counters=None, rng: str = "reference") -> np.ndarray:
    """uint64 deviates at key.counter + counters (rng.py:115-120), on the GPU."""
    if counters is None:
        counters = np.zeros(1, dtype=np.uint64)
    shape = np.shape(counters)
    dc, _ = _device_counters(counters)
    out = _lib.empty(dc.numel(), dtype=_lib.torch().int64)
    _lib.check(_lib.lib().hk_rng_raw64(_lib.make_key(key, rng_mode(rng)), _lib.ptr(dc), dc.numel(),
                                       _lib.ptr(out), _lib.stream_ptr()), "hk_rng_raw64")
    return out.cpu().numpy().view(np.uint64).reshape(shape)


def uniform_array(key: RngKey, counters, rng: str = "reference") -> np.ndarray:
    """Uniform [0, 1) deviates at key.counter + counters (rng.py:123-125), on the GPU."""
    shape = np.shape(counters)
    dc, _ = _device_counters(counters)
    out = _lib.empty(dc.numel())
    _lib.check(_lib.lib().hk_rng_uniform(_lib.make_key(key, rng_mode(rng)), _lib.ptr(dc), dc.numel(),
                                         _lib.ptr(out), _lib.stream_ptr()), "hk_rng_uniform")
    return out.cpu().numpy().reshape(shape)


def uniform(key: RngKey, rng: str = "reference") -> float:
    """Single uniform [0, 1) deviate addressed by the key (rng.py:128-130)."""
    return float(uniform_array(key, np.zeros(1, dtype=np.uint64), rng)[0])


PROPOSAL_BLOCK = 1 << 16   # rng.py:42 -- proposal draws reserved per accepted event


def _lattice(region: BoundedRegion, n: int) -> np.ndarray:
    """Generalised-golden-ratio lattice x_i = frac((i+1) alpha) (rng.py:154-164)."""
    d = region.dim
    phi = 1.0
    for _ in range(32):
        phi = (1.0 + phi) ** (1.0 / (d + 1))
    alpha = np.array([np.mod(1.0 / phi ** (k + 1), 1.0) for k in range(d)])
    u = np.mod(np.arange(1, n + 1)[:, None] * alpha[None, :], 1.0)
    return region.lower[None, :] + u * (region.upper - region.lower)[None, :]


def estimate_ceiling(expr, region: BoundedRegion, scan: int = 10_000) -> float:
    """1.1 x the max of expr over a quasi-random scan (rng.py:167-174); the
    scan points are evaluated on the GPU."""
    from .functors import map_evaluate  # noqa: PLC0415 -- import cycle
    from .store import ColumnSchema, ColumnStore  # noqa: PLC0415

    pts = _lattice(region, scan)
    names = [f"x{k}" for k in range(region.dim)]
    store = ColumnStore.from_columns(ColumnSchema.real64(*names), [pts[:, k] for k in range(region.dim)])
    m = float(np.max(map_evaluate(expr, store, names)))
    if not np.isfinite(m) or m <= 0.0:
        raise ValueError("cannot estimate a positive ceiling for the density")
    return 1.1 * m


def sample_pdf(expr, region: BoundedRegion, n: int, key: RngKey, ceiling: float | None = None,
               workers: int | None = 1):
    """n points distributed as expr on region by accept-reject (rng.py:177-242),
    one GPU thread per accepted event; returns a device ColumnStore x0..x{d-1}."""
    from .functors import compile_program  # noqa: PLC0415
    from .store import ColumnSchema, ColumnStore  # noqa: PLC0415

    d = region.dim
    if expr.arity != d:
        raise ValueError(f"expression consumes {expr.arity} arguments, region has {d}")
    if ceiling is None:
        ceiling = estimate_ceiling(expr, region)
    if ceiling <= 0:
        raise ValueError("ceiling must be positive")
    prog = compile_program(expr.lower([("col", k) for k in range(d)]))
    lo = region.lower.astype(np.float64)
    span = (region.upper - region.lower).astype(np.float64)
    max_rounds = PROPOSAL_BLOCK // (d + 1)
    cols = [_lib.empty(n) for _ in range(d)]
    bad = _lib.bad_cells(2)
    if n:
        lo_c = (ctypes.c_double * d)(*lo)
        span_c = (ctypes.c_double * d)(*span)
        _lib.check(_lib.lib().hk_sample_pdf(prog, d, lo_c, span_c, float(ceiling), _lib.make_key(key),
                                            0, int(n), max_rounds, _lib.ptr_array(cols), _lib.ptr(bad),
                                            _lib.stream_ptr()), "hk_sample_pdf")
        over, dry = _lib.read_bad(bad)
        batch_dry = dry // 65536 if dry != _lib.HK_NO_BAD_ROW else None
        if over != _lib.HK_NO_BAD_ROW and (batch_dry is None or (over >> 40) <= batch_dry):
            ev = ((over >> 40) << 16) | (over & 0xFFFF)
            t = (over >> 24) & 0xFFFF
            c0 = (ev + _lib.u64(key.counter)) * PROPOSAL_BLOCK + t * (d + 1)
            u = uniform_array(key.at(0), np.arange(c0, c0 + d, dtype=np.uint64))
            pt = lo + u * span
            from .functors import map_evaluate  # noqa: PLC0415
            names = [f"x{k}" for k in range(d)]
            one = ColumnStore.from_columns(ColumnSchema.real64(*names), [pt[k:k + 1] for k in range(d)])
            val = np.float64(map_evaluate(expr, one, names)[0])
            raise CeilingError(f"density {val!r} exceeds ceiling {ceiling!r} at point {tuple(pt)}")
        if dry != _lib.HK_NO_BAD_ROW:
            raise RuntimeError(f"acceptance too low: no accept within {max_rounds} proposals "
                               f"for some events (ceiling {ceiling!r})")
    schema = ColumnSchema.real64(*(f"x{k}" for k in range(d)))
    return ColumnStore._from_device(schema, cols)
