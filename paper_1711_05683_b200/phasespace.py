"""n-body phase-space generation on B200 -- drop-in for the reference's
phasespace module (phasespace.py:1-349).

Same names, signatures, defaults, exception types and messages as the
reference; the bodies launch the sm_100a kernels in libhepkit_cuda.so:

* phsp_generate ....... hk_phsp_generate (one thread per event, register-
                        resident GENBOD event, SoA fp64 stores, fused weight
                        moments)
* phsp_decay_chain .... hk_phsp_decay_chain (standalone) /
                        phsp_generate_chain -> hk_phsp_generate_chain (fused)
* phsp_average ........ hk_phsp_moments + hk_fold_partials
* phsp_integrate ...... hk_phsp_integrate (generation -> f -> moments, no store)
* phsp_unweight ....... hk_unweight_flags + hk_scan_counts + hk_compact

Events are addressed by a global row index: row r draws the RNG counters
(r + key.counter) * D + j (phasespace.py:105-109), so a shard [a, b) computed
on any GPU is bit-identical to rows a..b of a one-shot run.
"""

from __future__ import annotations

import ctypes
import functools
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .functors import (EvaluationError, FunctorExpr, columns_used, eval_node, lower_average,
                       match_pair_integrand)
from .integrate import IntegrationResult
from .kinematics import MASS_TOLERANCE, BelowThreshold, FourVector, breakup_momentum, invariant_mass
from .rng import RngKey, rng_mode
from .store import ColumnSchema, ColumnStore

EVAL_BATCH = 16 * _lib.HK_CHUNK   # parallel.py:21 -- error-attribution granularity


@dataclass(frozen=True)
class DecaySpec:
    """Mother mass and ordered daughter masses in GeV (phasespace.py:36-57)."""

    mother_mass: float
    daughter_masses: tuple[float, ...]

    def __post_init__(self):
        object.__setattr__(self, "daughter_masses", tuple(float(m) for m in self.daughter_masses))
        ms = self.daughter_masses
        if len(ms) < 2:
            raise ValueError("a decay needs at least two daughters")
        if any(m < 0 for m in ms):
            raise ValueError("daughter masses must be non-negative")
        if not self.mother_mass > sum(ms):
            raise BelowThreshold(f"mother mass {self.mother_mass} is not above the daughter "
                                 f"mass sum {sum(ms)}")

    @property
    def n(self) -> int:
        return len(self.daughter_masses)


@functools.lru_cache(maxsize=64)
def phsp_schema(n_daughters: int) -> ColumnSchema:
    """weight, p1_e, p1_px, p1_py, p1_pz, ... (phasespace.py:60-64)."""
    names = ["weight"]
    for k in range(1, n_daughters + 1):
        names.extend(f"p{k}_{c}" for c in ("e", "px", "py", "pz"))
    return ColumnSchema.real64(*names)


def _check_mother(spec: DecaySpec, mother: FourVector) -> float:
    m = invariant_mass(mother)
    if abs(m - spec.mother_mass) > MASS_TOLERANCE * spec.mother_mass:
        raise ValueError(f"mother mass {m!r} does not match spec mass {spec.mother_mass!r}")
    return m


def _column_block(n_cols: int, n: int, extra: int = 0):
    """n_cols device columns of n fp64 values carved out of ONE allocation
    (each column 256-byte aligned, so warp stores stay whole transactions),
    plus an `extra`-double tail for partials: one caching-allocator call
    instead of n_cols + 1 -- the host cost of small (C1-size) calls."""
    stride = (n + 31) // 32 * 32
    buf = _lib.empty(n_cols * stride + extra)
    return buf[: n_cols * stride].view(n_cols, stride), buf[n_cols * stride:]


def _columns(n_cols: int, n: int) -> list:
    return list(_column_block(n_cols, n)[0][:, :n].unbind(0))


@functools.lru_cache(maxsize=256)
def _decay_struct(spec: DecaySpec, mother: tuple, m_mother: float):
    """hk_decay_t per (spec, mother): read-only to the library, so shared."""
    return _lib.make_decay(spec, FourVector(*mother), m_mother)


@functools.lru_cache(maxsize=256)
def _checked_decay(spec: DecaySpec, mother: tuple):
    """(hk_decay_t, invariant mother mass) per (spec, mother four-vector); the
    mass check (phasespace.py:175-179) raises, and exceptions are not cached."""
    m_mother = _check_mother(spec, FourVector(*mother))
    return _decay_struct(spec, mother, m_mother), m_mother


# hk_key_t per (key, mode): RngKey is frozen and the library reads it as const
_key_struct = functools.lru_cache(maxsize=1024)(_lib.make_key)


def phsp_generate(spec: DecaySpec, mother: FourVector, n_events: int, key: RngKey,
                  workers: int | None = 1, *, rng: str = "reference",
                  row_offset: int = 0) -> ColumnStore:
    """Weighted n-body decays of ``mother`` (phasespace.py:162-188), on the GPU.

    Returns a device-resident ColumnStore in phsp_schema order.  ``workers``
    is accepted for API compatibility; results never depend on it.
    ``row_offset`` generates rows [row_offset, row_offset + n_events) of the
    run (a shard); ``rng="philox"`` selects the production Philox stream.
    The weight moments (sum w, sum w^2) are fused into the same pass and kept
    in ``store.meta["weight_partials"]``.
    """
    d, _ = _checked_decay(spec, (mother.e, mother.px, mother.py, mother.pz))
    n_events = int(n_events)
    if n_events < 0:
        raise ValueError(f"n_events must be >= 0, got {n_events}")
    k = _key_struct(key, rng_mode(rng))
    block, wpart = _column_block(4 * spec.n + 1, n_events, 2 * _lib.num_weight_slices(n_events))
    store = ColumnStore._from_block(phsp_schema(spec.n), block, n_events)
    if n_events:
        _lib.check(_lib.lib().hk_phsp_generate(d, k, _lib.u64(row_offset), n_events, _lib.ptr_rows(block),
                                               _lib.ptr(wpart), _lib.stream_ptr()), "hk_phsp_generate")
    _set_weight_partials(store, wpart)
    return store


def _set_weight_partials(store: ColumnStore, wpart) -> None:
    """Keep a generation's fused (sum w, sum w^2) warp-slice partials with the
    row count they describe (an empty shard keeps an empty tensor)."""
    store.meta["weight_partials"] = wpart
    store.meta["weight_partials_rows"] = len(store)


def _weight_partials(store: ColumnStore):
    """The fused weight partials when they still describe the store's rows."""
    parts = store.meta.get("weight_partials")
    if parts is None or store.meta.get("weight_partials_rows") != len(store):
        return None
    return parts


def phsp_generate_to_host(spec: DecaySpec, mother: FourVector, n_events: int, key: RngKey,
                          *, rng: str = "reference", row_offset: int = 0, out=None,
                          stage_bytes: int = 1 << 30):
    """phsp_generate straight into pinned HOST columns (the reference's memory
    space), generation overlapped with the device->host copies.

    Returns (ColumnStore with host columns, (sum w, sum w^2)).  ``out`` may
    pass preallocated pinned torch tensors (4n+1 of length n_events).
    """
    torch = _lib.torch()
    m_mother = _check_mother(spec, mother)
    d = _lib.make_decay(spec, mother, m_mother)
    k = _lib.make_key(key, rng_mode(rng))
    ncols = 4 * spec.n + 1
    if out is None:
        out = [torch.empty(n_events, dtype=torch.float64, pin_memory=True) for _ in range(ncols)]
    head = (2 * _lib.num_weight_slices(n_events) + 2 * _lib.HK_SUPERS + 2) * 8
    stage_bytes = max(int(stage_bytes), head + 2 * ncols * 8 * _lib.HK_CHUNK)
    sums = (ctypes.c_double * 2)()
    with _stage_lock:                     # one staging buffer per device, one user at a time
        stage = _stage_buffer(stage_bytes)
        _lib.check(_lib.lib().hk_phsp_generate_host(d, k, _lib.u64(row_offset), int(n_events),
                                                    _lib.ptr_array(out), sums, _lib.ptr(stage),
                                                    stage.numel(), _lib.stream_ptr()),
                   "hk_phsp_generate_host")
    store = ColumnStore.from_columns(phsp_schema(spec.n), [t.numpy() for t in out])
    return store, (sums[0], sums[1])


_stage_cache: dict = {}
_stage_lock = threading.Lock()


def _stage_buffer(nbytes: int):
    dev = _lib.device()
    buf = _stage_cache.get(dev)
    if buf is None or buf.numel() < nbytes:
        buf = _lib.torch().empty(int(nbytes), dtype=_lib.torch().uint8, device=dev)
        _stage_cache[dev] = buf
    return buf


def phsp_max_weight(spec: DecaySpec) -> float:
    """Upper bound on event weights (phasespace.py:191-203), host scalar."""
    ms = spec.daughter_masses
    T = spec.mother_mass - sum(ms)
    hi, lo, w = T + ms[0], 0.0, 1.0
    for k in range(1, spec.n):
        lo += ms[k - 1]
        hi += ms[k]
        w *= breakup_momentum(hi, lo, ms[k])
    return w


# ---------------------------------------------------------------------------
# weight integration (sum / mean / variance of the weight column)

@dataclass(frozen=True)
class WeightMoments:
    n: int
    sum_w: float
    sum_w2: float

    @property
    def mean(self) -> float:
        return self.sum_w / self.n

    @property
    def variance(self) -> float:
        """Population variance (np.var, ddof=0) from the two sums."""
        m = self.mean
        return max(self.sum_w2 / self.n - m * m, 0.0)


def phsp_weight_moments(block: ColumnStore) -> WeightMoments:
    """Sum, mean and variance of the weights.  Uses the moments fused into
    generation when present, else one device pass over the weight column."""
    n = len(block)
    if n == 0:
        raise ValueError("cannot integrate an empty block")
    parts = _weight_partials(block)
    if parts is None:
        prog = _weight_program()
        parts5 = _moment_partials(block, prog)
        tot = _lib.total(parts5, n, 5).cpu().numpy()
        return WeightMoments(n, float(tot[0]), float(tot[2]))
    tot = _lib.weight_totals(parts, n).cpu().numpy()
    return WeightMoments(n, float(tot[0]), float(tot[1]))


def _weight_program():
    from .functors import compile_program  # noqa: PLC0415
    return compile_program(("const", 1.0))


# ---------------------------------------------------------------------------
# averages

def _weighted_names(block: ColumnStore) -> list[str]:
    """Column names as the moment kernels see them: they read the weight from
    column 0 (phsp_schema order, phasespace.py:60-64).  The reference reads it
    by name (block.column("weight"), phasespace.py:310), so a store whose
    weight is elsewhere gets a copy of its pointer in front and the traced
    program's column indices shift by one."""
    names = list(block.schema.names)
    if "weight" not in names:
        raise KeyError("unknown column 'weight'")
    return names if names[0] == "weight" else ["\0weight", *names]


def _moment_partials(block: ColumnStore, prog, bad=None):
    n = len(block)
    names = _weighted_names(block)
    cols = block.device_columns([nm if nm != "\0weight" else "weight" for nm in names])
    parts = _lib.empty(5 * _lib.num_chunks(n))
    _lib.check(_lib.lib().hk_phsp_moments(_lib.ptr_array(cols), len(cols), n, prog, _lib.ptr(parts),
                                          _lib.ptr(bad) if bad is not None else None,
                                          _lib.stream_ptr()), "hk_phsp_moments")
    return parts


def _raise_program_error(bad: list[int], args, block_row) -> None:
    """Reference error precedence: the earliest 65536-row batch with a problem
    raises; inside it a zero divisor wins over a non-finite value
    (functors.py:200-207 runs inside expr.eval, before phasespace.py:314)."""
    div0, nonfin = bad
    if div0 == _lib.HK_NO_BAD_ROW and nonfin == _lib.HK_NO_BAD_ROW:
        return
    if div0 != _lib.HK_NO_BAD_ROW and (nonfin == _lib.HK_NO_BAD_ROW
                                       or div0 // EVAL_BATCH <= nonfin // EVAL_BATCH):
        vals = block_row(div0)
        point = tuple(eval_node(a, vals) for a in args)
        raise EvaluationError(f"division by zero at point {point}")
    raise EvaluationError(f"non-finite model value at event {nonfin}")


def _finish_average(tot, n: int) -> IntegrationResult:
    sw, swf, sw2, sw2f, sw2f2 = (float(v) for v in tot)
    if sw <= 0:
        raise ValueError("total weight is not positive")
    mu = swf / sw
    spread = max(sw2f2 - 2.0 * mu * sw2f + mu * mu * sw2, 0.0)
    return IntegrationResult(value=mu, error=math.sqrt(spread) / sw, iterations=1,
                             chi2_per_dof=0.0, calls_used=n)


def phsp_average(expr: FunctorExpr, block: ColumnStore, arg_builder,
                 workers: int | None = 1) -> IntegrationResult:
    """Weighted average of ``expr`` over the block (phasespace.py:291-349).

    ``arg_builder`` receives a dict of column arrays and returns the argument
    tuple; it is traced once symbolically and the composition runs on the GPU.
    """
    n = len(block)
    if n == 0:
        raise ValueError("cannot average over an empty block")
    names = _weighted_names(block)
    prog, args = lower_average(expr, arg_builder, names)
    bad = _lib.bad_cells(2)
    parts = _moment_partials(block, prog, bad)
    tot = _lib.total(parts, n, 5)
    flags = _lib.read_bad(bad)

    def row_values(r):
        return {c: float(block.device_column(names[c].lstrip("\0"))[r]) for c in columns_used(args)}

    _raise_program_error(flags, args, row_values)
    return _finish_average(tot.cpu().numpy(), n)


def phsp_integrate(expr: FunctorExpr, spec: DecaySpec, mother: FourVector, n_events: int,
                   key: RngKey, arg_builder, *, rng: str = "reference",
                   row_offset: int = 0, return_partials: bool = False):
    """Fused phsp_generate -> phsp_average with no event store (config C5).

    Equal (to the reduction's rounding) to
    ``phsp_average(expr, phsp_generate(spec, mother, n_events, key), arg_builder)``
    but reads and writes no event memory.  With ``return_partials`` the
    per-chunk moment partials (device tensor, 5 per 4096 rows) are returned
    instead.
    """
    n_events = int(n_events)
    if n_events == 0:
        raise ValueError("cannot average over an empty block")
    run = _IntegrateRun(expr, spec, mother, key, arg_builder, rng)
    parts, flags = run.partials(n_events, row_offset)
    run.raise_error(flags, row_offset)
    if return_partials:
        return parts
    tot = _lib.total(parts, n_events, 5)
    return _finish_average(tot.cpu().numpy(), n_events)


class _IntegrateRun:
    """One fused generate -> f -> moments run, split so that a sharded caller
    (parallel.sharded_integrate) can exchange partials and error rows before
    any rank raises."""

    def __init__(self, expr, spec, mother, key, arg_builder, rng):
        self.m_mother = _check_mother(spec, mother)
        self.spec, self.mother, self.key, self.rng = spec, mother, key, rng
        self.names = phsp_schema(spec.n).names
        self.prog, self.args, root = lower_average(expr, arg_builder, self.names, with_root=True)
        self.pair = match_pair_integrand(root, spec.n)   # Dalitz m^2_ij / BW(m^2_ij): specialised path

    def partials(self, n_events: int, row_offset: int):
        """(per-chunk partials, [first zero-divisor row, first non-finite row])
        of rows [row_offset, row_offset + n_events), rows global."""
        d = _lib.make_decay(self.spec, self.mother, self.m_mother)
        k = _lib.make_key(self.key, rng_mode(self.rng))
        bad = _lib.bad_cells(2)
        parts = _lib.empty(5 * _lib.num_chunks(n_events))
        if n_events:
            _lib.check(_lib.lib().hk_phsp_integrate(d, k, _lib.u64(row_offset), n_events, self.prog,
                                                    self.pair, _lib.ptr(parts), _lib.ptr(bad),
                                                    _lib.stream_ptr()), "hk_phsp_integrate")
        return parts, _lib.read_bad(bad)

    def raise_error(self, flags, base: int = 0) -> None:
        """The reference's exception for the first bad rows, if any; events
        are numbered from row `base` (the first row of the averaged block)."""
        def row_values(r):
            one = phsp_generate(self.spec, self.mother, 1, self.key, rng=self.rng, row_offset=r + base)
            return {c: float(one.device_column(self.names[c])[0]) for c in columns_used(self.args)}

        rel = [f if f == _lib.HK_NO_BAD_ROW else f - _lib.u64(base) for f in flags]
        _raise_program_error(rel, self.args, row_values)


# ---------------------------------------------------------------------------
# decay chains

def _chain_mass_error(k: int, fe, fx, fy, fz, M: float, j: int):
    e, x, y, z = (np.float64(v) for v in (fe, fx, fy, fz))
    fm = np.sqrt(np.maximum(e * e - x * x - y * y - z * z, 0.0))
    return ValueError(f"event {j}: daughter {k} mass {fm!r} does not match "
                      f"sub-decay mother mass {M!r}")


def phsp_decay_chain(block: ColumnStore, daughter_index: int, subspec: DecaySpec, key: RngKey,
                     workers: int | None = 1, *, rng: str = "reference",
                     row_offset: int = 0) -> ColumnStore:
    """Decay daughter ``daughter_index`` (1-based) of every event
    (phasespace.py:237-288), on the GPU.  Columns of the other daughters are
    shared with the input store (no copy)."""
    n_old = (len(block.schema) - 1) // 4
    if not 1 <= daughter_index <= n_old:
        raise ValueError(f"daughter index {daughter_index} out of range 1..{n_old}")
    k = daughter_index
    n = len(block)
    p4 = block.device_columns([f"p{k}_{c}" for c in ("e", "px", "py", "pz")])
    w_in = block.device_column("weight")
    sub = _lib.make_decay(subspec)
    w_out = _lib.empty(n)
    sub_cols = _columns(4 * subspec.n, n)
    if n:
        bad = _lib.bad_cells(1)
        _lib.check(_lib.lib().hk_phsp_decay_chain(
            _lib.ptr(w_in), _lib.ptr_array(p4), sub, _lib.make_key(key, rng_mode(rng)),
            _lib.u64(row_offset), n, _lib.ptr(w_out), _lib.ptr_array(sub_cols), _lib.ptr(bad),
            _lib.stream_ptr()), "hk_phsp_decay_chain")
        (first,) = _lib.read_bad(bad)
        if first != _lib.HK_NO_BAD_ROW:
            j = first - _lib.u64(row_offset)
            raise _chain_mass_error(k, *(float(t[j]) for t in p4), subspec.mother_mass, j)
    cols = [w_out]
    for i in range(1, n_old + 1):
        if i == k:
            cols.extend(sub_cols)
        else:
            cols.extend(block.device_columns([f"p{i}_{c}" for c in ("e", "px", "py", "pz")]))
    return ColumnStore._from_device(phsp_schema(n_old - 1 + subspec.n), cols)


def phsp_generate_chain(spec: DecaySpec, mother: FourVector, n_events: int, key: RngKey,
                        daughter_index: int, subspec: DecaySpec, sub_key: RngKey, *,
                        rng: str = "reference", row_offset: int = 0) -> ColumnStore:
    """Fused ``phsp_decay_chain(phsp_generate(spec, mother, n, key), k, subspec, sub_key)``
    (config C3): only the final-state columns are written."""
    m_mother = _check_mother(spec, mother)
    if not 1 <= daughter_index <= spec.n:
        raise ValueError(f"daughter index {daughter_index} out of range 1..{spec.n}")
    n_events = int(n_events)
    n_fin = spec.n - 1 + subspec.n
    cols = _columns(4 * n_fin + 1, n_events)
    store = ColumnStore._from_device(phsp_schema(n_fin), cols)
    if n_events == 0:
        return store
    mode = rng_mode(rng)
    wpart = _lib.empty(2 * _lib.num_weight_slices(n_events))
    bad = _lib.bad_cells(1)
    d, ds = _lib.make_decay(spec, mother, m_mother), _lib.make_decay(subspec)
    _lib.check(_lib.lib().hk_phsp_generate_chain(
        d, _lib.make_key(key, mode), int(daughter_index), ds, _lib.make_key(sub_key, mode),
        _lib.u64(row_offset), n_events, _lib.ptr_array(cols), _lib.ptr(wpart), _lib.ptr(bad), _lib.stream_ptr()),
        "hk_phsp_generate_chain")
    if _lib.lib().hk_chain_fixed_frame_mass(d, int(daughter_index), ds) > 0.0:
        # the host proved no event can fail the mass check: no read-back, the
        # call stays asynchronous like phsp_generate
        _set_weight_partials(store, wpart)
        return store
    (first,) = _lib.read_bad(bad)
    if first != _lib.HK_NO_BAD_ROW:
        j = first - _lib.u64(row_offset)
        parent = phsp_generate(spec, mother, 1, key, rng=rng, row_offset=first)
        p4 = [float(parent.device_column(f"p{daughter_index}_{c}")[0]) for c in ("e", "px", "py", "pz")]
        raise _chain_mass_error(daughter_index, *p4, subspec.mother_mass, j)
    _set_weight_partials(store, wpart)
    return store


# ---------------------------------------------------------------------------
# unweighting and device-side selection

def _compact(block: ColumnStore, flags, counts, weight_col: int) -> ColumnStore:
    n = len(block)
    nch = _lib.num_chunks(n)
    torch = _lib.torch()
    offsets = _lib.empty(nch, dtype=torch.int64)
    total = _lib.empty(1, dtype=torch.int64)
    _lib.check(_lib.lib().hk_scan_counts(_lib.ptr(counts), nch, _lib.ptr(offsets), _lib.ptr(total),
                                         _lib.stream_ptr()), "hk_scan_counts")
    m = int(total.item())
    cols_in = block.device_columns()
    cols_out = _columns(len(cols_in), m)
    if m:
        _lib.check(_lib.lib().hk_compact(_lib.ptr_array(cols_in), len(cols_in), n, _lib.ptr(flags),
                                         _lib.ptr(offsets), _lib.ptr_array(cols_out), weight_col,
                                         _lib.stream_ptr()), "hk_compact")
    return ColumnStore._from_device(block.schema, cols_out)


def _device_select(block: ColumnStore, mask: np.ndarray) -> ColumnStore:
    """where_mask for device stores: order-preserving GPU compaction."""
    torch = _lib.torch()
    n = len(block)
    flags = torch.from_numpy(mask.astype(np.uint8)).to(_lib.device())
    counts = torch.from_numpy(
        np.add.reduceat(mask.astype(np.int64), np.arange(0, max(n, 1), _lib.HK_CHUNK))
        if n else np.zeros(0, dtype=np.int64)).to(_lib.device())
    return _compact(block, flags, counts, -1)


def phsp_unweight(block: ColumnStore, w_max: float, key: RngKey,
                  workers: int | None = 1, *, row_offset: int = 0) -> ColumnStore:
    """Accept event i iff u_i * w_max < weight_i; accepted weights become 1
    (phasespace.py:206-234).  Order preserved; w > w_max names the event."""
    n = len(block)
    torch = _lib.torch()
    if n == 0:
        return ColumnStore._from_device(block.schema, _columns(len(block.schema), 0))
    w = block.device_column("weight")
    flags = _lib.empty(n, dtype=torch.uint8)
    counts = _lib.empty(_lib.num_chunks(n), dtype=torch.int64)
    bad = _lib.bad_cells(1)
    _lib.check(_lib.lib().hk_unweight_flags(_lib.ptr(w), n, float(w_max), _lib.make_key(key),
                                            _lib.u64(row_offset), _lib.ptr(flags), _lib.ptr(counts),
                                            _lib.ptr(bad), _lib.stream_ptr()), "hk_unweight_flags")
    (first,) = _lib.read_bad(bad)
    if first != _lib.HK_NO_BAD_ROW:
        j = first - _lib.u64(row_offset)
        raise ValueError(f"event {j} weight {np.float64(float(w[j]))!r} exceeds w_max {w_max!r}")
    return _compact(block, flags, counts, block.schema.names.index("weight"))


def _map_program(prog, cols: list, n: int) -> np.ndarray:
    out = _lib.empty(n)
    if n:
        bad = _lib.bad_cells(1)
        _lib.check(_lib.lib().hk_map_program(_lib.ptr_array(cols), len(cols), n, prog, _lib.ptr(out),
                                             _lib.ptr(bad), _lib.stream_ptr()), "hk_map_program")
        (first,) = _lib.read_bad(bad)
        if first != _lib.HK_NO_BAD_ROW:
            point = tuple(float(c[first]) for c in cols)
            raise EvaluationError(f"division by zero at point {point}")
    return out.cpu().numpy()
