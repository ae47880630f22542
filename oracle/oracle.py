"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
`--impl reference`) may import this module.  The product package
(paper_1711_05683_b200) never does: it fails loudly without its CUDA library.

Two halves:

* ``libhk_oracle.so`` (hk_oracle.c, built with -ffp-contract=off): scalar C
  restatement of the generator / chain / RNG.  Bit-exact against the
  reference's golden vectors (tests/test_oracle_golden.py).
* numpy restatements of the reductions, written with the same numpy ufunc
  sequence, chunking (4096 rows, parallel.py:18) and left fold
  (parallel.py:86-92) as the reference, so their bits match the reference:
    - phsp_average moments ........ phasespace.py:291-349
    - extended NLL ................ fitting.py:175-210 (density :160-166,
                                    Gaussian functors.py:137-143,
                                    exponential functors.py:157-161)
    - analytic norms .............. fitting.py:103-123
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhk_oracle.so")
CHUNK = 4096  # parallel.py:18

_lib = None
_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile the C oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.hko_mix64.restype = _u64
        L.hko_mix64.argtypes = [_u64]
        L.hko_base.restype = _u64
        L.hko_base.argtypes = [_u64, _u64]
        L.hko_raw64.restype = None
        L.hko_raw64.argtypes = [_u64, _u64, ctypes.c_void_p, _i64, ctypes.c_void_p]
        L.hko_uniform.restype = None
        L.hko_uniform.argtypes = [_u64, _u64, ctypes.c_void_p, _i64, ctypes.c_void_p]
        L.hko_generate.restype = ctypes.c_int
        L.hko_generate.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                   ctypes.c_int, ctypes.c_void_p, ctypes.c_double, _u64, _u64,
                                   _u64, _i64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.hko_decay_chain.restype = _i64
        L.hko_decay_chain.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_void_p, _u64, _u64, _u64, _i64, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.hko_philox_rows.restype = None
        L.hko_philox_rows.argtypes = [ctypes.c_void_p, _i64, ctypes.c_void_p]
        L.hko_philox_raw64.restype = None
        L.hko_philox_raw64.argtypes = [_u64, _u64, ctypes.c_void_p, _i64, ctypes.c_void_p]
        L.hko_unweight_flags.restype = None
        L.hko_unweight_flags.argtypes = [ctypes.c_void_p, _i64, ctypes.c_double, _u64, _u64, _u64,
                                         ctypes.c_void_p]
        _lib = L
    return _lib


def u64(v: int) -> int:
    return int(v) % (1 << 64)


def base(seed: int, stream: int) -> int:
    return int(lib().hko_base(u64(seed), u64(stream)))


def raw64(seed: int, stream: int, counter: int, counters) -> np.ndarray:
    c = np.ascontiguousarray(counters, dtype=np.uint64)
    out = np.empty(c.shape, dtype=np.uint64)
    lib().hko_raw64(base(seed, stream), u64(counter), c.ctypes.data, c.size, out.ctypes.data)
    return out


def uniform(seed: int, stream: int, counter: int, counters) -> np.ndarray:
    c = np.ascontiguousarray(counters, dtype=np.uint64)
    out = np.empty(c.shape, dtype=np.float64)
    lib().hko_uniform(base(seed, stream), u64(counter), c.ctypes.data, c.size, out.ctypes.data)
    return out


def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 blocks: ctr (rows x 4 uint32), key (rows x 2 uint32) -> rows x 4."""
    ctr = np.asarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.asarray(key, dtype=np.uint32).reshape(-1, 2)
    rows = np.ascontiguousarray(np.concatenate([ctr, key], axis=1))
    out = np.empty((rows.shape[0], 4), dtype=np.uint32)
    lib().hko_philox_rows(rows.ctypes.data, rows.shape[0], out.ctypes.data)
    return out


def philox_raw64(seed: int, stream: int, counter: int, counters) -> np.ndarray:
    """hk_rng_raw64 in Philox mode: counter c -> words 0-1 of block (c lo, c hi, 0, tag)."""
    c = np.ascontiguousarray(counters, dtype=np.uint64)
    out = np.empty(c.shape, dtype=np.uint64)
    lib().hko_philox_raw64(base(seed, stream), u64(counter), c.ctypes.data, c.size, out.ctypes.data)
    return out


def schema(n: int) -> list[str]:
    names = ["weight"]
    for k in range(1, n + 1):
        names += [f"p{k}_e", f"p{k}_px", f"p{k}_py", f"p{k}_pz"]
    return names


def _mass_terms(masses: Sequence[float], M: float) -> tuple[np.ndarray, float, np.ndarray]:
    # phasespace.py:94-97 -- numpy does these sums; keep its rounding
    m = np.asarray([float(x) for x in masses], dtype=np.float64)
    return m, float(M - float(np.sum(m))), np.ascontiguousarray(np.cumsum(m))


def _ptrs(cols: list[np.ndarray]):
    arr = (ctypes.c_void_p * len(cols))(*[c.ctypes.data for c in cols])
    return arr


def invariant_mass(e: float, px: float, py: float, pz: float) -> float:
    m2 = e ** 2 - (px ** 2 + py ** 2 + pz ** 2)
    return math.sqrt(max(0.0, m2))


RNG_MODES = {"reference": 0, "philox": 1}


def generate(masses, M, n_events, seed, stream, counter=0, mother=None, ev_begin=0,
             threads=1, rng: str = "reference") -> dict[str, np.ndarray]:
    """Rows [ev_begin, ev_begin+n_events) of phsp_generate as a name->column dict
    (rng="philox": the CUDA path's production stream, hko_philox4x32_10)."""
    m, T, csum = _mass_terms(masses, M)
    n = len(m)
    mother = (float(M), 0.0, 0.0, 0.0) if mother is None else tuple(float(v) for v in mother)
    moving = mother[1] != 0.0 or mother[2] != 0.0 or mother[3] != 0.0
    m_mother = invariant_mass(*mother)
    mom = np.asarray(mother, dtype=np.float64)
    cols = [np.empty(n_events) for _ in range(4 * n + 1)]
    rc = lib().hko_generate(n, m.ctypes.data, T, csum.ctypes.data, int(moving), mom.ctypes.data,
                            m_mother, base(seed, stream), u64(counter), u64(ev_begin),
                            int(n_events), _ptrs(cols), int(threads), RNG_MODES[rng])
    if rc != 0:
        raise ValueError(f"oracle generate failed rc={rc}")
    return dict(zip(schema(n), cols))


def decay_chain(block: dict[str, np.ndarray], k: int, sub_masses, M_sub, seed, stream,
                counter=0, ev_begin=0, threads=1, rng: str = "reference") -> dict[str, np.ndarray]:
    n_old = (len(block) - 1) // 4
    m, T, csum = _mass_terms(sub_masses, M_sub)
    n_sub = len(m)
    nev = len(block["weight"])
    p4 = [np.ascontiguousarray(block[f"p{k}_{c}"]) for c in ("e", "px", "py", "pz")]
    w_in = np.ascontiguousarray(block["weight"])
    out_w = np.empty(nev)
    out = [np.empty(nev) for _ in range(4 * n_sub)]
    bad = lib().hko_decay_chain(w_in.ctypes.data, _ptrs(p4), n_sub, m.ctypes.data, float(M_sub),
                                T, csum.ctypes.data, base(seed, stream), u64(counter),
                                u64(ev_begin), nev, out_w.ctypes.data, _ptrs(out), int(threads),
                                RNG_MODES[rng])
    if bad >= 0:
        raise ValueError(f"event {bad}: daughter {k} mass does not match sub-decay mother mass")
    cols = [out_w]
    for i in range(1, n_old + 1):
        if i == k:
            cols += out
        else:
            cols += [block[f"p{i}_{c}"] for c in ("e", "px", "py", "pz")]
    return dict(zip(schema(n_old - 1 + n_sub), cols))


def unweight_accept(w: np.ndarray, w_max: float, seed, stream, counter=0, ev_begin=0) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.float64)
    out = np.empty(w.shape, dtype=np.uint8)
    lib().hko_unweight_flags(w.ctypes.data, w.size, float(w_max), base(seed, stream),
                             u64(counter), u64(ev_begin), out.ctypes.data)
    return out.astype(bool)


# ---------------------------------------------------------------------------
# reductions (numpy, reference chunking and fold order)

def chunk_windows(n: int, chunk: int = CHUNK):
    return [(a, min(a + chunk, n)) for a in range(0, n, chunk)]


def average(w: np.ndarray, f: np.ndarray) -> tuple[float, float, tuple]:
    """phsp_average's value/error (phasespace.py:319-349) from w and f columns."""
    sw = swf = sw2 = sw2f = sw2f2 = 0.0
    for a, b in chunk_windows(len(w)):
        ws, fs = w[a:b], f[a:b]
        sw += float(np.sum(ws))
        swf += float(np.sum(ws * fs))
        sw2 += float(np.sum(ws * ws))
        sw2f += float(np.sum(ws * ws * fs))
        sw2f2 += float(np.sum(ws * ws * fs * fs))
    mu = swf / sw
    spread = max(sw2f2 - 2.0 * mu * sw2f + mu * mu * sw2, 0.0)
    return mu, math.sqrt(spread) / sw, (sw, swf, sw2, sw2f, sw2f2)


def pair_mass2(block: dict[str, np.ndarray], i: int, j: int) -> np.ndarray:
    """m^2 of daughters i+j, same ufunc order as test_phasespace.py:196-201."""
    e = block[f"p{i}_e"] + block[f"p{j}_e"]
    px = block[f"p{i}_px"] + block[f"p{j}_px"]
    py = block[f"p{i}_py"] + block[f"p{j}_py"]
    pz = block[f"p{i}_pz"] + block[f"p{j}_pz"]
    return e * e - px * px - py * py - pz * pz


def breit_wigner(s: np.ndarray, m0: float, g0: float) -> np.ndarray:
    return 1.0 / ((s - m0 * m0) ** 2 + (m0 * m0) * (g0 * g0))


_SQRT_2PI = math.sqrt(2.0 * math.pi)


def gaussian_norm(mu, sigma, lo, hi) -> float:
    rt2 = math.sqrt(2.0)
    return 0.5 * (math.erf((hi - mu) / (sigma * rt2)) - math.erf((lo - mu) / (sigma * rt2)))


def exponential_norm(tau, lo, hi) -> float:
    return tau * (math.exp(-lo / tau) - math.exp(-hi / tau))


def density(x: np.ndarray, components) -> np.ndarray:
    """sum_k N_k * shape_k(x) / norm_k with the reference's ufunc order.

    components: sequence of ("gauss", N, mu, sigma, norm) / ("exp", N, tau, norm).
    """
    total = None
    for c in components:
        if c[0] == "gauss":
            _, N, mu, s, norm = c
            z = (x - mu) / s
            shape = np.exp(-0.5 * z * z) / (s * _SQRT_2PI)
        elif c[0] == "exp":
            _, N, tau, norm = c
            shape = np.exp(-np.asarray(x, dtype=float) / tau)
        else:
            raise ValueError(c[0])
        term = N * (shape / norm)
        total = term if total is None else total + term
    return total


def nll(x: np.ndarray, components) -> float:
    """Extended NLL (fitting.py:175-210) over x; raises like the reference."""
    d = density(x, components)
    bad = ~(d > 0) | ~np.isfinite(d)
    if np.any(bad):
        j = int(np.argmax(bad))
        raise ValueError(f"model density {d[j]!r} is not positive at event {j}")
    logs = np.log(d)
    acc = None
    for a, b in chunk_windows(len(x)):
        s = float(np.sum(logs[a:b]))
        acc = s if acc is None else acc + s
    return sum(c[1] for c in components) - acc


def gauss_exp_components(mu, sigma, tau, n_sig, n_bkg, lo=0.0, hi=10.0):
    return [("gauss", n_sig, mu, sigma, gaussian_norm(mu, sigma, lo, hi)),
            ("exp", n_bkg, tau, exponential_norm(tau, lo, hi))]
