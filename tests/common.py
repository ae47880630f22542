"""Test helpers: pinned inputs, tolerance checks, a numpy emulation of the
device program interpreter (to test lowering on the CPU)."""

from __future__ import annotations

import numpy as np

B0_MASS = 5.27966
B0_DAUGHTERS = (3.0969, 0.493677, 0.13957039)     # J/psi, K, pi
M_JPSI = 3.0969
M_MU = 0.1056583755


def assert_block_parity(got: np.ndarray, ref: np.ndarray, n_daughters: int, what: str = "") -> None:
    """Parity definition of SURVEY.md 8(c): weights <= 1e-12 relative (expected
    bit-exact), four-momentum components |dc| <= 1e-12 * E_daughter(ref);
    NaN positions must coincide."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    nan_g, nan_r = np.isnan(got), np.isnan(ref)
    assert np.array_equal(nan_g, nan_r), f"{what}: NaN pattern differs"
    w_g, w_r = got[0], ref[0]
    ok = ~nan_r[0]
    rel = np.abs(w_g[ok] - w_r[ok]) / np.maximum(np.abs(w_r[ok]), 1e-300)
    assert rel.size == 0 or rel.max() <= 1e-12, f"{what}: weight rel err {rel.max()}"
    for j in range(n_daughters):
        e_ref = np.abs(ref[1 + 4 * j])
        for c in range(4):
            row = 1 + 4 * j + c
            m = ~nan_r[row] & ~nan_r[1 + 4 * j]
            d = np.abs(got[row][m] - ref[row][m])
            lim = 1e-12 * np.maximum(e_ref[m], 1e-300)
            assert np.all(d <= lim), f"{what}: daughter {j + 1} comp {c} max |d|/E {np.max(d / lim) * 1e-12}"


def run_program_numpy(prog, cols: list[np.ndarray], want_slots: bool = False):
    """Vectorised emulation of hk::run_program (csrc/hk_device.cuh):
    (result, zero-divisor mask[, the final slot values])."""
    from paper_1711_05683_b200 import _lib as L

    n = len(cols[0])
    r = [None] * L.HK_MAX_SLOTS
    div0 = np.zeros(n, dtype=bool)
    with np.errstate(all="ignore"):
        for i in range(prog.n_ops):
            op, a, b = prog.op[i], prog.a[i], prog.b[i]
            if op == L.OP_COL:
                v = np.asarray(cols[a], dtype=np.float64)
            elif op == L.OP_CONST:
                v = np.full(n, prog.cst[i])
            elif op == L.OP_ADD:
                v = r[a] + r[b]
            elif op == L.OP_SUB:
                v = r[a] - r[b]
            elif op == L.OP_MUL:
                v = r[a] * r[b]
            elif op == L.OP_DIV:
                div0 |= r[b] == 0
                v = r[a] / r[b]
            elif op == L.OP_NEG:
                v = -r[a]
            elif op == L.OP_SQRT:
                v = np.sqrt(r[a])
            elif op == L.OP_EXP:
                v = np.exp(r[a])
            elif op == L.OP_LOG:
                v = np.log(r[a])
            elif op == L.OP_GAUSS:
                z = (r[a] - prog.cst[i]) / prog.cst2[i]
                v = np.exp(-0.5 * z * z) / (prog.cst2[i] * 2.5066282746310002)
            elif op == L.OP_EXPO:
                v = np.exp(-r[a] / prog.cst[i])
            elif op == L.OP_BW:
                m0, g0 = prog.cst[i], prog.cst2[i]
                t = r[a] - m0 * m0
                v = 1.0 / (t * t + (m0 * m0) * (g0 * g0))
            elif op == L.OP_ADD0:
                v = r[a] + 0.0
            elif op == L.OP_UDIV:
                v = r[a] / r[b]
            elif op == L.OP_SQUARE:
                v = r[a] * r[a]
            else:
                raise ValueError(op)
            r[prog.dst[i]] = v
    return (r[prog.result], div0, r) if want_slots else (r[prog.result], div0)


def m12sq_builder(cols):
    """The reference's own pinned integrand argument (test_phasespace.py:196-201)."""
    e = cols["p1_e"] + cols["p2_e"]
    px = cols["p1_px"] + cols["p2_px"]
    py = cols["p1_py"] + cols["p2_py"]
    pz = cols["p1_pz"] + cols["p2_pz"]
    return (e * e - px * px - py * py - pz * pz,)


def m23sq_builder(cols):
    e = cols["p2_e"] + cols["p3_e"]
    px = cols["p2_px"] + cols["p3_px"]
    py = cols["p2_py"] + cols["p3_py"]
    pz = cols["p2_pz"] + cols["p3_pz"]
    return (e * e - px * px - py * py - pz * pz,)


def jit_cases(hk):
    """(name, expr, arg_builder) over the phase-space schema covering every
    program opcode -- shared by the specialisation tests (host + GPU)."""
    import numpy as np

    mean, sigma, tau = hk.Parameter("mean", 3.0), hk.Parameter("sigma", 0.4), hk.Parameter("tau", 1.7)
    return [
        ("m12sq", hk.identity(), m12sq_builder),
        ("bw_m23sq", hk.breit_wigner(0.89555, 0.0473), m23sq_builder),
        ("gauss_e1", hk.shape_gaussian(mean, sigma), lambda c: (c["p1_e"],)),
        ("expo_e3", hk.shape_exponential(tau), lambda c: (c["p3_e"],)),
        ("product", hk.identity() * hk.identity(), m12sq_builder),
        ("ratio", hk.identity(), lambda c: (c["p1_e"] / c["p2_pz"],)),
        ("transcendental", hk.identity(),
         lambda c: (np.log(c["p1_e"]) + np.sqrt(c["p2_e"]) * np.exp(-c["p3_e"]),)),
        ("coordinate", hk.coordinate(1, 2), lambda c: (c["p1_e"], c["p2_px"])),
        ("square_neg", hk.identity(), lambda c: (-(c["p1_px"] ** 2) - c["weight"],)),
        ("constant", hk.constant(2.5), lambda c: (c["p1_e"],)),
        ("checked_div", hk.combine("/", hk.identity(), hk.constant(3.0)), m12sq_builder),
    ]
