"""CPU tests: the C ABI surface, host-side logic, and program lowering
(checked with a numpy emulation of the device interpreter against the oracle)."""

from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS, m12sq_builder, m23sq_builder, run_program_numpy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions() -> set[str]:
    text = open(os.path.join(ROOT, "include", "hepkit_cuda.h")).read()
    return set(re.findall(r"^(?:int|int32_t|int64_t|double)\s+(hk_\w+)\(", text, flags=re.M))


def test_library_exports_every_declared_symbol(hk):
    from paper_1711_05683_b200 import _lib
    lib = _lib.load_library()
    declared = _header_functions()
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.hk_abi_version() == 1
    assert lib.hk_num_chunks(0) == 0
    assert lib.hk_num_chunks(4096) == 1
    assert lib.hk_num_chunks(4097) == 2
    assert lib.hk_num_chunks(10**10) == (10**10 + 4095) // 4096


def test_every_entry_point_marshals_and_validates(hk):
    """Call each C entry point through the ctypes signatures with empty work
    (validation runs, no kernel is launched) -- catches ABI drift on the CPU."""
    from paper_1711_05683_b200 import _lib
    L = _lib.load_library()
    spec = hk.DecaySpec(5.27966, (3.0969, 0.493677, 0.13957039))
    d = _lib.make_decay(spec)
    k = _lib.make_key(hk.RngKey(1, 1))
    cols = (ctypes.c_void_p * 65)(*([1] * 65))
    prog = hk.functors.compile_program(("add", ("col", 1), ("const", 2.0)))
    model = _lib.hk_model_t()
    model.n_comp, model.kind[0], model.yield_[0], model.norm[0], model.p0[0], model.p1[0] = 1, 0, 1.0, 1.0, 0.0, 1.0
    dummy = ctypes.create_string_buffer(1 << 16)
    dp = ctypes.addressof(dummy)
    two = (ctypes.c_double * 2)()
    OK = _lib.HK_OK
    assert L.hk_rng_raw64(k, None, 0, None, None) == OK
    assert L.hk_rng_uniform(k, None, 0, None, None) == OK
    assert L.hk_phsp_generate(d, k, 0, 0, cols, None, None) == OK
    assert L.hk_phsp_generate_host(d, k, 0, 0, cols, two, dp, len(dummy), None) == OK
    assert L.hk_phsp_decay_chain(dp, cols, d, k, 0, 0, dp, cols, None, None) == OK
    assert L.hk_phsp_generate_chain(d, k, 1, d, k, 0, 0, cols, None, None, None) == OK
    assert L.hk_phsp_moments(cols, 13, 0, prog, dp, None, None) == OK
    assert L.hk_phsp_integrate(d, k, 0, 0, prog, None, dp, None, None) == OK
    pair = _lib.hk_pair_integrand_t(_lib.HK_PAIR_BW, 1, 2, 0, 0.89555, 0.0473)
    assert L.hk_phsp_integrate(d, k, 0, 0, None, pair, dp, None, None) == OK
    pair.i = 5
    assert L.hk_phsp_integrate(d, k, 0, 10, None, pair, dp, None, None) == _lib.HK_EINVAL
    assert L.hk_map_program(cols, 13, 0, prog, dp, None, None) == OK
    assert L.hk_nll_partials(dp, 0, model, dp, None, None) == OK
    assert L.hk_model_density(dp, 0, model, dp, None) == OK
    assert L.hk_yield_partials(dp, 0, model, dp, None, None) == OK
    assert L.hk_unweight_flags(dp, 0, 1.0, k, 0, dp, dp, None, None) == OK
    assert L.hk_compact(cols, 13, 0, dp, dp, cols, 0, None) == OK
    lo = (ctypes.c_double * 1)(0.0)
    assert L.hk_sample_pdf(prog, 1, lo, lo, 1.0, k, 0, 0, 10, cols, dp, None) == OK
    assert L.hk_fold_segments(None, 0, 8, 2, None, None) == OK
    assert L.hk_fold_segments(dp, 4, 0, 2, dp, None) == _lib.HK_EINVAL
    assert L.hk_csv_scratch_bytes(0, 13) == 0
    assert L.hk_csv_scratch_bytes(1000, 13) > 1000 * 13 * 24
    text_len = ctypes.c_int64(-1)
    assert L.hk_format_csv(cols, 13, 0, None, None, 0, ctypes.byref(text_len), None) == OK
    assert text_len.value == 0
    assert L.hk_format_csv(cols, 13, 10, dp, dp, 100, ctypes.byref(text_len), None) == _lib.HK_EINVAL
    assert "capacity" in _lib.last_error()
    # validation errors come back as HK_EINVAL with a message
    assert L.hk_nll_eval(dp, 0, model, dp, two, ctypes.byref(ctypes.c_uint64()), None) == _lib.HK_EINVAL
    assert "empty" in _lib.last_error()
    bad = _lib.make_decay(spec)
    bad.n = 1
    assert L.hk_phsp_generate(bad, k, 0, 10, cols, None, None) == _lib.HK_EINVAL
    assert "daughter count" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(L.hk_phsp_generate(bad, k, 0, 10, cols, None, None), "generate")
    nd, sm = ctypes.c_int(-1), ctypes.c_int(-1)
    assert L.hk_device_info(ctypes.byref(nd), ctypes.byref(sm)) == OK
    assert nd.value >= 0


def test_clique_lifetime_validation(hk):
    """hk_init / hk_shutdown / the clique collectives: argument and state
    checks run on the host (no device, no NCCL needed)."""
    import torch
    from paper_1711_05683_b200 import _lib
    L = _lib.load_library()
    bufs = (ctypes.c_void_p * 1)(1)
    if not torch.cuda.is_available():
        assert L.hk_init(1) == _lib.HK_EINVAL
        assert "visible" in _lib.last_error()
        with pytest.raises(ValueError):
            _lib.init(1)
    assert L.hk_init(0) == _lib.HK_EINVAL
    assert L.hk_shutdown() == _lib.HK_OK      # idempotent, nothing to release
    assert L.hk_clique_size() == 0
    assert L.hk_allreduce_partials(bufs, 1, 4, None) == _lib.HK_EINVAL
    assert "hk_init" in _lib.last_error()
    assert L.hk_allgather_partials(bufs, bufs, 1, 4, None) == _lib.HK_EINVAL
    assert "hk_init" in _lib.last_error()


def test_struct_layouts_match_header(hk, tmp_path):
    """Every ctypes mirror has the C compiler's size and field offsets for the
    structs include/hepkit_cuda.h declares."""
    import shutil
    import subprocess
    from paper_1711_05683_b200 import _lib
    cc = shutil.which("gcc")
    if cc is None:
        pytest.skip("no host compiler")
    structs = {"hk_key_t": _lib.hk_key_t, "hk_decay_t": _lib.hk_decay_t, "hk_program_t": _lib.hk_program_t,
               "hk_model_t": _lib.hk_model_t, "hk_pair_integrand_t": _lib.hk_pair_integrand_t,
               "hk_density_t": _lib.hk_density_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hepkit_cuda.h"', "int main(void) {"]
    want = []
    for cname, py in structs.items():
        lines.append(f'printf("%zu\\n", sizeof({cname}));')
        want.append(ctypes.sizeof(py))
        for fname, _ in py._fields_:
            cfield = "yield" if fname == "yield_" else fname
            lines.append(f'printf("%zu\\n", offsetof({cname}, {cfield}));')
            want.append(getattr(py, fname).offset)
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == want


def test_no_device_fails_loudly(hk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(hk.DeviceUnavailable):
        hk.phsp_generate(hk.DecaySpec(1.0, (0.1, 0.2)), hk.FourVector.at_rest(1.0), 10, hk.RngKey(1, 1))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1711_05683_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("Oracle", ""), f


class TestHostKinematics:
    def test_breakup_known_answers(self, hk, golden):
        _, s = golden
        assert hk.breakup_momentum(2.0, 0.5, 0.3) == s["kat"]["breakup_2_05_03"] == 0.9119210492142398
        assert hk.breakup_momentum(1.0, 0.5, 0.5) == 0.0
        assert hk.breakup_momentum(1.0, 0.0, 0.0) == 0.5
        with pytest.raises(hk.BelowThreshold):
            hk.breakup_momentum(0.9, 0.5, 0.5)

    def test_max_weight_matches_reference(self, hk, golden):
        _, s = golden
        for b in s["gen_blocks"]:
            assert hk.phsp_max_weight(hk.DecaySpec(b["M"], tuple(b["masses"]))) == b["max_weight"]

    def test_decay_spec_validation(self, hk):
        with pytest.raises(hk.BelowThreshold):
            hk.DecaySpec(1.0, (0.5, 0.5))
        with pytest.raises(ValueError):
            hk.DecaySpec(1.0, (0.5,))
        with pytest.raises(ValueError):
            hk.DecaySpec(1.0, (0.5, -0.1))

    def test_boost_into_z(self, hk):
        beta = 0.6
        g = 1 / math.sqrt(1 - beta * beta)
        v = hk.boost_into(hk.FourVector(1.0, 0.0, 0.0, 0.0), hk.FourVector(g, 0.0, 0.0, g * beta))
        assert v.e == pytest.approx(g, rel=1e-15)
        assert v.pz == pytest.approx(g * beta, rel=1e-15)

    def test_schema(self, hk):
        assert hk.phsp_schema(2).names == ("weight", "p1_e", "p1_px", "p1_py", "p1_pz",
                                           "p2_e", "p2_px", "p2_py", "p2_pz")


class TestLowering:
    """Lowered programs, run by a numpy emulation of the kernel interpreter,
    reproduce the reference integrands on oracle blocks."""

    def _block(self, oracle, n=20_000):
        return oracle.generate(B0_DAUGHTERS, B0_MASS, n, 5, 1)

    def test_pair_mass_identity_bit_exact(self, hk, oracle):
        from paper_1711_05683_b200.functors import lower_average
        blk = self._block(oracle)
        names = hk.phsp_schema(3).names
        prog, _ = lower_average(hk.identity(), m12sq_builder, names)
        f, div0 = run_program_numpy(prog, [blk[n] for n in names])
        assert np.array_equal(f, oracle.pair_mass2(blk, 1, 2) + 0.0)
        assert not div0.any()

    def test_breit_wigner_builtin(self, hk, oracle):
        from paper_1711_05683_b200.functors import lower_average
        blk = self._block(oracle)
        names = hk.phsp_schema(3).names
        prog, _ = lower_average(hk.breit_wigner(0.89555, 0.0473), m23sq_builder, names)
        f, _ = run_program_numpy(prog, [blk[n] for n in names])
        ref = oracle.breit_wigner(oracle.pair_mass2(blk, 2, 3), 0.89555, 0.0473)
        assert np.array_equal(f, ref)

    def test_algebra_and_composition(self, hk, oracle):
        from paper_1711_05683_b200.functors import lower_average
        blk = self._block(oracle, 5000)
        names = hk.phsp_schema(3).names
        mu, s, tau = hk.Parameter("mu", 10.0), hk.Parameter("s", 2.0), hk.Parameter("tau", 3.0)
        g = hk.shape_gaussian(mu, s)
        e = hk.shape_exponential(tau)
        expr = hk.compose(g + e * hk.identity(), [hk.identity()]) / (hk.identity() + hk.constant(1.0))
        prog, _ = lower_average(expr, m12sq_builder, names)
        f, _ = run_program_numpy(prog, [blk[n] for n in names])
        x = oracle.pair_mass2(blk, 1, 2)
        ref = expr.eval((x,))
        assert np.array_equal(f, ref)

    def test_closure_tracing(self, hk, oracle):
        from paper_1711_05683_b200.functors import lower_average
        blk = self._block(oracle, 3000)
        names = hk.phsp_schema(3).names
        clo = hk.wrap_closure(lambda x, p: np.sqrt(x[0]) * 2.0 + x[0] ** 2 - np.log(x[0]))
        prog, _ = lower_average(clo, m12sq_builder, names)
        f, _ = run_program_numpy(prog, [blk[n] for n in names])
        x = oracle.pair_mass2(blk, 1, 2) + 0.0
        assert np.array_equal(f, np.sqrt(x) * 2.0 + x ** 2 - np.log(x))

    def test_untraceable_raises(self, hk):
        from paper_1711_05683_b200.functors import lower_average
        names = hk.phsp_schema(3).names
        bad = hk.wrap_closure(lambda x, p: np.where(x[0] > 1, 1.0, 0.0))
        with pytest.raises(NotImplementedError):
            lower_average(bad, m12sq_builder, names)
        with pytest.raises(NotImplementedError):
            lower_average(hk.identity(), lambda cols: (np.sin(cols["p1_e"]),), names)

    def test_pair_integrand_recognition(self, hk):
        from paper_1711_05683_b200 import _lib
        from paper_1711_05683_b200.functors import lower_average, match_pair_integrand
        names = hk.phsp_schema(3).names
        _, _, root = lower_average(hk.identity(), m12sq_builder, names, with_root=True)
        p = match_pair_integrand(root, 3)
        assert p is not None and (p.kind, p.i, p.j) == (_lib.HK_PAIR_MASS2, 0, 1)
        _, _, root = lower_average(hk.breit_wigner(0.89555, 0.0473), m23sq_builder, names, with_root=True)
        p = match_pair_integrand(root, 3)
        assert (p.kind, p.i, p.j, p.m0, p.g0) == (_lib.HK_PAIR_BW, 1, 2, 0.89555, 0.0473)
        # anything else stays on the generic interpreter
        _, _, root = lower_average(hk.identity() * hk.identity(), m12sq_builder, names, with_root=True)
        assert match_pair_integrand(root, 3) is None
        _, _, root = lower_average(hk.identity(), lambda c: (c["p1_e"] * c["p2_e"],), names, with_root=True)
        assert match_pair_integrand(root, 3) is None

    def test_program_register_budget(self, hk):
        from paper_1711_05683_b200.functors import compile_program
        node = ("col", 0)
        for k in range(1, 20):     # long dependent chain: needs 2 live slots
            node = ("add", node, ("col", k % 13))
        prog = compile_program(node)
        assert max(prog.dst[i] for i in range(prog.n_ops)) < 4


class TestHostFit:
    def test_minimize_quadratic(self, hk):
        a = hk.Parameter("a", 0.0, step=0.5)
        res = hk.minimize(lambda ps: (ps["a"].value - 3.0) ** 2, hk.ParamSet([a]))
        assert res.status is hk.FitStatus.CONVERGED
        assert a.value == pytest.approx(3.0, abs=1e-4)
        assert res.errors["a"] == pytest.approx(0.7071067811865475, rel=1e-4)

    def test_constant_shift_invariance(self, hk):
        base = lambda ps: (ps["a"].value - 2.0) ** 4 + (ps["a"].value + 1.0) ** 2  # noqa: E731
        a1 = hk.Parameter("a", 0.3, step=0.4)
        r1 = hk.minimize(base, hk.ParamSet([a1]))
        a2 = hk.Parameter("a", 0.3, step=0.4)
        r2 = hk.minimize(lambda ps: base(ps) + 4.0, hk.ParamSet([a2]))
        assert a2.value == a1.value and r2.nll_min == r1.nll_min + 4.0

    def test_bounded_and_fixed(self, hk):
        obj = lambda ps: (ps["a"].value - 1.5) ** 2 + 0.7  # noqa: E731
        free = hk.Parameter("a", 0.2, step=0.3)
        rf = hk.minimize(obj, hk.ParamSet([free]))
        bnd = hk.Parameter("a", 0.2, step=0.3, lower=-5.0, upper=5.0)
        rb = hk.minimize(obj, hk.ParamSet([bnd]))
        assert bnd.value == pytest.approx(free.value, abs=5e-4)
        assert rb.nll_min == pytest.approx(rf.nll_min, abs=1e-7)
        b = hk.Parameter("b", 2.5, fixed=True)
        hk.minimize(lambda ps: (ps["a"].value - 1.0) ** 2 + ps["b"].value,
                    hk.ParamSet([hk.Parameter("a", 0.0, step=0.5), b]))
        assert b.value == 2.5

    def test_rosenbrock_and_max_iterations(self, hk):
        x, y = hk.Parameter("x", -1.0, step=0.2), hk.Parameter("y", 1.5, step=0.2)
        res = hk.minimize(lambda ps: (1 - ps["x"].value) ** 2 + 5.0 * (ps["y"].value - ps["x"].value ** 2) ** 2,
                          hk.ParamSet([x, y]), max_iterations=5000)
        assert res.status is hk.FitStatus.CONVERGED
        assert x.value == pytest.approx(1.0, abs=1e-3) and y.value == pytest.approx(1.0, abs=1e-3)
        a = hk.Parameter("a", 100.0, step=0.001)
        r = hk.minimize(lambda ps: abs(ps["a"].value), hk.ParamSet([a]), max_iterations=3)
        assert r.status is hk.FitStatus.MAX_ITERATIONS and r.errors is None

    def test_numeric_errors_correlated(self, hk):
        H = np.array([[2.0, 0.6], [0.6, 1.0]])
        ps = hk.ParamSet([hk.Parameter("x", 0.0), hk.Parameter("y", 0.0)])
        err = hk.numeric_errors(lambda p: 0.5 * float(np.array([p["x"].value, p["y"].value]) @ H
                                                      @ np.array([p["x"].value, p["y"].value])), ps)
        cov = np.linalg.inv(H)
        assert err["x"] == pytest.approx(math.sqrt(cov[0, 0]), rel=1e-5)
        assert hk.numeric_errors(lambda p: -p["x"].value ** 2, hk.ParamSet([hk.Parameter("x", 0.0)])) is None

    def test_norms(self, hk):
        e = hk.shape_exponential(hk.Parameter("tau", 1.0))
        pdf = hk.make_pdf(e, hk.exponential_norm(e), hk.BoundedRegion(((0.0, 10.0),)))
        assert pdf.norm() == pytest.approx(0.9999546000702375, rel=1e-14)
        g = hk.shape_gaussian(hk.Parameter("m", 0.0), hk.Parameter("s", 1.0))
        pg = hk.make_pdf(g, hk.gaussian_norm(g), hk.BoundedRegion(((-10.0, 10.0),)))
        assert pg.value((0.0,)) == pytest.approx(0.3989422804014327, rel=1e-13)
        for _ in range(3):
            pg.value((1.0,))
        assert pg.norm_computations == 1


class TestStoreAndSharding:
    def test_store_host_ops(self, hk, tmp_path):
        s = hk.ColumnStore(hk.ColumnSchema.real64("a", "b"))
        for i in range(10):
            s.push((float(i), float(i * i)))
        assert len(s) == 10 and s.row(3) == (3.0, 9.0)
        sel = s.where_mask(np.arange(10) % 3 == 0)
        assert sel.column("a").tolist() == [0.0, 3.0, 6.0, 9.0]
        p = tmp_path / "x.csv"
        s.write_csv(str(p))
        back = hk.read_csv(str(p))
        assert np.array_equal(back.column("b"), s.column("b"))
        with pytest.raises(ValueError):
            hk.ColumnSchema.real64("a", "a")

    def test_shard_ranges_cover_and_align(self):
        from paper_1711_05683_b200.parallel import CHUNK, shard_range
        for n in (0, 1, 4095, 4096, 4097, 10**6, 10**8 + 17):
            for world in (1, 2, 3, 4, 8):
                rs = [shard_range(n, r, world) for r in range(world)]
                assert rs[0][0] == 0 and rs[-1][1] == n
                for (a0, b0), (a1, _) in zip(rs, rs[1:]):
                    assert b0 == a1
                for a, b in rs:
                    assert a % CHUNK == 0 and a <= b


@pytest.mark.parametrize("lang,std", [("c", "-std=c99"), ("c++", "-std=c++17")])
def test_header_is_plain_c_and_cpp(lang, std):
    """include/hepkit_cuda.h is the drop-in boundary for C / cgo / JNI hosts:
    it must compile as pedantic C99 and as C++ with no CUDA or torch types."""
    import shutil
    import subprocess
    cc = shutil.which("gcc" if lang == "c" else "g++")
    if cc is None:
        pytest.skip("no host compiler")
    hdr = os.path.join(ROOT, "include", "hepkit_cuda.h")
    r = subprocess.run([cc, std, "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only", "-x", lang, hdr],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_chain_fixed_frame_mass_predicate(hk):
    """hk_chain_fixed_frame_mass (host only): m_k for the C3 chain (J/psi,
    gamma <= 1.2), 0 for a sub-decay mother off by more than a quarter of the
    mismatch tolerance, a massless daughter, or a daughter boosted beyond
    gamma 4 (the pion of B0 -> J/psi K pi)."""
    from paper_1711_05683_b200 import _lib
    L = _lib.load_library()
    spec = _lib.make_decay(hk.DecaySpec(B0_MASS, B0_DAUGHTERS))
    jpsi = B0_DAUGHTERS[0]
    assert L.hk_chain_fixed_frame_mass(spec, 1, _lib.make_decay(hk.DecaySpec(jpsi, (0.105, 0.105)))) == jpsi
    near = _lib.make_decay(hk.DecaySpec(jpsi * (1 + 0.2e-9), (0.105, 0.105)))
    assert L.hk_chain_fixed_frame_mass(spec, 1, near) == jpsi
    off = _lib.make_decay(hk.DecaySpec(jpsi * (1 + 0.5e-9), (0.105, 0.105)))
    assert L.hk_chain_fixed_frame_mass(spec, 1, off) == 0.0
    pion = _lib.make_decay(hk.DecaySpec(B0_DAUGHTERS[2], (0.0, 0.0)))
    assert L.hk_chain_fixed_frame_mass(spec, 3, pion) == 0.0
    massless = _lib.make_decay(hk.DecaySpec(2.0, (0.0, 0.5)))
    assert L.hk_chain_fixed_frame_mass(massless, 1, _lib.make_decay(hk.DecaySpec(0.3, (0.1, 0.1)))) == 0.0
    assert L.hk_chain_fixed_frame_mass(spec, 4, pion) == 0.0


def test_python_constants_match_header(hk):
    """Every integer #define of include/hepkit_cuda.h that _lib mirrors has
    the header's value (sizes, limits, sentinels)."""
    import os
    import re
    from paper_1711_05683_b200 import _lib
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "include", "hepkit_cuda.h")).read()
    seen = 0
    for name, value in re.findall(r"#define\s+(HK_\w+)\s+(0x[0-9A-Fa-f]+|\d+)\b", text):
        if hasattr(_lib, name):
            assert getattr(_lib, name) == int(value, 0), name
            seen += 1
    assert seen >= 8
    assert _lib.HK_SUPERS == 1024
