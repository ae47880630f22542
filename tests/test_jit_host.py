"""CPU tests of functor specialisation (csrc/hk_jit.cu): every opcode's
emitted CUDA compiles with NVRTC for sm_100a -- no GPU needed.  Bitwise
equality with the interpreter is tests/test_jit_gpu.py."""

from __future__ import annotations

import pytest

from tests.common import jit_cases


def _nvrtc_present() -> bool:
    import ctypes
    for name in ("/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12"):
        try:
            ctypes.CDLL(name)
            return True
        except OSError:
            pass
    return False


def _programs(hk):
    from paper_1711_05683_b200.functors import lower_average
    names = hk.phsp_schema(3).names
    return [(name, lower_average(expr, builder, names)[0]) for name, expr, builder in jit_cases(hk)]


def test_cases_cover_every_opcode(hk):
    from paper_1711_05683_b200 import _lib
    seen = set()
    for _, prog in _programs(hk):
        seen.update(prog.op[i] for i in range(prog.n_ops))
    assert seen == set(range(_lib.OP_COL, _lib.OP_UDIV + 1)), sorted(seen)


def test_emitted_source_is_straight_line(hk):
    from paper_1711_05683_b200 import _lib
    for name, prog in _programs(hk):
        src = _lib.jit_source(prog)
        assert "hk_jit_moments" in src and "hk_jit_map" in src, name
        body = src.split("double hk_f(")[1].split("\n}\n")[0]
        assert body.count("const double v") == prog.n_ops, name
        assert "switch" not in body and "for (" not in body, name


@pytest.mark.skipif(not _nvrtc_present(), reason="NVRTC not in this image")
def test_every_program_compiles_for_sm100a(hk):
    from paper_1711_05683_b200 import _lib
    for name, prog in _programs(hk):
        assert _lib.jit_compile(prog) > 1000, name


def test_mode_switch_and_validation(hk):
    from paper_1711_05683_b200 import _lib
    prev = _lib.set_jit_mode(_lib.JIT_OFF)
    try:
        assert _lib.set_jit_mode(_lib.JIT_AUTO) == _lib.JIT_OFF
        with pytest.raises(ValueError):
            _lib.set_jit_mode(7)
        with _lib.jit_mode(_lib.JIT_ALWAYS):
            assert _lib.set_jit_mode(_lib.JIT_ALWAYS) == _lib.JIT_ALWAYS
        assert _lib.set_jit_mode(_lib.JIT_AUTO) == _lib.JIT_AUTO
    finally:
        _lib.set_jit_mode(prev)
    assert _lib.load_library().hk_jit_count() >= 0


@pytest.mark.skipif(not _nvrtc_present(), reason="NVRTC not in this image")
def test_fused_generator_module_compiles(hk):
    """The fused generate+integrate module: the embedded device headers compile
    under NVRTC for every templated final state and both RNG modes."""
    from paper_1711_05683_b200 import _lib
    progs = dict(_programs(hk))
    src = _lib.jit_source(progs["transcendental"], 3, _lib.HK_RNG_REFERENCE)
    assert "integrate_chunks<3, 0, hk::JitIntegrand>" in src
    assert "__ldg" not in src.split("struct JitIntegrand")[1]      # event from registers, not HBM
    for n, mode in ((2, 0), (3, 0), (3, 1), (8, 1)):
        assert _lib.jit_compile(progs["gauss_e1"], n, mode) > 1000, (n, mode)
    with pytest.raises(ValueError):
        _lib.jit_compile(progs["gauss_e1"], 9, 0)
