"""ctypes binding of libhepkit_cuda.so (include/hepkit_cuda.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
hot-path call raises :class:`DeviceUnavailable`.  Device memory, streams and
(multi-GPU) collectives come from PyTorch; all arithmetic on the hot path is
in the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HK_LIB_PATH") or os.path.join(HERE, "libhepkit_cuda.so")

HK_OK, HK_EINVAL, HK_ECUDA, HK_EDOMAIN, HK_EUNSUPPORTED = 0, 1, 2, 3, 4
HK_CHUNK = 4096
HK_MAX_DAUGHTERS = 16
HK_MAX_PROGRAM = 256
HK_MAX_SLOTS = 32
HK_MAX_COMPONENTS = 8
HK_MAX_POINTS = 64
HK_NO_BAD_ROW = (1 << 64) - 1
HK_RNG_REFERENCE, HK_RNG_PHILOX = 0, 1
HK_SHAPE_GAUSS, HK_SHAPE_EXPO = 0, 1

# opcodes (enum hk_opcode)
OP_COL, OP_CONST, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG, OP_SQRT, OP_EXP, OP_LOG = range(10)
OP_GAUSS, OP_EXPO, OP_BW, OP_ADD0, OP_SQUARE, OP_UDIV = range(10, 16)

# symbols the header declares; tests check the .so exports every one
EXPORTS = (
    "hk_abi_version", "hk_last_error", "hk_device_info", "hk_num_chunks",
    "hk_rng_raw64", "hk_rng_uniform",
    "hk_phsp_generate", "hk_phsp_generate_host", "hk_phsp_decay_chain", "hk_phsp_generate_chain",
    "hk_chain_fixed_frame_mass", "hk_column_stats", "hk_column_stats_work_doubles",
    "hk_phsp_moments", "hk_map_program", "hk_phsp_integrate", "hk_fold_partials",
    "hk_nll_partials", "hk_nll_eval", "hk_model_density",
    "hk_yield_partials", "hk_splot_weights",
    "hk_sample_pdf", "hk_unweight_flags", "hk_compact", "hk_scan_counts",
    "hk_set_jit_mode", "hk_jit_count", "hk_jit_source", "hk_jit_compile",
    "hk_csv_scratch_bytes", "hk_format_csv", "hk_nll_work_doubles", "hk_fold_segments",
    "hk_init", "hk_shutdown", "hk_clique_size", "hk_allreduce_partials", "hk_allgather_partials",
    "hk_fold_supers", "hk_philox4x32_10",
    "hk_nll_program_eval", "hk_ratio_partials_program", "hk_splot_weights_program", "hk_nll_combine",
    "hk_nll_eval_many", "hk_nll_many_work_doubles",
    "hk_fcn_session_start", "hk_fcn_session_eval", "hk_fcn_session_stop", "hk_fcn_session_device_ns",
)


class DeviceUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is not available (no CPU fallback)."""


class KernelError(RuntimeError):
    """A library call failed for a reason other than a per-event domain error."""


class hk_key_t(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("stream", ctypes.c_uint64),
                ("counter", ctypes.c_uint64), ("mode", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class hk_decay_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("moving", ctypes.c_int32),
                ("mother_mass", ctypes.c_double), ("T", ctypes.c_double),
                ("masses", ctypes.c_double * HK_MAX_DAUGHTERS),
                ("csum", ctypes.c_double * HK_MAX_DAUGHTERS),
                ("mother", ctypes.c_double * 4), ("m_mother", ctypes.c_double)]


class hk_program_t(ctypes.Structure):
    _fields_ = [("n_ops", ctypes.c_int32), ("result", ctypes.c_int32),
                ("op", ctypes.c_int32 * HK_MAX_PROGRAM), ("dst", ctypes.c_int32 * HK_MAX_PROGRAM),
                ("a", ctypes.c_int32 * HK_MAX_PROGRAM), ("b", ctypes.c_int32 * HK_MAX_PROGRAM),
                ("cst", ctypes.c_double * HK_MAX_PROGRAM), ("cst2", ctypes.c_double * HK_MAX_PROGRAM)]


class hk_model_t(ctypes.Structure):
    _fields_ = [("n_comp", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("kind", ctypes.c_int32 * HK_MAX_COMPONENTS),
                ("yield_", ctypes.c_double * HK_MAX_COMPONENTS),
                ("norm", ctypes.c_double * HK_MAX_COMPONENTS),
                ("p0", ctypes.c_double * HK_MAX_COMPONENTS),
                ("p1", ctypes.c_double * HK_MAX_COMPONENTS),
                ("has_stats", ctypes.c_int32), ("_pad2", ctypes.c_int32), ("x_count", ctypes.c_int64),
                ("x_min", ctypes.c_double), ("x_max", ctypes.c_double), ("x_sum", ctypes.c_double)]


HK_FCN_MAX_OBS = 8


class hk_density_t(ctypes.Structure):
    _fields_ = [("n_obs", ctypes.c_int32), ("n_comp", ctypes.c_int32),
                ("pdf_slot", ctypes.c_int32 * HK_MAX_COMPONENTS),
                ("yield_", ctypes.c_double * HK_MAX_COMPONENTS),
                ("program", hk_program_t)]


HK_PAIR_NONE, HK_PAIR_MASS2, HK_PAIR_BW = 0, 1, 2


class hk_pair_integrand_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("i", ctypes.c_int32), ("j", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("m0", ctypes.c_double), ("g0", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int32
_D = ctypes.POINTER(hk_decay_t)      # structs: ctypes passes byref automatically
_K = ctypes.POINTER(hk_key_t)
_F = ctypes.POINTER(hk_program_t)
_M = ctypes.POINTER(hk_model_t)
_DM = ctypes.POINTER(hk_density_t)
_PP = ctypes.POINTER(ctypes.c_void_p)  # double* const* column-pointer arrays
_PD = ctypes.POINTER(ctypes.c_double)  # host doubles
_PU = ctypes.POINTER(ctypes.c_uint64)  # host u64
_INT = ctypes.c_int
_SIGS = {
    "hk_abi_version": (_INT, []),
    "hk_last_error": (_INT, [ctypes.c_char_p, ctypes.c_size_t]),
    "hk_device_info": (_INT, [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "hk_num_chunks": (_I64, [_I64]),
    "hk_rng_raw64": (_INT, [_K, _P, _I64, _P, _P]),
    "hk_rng_uniform": (_INT, [_K, _P, _I64, _P, _P]),
    "hk_philox4x32_10": (_INT, [_P, _I64, _P, _P]),
    "hk_phsp_generate": (_INT, [_D, _K, _U64, _I64, _PP, _P, _P]),
    "hk_phsp_generate_host": (_INT, [_D, _K, _U64, _I64, _PP, _PD, _P, ctypes.c_size_t, _P]),
    "hk_phsp_decay_chain": (_INT, [_P, _PP, _D, _K, _U64, _I64, _P, _PP, _P, _P]),
    "hk_phsp_generate_chain": (_INT, [_D, _K, _I32, _D, _K, _U64, _I64, _PP, _P, _P, _P]),
    "hk_chain_fixed_frame_mass": (ctypes.c_double, [_D, _I32, _D]),
    "hk_column_stats": (_INT, [_P, _I64, _P, _PD, _P]),
    "hk_column_stats_work_doubles": (_I64, [_I64]),
    "hk_phsp_moments": (_INT, [_PP, _I32, _I64, _F, _P, _P, _P]),
    "hk_phsp_integrate": (_INT, [_D, _K, _U64, _I64, _F, ctypes.POINTER(hk_pair_integrand_t), _P, _P, _P]),
    "hk_map_program": (_INT, [_PP, _I32, _I64, _F, _P, _P, _P]),
    "hk_fold_partials": (_INT, [_P, _I64, _I32, _P, _P]),
    "hk_nll_partials": (_INT, [_P, _I64, _M, _P, _P, _P]),
    "hk_nll_eval": (_INT, [_P, _I64, _M, _P, _PD, _PU, _P]),
    "hk_nll_program_eval": (_INT, [_PP, _I64, _DM, _P, _PD, _PU, _PU, _P]),
    "hk_ratio_partials_program": (_INT, [_PP, _I64, _DM, _P, _P, _P]),
    "hk_nll_combine": (_INT, [_P, _I32, _PD, _PU, _PU, _P]),
    "hk_nll_eval_many": (_INT, [_P, _I64, _M, _I32, _P, _PD, _PU, _P]),
    "hk_nll_many_work_doubles": (_I64, [_I64, _I32]),
    "hk_fcn_session_start": (_INT, [_P, _I64, _P, _I64]),
    "hk_fcn_session_eval": (_INT, [_M, _PD, _PU]),
    "hk_fcn_session_stop": (_INT, []),
    "hk_fcn_session_device_ns": (_I64, []),
    "hk_splot_weights_program": (_INT, [_PP, _I64, _DM, _PD, _PP, _P, _P]),
    "hk_model_density": (_INT, [_P, _I64, _M, _P, _P]),
    "hk_yield_partials": (_INT, [_P, _I64, _M, _P, _P, _P]),
    "hk_splot_weights": (_INT, [_P, _I64, _M, _PD, _PP, _P, _P]),
    "hk_unweight_flags": (_INT, [_P, _I64, ctypes.c_double, _K, _U64, _P, _P, _P, _P]),
    "hk_compact": (_INT, [_PP, _I32, _I64, _P, _P, _PP, _I32, _P]),
    "hk_scan_counts": (_INT, [_P, _I64, _P, _P, _P]),
    "hk_sample_pdf": (_INT, [_F, _I32, _PD, _PD, ctypes.c_double, _K, _U64, _I64, _I32, _PP, _P, _P]),
    "hk_set_jit_mode": (_INT, [_I32]),
    "hk_jit_count": (_I64, []),
    "hk_jit_source": (_I64, [_F, _I32, _I32, ctypes.c_char_p, _I64]),
    "hk_jit_compile": (_INT, [_F, _I32, _I32, ctypes.POINTER(_I64)]),
    "hk_csv_scratch_bytes": (_I64, [_I64, _I32]),
    "hk_nll_work_doubles": (_I64, [_I64]),
    "hk_fold_segments": (_INT, [_P, _I64, _I32, _I32, _P, _P]),
    "hk_fold_supers": (_INT, [_P, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P]),
    "hk_format_csv": (_INT, [_PP, _I32, _I64, _P, _P, _I64, ctypes.POINTER(_I64), _P]),
    "hk_init": (_INT, [_I32]),
    "hk_shutdown": (_INT, []),
    "hk_clique_size": (_I32, []),
    "hk_allreduce_partials": (_INT, [_PP, _I32, _I64, _PP]),
    "hk_allgather_partials": (_INT, [_PP, _PP, _I32, _I64, _PP]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen the library and attach signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise DeviceUnavailable(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load_library().hk_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != HK_OK:
        msg = last_error()
        if rc == HK_EINVAL:
            raise ValueError(f"{what}: {msg}")
        if rc == HK_EUNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise KernelError(f"{what} failed (rc={rc}): {msg}")


_torch = None


def torch():
    """Import torch lazily (it is plumbing: allocation, streams, collectives)."""
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


_device_ok = False


def _require_device() -> None:
    global _device_ok
    if not _device_ok:
        if not torch().cuda.is_available():
            raise DeviceUnavailable("no CUDA device is visible; the hot path has no CPU fallback")
        load_library()
        _device_ok = True


def device():
    """The current CUDA device; raises when there is none (no CPU fallback)."""
    _require_device()
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def lib() -> ctypes.CDLL:
    _require_device()
    return _lib


_raw_stream = None
_get_device = None


def current_device() -> int:
    """Index of the current CUDA device (torch's C-level query when it exists:
    no Python wrapper layers on the FCN's per-call path)."""
    global _get_device
    if _get_device is None:
        t = torch()
        _get_device = getattr(t._C, "_cuda_getDevice", None) or t.cuda.current_device
    return _get_device()


def stream_ptr() -> int:
    """cudaStream_t of torch's current stream on the current device (honours
    `with torch.cuda.stream(...)`).  Uses torch's raw-stream query when it
    exists -- it skips building a Stream object (3 us -> 0.3 us per call)."""
    global _raw_stream
    t = torch()
    if _raw_stream is None:
        fn = getattr(t._C, "_cuda_getCurrentRawStream", None)
        _raw_stream = fn if fn is not None else False
    if _raw_stream:
        return _raw_stream(current_device())
    return t.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return t.data_ptr()


def ptr_array(tensors) -> ctypes.Array:
    arr = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    return arr


def ptr_rows(block) -> ctypes.Array:
    """Column pointers of a 2-D (columns x stride) fp64 block, without
    materialising per-column tensors."""
    base, step = block.data_ptr(), block.stride(0) * block.element_size()
    n = block.shape[0]
    return (ctypes.c_void_p * n)(*range(base, base + n * step, step))


def empty(n: int, dtype=None):
    _require_device()
    t = torch()
    return t.empty(int(n), dtype=dtype or t.float64, device="cuda")   # the current device


def bad_cells(k: int = 1):
    """k first-bad-row cells initialised to HK_NO_BAD_ROW."""
    t = torch()
    return t.full((k,), -1, dtype=t.int64, device=device())


def read_bad(cells) -> list[int]:
    return [int(v) % (1 << 64) for v in cells.cpu().tolist()]


def u64(v: int) -> int:
    return int(v) % (1 << 64)


def make_key(key, mode: int = HK_RNG_REFERENCE) -> hk_key_t:
    return hk_key_t(u64(key.seed), u64(key.stream), u64(key.counter), int(mode), 0)


def make_decay(spec, mother=None, m_mother=None) -> hk_decay_t:
    """hk_decay_t from a DecaySpec; T/csum with numpy like phasespace.py:94-97."""
    ms = np.asarray(spec.daughter_masses, dtype=np.float64)
    n = len(ms)
    if n > HK_MAX_DAUGHTERS:
        raise NotImplementedError(f"{n} daughters: the library supports up to {HK_MAX_DAUGHTERS}")
    d = hk_decay_t()
    d.n = n
    d.mother_mass = float(spec.mother_mass)
    d.T = float(spec.mother_mass - float(np.sum(ms)))
    csum = np.cumsum(ms)
    for i in range(n):
        d.masses[i] = float(ms[i])
        d.csum[i] = float(csum[i])
    if mother is None:
        d.moving = 0
        d.mother[:] = [float(spec.mother_mass), 0.0, 0.0, 0.0]
        d.m_mother = float(spec.mother_mass)
    else:
        d.moving = int(mother.px != 0.0 or mother.py != 0.0 or mother.pz != 0.0)
        d.mother[:] = [float(mother.e), float(mother.px), float(mother.py), float(mother.pz)]
        d.m_mother = float(m_mother)
    return d


def num_chunks(n: int) -> int:
    return (int(n) + HK_CHUNK - 1) // HK_CHUNK


HK_FCN_TILE = 4096   # rows per FCN partial (include/hepkit_cuda.h)
HK_WARP_SLICES = 8   # per-warp weight partials per chunk (generation kernels)


def num_weight_slices(n: int) -> int:
    """Number of (sum w, sum w^2) partials the generation kernels write for n rows."""
    return HK_WARP_SLICES * num_chunks(n)


def num_fcn_tiles(n: int) -> int:
    return (int(n) + HK_FCN_TILE - 1) // HK_FCN_TILE


def fold(partials, n_parts: int, width: int):
    """Deterministic device fold of (n_parts, width) partials -> (width,) tensor."""
    out = empty(width)
    check(lib().hk_fold_partials(ptr(partials) if n_parts else None, int(n_parts), int(width),
                                 ptr(out), stream_ptr()), "hk_fold_partials")
    return out


def fold_segments(partials, n_segments: int, seg_len: int, width: int):
    """Fixed-order fold of each run of seg_len partials -> (n_segments, width)."""
    out = empty(max(int(n_segments), 0) * width)
    if n_segments:
        check(lib().hk_fold_segments(ptr(partials), int(n_segments), int(seg_len), int(width), ptr(out),
                                     stream_ptr()), "hk_fold_segments")
    return out


HK_SUPERS = 1024     # super-chunks per run (include/hepkit_cuda.h)


def super_chunks(n_total: int, s_begin: int, s_end: int) -> tuple[int, int]:
    """Global chunk range [c0, c1) of supers [s_begin, s_end) of an n_total-row
    run: super s covers chunks [s N / S, (s+1) N / S), N = num_chunks(n_total)."""
    nch = num_chunks(n_total)
    return s_begin * nch // HK_SUPERS, s_end * nch // HK_SUPERS


def fold_supers(partials, n_total: int, s_begin: int, s_end: int, recs_per_chunk: int, width: int):
    """One record per super-chunk in [s_begin, s_end) from the local per-chunk
    partials (recs_per_chunk records of `width` doubles per chunk of the
    supers' chunk range) -> ((s_end - s_begin) * width,) tensor (hk_fold_supers)."""
    c0, c1 = super_chunks(n_total, s_begin, s_end)
    out = empty((s_end - s_begin) * width)
    if s_end > s_begin:
        p = ptr(partials) if c1 > c0 else None
        check(lib().hk_fold_supers(p, num_chunks(n_total), c0, c1 - c0, int(recs_per_chunk), int(width),
                                   int(s_begin), int(s_end - s_begin), ptr(out), stream_ptr()),
              "hk_fold_supers")
    return out


def total(partials, n: int, width: int, recs_per_chunk: int = 1):
    """Deterministic total of an n-row run's per-chunk partials: chunks ->
    HK_SUPERS super-chunks -> one fixed-tree fold.  The same two levels run
    sharded over any number of GPUs (parallel.py), so totals are bitwise
    independent of the GPU count."""
    return fold(fold_supers(partials, n, 0, HK_SUPERS, recs_per_chunk, width), HK_SUPERS, width)


def weight_chunk_partials(wpart, n: int):
    """A generation's per-warp-slice (sum w, sum w^2) -> one pair per 4096-row chunk."""
    return fold_segments(wpart, num_chunks(n), HK_WARP_SLICES, 2)


def weight_totals(wpart, n: int):
    """(sum w, sum w^2) of a generation: warp slices -> supers -> total, fixed order."""
    return total(wpart, n, 2, HK_WARP_SLICES)


JIT_OFF, JIT_ALWAYS, JIT_AUTO = 0, 1, 2
HK_JIT_MIN_ROWS = 1 << 22


def set_jit_mode(mode: int) -> int:
    """Functor specialisation policy (hk_set_jit_mode); returns the previous mode."""
    prev = load_library().hk_set_jit_mode(int(mode))
    if prev < 0:
        raise ValueError(last_error())
    return prev


class jit_mode:
    """``with jit_mode(JIT_OFF): ...`` -- scoped specialisation policy."""

    def __init__(self, mode: int):
        self.mode = mode
        self.prev = None

    def __enter__(self):
        self.prev = set_jit_mode(self.mode)
        return self

    def __exit__(self, *exc):
        set_jit_mode(self.prev)
        return False


def jit_source(program, n_daughters: int = 0, rng_mode: int = HK_RNG_REFERENCE) -> str:
    """CUDA source emitted for a lowered program (hk_jit_source): the
    stored-block module (n_daughters 0) or the fused generate+integrate one."""
    L = load_library()
    n = L.hk_jit_source(program, n_daughters, rng_mode, None, 0)
    if n < 0:
        raise ValueError(last_error())
    buf = ctypes.create_string_buffer(n + 1)
    L.hk_jit_source(program, n_daughters, rng_mode, buf, n + 1)
    return buf.value.decode()


def jit_compile(program, n_daughters: int = 0, rng_mode: int = HK_RNG_REFERENCE) -> int:
    """NVRTC-compile a module for sm_100a without a device; returns cubin bytes."""
    out = ctypes.c_int64(0)
    check(load_library().hk_jit_compile(program, n_daughters, rng_mode, ctypes.byref(out)),
          "hk_jit_compile")
    return out.value


# ---------------------------------------------------- lifetime + collectives
# For one process driving GPUs 0..n-1 (a C host's view of the reference's
# worker pool).  The drop-in API itself runs one process per GPU and uses
# torch.distributed (parallel.py); these are the C-ABI equivalents.

def init(n_devices: int = 1) -> None:
    """hk_init: NCCL clique over devices 0..n_devices-1 (NCCL dlopen'ed)."""
    check(load_library().hk_init(int(n_devices)), "hk_init")


def shutdown() -> None:
    """hk_shutdown: destroy the clique and release cached modules/buffers."""
    check(load_library().hk_shutdown(), "hk_shutdown")


def clique_size() -> int:
    return int(load_library().hk_clique_size())


def _clique_args(tensors):
    t = torch()
    n = tensors[0].numel()
    for g, x in enumerate(tensors):
        if x.dtype != t.float64 or not x.is_contiguous() or x.numel() != n:
            raise ValueError("partials must be contiguous fp64 tensors of equal length")
        if x.device.type != "cuda" or x.device.index != g:
            raise ValueError(f"partials[{g}] must live on cuda:{g}, found {x.device}")
    streams = (ctypes.c_void_p * len(tensors))(
        *[t.cuda.current_stream(x.device).cuda_stream for x in tensors])
    return n, streams


def allreduce_partials(bufs) -> None:
    """In-place sum across the clique (hk_allreduce_partials); bufs[g] on cuda:g."""
    n, streams = _clique_args(bufs)
    check(lib().hk_allreduce_partials(ptr_array(bufs), len(bufs), n, streams), "hk_allreduce_partials")


def allgather_partials(sends) -> list:
    """Every device gets all devices' partials in device order (hk_allgather_partials)."""
    n, streams = _clique_args(sends)
    t = torch()
    recv = [t.empty(len(sends) * n, dtype=t.float64, device=x.device) for x in sends]
    check(lib().hk_allgather_partials(ptr_array(sends), ptr_array(recv), len(sends), n, streams),
          "hk_allgather_partials")
    return recv
