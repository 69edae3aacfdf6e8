"""Thin Python binding of libvndf (include/vndf.h): argument marshalling only.

Every sampling step runs in the sm_100a kernels of ``libvndf.so``; this module
checks tensors, passes device pointers and the current CUDA stream, and raises
on a non-OK status.  There is no CPU fallback: if the shared library is missing
or fails to load, importing the sampling functions raises.

Names follow the C ABI.  Tensors are torch tensors: float32, contiguous, 1-D,
at least ``n`` elements, on one CUDA device (the host entry point takes CPU
tensors or numpy arrays instead).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvndf.so")

VNDF_OK = 0
VNDF_ERR_INVALID_ARGUMENT = 1
VNDF_ERR_CUDA = 2
VNDF_ERR_NOT_IMPLEMENTED = 3

# exported symbols of include/vndf.h (checked by tests/test_abi.py)
SYMBOLS = (
    "vndf_sample_cap", "vndf_sample_cap_pdf", "vndf_sample_heitz2018",
    "vndf_sample_cap_philox", "vndf_sample_heitz2018_philox", "vndf_sample_cap_philox_edge",
    "vndf_sample_heitz2018_philox_edge", "vndf_philox4x32_10",
    "vndf_sample_cap_pdf_host", "vndf_release_host_staging", "vndf_count_fixups", "vndf_count_fixups_philox",
    "vndf_set_launch_config", "vndf_status_string", "vndf_last_cuda_error", "vndf_version",
    "vndf_microbench", "vndf_sample_cap_reflect", "vndf_furnace", "vndf_pdf",
    "vndf_sample_cap_pdf_native", "vndf_histogram",
    "vndf_sample_cap_reflect_philox", "vndf_sample_heitz2018_reflect_philox",
    "vndf_sample_cap_philox_host", "vndf_microbench_trace", "vndf_init",
)


class VndfError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = f"{fn}: {status_string(status)}"
        if status == VNDF_ERR_CUDA:
            msg += f" (cudaError {last_cuda_error()})"
        super().__init__(msg)
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libvndf.so (fails loudly if it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, u64, u32, i32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                  ctypes.c_uint32, ctypes.c_int)
        for name in ("vndf_sample_cap",):
            getattr(L, name).argtypes = [P] * 10 + [i64, P]
        for name in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018", "vndf_sample_cap_pdf_host",
                     "vndf_sample_cap_pdf_native"):
            getattr(L, name).argtypes = [P] * 11 + [i64, P]
        for name in ("vndf_sample_cap_philox", "vndf_sample_heitz2018_philox", "vndf_sample_cap_philox_edge",
                     "vndf_sample_heitz2018_philox_edge"):
            getattr(L, name).argtypes = [u64, u64, i64, P, P, P, P, P]
        L.vndf_philox4x32_10.argtypes = [u64, u64, i64, u32, P, P]
        L.vndf_count_fixups.argtypes = [P] * 7 + [i64, P, P]
        L.vndf_count_fixups_philox.argtypes = [u64, u64, i64, P, P]
        L.vndf_set_launch_config.argtypes = [i32, i32, i32]
        L.vndf_release_host_staging.argtypes = []
        L.vndf_microbench.argtypes = [i32, u64, i64, i32, P, P]
        L.vndf_microbench_trace.argtypes = [i32, u64, i64, i32, P, P, P]
        L.vndf_init.argtypes = [i32]
        L.vndf_sample_cap_philox_host.argtypes = [u64, u64, i64, P, P, P, P, P]
        L.vndf_sample_cap_reflect.argtypes = [P] * 12 + [i64, P]
        for name in ("vndf_sample_cap_reflect_philox", "vndf_sample_heitz2018_reflect_philox"):
            getattr(L, name).argtypes = [u64, u64, i64, P, P, P, P, P, P]
        L.vndf_pdf.argtypes = [P] * 9 + [i64, P]
        f32_ = ctypes.c_float
        L.vndf_histogram.argtypes = [i32, i32, f32_, f32_, f32_, f32_, f32_, u64, u64, i64, i32, i32, P, P]
        f32 = ctypes.c_float
        L.vndf_furnace.argtypes = [i32, f32, f32, f32, f32, f32, u64, u64, i64, P, P]
        L.vndf_status_string.argtypes = [i32]
        L.vndf_status_string.restype = ctypes.c_char_p
        L.vndf_last_cuda_error.argtypes = []
        L.vndf_version.argtypes = []
        for name in SYMBOLS:
            if name != "vndf_status_string":
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().vndf_status_string(status).decode()


def last_cuda_error() -> int:
    return lib().vndf_last_cuda_error()


def version() -> int:
    return lib().vndf_version()


def _check(fn: str, status: int) -> None:
    if status != VNDF_OK:
        raise VndfError(fn, status)


# ------------------------------------------------------------- marshalling --
# Kept lean: a call's host cost is paid per launch (tools/binding_overhead.py).
_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def _dev_ptr(t, n: int, name: str, dtype=None, device=None):
    """(device pointer as int, CUDA device index) of a checked tensor."""
    if t is None:
        return None, device
    torch = _t()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor")
    want = dtype or torch.float32
    if t.dtype != want:
        raise TypeError(f"{name}: expected {want}, got {t.dtype}")
    d = t.get_device()
    if d < 0:
        raise ValueError(f"{name}: expected a CUDA tensor")
    if not t.is_contiguous() or t.numel() < n:
        raise ValueError(f"{name}: expected a contiguous tensor with >= {n} elements")
    if device is not None and d != device:
        raise ValueError(f"{name}: all tensors must be on cuda:{device}")
    return t.data_ptr(), d


def _stream(stream, device):
    """Raw cudaStream_t: the given stream, else the current stream of `device`
    (a CUDA device index, or None for the current device)."""
    torch = _t()
    if stream is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # skips the Stream object
        if raw is not None:
            return raw(torch.cuda.current_device() if device is None else device)
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _n(n, t) -> int:
    return int(t.numel()) if n is None else int(n)


def _stream_call(fn, tensors, names, n, stream):
    dev = None
    ptrs = []
    for t, nm in zip(tensors, names):
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    _check(fn, getattr(lib(), fn)(*ptrs, n, _stream(stream, dev)))


_IN = ("wi_x", "wi_y", "wi_z", "alpha_x", "alpha_y", "u1", "u2")


def vndf_sample_cap(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, n=None, stream=None):
    """Listing 1 + Listing 3: h only."""
    n = _n(n, wi_x)
    _stream_call("vndf_sample_cap", (wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z),
                 _IN + ("h_x", "h_y", "h_z"), n, stream)


def vndf_sample_cap_pdf(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf,
                        n=None, stream=None):
    """Listing 1 + Listing 3 plus the Eq. 1 pdf."""
    n = _n(n, wi_x)
    _stream_call("vndf_sample_cap_pdf",
                 (wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf),
                 _IN + ("h_x", "h_y", "h_z", "pdf"), n, stream)


def vndf_sample_cap_pdf_native(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf=None,
                               n=None, stream=None):
    """NEXT-3: the paper's native below-horizon handling (Fig. 4), no flip."""
    n = _n(n, wi_x)
    dev = None
    ptrs = []
    for t, nm in zip((wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf),
                     _IN + ("h_x", "h_y", "h_z", "pdf")):
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    _check("vndf_sample_cap_pdf_native", lib().vndf_sample_cap_pdf_native(*ptrs, n, _stream(stream, dev)))


def vndf_sample_heitz2018(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf=None,
                          n=None, stream=None):
    """Listing 1 + Listing 2, the same-harness baseline."""
    n = _n(n, wi_x)
    dev = None
    ptrs = []
    for t, nm in zip((wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf),
                     _IN + ("h_x", "h_y", "h_z", "pdf")):
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    _check("vndf_sample_heitz2018", lib().vndf_sample_heitz2018(*ptrs, n, _stream(stream, dev)))


def _philox_call(fn, seed, first_index, n, h_x, h_y, h_z, pdf, stream):
    dev = None
    ptrs = []
    for t, nm in zip((h_x, h_y, h_z, pdf), ("h_x", "h_y", "h_z", "pdf")):
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    _check(fn, getattr(lib(), fn)(int(seed), int(first_index), int(n), *ptrs, _stream(stream, dev)))


def vndf_sample_cap_philox(seed, first_index, n, h_x, h_y, h_z, pdf=None, stream=None):
    """Fused Philox4x32-10 inputs + spherical-cap sampling + pdf (config 4)."""
    _philox_call("vndf_sample_cap_philox", seed, first_index, n, h_x, h_y, h_z, pdf, stream)


def vndf_sample_heitz2018_philox(seed, first_index, n, h_x, h_y, h_z, pdf=None, stream=None):
    _philox_call("vndf_sample_heitz2018_philox", seed, first_index, n, h_x, h_y, h_z, pdf, stream)


def vndf_sample_cap_philox_edge(seed, first_index, n, h_x, h_y, h_z, pdf=None, stream=None):
    """Fused Philox4x32-10 inputs of the config-5 edge mix + spherical-cap sampling + pdf."""
    _philox_call("vndf_sample_cap_philox_edge", seed, first_index, n, h_x, h_y, h_z, pdf, stream)


def vndf_sample_heitz2018_philox_edge(seed, first_index, n, h_x, h_y, h_z, pdf=None, stream=None):
    _philox_call("vndf_sample_heitz2018_philox_edge", seed, first_index, n, h_x, h_y, h_z, pdf, stream)


def vndf_philox4x32_10(seed, first_index, n, block, words, stream=None):
    """Raw Philox words (int32 tensor of >= 4n elements, bit pattern = uint32)."""
    import torch
    p, dev = _dev_ptr(words, 4 * int(n), "words", dtype=torch.int32)
    _check("vndf_philox4x32_10", lib().vndf_philox4x32_10(int(seed), int(first_index), int(n),
                                                          int(block), p, _stream(stream, dev)))


def vndf_count_fixups(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, count, n=None, stream=None):
    """Adds to count[0] (int64 CUDA tensor) the number of float64 fix-ups."""
    import torch
    n = _n(n, wi_x)
    dev = None
    ptrs = []
    for t, nm in zip((wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2), _IN):
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    c, _ = _dev_ptr(count, 1, "count", dtype=torch.int64, device=dev)
    _check("vndf_count_fixups", lib().vndf_count_fixups(*ptrs, n, c, _stream(stream, dev)))


def vndf_count_fixups_philox(seed, first_index, n, count, stream=None):
    import torch
    c, dev = _dev_ptr(count, 1, "count", dtype=torch.int64)
    _check("vndf_count_fixups_philox",
           lib().vndf_count_fixups_philox(int(seed), int(first_index), int(n), c, _stream(stream, dev)))


def vndf_sample_cap_pdf_host(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf=None,
                             n=None, stream=None):
    """End-to-end call on HOST buffers (CPU torch tensors, ideally pinned, or
    numpy arrays); blocking.  Copies and kernel overlap inside libvndf.
    pdf=None: h only (config 3's end-to-end form)."""
    import numpy as np
    import torch
    arrs = (wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, h_x, h_y, h_z, pdf)
    names = _IN + ("h_x", "h_y", "h_z", "pdf")
    n = int(len(wi_x)) if n is None else int(n)
    ptrs = []
    for a, nm in zip(arrs, names):
        if a is None and nm == "pdf":
            ptrs.append(ctypes.c_void_p(0))
        elif isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous() or a.numel() < n:
                raise ValueError(f"{nm}: expected a contiguous float32 CPU tensor of >= {n} elements")
            ptrs.append(ctypes.c_void_p(a.data_ptr()))
        elif isinstance(a, np.ndarray):
            if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"] or a.size < n:
                raise ValueError(f"{nm}: expected a contiguous float32 array of >= {n} elements")
            ptrs.append(ctypes.c_void_p(a.ctypes.data))
        else:
            raise TypeError(f"{nm}: expected a torch CPU tensor or numpy array")
    if stream is None:
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    else:
        st = _stream(stream, None)
    _check("vndf_sample_cap_pdf_host", lib().vndf_sample_cap_pdf_host(*ptrs, n, st))


def _host_ptr(a, n: int, name: str):
    import numpy as np
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float32 or not a.is_contiguous() or a.numel() < n:
            raise ValueError(f"{name}: expected a contiguous float32 CPU tensor of >= {n} elements")
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"] or a.size < n:
            raise ValueError(f"{name}: expected a contiguous float32 array of >= {n} elements")
        return ctypes.c_void_p(a.ctypes.data)
    raise TypeError(f"{name}: expected a torch CPU tensor or numpy array")


def vndf_sample_cap_philox_host(seed, first_index, n, h_x, h_y, h_z, pdf=None, stream=None):
    """End-to-end config-4 call writing HOST buffers (CPU tensors, ideally
    pinned: the kernel then writes them in place); blocking."""
    import torch
    n = int(n)
    ptrs = [_host_ptr(a, n, nm) for a, nm in ((h_x, "h_x"), (h_y, "h_y"), (h_z, "h_z"))]
    ptrs.append(_host_ptr(pdf, n, "pdf") if pdf is not None else None)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream) if stream is None else _stream(stream, None)
    _check("vndf_sample_cap_philox_host",
           lib().vndf_sample_cap_philox_host(int(seed), int(first_index), n, *ptrs, st))


def vndf_sample_cap_reflect(wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, wo_x, wo_y, wo_z, pdf, weight,
                            n=None, stream=None):
    """Appendix steps (1)-(2): reflected direction, Eq. 20 pdf, G2/G1 weight."""
    n = _n(n, wi_x)
    _stream_call("vndf_sample_cap_reflect",
                 (wi_x, wi_y, wi_z, alpha_x, alpha_y, u1, u2, wo_x, wo_y, wo_z, pdf, weight),
                 _IN + ("wo_x", "wo_y", "wo_z", "pdf", "weight"), n, stream)


def _philox_reflect_call(fn, seed, first_index, n, wo_x, wo_y, wo_z, pdf, weight, stream):
    dev = None
    ptrs = []
    for t, nm in zip((wo_x, wo_y, wo_z, pdf, weight), ("wo_x", "wo_y", "wo_z", "pdf", "weight")):
        if t is None:
            raise ValueError(f"{nm}: required")
        p, dev = _dev_ptr(t, n, nm, device=dev)
        ptrs.append(p)
    _check(fn, getattr(lib(), fn)(int(seed), int(first_index), int(n), *ptrs, _stream(stream, dev)))


def vndf_sample_cap_reflect_philox(seed, first_index, n, wo_x, wo_y, wo_z, pdf, weight, stream=None):
    """NEXT-2 fused: config-4 inputs in-kernel, reflected direction, Eq. 20 pdf, G2/G1 weight."""
    _philox_reflect_call("vndf_sample_cap_reflect_philox", seed, first_index, n, wo_x, wo_y, wo_z, pdf,
                         weight, stream)


def vndf_sample_heitz2018_reflect_philox(seed, first_index, n, wo_x, wo_y, wo_z, pdf, weight, stream=None):
    _philox_reflect_call("vndf_sample_heitz2018_reflect_philox", seed, first_index, n, wo_x, wo_y, wo_z, pdf,
                         weight, stream)


def vndf_pdf(h_x, h_y, h_z, wi_x, wi_y, wi_z, alpha_x, alpha_y, pdf, n=None, stream=None):
    """NEXT-4: Eq. 1 at caller-provided h."""
    n = _n(n, h_x)
    _stream_call("vndf_pdf", (h_x, h_y, h_z, wi_x, wi_y, wi_z, alpha_x, alpha_y, pdf),
                 ("h_x", "h_y", "h_z", "wi_x", "wi_y", "wi_z", "alpha_x", "alpha_y", "pdf"), n, stream)


def vndf_histogram(method, mode, wi, alpha, seed, n, nt, nphi, counts, first_index=0, stream=None):
    """NEXT-3 device histogram (counts: int64 CUDA tensor of nt * nphi, added to)."""
    import torch
    p, dev = _dev_ptr(counts, int(nt) * int(nphi), "counts", dtype=torch.int64)
    _check("vndf_histogram", lib().vndf_histogram(int(method), int(mode), float(wi[0]), float(wi[1]),
                                                  float(wi[2]), float(alpha[0]), float(alpha[1]), int(seed),
                                                  int(first_index), int(n), int(nt), int(nphi), p,
                                                  _stream(stream, dev)))


def vndf_furnace(method, wi, alpha, seed, n, sums, first_index=0, stream=None):
    """Eq. 19 white-furnace estimator; sums: float64 CUDA tensor of 2 (sum, sum of squares)."""
    import torch
    p, dev = _dev_ptr(sums, 2, "sums", dtype=torch.float64)
    _check("vndf_furnace", lib().vndf_furnace(int(method), float(wi[0]), float(wi[1]), float(wi[2]),
                                              float(alpha[0]), float(alpha[1]), int(seed), int(first_index),
                                              int(n), p, _stream(stream, dev)))


MICROBENCH_CAP, MICROBENCH_HEITZ, MICROBENCH_CAP_LITERAL = 0, 1, 2


def vndf_microbench(method, seed, lanes, iters, checksum, stream=None):
    """NEXT-1 sampler-only microbenchmark: per-lane checksums."""
    p, dev = _dev_ptr(checksum, int(lanes), "checksum")
    _check("vndf_microbench", lib().vndf_microbench(int(method), int(seed), int(lanes), int(iters), p,
                                                    _stream(stream, dev)))


def vndf_microbench_trace(method, seed, lanes, iters, checksum, trace, stream=None):
    """NEXT-1 with every call recorded: trace (float32, >= 4 lanes iters) gets
    (h.x, h.y, h.z, flag) per call, lane-major."""
    p, dev = _dev_ptr(checksum, int(lanes), "checksum")
    t, _ = _dev_ptr(trace, 4 * int(lanes) * int(iters), "trace", device=dev)
    _check("vndf_microbench_trace", lib().vndf_microbench_trace(int(method), int(seed), int(lanes), int(iters),
                                                                p, t, _stream(stream, dev)))


def vndf_init(device: int = -1):
    """Start libvndf's CUDA state on `device` now (vndf.h): later calls only enqueue."""
    _check("vndf_init", lib().vndf_init(int(device)))


def vndf_release_host_staging():
    _check("vndf_release_host_staging", lib().vndf_release_host_staging())


def vndf_set_launch_config(vector_width: int = 0, block_size: int = 0, blocks_per_sm: int = 0):
    _check("vndf_set_launch_config", lib().vndf_set_launch_config(vector_width, block_size, blocks_per_sm))


# ------------------------------------------------------------ conveniences --
def empty_outputs(n: int, device="cuda", pdf: bool = True):
    """Allocate (h_x, h_y, h_z[, pdf]) float32 device planes of length n."""
    import torch
    k = 4 if pdf else 3
    return tuple(torch.empty(n, dtype=torch.float32, device=device) for _ in range(k))
