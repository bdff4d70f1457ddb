"""ctypes binding of ``libqttb200.so`` (the C ABI in include/qtt_b200.h).

There is no CPU fallback: importing works without a GPU (so the host-side
modules and the symbol table can be inspected), but every compute entry
point raises when the shared library or a CUDA device is missing.
"""

from __future__ import annotations

import concurrent.futures
import ctypes
import os

import torch

MAX_CORES = 64
_LIB_PATH = os.environ.get(
    "QTT_LIB_PATH",  # A/B builds of the same library (tools/)
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libqttb200.so"))

QTT_OK, QTT_EINVAL, QTT_ECUDA, QTT_EWORKSPACE, QTT_EUNSUPPORTED = range(5)

# Every symbol declared in include/qtt_b200.h (checked by tests/test_abi.py).
EXPORTS = (
    "qtt_version",
    "qtt_launch_count",
    "qtt_profile_gemm",
    "qtt_profile_gemm_read",
    "qtt_profile_gemm_shape",
    "qtt_layout_size",
    "qtt_release_cached",
    "qtt_thread_shared_pool",
    "qtt_matvec",
    "qtt_matmat",
    "qtt_hadamard",
    "qtt_add",
    "qtt_zkron",
    "qtt_diag",
    "qtt_transpose",
    "qtt_scale",
    "qtt_round",
    "qtt_round_to_host",
    "qtt_decompose",
    "qtt_norm",
    "qtt_dot",
    "qtt_contract",
    "qtt_dense_apply",
    "qtt_zorder_permutation",
    "qtt_zorder_dof_permutation",
    "qtt_z_index",
    "qtt_element_grids",
    "qtt_dense_solve",
    "qtt_local_gmres",
    "qtt_local_apply",
    "qtt_gemm",
    "qtt_gemm_structured",
    "qtt_qr",
    "qtt_svd",
)


class Layout(ctypes.Structure):
    """Mirror of ``qtt_layout``."""

    _fields_ = [
        ("d", ctypes.c_int32),
        ("is_matrix", ctypes.c_int32),
        ("ranks", ctypes.c_int64 * (MAX_CORES + 1)),
        ("rows", ctypes.c_int64 * MAX_CORES),
        ("cols", ctypes.c_int64 * MAX_CORES),
        ("offsets", ctypes.c_int64 * MAX_CORES),
    ]


class QTTError(RuntimeError):
    pass


_lib = None


def library_path() -> str:
    return _LIB_PATH


def load():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise QTTError(
                f"libqttb200.so not built ({_LIB_PATH}); run `make` or "
                "`python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(_LIB_PATH)
        lib.qtt_version.restype = ctypes.c_char_p
        lib.qtt_layout_size.restype = ctypes.c_int64
        lib.qtt_launch_count.restype = ctypes.c_longlong
        for name in EXPORTS:
            if name not in ("qtt_version", "qtt_layout_size", "qtt_launch_count"):
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise QTTError("paper_2501_07778_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def check(status: int, what: str) -> None:
    if status == QTT_OK:
        return
    names = {
        QTT_EINVAL: "invalid argument",
        QTT_ECUDA: "CUDA error",
        QTT_EWORKSPACE: "output buffer too small",
        QTT_EUNSUPPORTED: "size outside the kernel envelope",
    }
    msg = f"{what}: {names.get(status, status)}"
    if status == QTT_EINVAL:
        raise ValueError(msg)
    raise QTTError(msg)


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def align(n: int) -> int:
    return (n + 31) // 32 * 32


def launch_count() -> int:
    return int(load().qtt_launch_count())


def release_cached() -> None:
    """Return cached device memory of BOTH allocators (torch's caching
    allocator and the library's stream-ordered pool) to the driver.  The two
    caches cannot serve each other, so when allocations grow step by step
    (AMEn local systems of tens of GB) each must be trimmed before the other
    allocates."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    call("qtt_release_cached", stream_handle())


def gemm_profile_start() -> None:
    call("qtt_profile_gemm", ctypes.c_int32(1))


def gemm_profile_stop() -> tuple:
    """(flops, ms, launches) of the GEMMs since gemm_profile_start()."""
    f, ms, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    call("qtt_profile_gemm_read", ctypes.byref(f), ctypes.byref(ms), ctypes.byref(n))
    call("qtt_profile_gemm", ctypes.c_int32(0))
    return f.value, ms.value, n.value


def gemm_profile_shapes(count: int) -> list:
    """Dispatch records of the last ``count`` profiled GEMM launches, each a
    dict (m, n, k, batch, flags, splits, bm); call before gemm_profile_stop."""
    out = []
    buf = (ctypes.c_int64 * 7)()
    for i in range(-count, 0):
        call("qtt_profile_gemm_shape", ctypes.c_int64(i), buf)
        out.append(dict(zip(("m", "n", "k", "batch", "flags", "splits", "bm"), list(buf))))
    return out


_WORKERS: list = []
_STREAMS: list = []


class _Worker:
    """One host thread bound to one chain slot: slot i always runs on thread i
    with stream i, so the library's per-thread state (private memory pool,
    look-ahead side stream) stays with the chain."""

    def __init__(self, idx: int):
        import queue
        import threading

        self.q = queue.SimpleQueue()
        self.t = threading.Thread(target=self._loop, name=f"qtt-chain-{idx}", daemon=True)
        self.t.start()

    def _loop(self):
        # concurrent chains share the device's default pool (fastest while they
        # all run); the caller's thread keeps its private pool (csrc/common.cuh)
        load().qtt_thread_shared_pool(ctypes.c_int32(1))
        while True:
            fut, fn, args = self.q.get()
            if not fut.set_running_or_notify_cancel():
                continue
            try:
                fut.set_result(fn(*args))
            except BaseException as exc:  # delivered to the submitting thread
                fut.set_exception(exc)

    def submit(self, fn, *args):
        fut = concurrent.futures.Future()
        self.q.put((fut, fn, args))
        return fut


def run_concurrent(jobs):
    """Run independent TT chains (fn(arg) -> TT object) concurrently, one CUDA stream
    and one host thread each (the C-ABI calls release the GIL; each chain's
    host synchronisations then overlap the others' kernels).  Inputs were
    produced on the caller's stream, which every chain stream waits for; the
    caller's stream waits for all chains before the results are used."""
    global _WORKERS, _STREAMS
    import threading

    if threading.current_thread().name.startswith("qtt-chain-"):
        # nested use from inside a chain: its own slot would wait on itself
        return [fn(arg) for fn, arg in jobs]
    dev = torch.cuda.current_device()
    while len(_WORKERS) < len(jobs):
        _WORKERS.append(_Worker(len(_WORKERS)))
    if len(_STREAMS) < len(jobs) or _STREAMS[0].device.index != dev:
        # callers order their jobs longest first: the earlier a chain, the
        # higher its stream priority, so the critical (longest) chain is not
        # queued behind the short chains' kernels (QTT_CHAIN_PRIORITY=0: flat)
        levels = 1
        if os.environ.get("QTT_CHAIN_PRIORITY", "1") != "0":
            try:
                lo, hi = torch.cuda.Stream.priority_range()  # (least, greatest), e.g. (0, -5)
                levels = abs(hi - lo) + 1
            except Exception:
                levels = 2
        _STREAMS = [torch.cuda.Stream(device=dev, priority=-max(levels - 1 - i, 0))
                    for i in range(max(12, len(jobs)))]
    main = torch.cuda.current_stream()

    def run(fn, arg, stream):
        torch.cuda.set_device(dev)
        stream.wait_stream(main)
        with torch.cuda.stream(stream):
            out = fn(arg)
        for item in (out if isinstance(out, tuple) else (out,)):
            t = getattr(item, "data", item)
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(main)
        return out

    futs = [_WORKERS[i].submit(run, fn, arg, _STREAMS[i]) for i, (fn, arg) in enumerate(jobs)]
    # wait for EVERY chain before joining the streams: if one job raises, the
    # others must not keep reading or writing memory the caller may free
    concurrent.futures.wait(futs)
    try:
        return [f.result() for f in futs]
    finally:
        for i in range(len(jobs)):
            main.wait_stream(_STREAMS[i])
