"""Thin ctypes binding of libtomoq.so (include/tomoq.h): argument marshalling only.

Every computation runs in the library's sm_100a kernels.  There is no CPU or
PyTorch fallback: if the in-tree libtomoq.so is missing this module raises.
torch supplies device memory (tensor data pointers), streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TQ_LIB_PATH") or os.path.join(HERE, "libtomoq.so")  # override: A/B timing tools only
HEADER = os.path.join(os.path.dirname(HERE), "include", "tomoq.h")

SPLIT_RR, SPLIT_CONTIG = 0, 1
RULE_GRAPH, RULE_PAPER, RULE_CONSENSUS = 0, 1, 2
PROJ_JOSEPH, PROJ_SIDDON = 0, 1
INNER_GD, INNER_CG = 0, 1
Q_NONE, Q_KMEANS, Q_DCT, Q_ALT = 0, 1, 2, 3
STATUS = {0: "TQ_OK", 1: "TQ_EINVAL", 2: "TQ_ENOMEM", 3: "TQ_ECUDA", 4: "TQ_ENCCL",
          5: "TQ_EDIVERGED", 6: "TQ_ESTATE"}


class TomoQError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Geometry(C.Structure):
    _fields_ = [("image_side", C.c_int32), ("n_angles", C.c_int32), ("n_det", C.c_int32),
                ("projector", C.c_int32), ("angles_rad", C.POINTER(C.c_double))]


def _geom(N, n_angles, n_det, projector, angles):
    """Geometry + the array it points to (kept alive by the caller)."""
    if angles is None:
        return Geometry(N, n_angles, n_det, projector, None), None
    a = np.ascontiguousarray(angles, np.float64)
    if a.size != n_angles:
        raise ValueError("angles: n_angles values expected")
    return Geometry(N, n_angles, n_det, projector, a.ctypes.data_as(C.POINTER(C.c_double))), a


class Graph(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_edges", C.c_int32), ("edges", C.POINTER(C.c_int32)),
                ("angle_split", C.c_int32), ("node_rank", C.POINTER(C.c_int32)), ("rule", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("rho", C.c_double), ("inner", C.c_int32), ("e1", C.c_int32),
                ("eta1", C.POINTER(C.c_double)), ("e2", C.c_int32), ("eta2", C.c_double),
                ("stop_tol", C.c_double)]


class Quant(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k", C.c_int32), ("lloyd_iters", C.c_int32),
                ("quality", C.c_int32), ("keep_labels", C.c_int32), ("jpeg_restart", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("iters", C.c_int64), ("local_nodes", C.c_int32), ("world", C.c_int32),
                ("payload_bytes_logical", C.c_int64), ("nccl_bytes_sent", C.c_int64),
                ("nccl_bytes_recv", C.c_int64), ("kernel_launches", C.c_int64),
                ("ms_last_run", C.c_double), ("iters_last_run", C.c_int64), ("rel_change_last", C.c_double),
                ("phase_valid", C.c_int32), ("node_groups", C.c_int32), ("phase_ms", C.c_double * 4)]


_lib = None
_vp, _i32, _i64, _d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "tq_nccl_unique_id": [_vp],
    "tq_loopback_id": [_vp],
    "tq_create": [C.POINTER(Geometry), C.POINTER(Graph), _i32, _i32, _i32, _vp, _i32, _i32, C.POINTER(_vp)],
    "tq_set_params": [_vp, C.POINTER(Params)],
    "tq_set_quantizer": [_vp, C.POINTER(Quant)],
    "tq_set_sinogram": [_vp, _i32, _i32, _vp, _i64, _i32],
    "tq_set_sinogram_stream": [_vp, _i32, _i32, _vp, _i64, _vp],
    "tq_run": [_vp, _i32, _vp],
    "tq_run_async": [_vp, _i32, _vp],
    "tq_wait": [_vp],
    "tq_get_image": [_vp, _i32, _i32, _vp, _i64, _i32],
    "tq_get_image_async": [_vp, _i32, _i32, _vp, _i64, _i32, _vp],
    "tq_export_state": [_vp, _i32, _i32, _vp, _i64],
    "tq_import_state": [_vp, _i32, _i32, _vp, _i64],
    "tq_export_labels": [_vp, _i32, _i32, _vp, _i64],
    "tq_get_stats": [_vp, C.POINTER(Stats)],
    "tq_set_profiling": [_vp, _i32],
    "tq_debug_guard_check": [],
    "tq_debug_transport_check": [_vp, _i32, _i32, _i32, _i64, _i64, _i32],
    "tq_get_node_bytes": [_vp, _i32, _i32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "tq_launch_component": [_vp, _i32, _i32, _vp, C.POINTER(C.c_int64)],
    "tq_partition_angles": [_i32, _i32, _i32, _vp, _vp],
    "tq_exchange_plan": [C.POINTER(Graph), _i32, _i32, _vp, _i32, _vp, _vp, _i32, _vp],
    "tq_project": [C.POINTER(Geometry), _vp, _i32, _vp, _vp, _i32, _vp],
    "tq_backproject": [C.POINTER(Geometry), _vp, _i32, _vp, _vp, _i32, _vp],
    "tq_local_solve": [C.POINTER(Geometry), _vp, _i32, _vp, _vp, _d, _i32, _i32, _d, _vp, _i32, _vp],
    "tq_kmeans_encode": [_vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "tq_kmeans_decode": [_vp, _vp, _i64, _i32, _vp, _vp],
    "tq_dct_encode": [_vp, _i32, _i32, _i32, _vp, _vp, _vp],
    "tq_dct_decode": [_vp, _vp, _i32, _i32, _i32, _vp, _vp],
    "tq_jpeg_encode": [_vp, _i64, _i32, _vp, _i64, C.POINTER(C.c_int64), _vp],
    "tq_jpeg_decode": [_vp, _i64, _i64, _i32, _vp, _vp],
}


def lib() -> C.CDLL:
    """Load the in-tree libtomoq.so (built by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_2410_06106_b200.build")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.tq_last_error.argtypes = [_vp]
        L.tq_last_error.restype = C.c_char_p
        L.tq_last_error_global.argtypes = []
        L.tq_last_error_global.restype = C.c_char_p
        L.tq_destroy.argtypes = [_vp]
        L.tq_destroy.restype = None
        L.tq_payload_bytes.argtypes = [_i32, _i32, _i64, _i32]
        L.tq_payload_bytes.restype = C.c_int64
        _lib = L
    return _lib


def _check(code, ctx=None):
    if code != 0:
        L = lib()
        msg = (L.tq_last_error(ctx) if ctx else L.tq_last_error_global()) or b""
        raise TomoQError(code, msg.decode(errors="replace"))


def _i32arr(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _graph(n_nodes, edges, split, rule, node_rank=None):
    e = _i32arr(np.asarray(edges, np.int32).reshape(-1, 2).ravel() if len(edges) else np.zeros(2))
    nr = None if node_rank is None else _i32arr(node_rank)
    g = Graph(n_nodes, len(edges), e.ctypes.data_as(C.POINTER(C.c_int32)), split,
              nr.ctypes.data_as(C.POINTER(C.c_int32)) if nr is not None else None, rule)
    return g, (e, nr)


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


# --------------------------------------------------------------------- host plans
def partition_angles(n_angles: int, n_nodes: int, split: int):
    off = np.zeros(n_nodes + 1, np.int32)
    idx = np.zeros(n_angles, np.int32)
    _check(lib().tq_partition_angles(n_angles, n_nodes, split, off.ctypes.data, idx.ctypes.data))
    return off, idx


def exchange_plan(n_nodes, edges, rule, rank, world, node_rank=None):
    g, keep = _graph(n_nodes, edges, SPLIT_RR, rule, node_rank)
    cap = max(1, n_nodes * world)
    s = np.zeros(2 * cap, np.int32)
    r = np.zeros(2 * cap, np.int32)
    ns, nr = C.c_int32(), C.c_int32()
    _check(lib().tq_exchange_plan(C.byref(g), rank, world, s.ctypes.data, cap, C.addressof(ns),
                                  r.ctypes.data, cap, C.addressof(nr)))
    return ([tuple(x) for x in s[:2 * ns.value].reshape(-1, 2)],
            [tuple(x) for x in r[:2 * nr.value].reshape(-1, 2)])


def payload_bytes(kind: int, k: int, n: int, precision: int = 0) -> int:
    return int(lib().tq_payload_bytes(kind, k, n, precision))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().tq_nccl_unique_id(buf))
    return bytes(buf)


def debug_guard_check():
    """tq_debug_guard_check: raises if a guard band (TQ_GUARD=1) was overwritten."""
    _check(lib().tq_debug_guard_check())


def debug_transport_check(tid: bytes, rank: int, world: int, device: int = 0, nbytes: int = 1 << 20,
                          n_doubles: int = 1 << 16, rounds: int = 2):
    """tq_debug_transport_check: every operation of the transport `tid` (NCCL or loopback id)
    on a synthetic plan, results compared with exact host values; raises on a mismatch."""
    buf = (C.c_uint8 * 128).from_buffer_copy(tid)
    _check(lib().tq_debug_transport_check(buf, rank, world, device, nbytes, n_doubles, rounds))


def loopback_id() -> bytes:
    """An in-process world id (tq_loopback_id): pass it as `nccl_id` to the `world`
    contexts of one process (one thread per rank)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().tq_loopback_id(buf))
    return bytes(buf)


# --------------------------------------------------------------------- context
class Context:
    """One rank's ADMM context (tq_create)."""

    def __init__(self, N, n_angles, n_det, n_nodes, edges, split=SPLIT_RR, rule=RULE_GRAPH,
                 n_slices=1, rank=0, world=1, nccl_id: bytes | None = None, precision=0,
                 device=0, node_rank=None, projector=PROJ_JOSEPH, angles=None):
        self.N, self.n = N, N * N
        self.precision = precision
        geom, _keep_angles = _geom(N, n_angles, n_det, projector, angles)
        g, self._keep = _graph(n_nodes, edges, split, rule, node_rank)
        h = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
        code = lib().tq_create(C.byref(geom), C.byref(g), n_slices, rank, world, idbuf, precision,
                               device, C.byref(h))
        _check(code)
        self.h = h

    def _c(self, code):
        _check(code, self.h)

    def set_params(self, rho, inner=INNER_CG, e1=5, eta1=None, e2=10, eta2=0.2, stop_tol=0.0):
        self._eta1 = None if eta1 is None else np.ascontiguousarray(eta1, np.float64)
        p = Params(rho, inner, e1, self._eta1.ctypes.data_as(C.POINTER(C.c_double)) if eta1 is not None else None,
                   e2, eta2, stop_tol)
        self._c(lib().tq_set_params(self.h, C.byref(p)))

    def set_quantizer(self, kind, k=16, lloyd=10, quality=50, keep_labels=False, jpeg_restart=0):
        q = Quant(kind, k, lloyd, quality, int(bool(keep_labels)), int(jpeg_restart))
        self._c(lib().tq_set_quantizer(self.h, C.byref(q)))

    def set_sinogram(self, slice_, sino, node=-1):
        """sino: numpy array (host) or torch CUDA tensor, fp32."""
        try:
            import torch
            if isinstance(sino, torch.Tensor):
                t = sino.detach().contiguous().to(torch.float32)
                if t.is_cuda:  # ordered after torch's pending writes to t (its current stream)
                    self._c(lib().tq_set_sinogram_stream(self.h, slice_, node, t.data_ptr(), t.numel(),
                                                         _stream(None)))
                else:
                    self._c(lib().tq_set_sinogram(self.h, slice_, node, t.data_ptr(), t.numel(), 0))
                return
        except ImportError:
            pass
        a = np.ascontiguousarray(sino, np.float32)
        self._c(lib().tq_set_sinogram(self.h, slice_, node, a.ctypes.data, a.size, 0))

    def run(self, iters, stream=None):
        self._c(lib().tq_run(self.h, iters, _stream(stream) if stream is not None else None))

    def run_async(self, iters, stream=None):
        """Enqueue `iters` iterations without waiting (tq_run_async); `wait()` (or any
        call that waits) reports their divergence check."""
        self._c(lib().tq_run_async(self.h, iters, _stream(stream) if stream is not None else None))

    def wait(self):
        self._c(lib().tq_wait(self.h))

    def image(self, slice_=0, node=-1, out=None, host_out=None):
        """Host numpy image; or into a CUDA tensor `out` / a (pinned) host tensor
        `host_out` (fp32, N*N elements)."""
        if out is not None:
            self._c(lib().tq_get_image(self.h, slice_, node, out.data_ptr(), self.n, 1))
            return out
        if host_out is not None:
            self._c(lib().tq_get_image(self.h, slice_, node, host_out.data_ptr(), self.n, 0))
            return host_out
        a = np.zeros(self.n, np.float32)
        self._c(lib().tq_get_image(self.h, slice_, node, a.ctypes.data, self.n, 0))
        return a.reshape(self.N, self.N)

    def image_async(self, out, stream, slice_=0, node=-1):
        """Enqueue the image copy into `out` (pinned host or CUDA fp32 tensor, N*N) on the
        torch CUDA `stream`; it is there once `stream` completes (tq_get_image_async)."""
        self._c(lib().tq_get_image_async(self.h, slice_, node, out.data_ptr(), self.n, 1 if out.is_cuda else 0,
                                         _stream(stream)))
        return out

    def export_state(self, slice_, node):
        buf = np.zeros(3 * self.n, np.float64)
        self._c(lib().tq_export_state(self.h, slice_, node, buf.ctypes.data, buf.size))
        return buf.reshape(3, self.n)

    def import_state(self, slice_, node, state):
        buf = np.ascontiguousarray(np.asarray(state, np.float64).reshape(-1))
        self._c(lib().tq_import_state(self.h, slice_, node, buf.ctypes.data, buf.size))

    def labels(self, slice_, node, length):
        buf = np.zeros(length, np.int32)
        self._c(lib().tq_export_labels(self.h, slice_, node, buf.ctypes.data, length))
        return buf

    def launch_component(self, component, reps=1, stream=None) -> int:
        """Enqueue `reps` launches of one component (profiling hook); returns the
        algorithmic units per launch."""
        u = C.c_int64()
        self._c(lib().tq_launch_component(self.h, component, reps,
                                          _stream(stream) if stream is not None else None, C.byref(u)))
        return u.value

    def stats(self) -> dict:
        s = Stats()
        self._c(lib().tq_get_stats(self.h, C.byref(s)))
        out = {f: getattr(s, f) for f, _ in Stats._fields_}
        out["phase_ms"] = list(s.phase_ms)
        return out

    def set_profiling(self, on=True):
        self._c(lib().tq_set_profiling(self.h, int(bool(on))))

    def node_bytes(self, slice_, node):
        """(sent, received) bytes of a local node in the last iteration (tq_get_node_bytes)."""
        a, b = C.c_int64(), C.c_int64()
        self._c(lib().tq_get_node_bytes(self.h, slice_, node, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None):
            lib().tq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------- stateless kernels
def _prec(t):
    import torch
    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise TypeError("float32 or float64 tensors only")


def project(img, n_angles, n_det, sel=None, stream=None, projector=PROJ_JOSEPH, angles=None):
    """A img for the selected angles; img: CUDA tensor N x N (fp32/fp64)."""
    import torch
    N = img.shape[-1]
    sel = _i32arr(np.arange(n_angles) if sel is None else sel)
    out = torch.empty((len(sel), n_det), dtype=img.dtype, device=img.device)
    g, _keep = _geom(N, n_angles, n_det, projector, angles)
    _check(lib().tq_project(C.byref(g), sel.ctypes.data, len(sel), img.contiguous().data_ptr(),
                            out.data_ptr(), _prec(img), _stream(stream)))
    return out


def backproject(sino, N, n_angles, sel=None, stream=None, projector=PROJ_JOSEPH, angles=None):
    import torch
    sel = _i32arr(np.arange(n_angles) if sel is None else sel)
    out = torch.empty((N, N), dtype=sino.dtype, device=sino.device)
    g, _keep = _geom(N, n_angles, sino.shape[-1], projector, angles)
    _check(lib().tq_backproject(C.byref(g), sel.ctypes.data, len(sel), sino.contiguous().data_ptr(),
                                out.data_ptr(), _prec(sino), _stream(stream)))
    return out


def local_solve(d, bprime, c, e1, x0, n_angles, sel, inner=INNER_CG, eta=0.0, stream=None,
                projector=PROJ_JOSEPH):
    x = x0.clone().contiguous()
    N = x.shape[-1]
    sel = _i32arr(sel)
    g, _keep = _geom(N, n_angles, d.shape[-1], projector, None)
    _check(lib().tq_local_solve(C.byref(g), sel.ctypes.data, len(sel), d.contiguous().data_ptr(),
                                bprime.contiguous().data_ptr(), float(c), inner, e1, float(eta),
                                x.data_ptr(), _prec(x), _stream(stream)))
    return x


def kmeans_encode(v, k, iters, want_labels=True, stream=None):
    import torch
    v = v.contiguous().view(-1)
    n = v.numel()
    B = max(0, int(np.ceil(np.log2(k)))) if k > 1 else 0
    cen = torch.empty(k, dtype=torch.float32, device=v.device)
    planes = torch.zeros(max(1, ((n + 31) // 32) * B), dtype=torch.int32, device=v.device)
    lab = torch.empty(n, dtype=torch.int32, device=v.device) if want_labels else None
    _check(lib().tq_kmeans_encode(v.data_ptr(), n, k, iters, cen.data_ptr(), planes.data_ptr(),
                                  lab.data_ptr() if lab is not None else None, _stream(stream)))
    return cen, planes, lab


def kmeans_decode(cen, planes, n, k, stream=None):
    import torch
    out = torch.empty(n, dtype=torch.float32, device=cen.device)
    _check(lib().tq_kmeans_decode(cen.data_ptr(), planes.data_ptr(), n, k, out.data_ptr(), _stream(stream)))
    return out


def dct_encode(v, quality, stream=None):
    import torch
    rows, cols = v.shape
    coef = torch.empty(rows * cols, dtype=torch.int16, device=v.device)
    mm = torch.empty(2, dtype=torch.float32, device=v.device)
    _check(lib().tq_dct_encode(v.contiguous().data_ptr(), rows, cols, quality, coef.data_ptr(),
                               mm.data_ptr(), _stream(stream)))
    return coef, mm


def jpeg_encode(coef, restart, stream=None):
    """Baseline JPEG Huffman entropy coding of int16 coefficient blocks (device tensor,
    tq_dct_encode order) with an RSTm marker every `restart` blocks -> uint8 device tensor."""
    import torch
    coef = coef.contiguous().view(-1)
    nb = coef.numel() // 64
    cap = 2 * coef.numel()
    out = torch.empty(max(1, cap), dtype=torch.uint8, device=coef.device)
    n = C.c_int64()
    _check(lib().tq_jpeg_encode(coef.data_ptr(), nb, restart, out.data_ptr(), cap, C.byref(n), _stream(stream)))
    return out[:n.value]


def jpeg_decode(stream_bytes, n_blocks, restart, stream=None):
    import torch
    coef = torch.empty(64 * n_blocks, dtype=torch.int16, device=stream_bytes.device)
    _check(lib().tq_jpeg_decode(stream_bytes.contiguous().data_ptr(), stream_bytes.numel(), n_blocks, restart,
                                coef.data_ptr(), _stream(stream)))
    return coef


def dct_decode(coef, mm, rows, cols, quality, stream=None):
    import torch
    out = torch.empty((rows, cols), dtype=torch.float32, device=coef.device)
    _check(lib().tq_dct_decode(coef.data_ptr(), mm.data_ptr(), rows, cols, quality, out.data_ptr(),
                               _stream(stream)))
    return out
