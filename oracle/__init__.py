"""fp64 CPU oracle (ctypes wrapper around oracle.c).

TEST INFRASTRUCTURE ONLY: may be imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, nothing else.  Shares no code
with the CUDA path.  Each function cites the PAPER.md passage it follows (see
oracle.c for the line-level citations).

Parity status: every exported function is pinned by a
`-m "not gpu"` test in tests/test_oracle_*.py against a closed form, a textbook
routine, a brute-force construction or a value printed in the paper.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "_liboracle.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_sp = np.ctypeslib.ndpointer(dtype=np.int16, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile oracle.c (plain gcc, IEEE fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.or_angles.argtypes = [C.c_int, _dp, _dp, _dp, _ip, _dp]
        L.or_project.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp]
        L.or_project_t.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _ip, _dp, _dp]
        L.or_backproject_t.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _ip, _dp, _dp]
        L.or_project_siddon_t.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _ip, _dp, _dp]
        L.or_backproject_siddon_t.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, _ip, _dp, _dp]
        L.or_backproject.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp]
        L.or_gd.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp, C.c_double,
                            C.c_double, C.c_int, _dp]
        L.or_cg.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp, C.c_double,
                            C.c_int, _dp]
        L.or_kmeans_encode.argtypes = [_fp, C.c_long, C.c_int, C.c_int, _fp, _ip]
        L.or_kmeans_decode.argtypes = [_fp, _ip, C.c_long, _fp]
        L.or_dct_qtable.argtypes = [C.c_int, _ip]
        L.or_dct_cmatrix.argtypes = [_ip]
        L.or_dct_encode.argtypes = [_fp, C.c_int, C.c_int, C.c_int, _sp, _fp]
        L.or_dct_decode.argtypes = [_sp, _fp, C.c_int, C.c_int, C.c_int, _fp, C.c_void_p]
        L.or_project_siddon.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp]
        L.or_backproject_siddon.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _dp, _dp]
        L.or_jpeg_tables.argtypes = [_up, _up, _up, _up]
        L.or_jpeg_zigzag.argtypes = [_ip]
        L.or_jpeg_encode.argtypes = [_sp, C.c_long, C.c_int, _up, C.c_long]
        L.or_jpeg_encode.restype = C.c_long
        L.or_jpeg_decode.argtypes = [_up, C.c_long, C.c_long, C.c_int, _sp]
        L.or_jpeg_decode.restype = C.c_int
        L.or_partition_angles.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip]
        L.or_partition_rows.argtypes = [C.c_int, C.c_int, _ip]
        L.or_admm_run.restype = C.c_long
        L.or_admm_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, C.c_int, _ip,
                                  C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                  C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int,
                                  _dp, _dp, _dp, C.c_int, C.c_int, C.c_void_p, C.c_double,
                                  C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.or_alg3.restype = C.c_double
        L.or_alg3.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int]
        L.or_memory_model.restype = C.c_double
        L.or_memory_model.argtypes = [C.c_int, C.c_double, C.c_double]
        L.or_comm_model.restype = C.c_double
        L.or_comm_model.argtypes = [C.c_int, C.c_double]
        _lib = L
    return _lib


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# ----------------------------------------------------------------- geometry / projector
def angles(n_ang: int):
    th, cs, sn, m = (np.zeros(n_ang) for _ in range(4))
    xm = np.zeros(n_ang, np.int32)
    lib().or_angles(n_ang, th, cs, sn, xm, m)
    return th, cs, sn, xm, m


def _theta(theta, n_ang):
    if theta is None:
        return None, None
    t = _f64(theta).ravel()
    assert t.size == n_ang
    return t.ctypes.data, t


def project(img, n_ang: int, n_det: int, sel=None, theta=None):
    """A img for the selected angles (Eq. 2, Joseph discretisation).
    theta: explicit angles in radians (None: pi a / n_ang)."""
    img = _f64(img)
    N = img.shape[0]
    sel = _i32(np.arange(n_ang) if sel is None else sel)
    out = np.zeros((len(sel), n_det))
    tp, _keep = _theta(theta, n_ang)
    lib().or_project_t(N, n_det, n_ang, tp, len(sel), sel, img, out)
    return out


def project_siddon(img, n_ang: int, n_det: int, sel=None, theta=None):
    """A img with P_ji = length of ray j inside pixel i (Siddon's
    algorithm, R-26)."""
    img = _f64(img)
    N = img.shape[0]
    sel = _i32(np.arange(n_ang) if sel is None else sel)
    out = np.zeros((len(sel), n_det))
    tp, _keep = _theta(theta, n_ang)
    lib().or_project_siddon_t(N, n_det, n_ang, tp, len(sel), sel, img, out)
    return out


def backproject_siddon(sino, N: int, n_ang: int, sel=None, theta=None):
    sino = _f64(sino)
    sel = _i32(np.arange(n_ang) if sel is None else sel)
    n_det = sino.shape[-1]
    out = np.zeros((N, N))
    tp, _keep = _theta(theta, n_ang)
    lib().or_backproject_siddon_t(N, n_det, n_ang, tp, len(sel), sel, sino.reshape(len(sel), n_det), out)
    return out


def backproject(sino, N: int, n_ang: int, sel=None, theta=None):
    """A^T sino (the transpose in Alg. 1/2)."""
    sino = _f64(sino)
    sel = _i32(np.arange(n_ang) if sel is None else sel)
    n_det = sino.shape[-1]
    out = np.zeros((N, N))
    tp, _keep = _theta(theta, n_ang)
    lib().or_backproject_t(N, n_det, n_ang, tp, len(sel), sel, sino.reshape(len(sel), n_det), out)
    return out


def cg(d, bprime, c: float, e1: int, x0, n_ang: int, sel):
    x = _f64(x0).copy()
    N = x.shape[0]
    sel = _i32(sel)
    d = _f64(d).reshape(len(sel), -1)
    lib().or_cg(N, d.shape[1], n_ang, len(sel), sel, d, _f64(bprime), c, e1, x)
    return x


def gd(d, bprime, c: float, eta: float, e1: int, x0, n_ang: int, sel):
    x = _f64(x0).copy()
    N = x.shape[0]
    sel = _i32(sel)
    d = _f64(d).reshape(len(sel), -1)
    lib().or_gd(N, d.shape[1], n_ang, len(sel), sel, d, _f64(bprime), c, eta, e1, x)
    return x


# ----------------------------------------------------------------- quantizers
def kmeans_encode(v, K: int, iters: int):
    v = _f32(v).ravel()
    cen = np.zeros(K, np.float32)
    lab = np.zeros(v.size, np.int32)
    lib().or_kmeans_encode(v, v.size, K, iters, cen, lab)
    return cen, lab


def kmeans_decode(cen, lab):
    lab = _i32(lab)
    out = np.zeros(lab.size, np.float32)
    lib().or_kmeans_decode(_f32(cen), lab, lab.size, out)
    return out


def dct_qtable(quality: int):
    q = np.zeros(64, np.int32)
    lib().or_dct_qtable(quality, q)
    return q.reshape(8, 8)


def dct_cmatrix():
    c = np.zeros(64, np.int32)
    lib().or_dct_cmatrix(c)
    return c.reshape(8, 8)


def dct_encode(v, quality: int):
    v = _f32(v)
    rows, cols = v.shape
    coef = np.zeros(rows * cols, np.int16)
    mm = np.zeros(2, np.float32)
    lib().or_dct_encode(v, rows, cols, quality, coef, mm)
    return coef, mm


def dct_decode(coef, mm, rows: int, cols: int, quality: int, return_samples: bool = False):
    out = np.zeros((rows, cols), np.float32)
    smp = np.zeros((rows, cols), np.uint8)
    lib().or_dct_decode(np.ascontiguousarray(coef, dtype=np.int16), _f32(mm), rows, cols,
                        quality, out, smp.ctypes.data if return_samples else None)
    return (out, smp) if return_samples else out


# ----------------------------------------------------------------- JPEG entropy coding (NEXT-2)
def jpeg_tables():
    """(dc_bits, dc_val, ac_bits, ac_val) as the oracle stores them (T.81 Tables K.3, K.5)."""
    t = [np.zeros(16, np.uint8), np.zeros(12, np.uint8), np.zeros(16, np.uint8), np.zeros(162, np.uint8)]
    lib().or_jpeg_tables(*t)
    return tuple(t)


def jpeg_zigzag():
    z = np.zeros(64, np.int32)
    lib().or_jpeg_zigzag(z)
    return z


def jpeg_encode(coef, restart: int = 0) -> bytes:
    """Baseline JPEG Huffman entropy coding (T.81 F.1.2) of int16 blocks [nblocks*64]
    (natural order, raster block order) with a restart marker every `restart` blocks."""
    c = np.ascontiguousarray(coef, dtype=np.int16).ravel()
    nb = c.size // 64
    cap = 16 + nb * 512 + 4 * (nb // max(1, restart) + 1)
    out = np.zeros(cap, np.uint8)
    n = lib().or_jpeg_encode(c, nb, restart, out, cap)
    if n < 0:
        raise ValueError("jpeg_encode: value outside the baseline categories")
    return out[:n].tobytes()


def jpeg_decode(stream: bytes, nblocks: int, restart: int = 0):
    buf = np.frombuffer(bytes(stream), np.uint8).copy() if len(stream) else np.zeros(1, np.uint8)
    coef = np.zeros(nblocks * 64, np.int16)
    if lib().or_jpeg_decode(buf, len(stream), nblocks, restart, coef) != 0:
        raise ValueError("jpeg_decode: malformed stream")
    return coef


# ----------------------------------------------------------------- partitions / models
def partition_angles(n_ang: int, M: int, contiguous: bool):
    off = np.zeros(M + 1, np.int32)
    idx = np.zeros(n_ang, np.int32)
    lib().or_partition_angles(n_ang, M, int(bool(contiguous)), off, idx)
    return off, idx


def partition_rows(N: int, M: int):
    off = np.zeros(M + 1, np.int32)
    lib().or_partition_rows(N, M, off)
    return off


def alg3(x: float, u: float, lam: float, rho: float, eta2: float, e2: int) -> float:
    """Alg. 3 on one element."""
    return lib().or_alg3(x, u, lam, rho, eta2, e2)


def memory_model(M: int, D: float, X: float) -> float:
    return lib().or_memory_model(M, D, X)


def comm_model(M: int, X: float) -> float:
    return lib().or_comm_model(M, X)


# ----------------------------------------------------------------- ADMM
class OracleADMM:
    """The ADMM outer loop (Alg. 4 PAPER.md:207-229 / DESIGN.md R-7) on one slice.
    rule 0 graph (R-7), 1 paper (eq:solve_u..eq:solve_lamda), 2 consensus (P:121-131,
    segment-sharded with Q per segment).

    State: X (private x_i / u_m), L (alpha_i / lambda_m), XH (graph: xhat_i per node;
    paper / consensus: x in XH[0])."""

    def __init__(self, N, n_det, n_ang, M, edges, sino_full, split_contig, rule=0, inner=1,
                 e1=5, rho=1.0, eta1=None, e2=10, eta2=0.2, qkind=0, K=16, lloyd=10,
                 quality=50, threads=1, projector=0, theta=None, stop_tol=0.0):
        self.N, self.n_det, self.n_ang, self.M = N, n_det, n_ang, M
        self.projector = projector  # 0 Joseph (R-1), 1 Siddon (R-26, NEXT-3)
        self.theta = None if theta is None else _f64(theta).ravel()  # explicit angles (radians)
        self.stop_tol = float(stop_tol)  # P:330 stopping criterion (R-13); 0 = fixed count
        self.last_change = -1.0
        if qkind == 2:  # the DCT codec works on whole 8x8 blocks (R-18)
            rows = N // M if rule in (1, 2) else N
            if N % 8 or rows % 8 or (rule in (1, 2) and N % M):
                raise ValueError("DCT quantizer needs 8 | N and 8 | segment rows")
        self.off, self.idx = partition_angles(n_ang, M, split_contig)
        sino_full = np.asarray(sino_full, np.float64).reshape(n_ang, n_det)
        self.d = _f64(np.concatenate([sino_full[self.idx[self.off[m]:self.off[m + 1]]].ravel()
                                      for m in range(M)]))
        self.edges = _i32(np.asarray(edges, np.int32).reshape(-1, 2).ravel() if len(edges) else
                          np.zeros(2, np.int32))
        self.n_edges = len(edges)
        self.rule, self.inner, self.e1, self.rho = rule, inner, e1, rho
        self.eta1 = None if eta1 is None else _f64(eta1)
        self.e2, self.eta2 = e2, eta2
        self.qkind, self.K, self.lloyd, self.quality = qkind, K, lloyd, quality
        self.threads = threads
        n = N * N
        self.X = np.zeros((M, n))
        self.L = np.zeros((M, n))
        self.XH = np.zeros((M if rule == 0 else 1, n))  # rule 1 (paper) and 2 (consensus): x
        self.iters = 0
        self.bytes_per_iter = 0

    def run(self, iters: int):
        done, change = C.c_int(0), C.c_double(-1.0)
        self.bytes_per_iter = lib().or_admm_run(
            self.N, self.n_det, self.n_ang, self.M, self.off, self.idx, self.n_edges, self.edges,
            self.rule, self.inner, self.e1, self.rho,
            None if self.eta1 is None else self.eta1.ctypes.data, self.e2, self.eta2,
            self.qkind, self.K, self.lloyd, self.quality, self.d, iters, self.X, self.L, self.XH,
            self.threads, self.projector, None if self.theta is None else self.theta.ctypes.data,
            self.stop_tol, C.byref(done), C.byref(change))
        self.iters += done.value
        self.last_run_iters = done.value
        self.last_change = change.value
        return self

    def image(self):
        """graph rule: mean over nodes of the private x_i (R-22); paper rule: x."""
        N = self.N
        if self.rule == 0:
            return self.X.mean(axis=0).reshape(N, N)
        return self.XH[0].reshape(N, N).copy()
