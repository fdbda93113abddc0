"""B200-native Gauss-Newton Hessian-vector products for FWI (arxiv 2507.10804).

Thin Python binding of the C ABI in `include/hv.h` (libhv.so, built in-tree by
`python -m paper_2507_10804_b200.build`). The binding only marshals arguments: every step of
forward / gradient / hessvec / psido_apply runs in the library's sm_100a kernels. There is no
CPU fallback — importing works without a GPU, but creating a `Solver` on a machine without an
sm_100 device raises `HVError` (status HV_ECUDA).

Arrays may be numpy arrays (host; the library copies them in/out inside the call, which is
what the end-to-end bench measures) or torch CUDA tensors (device; zero-copy, work ordered on
torch's current stream: a non-default stream is bound with hv_set_stream, and on torch's default
stream the library's own stream first waits for the legacy default stream). Layout: [nz][nx]
float32 row-major; data [shot][nt][nrec]; probes [K][nz][nx].
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = ["Solver", "HVError", "lib", "STORE", "psido_apply"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HV_LIB") or os.path.join(_HERE, "libhv.so")  # HV_LIB: tuning variants only

HV_OK, HV_EINVAL, HV_EGRID, HV_ECFL, HV_ENOMEM, HV_ECUDA, HV_ESTATE, HV_ENCCL = range(8)
STATUS = {0: "HV_OK", 1: "HV_EINVAL", 2: "HV_EGRID", 3: "HV_ECFL", 4: "HV_ENOMEM", 5: "HV_ECUDA", 6: "HV_ESTATE",
          7: "HV_ENCCL"}
STORE = {"auto": 0, "full": 1, "checkpoint": 2, "boundary": 3}


class HVError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class HvConfig(ctypes.Structure):
    _fields_ = [
        ("nz", ctypes.c_int32), ("nx", ctypes.c_int32), ("h", ctypes.c_float), ("dt", ctypes.c_float),
        ("nt", ctypes.c_int32), ("sponge", ctypes.c_int32), ("v_ref", ctypes.c_float),
        ("nsrc", ctypes.c_int32), ("src_iz", ctypes.POINTER(ctypes.c_int32)),
        ("src_ix", ctypes.POINTER(ctypes.c_int32)),
        ("nrec", ctypes.c_int32), ("rec_iz", ctypes.POINTER(ctypes.c_int32)),
        ("rec_ix", ctypes.POINTER(ctypes.c_int32)),
        ("wavelet", ctypes.POINTER(ctypes.c_float)),
        ("src_begin", ctypes.c_int32), ("src_end", ctypes.c_int32),
        ("store", ctypes.c_int32), ("ckpt_interval", ctypes.c_int32),
        ("shot_batch", ctypes.c_int32), ("field_group", ctypes.c_int32),
        ("device", ctypes.c_int32), ("mem_budget", ctypes.c_size_t), ("nccl_comm", ctypes.c_void_p),
    ]


class HvStats(ctypes.Structure):
    _fields_ = [
        ("kernel_launches", ctypes.c_int64), ("graph_launches", ctypes.c_int64),
        ("shot_batch", ctypes.c_int32), ("field_group", ctypes.c_int32), ("store", ctypes.c_int32),
        ("ckpt_interval", ctypes.c_int32), ("bytes_per_shot", ctypes.c_double),
        ("ms_forward", ctypes.c_double), ("ms_backward", ctypes.c_double), ("ms_total", ctypes.c_double),
        ("fwd_kernel", ctypes.c_int32), ("bwd_kernel", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libhv.so (fails loudly if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2507_10804_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, fp, ip = ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p
        L.hv_create.argtypes = [ctypes.POINTER(HvConfig), ctypes.POINTER(ctypes.c_void_p)]
        L.hv_destroy.argtypes = [vp]
        L.hv_set_stream.argtypes = [vp, vp]
        L.hv_forward.argtypes = [vp, fp, fp]
        L.hv_forward_shot.argtypes = [vp, fp, i32, fp]
        L.hv_misfit.argtypes = [vp, fp, fp, ctypes.POINTER(ctypes.c_double)]
        L.hv_set_comm.argtypes = [vp, vp]
        L.hv_nccl_unique_id.argtypes = [vp]
        L.hv_nccl_comm_create.argtypes = [i32, i32, vp, i32, ctypes.POINTER(ctypes.c_void_p)]
        L.hv_nccl_comm_destroy.argtypes = [vp]
        L.hv_gradient.argtypes = [vp, fp, fp, fp, ctypes.POINTER(ctypes.c_double)]
        L.hv_hessvec.argtypes = [vp, fp, i32, fp, fp]
        L.hv_gradient_hessvec.argtypes = [vp, fp, fp, i32, fp, fp, ctypes.POINTER(ctypes.c_double), fp]
        L.hv_psido_apply.argtypes = [vp, i32, i32, i32, fp, fp, fp, fp, i32]
        L.hv_psf_rows.argtypes = [vp, i32, i32, i32, fp, i32, ip, ip, ip, i32, fp]
        L.hv_psf_weights.argtypes = [vp, i32, i32, i32, ip, i32, ip, fp]
        L.hv_pdo_columns.argtypes = [vp, i32, i32, fp, i32, ip, ip, ctypes.c_float, fp]
        L.hv_pdo_weights.argtypes = [vp, i32, i32, ctypes.c_float, ctypes.c_float, i32, fp, fp]
        L.hv_highpass.argtypes = [vp, i32, i32, ctypes.c_float, ctypes.c_float, ctypes.c_float, i32, fp, fp]
        L.hv_lowrank_geneig.argtypes = [vp, fp, i32, i32, fp, i32, ctypes.c_double, ctypes.c_double, fp, fp]
        L.hv_psf_plus.argtypes = [vp, i32, i32, i32, fp, fp, i32, fp, ip, ip, i32, fp, fp,
                                  ctypes.POINTER(ctypes.c_double)]
        L.hv_get_stats.argtypes = [vp, ctypes.POINTER(HvStats)]
        L.hv_last_error.argtypes = [vp]
        L.hv_last_error.restype = ctypes.c_char_p
        for name in ("hv_create", "hv_destroy", "hv_set_stream", "hv_forward", "hv_forward_shot", "hv_misfit",
                     "hv_set_comm", "hv_nccl_unique_id", "hv_nccl_comm_create", "hv_nccl_comm_destroy",
                     "hv_gradient", "hv_hessvec",
                     "hv_gradient_hessvec", "hv_psido_apply", "hv_get_stats", "hv_psf_rows", "hv_psf_weights",
                     "hv_pdo_columns", "hv_pdo_weights", "hv_highpass", "hv_lowrank_geneig", "hv_psf_plus"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Arr:
    """Marshal one array argument: (pointer, keep-alive, is_device)."""

    def __init__(self, x, dtype=np.float32, shape: Optional[Sequence[int]] = None, name: str = "array"):
        if _is_torch(x):
            import torch
            tdt = {np.float32: torch.float32, np.complex64: torch.complex64}[dtype]
            if x.dtype != tdt:
                raise TypeError(f"{name}: expected {tdt}, got {x.dtype}")
            x = x.contiguous()
            self.device = x.is_cuda
            self.ptr = ctypes.c_void_p(x.data_ptr())
        else:
            x = np.ascontiguousarray(x, dtype=dtype)
            self.device = False
            self.ptr = ctypes.c_void_p(x.ctypes.data)
        if shape is not None and tuple(x.shape) != tuple(shape):
            raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(x.shape)}")
        self.obj = x


def _empty_like_kind(ref: _Arr, shape, dtype=np.float32):
    if _is_torch(ref.obj):
        import torch
        return torch.empty(tuple(shape), dtype=torch.float32, device=ref.obj.device)
    return np.empty(tuple(shape), dtype=dtype)


class Solver:
    """One hv_ctx: the acquisition of a shot shard [src_begin, src_end) on one GPU."""

    def __init__(self, *, nz: int, nx: int, h: float, dt: float, nt: int, sponge: int, v_ref: float,
                 src: np.ndarray, rec: np.ndarray, wavelet: np.ndarray, src_begin: int = 0,
                 src_end: Optional[int] = None, store: str = "auto", ckpt_interval: int = 0,
                 shot_batch: int = 0, field_group: int = 0, device: int = 0, mem_budget: int = 0,
                 nccl_comm: Optional[int] = None):
        L = lib()
        self._src = np.ascontiguousarray(src, dtype=np.int32)
        self._rec = np.ascontiguousarray(rec, dtype=np.int32)
        self._siz, self._six = np.ascontiguousarray(self._src[:, 0]), np.ascontiguousarray(self._src[:, 1])
        self._riz, self._rix = np.ascontiguousarray(self._rec[:, 0]), np.ascontiguousarray(self._rec[:, 1])
        self._wav = np.ascontiguousarray(wavelet, dtype=np.float32)
        i32p = ctypes.POINTER(ctypes.c_int32)
        cfg = HvConfig(
            nz=nz, nx=nx, h=h, dt=dt, nt=nt, sponge=sponge, v_ref=v_ref, nsrc=len(self._src),
            src_iz=self._siz.ctypes.data_as(i32p), src_ix=self._six.ctypes.data_as(i32p),
            nrec=len(self._rec), rec_iz=self._riz.ctypes.data_as(i32p), rec_ix=self._rix.ctypes.data_as(i32p),
            wavelet=self._wav.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
            src_begin=src_begin, src_end=(len(self._src) if src_end is None else src_end),
            store=STORE[store] if isinstance(store, str) else int(store), ckpt_interval=ckpt_interval,
            shot_batch=shot_batch, field_group=field_group, device=device, mem_budget=mem_budget,
            nccl_comm=nccl_comm)
        h_ = ctypes.c_void_p()
        st = L.hv_create(ctypes.byref(cfg), ctypes.byref(h_))
        if st != HV_OK:
            raise HVError(st, "hv_create failed (see stderr)")
        self._h = h_
        self.nz, self.nx, self.nt, self.nrec = nz, nx, nt, len(self._rec)
        self.src_begin = src_begin
        self.src_end = len(self._src) if src_end is None else src_end
        self.nloc = self.src_end - self.src_begin
        self.device = device

    @classmethod
    def from_workload(cls, wl, **kw) -> "Solver":
        return cls(nz=wl.nz, nx=wl.nx, h=wl.h, dt=wl.dt, nt=wl.nt, sponge=wl.W, v_ref=wl.v_ref,
                   src=wl.src, rec=wl.rec, wavelet=wl.wavelet, **kw)

    def close(self):
        if getattr(self, "_h", None):
            lib().hv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != HV_OK:
            raise HVError(st, lib().hv_last_error(self._h).decode())

    def _stream(self, *arrs):
        if any(a.device for a in arrs):
            import torch
            lib().hv_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        else:
            lib().hv_set_stream(self._h, None)

    # ---------------------------------------------------------------- the paper's calls

    def forward(self, m, out=None):
        """d = f(m) for the shard: [nloc][nt][nrec]."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        shape = (self.nloc, self.nt, self.nrec)
        o = _Arr(out if out is not None else _empty_like_kind(a, shape), shape=shape, name="d")
        self._stream(a, o)
        self._check(lib().hv_forward(self._h, a.ptr, o.ptr))
        return o.obj

    def forward_shot(self, m, isrc: int, out=None):
        """d = f(m) for ONE shot, global index isrc in [src_begin, src_end): [nt][nrec]."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        shape = (self.nt, self.nrec)
        o = _Arr(out if out is not None else _empty_like_kind(a, shape), shape=shape, name="d")
        self._stream(a, o)
        self._check(lib().hv_forward_shot(self._h, a.ptr, int(isrc), o.ptr))
        return o.obj

    def misfit(self, m, d_obs) -> float:
        """Phi_d(m) = 1/2 sum (f(m) - d_obs)^2 over the shard: forward + residual only, no adjoint (the
        likelihood each gpCN proposal evaluates)."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        d = _Arr(d_obs, shape=(self.nloc, self.nt, self.nrec), name="d_obs")
        phi = ctypes.c_double(0.0)
        self._stream(a, d)
        self._check(lib().hv_misfit(self._h, a.ptr, d.ptr, ctypes.byref(phi)))
        return phi.value

    def set_comm(self, comm: Optional[int]):
        """Attach a NCCL communicator (from `nccl_comm_create`): g, H·v and phi are then summed over the ranks
        in-library. None detaches it (rank-local partial sums)."""
        self._check(lib().hv_set_comm(self._h, ctypes.c_void_p(comm) if comm else None))

    def gradient(self, m, d_obs, out=None):
        """(phi, g): misfit and its gradient F*(f(m) - d_obs) over the shard."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        d = _Arr(d_obs, shape=(self.nloc, self.nt, self.nrec), name="d_obs")
        o = _Arr(out if out is not None else _empty_like_kind(a, (self.nz, self.nx)), shape=(self.nz, self.nx),
                 name="g")
        phi = ctypes.c_double(0.0)
        self._stream(a, d, o)
        self._check(lib().hv_gradient(self._h, a.ptr, d.ptr, o.ptr, ctypes.byref(phi)))
        return phi.value, o.obj

    def hessvec(self, m, V, out=None):
        """H_d [v_1..v_K] over the shard: V, HV [K][nz][nx]."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        K = int(V.shape[0])
        v = _Arr(V, shape=(K, self.nz, self.nx), name="V")
        o = _Arr(out if out is not None else _empty_like_kind(v, (K, self.nz, self.nx)),
                 shape=(K, self.nz, self.nx), name="HV")
        self._stream(a, v, o)
        self._check(lib().hv_hessvec(self._h, a.ptr, K, v.ptr, o.ptr))
        return o.obj

    def gradient_hessvec(self, m, d_obs, V):
        """(phi, g, HV) in one fused pass (1 + K forward fields, 1 + K adjoint fields)."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        d = _Arr(d_obs, shape=(self.nloc, self.nt, self.nrec), name="d_obs")
        K = int(V.shape[0])
        v = _Arr(V, shape=(K, self.nz, self.nx), name="V")
        g = _Arr(_empty_like_kind(a, (self.nz, self.nx)), name="g")
        o = _Arr(_empty_like_kind(v, (K, self.nz, self.nx)), name="HV")
        phi = ctypes.c_double(0.0)
        self._stream(a, d, v, g, o)
        self._check(lib().hv_gradient_hessvec(self._h, a.ptr, d.ptr, K, v.ptr, g.ptr, ctypes.byref(phi), o.ptr))
        return phi.value, g.obj, o.obj

    def psido_apply(self, a, b, v, mode: int = 0, out=None):
        """Low-rank-symbol PsiDO apply: a [r][nz][nx] real (or complex64: PSF+ factors),
        b [r][nz][nx] complex64, v [nz][nx]; mode 0 apply, 1 adjoint, 2 symmetrised."""
        r, nz, nx = (int(s) for s in a.shape)
        cplx = np.iscomplexobj(a) if not _is_torch(a) else a.is_complex()
        A = _Arr(a, dtype=np.complex64 if cplx else np.float32, shape=(r, nz, nx), name="a")
        mode = int(mode) | (4 if cplx else 0)
        B = _Arr(b, dtype=np.complex64, shape=(r, nz, nx), name="b")
        Vv = _Arr(v, shape=(nz, nx), name="v")
        o = _Arr(out if out is not None else _empty_like_kind(Vv, (nz, nx)), shape=(nz, nx), name="out")
        self._stream(A, B, Vv, o)
        self._check(lib().hv_psido_apply(self._h, nz, nx, r, A.ptr, B.ptr, Vv.ptr, o.ptr, int(mode)))
        return o.obj

    # ---------------------------------------------------------------- probe -> symbol assembly (N1)

    def _cempty(self, ref: _Arr, shape):
        if _is_torch(ref.obj):
            import torch
            return torch.empty(tuple(shape), dtype=torch.complex64, device=ref.obj.device)
        return np.empty(tuple(shape), dtype=np.complex64)

    def psf_rows(self, responses, points, batch_of, radius: int):
        """Symbol rows conj(DFT(p_k)) [np][nz][nx] complex64 from PSF responses [nb][nz][nx]."""
        nb, nz, nx = (int(d) for d in responses.shape)
        R = _Arr(responses, shape=(nb, nz, nx), name="responses")
        pts = np.ascontiguousarray(np.asarray(points, dtype=np.int32).reshape(-1, 2))
        iz, ix = np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1])
        b = np.ascontiguousarray(np.asarray(batch_of, dtype=np.int32))
        out = _Arr(self._cempty(R, (len(pts), nz, nx)), dtype=np.complex64, name="rows")
        self._stream(R, out)
        self._check(lib().hv_psf_rows(self._h, nz, nx, nb, R.ptr, len(pts), iz.ctypes.data, ix.ctypes.data,
                                      b.ctypes.data, int(radius), out.ptr))
        return out.obj

    def psf_weights(self, nz: int, nx: int, lat_z, lat_x, like=None):
        """Bilinear hat weights [len(lat_z) * len(lat_x)][nz][nx]."""
        lz = np.ascontiguousarray(np.asarray(lat_z, dtype=np.int32))
        lx = np.ascontiguousarray(np.asarray(lat_x, dtype=np.int32))
        ref = _Arr(like if like is not None else np.zeros(1, np.float32), name="like")
        out = _Arr(_empty_like_kind(ref, (len(lz) * len(lx), nz, nx)), name="w")
        self._stream(out)
        self._check(lib().hv_psf_weights(self._h, nz, nx, len(lz), lz.ctypes.data, len(lx), lx.ctypes.data, out.ptr))
        return out.obj

    def pdo_columns(self, response, freq_idx, mask_radius: float):
        """Symbol columns [r][nz][nx] complex64 by spectral separation."""
        nz, nx = (int(d) for d in response.shape)
        R = _Arr(response, shape=(nz, nx), name="response")
        f = np.ascontiguousarray(np.asarray(freq_idx, dtype=np.int32).reshape(-1, 2))
        kz, kx = np.ascontiguousarray(f[:, 0]), np.ascontiguousarray(f[:, 1])
        out = _Arr(self._cempty(R, (len(f), nz, nx)), dtype=np.complex64, name="cols")
        self._stream(R, out)
        self._check(lib().hv_pdo_columns(self._h, nz, nx, R.ptr, len(f), kz.ctypes.data, kx.ctypes.data,
                                         float(mask_radius), out.ptr))
        return out.obj

    def pdo_weights(self, nz: int, nx: int, h: float, rho0: float, thetas, like=None):
        """Frequency weights (|xi| / rho0) t(theta - theta_k) [r][nz][nx] complex64."""
        th = np.ascontiguousarray(np.asarray(thetas, dtype=np.float32))
        ref = _Arr(like if like is not None else np.zeros(1, np.float32), name="like")
        out = _Arr(self._cempty(ref, (len(th), nz, nx)), dtype=np.complex64, name="w")
        self._stream(out)
        self._check(lib().hv_pdo_weights(self._h, nz, nx, float(h), float(rho0), len(th), th.ctypes.data, out.ptr))
        return out.obj

    # ---------------------------------------------------------------- high-pass wrapper (N4)

    def highpass(self, V, h: float, cutoff: float, width: float, out=None):
        """Q v for V [K][nz][nx] (or [nz][nx]): raised-cosine high-pass multiplier."""
        squeeze = V.ndim == 2
        K, nz, nx = (1, *V.shape) if squeeze else tuple(int(d) for d in V.shape)
        v = _Arr(V.reshape(K, nz, nx) if squeeze else V, shape=(K, nz, nx), name="V")
        o = _Arr(out if out is not None else _empty_like_kind(v, (K, nz, nx)), shape=(K, nz, nx), name="out")
        self._stream(v, o)
        self._check(lib().hv_highpass(self._h, nz, nx, float(h), float(cutoff), float(width), K, v.ptr, o.ptr))
        return o.obj.reshape(nz, nx) if squeeze else o.obj

    def hessvec_highpass(self, m, V, h: float, cutoff: float, width: float):
        """Q H_d Q [v_1..v_K]: the high-pass-filtered Hessian the PSF / PDO approximations target."""
        return self.highpass(self.hessvec(m, self.highpass(V, h, cutoff, width)), h, cutoff, width)

    # ---------------------------------------------------------------- randomized generalized eigensolver (N2)

    def lowrank_geneig(self, m, Omega, r: int, power_iters: int = 1, delta: float = 1.0, gamma: float = 0.0):
        """Leading r pairs of H_d v = lambda R v, R = (delta I - gamma Delta)^2.
        Omega: [K][nz][nx] random probes, K >= r. Returns (evals float64 [r] descending, evecs [r][nz][nx])."""
        a = _Arr(m, shape=(self.nz, self.nx), name="m")
        K = int(Omega.shape[0])
        om = _Arr(Omega, shape=(K, self.nz, self.nx), name="Omega")
        ev = np.zeros(r, dtype=np.float64)
        V = _Arr(_empty_like_kind(om, (r, self.nz, self.nx)), name="evecs")
        self._stream(a, om, V)
        self._check(lib().hv_lowrank_geneig(self._h, a.ptr, int(r), K, om.ptr, int(power_iters), float(delta),
                                            float(gamma), ev.ctypes.data, V.ptr))
        return ev, V.obj

    # ---------------------------------------------------------------- PSF+ (N3)

    def psf_plus(self, rows, w, cols, col_idx, rank: int):
        """PSF+ factors (A [rank][nz][nx], B [rank][nz][nx]) complex64 and alpha."""
        nr, nz, nx = (int(d) for d in rows.shape)
        R = _Arr(rows, dtype=np.complex64, shape=(nr, nz, nx), name="rows")
        Wt = _Arr(w, shape=(nr, nz, nx), name="w")
        nc = int(cols.shape[0])
        C = _Arr(cols, dtype=np.complex64, shape=(nc, nz, nx), name="cols")
        f = np.ascontiguousarray(np.asarray(col_idx, dtype=np.int32).reshape(-1, 2))
        kz, kx = np.ascontiguousarray(f[:, 0]), np.ascontiguousarray(f[:, 1])
        A = _Arr(self._cempty(R, (rank, nz, nx)), dtype=np.complex64, name="A")
        B = _Arr(self._cempty(R, (rank, nz, nx)), dtype=np.complex64, name="B")
        alpha = ctypes.c_double(0.0)
        self._stream(R, Wt, C, A, B)
        self._check(lib().hv_psf_plus(self._h, nz, nx, nr, R.ptr, Wt.ptr, nc, C.ptr, kz.ctypes.data, kx.ctypes.data,
                                      int(rank), A.ptr, B.ptr, ctypes.byref(alpha)))
        return A.obj, B.obj, alpha.value

    def stats(self) -> dict:
        s = HvStats()
        self._check(lib().hv_get_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in HvStats._fields_}


def psido_apply(solver: Solver, a, b, v, mode: int = 0):
    return solver.psido_apply(a, b, v, mode)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; share it with the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().hv_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st != HV_OK:
        raise HVError(st, "hv_nccl_unique_id failed")
    return buf.raw


def nccl_comm_create(nranks: int, rank: int, uid: bytes, device: int) -> int:
    """A NCCL communicator for the library's in-library reductions (caller owns it: nccl_comm_destroy)."""
    if len(uid) != 128:
        raise ValueError("uid must be 128 bytes")
    buf = ctypes.create_string_buffer(uid, 128)
    out = ctypes.c_void_p()
    st = lib().hv_nccl_comm_create(int(nranks), int(rank), ctypes.cast(buf, ctypes.c_void_p), int(device),
                                   ctypes.byref(out))
    if st != HV_OK:
        raise HVError(st, "hv_nccl_comm_create failed")
    return int(out.value)


def nccl_comm_destroy(comm: int) -> None:
    st = lib().hv_nccl_comm_destroy(ctypes.c_void_p(comm))
    if st != HV_OK:
        raise HVError(st, "hv_nccl_comm_destroy failed")
