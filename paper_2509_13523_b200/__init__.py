"""swinflow-b200: B200-native (sm_100a) denoiser hot path of arxiv 2509.13523 (AERIS).

Thin ctypes mirror of the C-ABI in include/swinflow_capi.h, which itself mirrors the
reference's C++ API (proj/include/swinflow/swin.hpp `forward`, diffusion.hpp `solve_pf_ode`,
`forecast_step`, `rollout_ensemble`). There is no CPU fallback: if the CUDA library is missing
or no B200 is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, astuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWF_LIB") or os.path.join(_HERE, "_build", "libswinflow_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "swinflow_capi.h")

OK, ERR_NUMERICS, ERR_CONFIG, ERR_IO, ERR_CUDA = 0, 1, 2, 3, 4
PREC_BF16, PREC_FP32 = 0, 1
F32, F64 = 0, 1
OWN_CONTIGUOUS, OWN_ROUND_ROBIN = 0, 1


class SwfError(RuntimeError):
    def __init__(self, rc: int, msg: str):
        super().__init__(f"[rc={rc}] {msg}")
        self.rc = rc


class ConfigError(SwfError):
    pass


class NumericsError(SwfError):
    pass


class CudaError(SwfError):
    pass


class IoError(SwfError):
    pass


@dataclass
class ModelConfig:
    """swinflow::ModelConfig (model.hpp:21-62)."""
    hidden_dim: int
    n_heads: int
    ffn_dim: int
    n_layers: int
    blocks_per_layer: int = 1
    window_px: int = 8
    in_channels: int = 8
    out_channels: int = 3
    time_dim: int = 0

    def n_blocks(self) -> int:
        return self.n_layers * self.blocks_per_layer


@dataclass
class DiffusionConfig:
    """swinflow::DiffusionConfig (diffusion.hpp:29-46)."""
    sigma_d: float = 1.0
    sigma_min: float = 0.2
    sigma_max: float = 500.0
    solver_steps: int = 10
    churn: float = 0.0


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("hidden_dim", "n_heads", "ffn_dim", "n_layers", "blocks_per_layer",
                                        "window_px", "in_channels", "out_channels", "time_dim")]


class _DCfg(C.Structure):
    _fields_ = [("sigma_d", C.c_double), ("sigma_min", C.c_double), ("sigma_max", C.c_double),
                ("solver_steps", C.c_int), ("churn", C.c_double)]


class _LW(C.Structure):
    _fields_ = [("alpha_row", C.c_void_p), ("kappa", C.c_void_p)]


class _Std(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("state_mean", "state_std", "resid_mean", "resid_std", "forcing_mean",
                                          "forcing_std")]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    """Load the sm_100a library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"swinflow CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i, d, u64, ll = C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_longlong
        L.swf_last_error.restype = C.c_char_p
        L.swf_version.restype = C.c_char_p
        L.swf_create.argtypes = [vp, i, i, i, i, C.POINTER(vp)]
        L.swf_destroy.argtypes = [vp]
        L.swf_destroy.restype = None
        L.swf_set_topology.argtypes = [vp, i, i, i, i, i]
        L.swf_set_topology_devices.argtypes = [vp, i, i, i, i, vp]
        L.swf_group_size.argtypes = [vp]
        L.swf_group_rank.argtypes = [vp, i]
        L.swf_group_rank.restype = vp
        L.swf_ipc_handles.argtypes = [vp, vp]
        L.swf_connect_peers.argtypes = [vp, vp]
        L.swf_plan_owners.argtypes = [i, i, i, i, i, i, vp]
        L.swf_plan_exchange.argtypes = [i, i, i, i, i, i, i, i, vp]
        L.swf_plan_tokens.argtypes = [i, i, i, i, i, i, i, i, vp]
        L.swf_load_params.argtypes = [vp, vp, i, i]
        L.swf_load_params_flat.argtypes = [vp, vp, ll, i]
        L.swf_init_params.argtypes = [vp, u64, i, d]
        L.swf_load_checkpoint.argtypes = [vp, C.c_char_p]
        L.swf_verify_checkpoint.argtypes = [vp, C.c_char_p]
        L.swf_param_count.argtypes = [vp]
        L.swf_param_count.restype = ll
        L.swf_forward.argtypes = [vp, vp, d, vp, i]
        L.swf_forward_device.argtypes = [vp, vp, d, vp]
        L.swf_sync.argtypes = [vp]
        L.swf_stream.argtypes = [vp]
        L.swf_stream.restype = vp
        L.swf_solve_pf_ode.argtypes = [vp, vp, vp, vp, vp, u64, vp, C.POINTER(i), i]
        L.swf_forecast_step.argtypes = [vp, vp, vp, vp, vp, u64, u64, vp, i]
        L.swf_rollout_ensemble.argtypes = [vp, vp, vp, i, i, vp, vp, u64, u64, vp, i]
        L.swf_local_tokens.argtypes = [vp]
        L.swf_local_tokens.restype = ll
        L.swf_owned_pixels.argtypes = [vp, vp]
        L.swf_kernel_launches.argtypes = [vp]
        L.swf_kernel_launches.restype = ll
        L.swf_bench_kernel.argtypes = [vp, i, i, i, C.POINTER(d)]
        L.swf_profile.argtypes = [vp, i]
        L.swf_set_graphs.argtypes = [vp, i]
        L.swf_fnv1a64.argtypes = [vp, C.c_size_t, u64]
        L.swf_fnv1a64.restype = u64
        L.swf_param_array.argtypes = [vp, i, C.c_char_p, i, C.POINTER(ll), C.POINTER(ll)]
        L.swf_profile_read.argtypes = [vp, vp, vp, i]
        L.swf_profile_launches.argtypes = [vp, vp, vp, i, C.POINTER(i)]
        L.swf_noise_field.argtypes = [vp, u64, u64, i, d, vp]
        L.swf_selftest_gemm.argtypes = [i, ll, i, i, C.POINTER(d), C.POINTER(d)]
        L.swf_selftest_attention.argtypes = [i, i, i, i, i, i, i, i, vp, vp, vp, vp, i]
        L.swf_forward_hidden.argtypes = [vp, vp, d, i, vp, ll, vp, i]
        L.swf_block_window_forward.argtypes = [vp, i, i, i, d, vp, vp, i]
        L.swf_op_linear_cols.argtypes = [i, i, vp, i, i, vp, ll, vp]
        L.swf_op_prenorm_modulate.argtypes = [i, vp, i, ll, vp, vp, vp, vp, vp]
        L.swf_op_swiglu_fwd.argtypes = [i, i, vp, vp, vp, i, i, vp, ll, vp]
        L.swf_op_gemm_bf16.argtypes = [i, i, ll, ll, ll, vp, ll, vp, ll, vp, ll, i]
        L.swf_set_backward_precision.argtypes = [vp, i]
        L.swf_backward.argtypes = [vp, vp, d, vp, vp, vp, i]
        L.swf_diffusion_loss_sample.argtypes = [vp, vp, vp, vp, vp, vp, u64, vp, C.POINTER(d), vp, i]
        L.swf_train_accumulate.argtypes = [vp, vp, vp, vp, vp, vp, u64, u64, C.POINTER(d), i]
        L.swf_train_reset.argtypes = [vp]
        L.swf_train_grads.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(ll)]
        L.swf_train_read.argtypes = [vp, d, vp, i]
        L.swf_prefetch_chunked.argtypes = [vp, C.c_char_p, C.c_char_p]
        L.swf_forecast_step_chunked.argtypes = [vp, C.c_char_p, C.c_char_p, vp, vp, u64, u64, vp, i]
        L.swf_last_chunk_reads.argtypes = [vp]
        L.swf_last_chunk_reads.restype = ll
        L.swf_chunked_write.argtypes = [C.c_char_p, vp, i, i, i, i, i]
        L.swf_chunked_open.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.swf_chunked_close.argtypes = [vp]
        L.swf_chunked_close.restype = None
        L.swf_chunked_info.argtypes = [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i)]
        L.swf_chunked_read.argtypes = [vp, i, i, i, i, vp]
        L.swf_chunked_cover.argtypes = [vp, i, i, i, i, C.POINTER(ll)]
        L.swf_chunked_reads.argtypes = [vp]
        L.swf_chunked_reads.restype = ll
        L.swf_chunked_reset_reads.argtypes = [vp]
        L.swf_chunked_reset_reads.restype = None
        _lib = L
    return _lib


def _check(rc: int):
    if rc == OK:
        return
    msg = lib().swf_last_error().decode()
    cls = {ERR_NUMERICS: NumericsError, ERR_CONFIG: ConfigError, ERR_IO: IoError, ERR_CUDA: CudaError}.get(rc,
                                                                                                SwfError)
    raise cls(rc, msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float64:
        return F64
    if a.dtype == np.float32:
        return F32
    raise TypeError("fields must be float32 or float64")


def param_count(cfg: ModelConfig) -> int:
    return lib().swf_param_count(C.byref(_Cfg(*astuple(cfg))))


def selftest_gemm(M: int, N: int, K: int, device: int = 0):
    e, r = C.c_double(), C.c_double()
    _check(lib().swf_selftest_gemm(device, M, N, K, C.byref(e), C.byref(r)))
    return e.value, r.value


def selftest_attention(q, k, v, n_wy: int, n_wx: int, w: int, shift: int = 0, precision: int = PREC_BF16,
                       flags: int = 0, device: int = 0) -> np.ndarray:
    """The windowed attention kernel alone on q/k/v [n_win][heads][w*w][d] (fp32); returns
    [n_win][w*w][heads*d]. flags bit 0 disables the O rescale (negative control)."""
    q, k, v = (np.ascontiguousarray(a, np.float32) for a in (q, k, v))
    nwin, heads, s, dd = q.shape
    if nwin != n_wy * n_wx or s != w * w or k.shape != q.shape or v.shape != q.shape:
        raise ConfigError(ERR_CONFIG, "selftest_attention: q/k/v must be [n_wy*n_wx][heads][w*w][d]")
    o = np.zeros((nwin, s, heads * dd), np.float32)
    _check(lib().swf_selftest_attention(device, precision, n_wy, n_wx, w, shift, heads, dd, _p(q), _p(k), _p(v),
                                        _p(o), flags))
    return o


class ops:
    """The reference's ops leaves (swin.hpp:49-234) on the device. Matrices are numpy arrays in the
    reference's column-major storage: W (out x in) as W.reshape(in, out) [in][out], fields (C x n) as
    [n][C] rows."""

    @staticmethod
    def linear_cols(W, out: int, inp: int, X, precision: int = PREC_BF16, device: int = 0):
        W = np.ascontiguousarray(W, np.float32).reshape(-1)
        X = np.ascontiguousarray(X, np.float32)
        n = X.size // inp
        Y = np.zeros((n, out), np.float32)
        _check(lib().swf_op_linear_cols(device, precision, _p(W), out, inp, _p(X), n, _p(Y)))
        return Y

    @staticmethod
    def prenorm_modulate(X, g, a=None, b=None, gate=None, device: int = 0):
        X = np.ascontiguousarray(X, np.float32)
        n, h = X.shape
        Y = np.zeros_like(X)
        v = [None if t is None else np.ascontiguousarray(t, np.float32) for t in (g, a, b, gate)]
        _check(lib().swf_op_prenorm_modulate(device, _p(X), h, n, *[_p(t) for t in v], _p(Y)))
        return Y

    @staticmethod
    def swiglu_fwd(W_gate, W_up, W_down, h: int, f: int, X, precision: int = PREC_BF16, device: int = 0):
        W = [np.ascontiguousarray(t, np.float32).reshape(-1) for t in (W_gate, W_up, W_down)]
        X = np.ascontiguousarray(X, np.float32)
        n = X.size // h
        Y = np.zeros((n, h), np.float32)
        _check(lib().swf_op_swiglu_fwd(device, precision, *[_p(t) for t in W], h, f, _p(X), n, _p(Y)))
        return Y

    @staticmethod
    def gemm_bf16(A, B, mn_major: bool, C=None, accumulate: bool = False, device: int = 0):
        """The backward's tensor-core GEMM: returns C (+)= op(A) . op(B) in fp32 with bf16-rounded operands.
        K-major: A [M][K], B [N][K] (C = A B^T); MN-major: A [K][M], B [K][N] (C = A^T B)."""
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        if mn_major:
            (K, M), N = A.shape, B.shape[1]
        else:
            (M, K), N = A.shape, B.shape[0]
        C = np.zeros((M, N), np.float32) if C is None else np.ascontiguousarray(C, np.float32).copy()
        _check(lib().swf_op_gemm_bf16(device, int(mn_major), M, N, K, _p(A), A.shape[1], _p(B), B.shape[1], _p(C),
                                      N, int(accumulate)))
        return C


class Denoiser:
    """Device context for one model on one H x W grid (forward / solve / forecast)."""

    def __init__(self, cfg: ModelConfig, grid_h: int, grid_w: int, device: int = 0, precision: int = PREC_BF16,
                 topology: tuple | None = None, devices: list | None = None):
        """topology=(wp_a, wp_b, sp, rank, ownership): this process is one rank (connect the others with
        connect_peers / connect_peers_torch). devices=[dev of rank 0, dev of rank 1, ...] with
        topology=(wp_a, wp_b, sp, ownership): this one object drives every rank (single-process group,
        swf_set_topology_devices) and every call returns complete fields."""
        self.cfg, self.H, self.W, self.precision = cfg, grid_h, grid_w, precision
        self._c = C.c_void_p()
        dev0 = devices[0] if devices is not None else device
        _check(lib().swf_create(C.byref(_Cfg(*astuple(cfg))), grid_h, grid_w, dev0, precision,
                                C.byref(self._c)))
        self.wp_world, self.wp_rank = 1, 0  # ranks sharing this model's windows (WP x SP group)
        if devices is not None:
            wp_a, wp_b, sp, own = topology if topology is not None else (1, len(devices), 1, OWN_CONTIGUOUS)
            ids = (C.c_int * len(devices))(*devices)
            _check(lib().swf_set_topology_devices(self._c, wp_a, wp_b, sp, own, ids))
        elif topology is not None:
            wp_a, wp_b, sp, rank, own = topology
            _check(lib().swf_set_topology(self._c, wp_a, wp_b, sp, rank, own))
            self.wp_world, self.wp_rank = wp_a * wp_b * sp, rank

    def group_size(self) -> int:
        return lib().swf_group_size(self._c)

    def connect_peers(self, all_handles: bytes):
        buf = C.create_string_buffer(all_handles, len(all_handles))
        _check(lib().swf_connect_peers(self._c, buf))

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(320)
        _check(lib().swf_ipc_handles(self._c, buf))
        return buf.raw

    def connect_peers_torch(self, dist, group=None):
        """Exchange IPC handles with torch.distributed (any backend) over the WP group (default: the
        whole world, ranks in topology order) and map every peer."""
        mine = self.ipc_handles()
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, mine, group=group)
        self.connect_peers(b"".join(allh))

    def close(self):
        if self._c:
            lib().swf_destroy(self._c)
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- parameters (model.hpp:140-168 canonical order, col-major)
    def load_params(self, flat: np.ndarray):
        flat = np.ascontiguousarray(flat)
        _check(lib().swf_load_params_flat(self._c, _p(flat), flat.size, _dt(flat)))

    def load_checkpoint(self, base: str):
        """load_params(base, p) of the reference (checkpoint.hpp:84-89): .bin + .manifest."""
        _check(lib().swf_load_checkpoint(self._c, base.encode()))

    def init_params(self, seed: int, mode: int = 0, scale: float = 0.25):
        """init_parameters (mode 0) / init_parameters_random (mode 1) / bench weights (mode 2),
        generated on the device with the reference counter RNG (model.hpp:185-223)."""
        _check(lib().swf_init_params(self._c, seed, mode, scale))

    # ---- forward (swin.hpp:327-368)
    def forward(self, inp: np.ndarray, t: float) -> np.ndarray:
        inp = np.ascontiguousarray(inp)
        out = np.zeros((self.H * self.W, self.cfg.out_channels), inp.dtype)
        _check(lib().swf_forward(self._c, _p(inp), float(t), _p(out), _dt(inp)))
        return out

    def forward_hidden(self, inp: np.ndarray, t: float, n_blocks: int, pixels) -> np.ndarray:
        """Residual stream after the first n_blocks blocks (fp32) at the given pixels: [n_pix][h]."""
        inp = np.ascontiguousarray(inp)
        pix = np.ascontiguousarray(pixels, np.int64)
        out = np.zeros((pix.size, self.cfg.hidden_dim), np.float32)
        _check(lib().swf_forward_hidden(self._c, _p(inp), float(t), int(n_blocks), _p(pix), pix.size, _p(out),
                                        _dt(inp)))
        return out

    def block_window_forward(self, block: int, wy: int, wx: int, t: float, x_in: np.ndarray) -> np.ndarray:
        """block_window_forward (swin.hpp:306-325): one window's residual rows [w*w][h] (canonical
        token order) through block `block` of the loaded model at time t."""
        x_in = np.ascontiguousarray(x_in)
        out = np.zeros_like(x_in)
        _check(lib().swf_block_window_forward(self._c, block, wy, wx, float(t), _p(x_in), _p(out), _dt(x_in)))
        return out

    def forward_device(self, d_in: int, t: float, d_out: int):
        _check(lib().swf_forward_device(self._c, C.c_void_p(d_in), float(t), C.c_void_p(d_out)))

    def sync(self):
        _check(lib().swf_sync(self._c))

    @property
    def stream(self) -> int:
        return lib().swf_stream(self._c) or 0

    def local_tokens(self) -> int:
        n = lib().swf_local_tokens(self._c)
        if n < 0:
            _check(ERR_CUDA)
        return n

    KERNEL_CLASSES = ("encode_gemm", "rms_adaln", "qkv_gemm", "attention", "out_gemm", "gateup_gemm",
                      "down_gemm", "decode_gemm", "other")

    def set_backward_precision(self, precision: int):
        """PREC_BF16: the backward's linear-layer GEMMs on the tensor cores (bf16 operands, fp32
        accumulation); PREC_FP32: the FP32 validation mode (default)."""
        _check(lib().swf_set_backward_precision(self._c, precision))

    def set_graphs(self, enable: bool = True):
        """CUDA-graph replay of the sampler's evaluations (default on)."""
        _check(lib().swf_set_graphs(self._c, int(enable)))

    def profile(self, enable: bool = True):
        _check(lib().swf_profile(self._c, int(enable)))

    def profile_launches(self, max_n: int = 4096) -> list:
        cls = (C.c_int * max_n)()
        ms = (C.c_double * max_n)()
        n = C.c_int(0)
        _check(lib().swf_profile_launches(self._c, cls, ms, max_n, C.byref(n)))
        return [(self.KERNEL_CLASSES[cls[i]], ms[i]) for i in range(n.value)]

    def profile_read(self) -> dict:
        n = len(self.KERNEL_CLASSES)
        ms = (C.c_double * n)()
        cnt = (C.c_longlong * n)()
        _check(lib().swf_profile_read(self._c, ms, cnt, n))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(self.KERNEL_CLASSES)}

    def bench_kernel(self, name: str, block: int = 1, reps: int = 10) -> float:
        ms = C.c_double()
        _check(lib().swf_bench_kernel(self._c, self.KERNEL_CLASSES.index(name), block, reps, C.byref(ms)))
        return ms.value

    def kernel_launches(self) -> int:
        return lib().swf_kernel_launches(self._c)

    # ---- sampler (diffusion.hpp:207-339)
    def solve_pf_ode(self, x_init, x_prev_std, forcings_std, dc: DiffusionConfig, churn_key: int = 0):
        x_init = np.ascontiguousarray(x_init)
        dt = x_init.dtype
        out = np.zeros_like(x_init)
        fe = C.c_int(0)
        f = None if forcings_std is None else np.ascontiguousarray(forcings_std, dt)
        _check(lib().swf_solve_pf_ode(self._c, _p(x_init), _p(np.ascontiguousarray(x_prev_std, dt)), _p(f),
                                      C.byref(_DCfg(*astuple(dc))), churn_key, _p(out), C.byref(fe), _dt(x_init)))
        return out, fe.value

    def _stds(self, stds, dt):
        if stds is None:
            return None, []
        keep = [None if a is None else np.ascontiguousarray(a, dt) for a in stds]
        return _Std(*[None if a is None else a.ctypes.data for a in keep]), keep

    def forecast_step(self, x_prev_phys, forcing_phys, dc: DiffusionConfig, run_seed: int, event: int, stds=None):
        x_prev_phys = np.ascontiguousarray(x_prev_phys)
        dt = x_prev_phys.dtype
        st, keep = self._stds(stds, dt)
        out = np.zeros_like(x_prev_phys)
        f = None if forcing_phys is None else np.ascontiguousarray(forcing_phys, dt)
        _check(lib().swf_forecast_step(self._c, _p(x_prev_phys), _p(f), None if st is None else C.byref(st),
                                       C.byref(_DCfg(*astuple(dc))), run_seed, event, _p(out), _dt(x_prev_phys)))
        return out

    def rollout_ensemble(self, x_init_phys, forcings_phys, n_members, n_steps, dc, run_seed, rollout_id, stds=None):
        x = np.ascontiguousarray(x_init_phys)
        dt = x.dtype
        st, keep = self._stds(stds, dt)
        f = np.ascontiguousarray(np.stack(forcings_phys[:n_steps]), dt)
        out = np.zeros((n_members, n_steps) + x.shape, dt)
        _check(lib().swf_rollout_ensemble(self._c, _p(x), _p(f), n_members, n_steps,
                                          None if st is None else C.byref(st), C.byref(_DCfg(*astuple(dc))),
                                          run_seed, rollout_id, _p(out), _dt(x)))
        return out

    # ---- backward (swin.hpp:419-467), FP32 validation mode
    def backward(self, inp, t: float, d_output, want_input_grad: bool = True):
        """Parameter gradients (canonical flat order, column-major arrays) and input gradient of
        sum(d_output * forward(inp, t))."""
        inp = np.ascontiguousarray(inp)
        dt = inp.dtype
        dout = np.ascontiguousarray(d_output, dt)
        g = np.zeros(param_count(self.cfg), dt)
        din = np.zeros_like(inp) if want_input_grad else None
        _check(lib().swf_backward(self._c, _p(inp), t, _p(dout), _p(g), _p(din), _dt(inp)))
        return g, din

    # ---- training (diffusion.hpp:168-192, simulator.hpp:50-86; FP32 validation mode)
    def _lw(self, w, dt):
        a = np.ascontiguousarray(w.alpha_row, dt)
        k = np.ascontiguousarray(w.kappa, dt)
        if a.shape != (self.H,) or k.shape != (self.cfg.out_channels,):
            raise ConfigError(ERR_CONFIG, "loss weights: alpha_row needs H entries and kappa C_out entries")
        return _LW(_p(a), _p(k)), (a, k)

    def _train_fields(self, x_prev, x0, forcings, dt):
        f = [np.ascontiguousarray(v, dt) for v in (x_prev, x0)]
        fo = None if forcings is None else np.ascontiguousarray(forcings, dt)
        return f[0], f[1], fo

    def diffusion_loss_sample(self, x_prev, x0, forcings, w, dc: DiffusionConfig, t_key: int, z,
                              want_grads: bool = True):
        """(loss, parameter gradients) of diffusion_loss_sample for one standardized sample."""
        dt = np.asarray(x0).dtype if np.asarray(x0).dtype in (np.float32, np.float64) else np.float32
        xp, x0_, fo = self._train_fields(x_prev, x0, forcings, dt)
        zz = np.ascontiguousarray(z, dt)
        lw, keep = self._lw(w, dt)
        loss = C.c_double(0)
        g = np.zeros(param_count(self.cfg), dt) if want_grads else None
        _check(lib().swf_diffusion_loss_sample(self._c, _p(xp), _p(x0_), _p(fo), C.byref(lw),
                                               C.byref(_DCfg(*astuple(dc))), t_key, _p(zz), C.byref(loss), _p(g),
                                               _dt(x0_)))
        return loss.value, g

    def train_reset(self):
        _check(lib().swf_train_reset(self._c))

    def train_accumulate(self, x_prev, x0, forcings, w, dc: DiffusionConfig, run_seed: int, sample_id: int) -> float:
        """One microbatch (noise and t from the seed protocol); gradient added on the device."""
        dt = np.asarray(x0).dtype if np.asarray(x0).dtype in (np.float32, np.float64) else np.float32
        xp, x0_, fo = self._train_fields(x_prev, x0, forcings, dt)
        lw, keep = self._lw(w, dt)
        loss = C.c_double(0)
        _check(lib().swf_train_accumulate(self._c, _p(xp), _p(x0_), _p(fo), C.byref(lw),
                                          C.byref(_DCfg(*astuple(dc))), run_seed, sample_id, C.byref(loss),
                                          _dt(x0_)))
        return loss.value

    def train_grads_device(self):
        """(device pointer, element count) of the FP32 gradient accumulator."""
        ptr, n = C.c_void_p(), C.c_longlong()
        _check(lib().swf_train_grads(self._c, C.byref(ptr), C.byref(n)))
        return int(ptr.value), int(n.value)

    def train_read(self, scale: float = 1.0, dtype=np.float64) -> np.ndarray:
        g = np.zeros(param_count(self.cfg), dtype)
        _check(lib().swf_train_read(self._c, scale, _p(g), _dt(g)))
        return g

    def train_step(self, data, first_sample: int, dp: int, gas: int, w, dc: DiffusionConfig, run_seed: int,
                   group=None):
        """reference_train_step with data-parallel replicas on ranks (see train.py)."""
        from .train import train_step
        return train_step(self, data, first_sample, dp, gas, w, dc, run_seed, group)

    # ---- per-rank input loading from chunked containers (chunked_file.cpp:156-188)
    def prefetch_chunked(self, state_path: str, forcing_path: str | None = None):
        _check(lib().swf_prefetch_chunked(self._c, state_path.encode(), None if forcing_path is None
                                          else forcing_path.encode()))

    def forecast_step_chunked(self, state_path: str, forcing_path: str | None, dc: DiffusionConfig, run_seed: int,
                              event: int, stds=None, dtype=np.float32):
        st, keep = self._stds(stds, np.dtype(dtype))
        out = np.zeros((self.H * self.W, self.cfg.out_channels), dtype)
        _check(lib().swf_forecast_step_chunked(self._c, state_path.encode(),
                                               None if forcing_path is None else forcing_path.encode(),
                                               None if st is None else C.byref(st), C.byref(_DCfg(*astuple(dc))),
                                               run_seed, event, _p(out), 1 if np.dtype(dtype) == np.float64 else 0))
        return out

    def last_chunk_reads(self) -> int:
        return lib().swf_last_chunk_reads(self._c)

    def noise_field(self, run_seed: int, event: int, channels: int, sigma_d: float = 1.0) -> np.ndarray:
        out = np.zeros((self.H * self.W, channels), np.float32)
        _check(lib().swf_noise_field(self._c, run_seed, event, channels, sigma_d, _p(out)))
        return out


def write_chunked(path: str, field: np.ndarray, height: int, width: int, chunk_h: int, chunk_w: int):
    """write_chunked (chunked_file.cpp:44-99): field is [H*W][C] float32 (FieldTensor values)."""
    f = np.ascontiguousarray(field, np.float32)
    _check(lib().swf_chunked_write(path.encode(), _p(f), f.shape[1], height, width, chunk_h, chunk_w))


class ChunkedReader:
    """ChunkedReader (chunked_file.hpp:36-75) over the C-ABI: read_window_slice returns [h*w][C]."""

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(lib().swf_chunked_open(path.encode(), C.byref(h)))
        self._h = h
        v = [C.c_int() for _ in range(5)]
        _check(lib().swf_chunked_info(self._h, *[C.byref(x) for x in v]))
        self.channels, self.height, self.width, self.chunk_h, self.chunk_w = [x.value for x in v]

    def read_window_slice(self, y0: int, x0: int, h: int, w: int) -> np.ndarray:
        out = np.zeros((max(h, 0) * max(w, 0), self.channels), np.float32)
        _check(lib().swf_chunked_read(self._h, y0, x0, h, w, _p(out)))
        return out

    def read_full(self) -> np.ndarray:
        return self.read_window_slice(0, 0, self.height, self.width)

    def chunk_cover(self, y0: int, x0: int, h: int, w: int) -> int:
        n = C.c_longlong()
        _check(lib().swf_chunked_cover(self._h, y0, x0, h, w, C.byref(n)))
        return n.value

    def chunk_reads(self) -> int:
        return lib().swf_chunked_reads(self._h)

    def reset_chunk_reads(self):
        lib().swf_chunked_reset_reads(self._h)

    def close(self):
        if self._h:
            lib().swf_chunked_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def param_arrays(cfg: ModelConfig) -> list[tuple[str, int, int]]:
    """parameter_arrays (model.hpp:140-168): (name, rows, cols) in canonical order."""
    out, i = [], 0
    c = _Cfg(*astuple(cfg))
    buf, r, k = C.create_string_buffer(64), C.c_longlong(), C.c_longlong()
    while lib().swf_param_array(C.byref(c), i, buf, 64, C.byref(r), C.byref(k)) == OK:
        out.append((buf.value.decode(), r.value, k.value))
        i += 1
    return out


def fnv1a64(data, h: int = 0xcbf29ce484222325) -> int:
    """fnv1a64 of a bytes-like object or contiguous numpy array (host)."""
    a = np.ascontiguousarray(np.frombuffer(data, np.uint8) if isinstance(data, (bytes, bytearray)) else data)
    return int(lib().swf_fnv1a64(a.ctypes.data_as(C.c_void_p), a.nbytes, h))


def save_checkpoint(base: str, cfg: ModelConfig, arrays, dtype=None):
    """save_params / save_named_arrays (checkpoint.hpp:29-47, 78-81): `arrays` yields the canonical
    arrays (column-major) one at a time; writes base.manifest + base.bin. Every array is written in
    one element type -- `dtype` (np.float32 / np.float64), default the first array's -- as the
    reference's save_named_arrays<T> does; exactly the canonical number of arrays is required."""
    shapes = param_arrays(cfg)
    it = iter(arrays)
    off, dt = 0, None if dtype is None else np.dtype(dtype)
    if dt is not None and dt not in (np.float32, np.float64):
        raise ConfigError(ERR_CONFIG, "save_checkpoint: dtype must be float32 or float64")
    with open(base + ".bin", "wb") as fb, open(base + ".manifest", "w") as fm:
        for k, (name, r, c) in enumerate(shapes):
            try:
                a = next(it)
            except StopIteration:
                raise ConfigError(ERR_CONFIG, f"save_checkpoint: {k} arrays given, the model has {len(shapes)}") \
                    from None
            a = np.asarray(a)
            if dt is None:
                dt = np.dtype(np.float64) if a.dtype == np.float64 else np.dtype(np.float32)
            a = np.ascontiguousarray(a, dt)
            if a.size != r * c:
                raise ConfigError(ERR_CONFIG, f"save_checkpoint: `{name}` has {a.size} elements, expected {r}x{c}")
            if k == 0:
                fm.write("dtype f64\n" if dt == np.float64 else "dtype f32\n")
            fm.write(f"{name} {r}x{c} {off} {fnv1a64(a)}\n")
            fb.write(a.tobytes())
            off += a.nbytes
        if next(it, None) is not None:
            raise ConfigError(ERR_CONFIG, f"save_checkpoint: more arrays than the model's {len(shapes)}")


def verify_checkpoint(cfg: ModelConfig, base: str):
    """Host-only strict manifest + fnv1a64 check of a reference checkpoint (no GPU)."""
    _check(lib().swf_verify_checkpoint(C.byref(_Cfg(*astuple(cfg))), base.encode()))


def plan_owners(H: int, W: int, w: int, wp_a: int, wp_b: int, ownership: int = OWN_CONTIGUOUS) -> np.ndarray:
    own = np.zeros((H // w) * (W // w), np.int32)
    _check(lib().swf_plan_owners(H, W, w, wp_a, wp_b, ownership, _p(own)))
    return own


def plan_tokens(H: int, W: int, w: int, wp_a: int, wp_b: int, sp: int, rank: int,
                ownership: int = OWN_CONTIGUOUS) -> np.ndarray:
    """Pixel of every local token of `rank` (unshifted layout, device order), no GPU."""
    n = H * W // (wp_a * wp_b * sp)
    pix = np.zeros(n, np.int64)
    _check(lib().swf_plan_tokens(H, W, w, wp_a, wp_b, sp, ownership, rank, _p(pix)))
    return pix


def plan_exchange(H: int, W: int, w: int, wp_a: int, wp_b: int, ownership: int = OWN_CONTIGUOUS,
                  shift_from: int = 0, shift_to: int | None = None) -> np.ndarray:
    world = wp_a * wp_b
    sent = np.zeros((world, world), np.int64)
    _check(lib().swf_plan_exchange(H, W, w, wp_a, wp_b, ownership, shift_from, w // 2 if shift_to is None else shift_to,
                                   _p(sent)))
    return sent


def exported_symbols() -> list[str]:
    """Function names declared in include/swinflow_capi.h."""
    import re
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(swf_[a-z0-9_]+)\s*\(", src)))
from .train import DataSet, LossWeights, TrainStepResult, latitude_weights  # noqa: E402,F401
