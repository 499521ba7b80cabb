"""ctypes binding of the CPU oracle (oracle/swf_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, astuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class OracleError(RuntimeError):
    def __init__(self, rc: int, msg: str):
        super().__init__(msg)
        self.rc = rc


class ConfigError(OracleError):
    pass


class NumericsError(OracleError):
    pass


@dataclass
class ModelConfig:
    """Mirror of swinflow::ModelConfig (model.hpp:21-62)."""
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

    def tdim(self) -> int:
        return self.time_dim if self.time_dim > 0 else self.hidden_dim


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("hidden_dim", "n_heads", "ffn_dim", "n_layers", "blocks_per_layer",
                                        "window_px", "in_channels", "out_channels", "time_dim")]


def _c(cfg: ModelConfig) -> _Cfg:
    return _Cfg(*astuple(cfg))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        L = _lib
        u64 = C.c_uint64
        L.orc_gaussian.restype = C.c_double
        L.orc_gaussian.argtypes = [u64, u64]
        L.orc_uniform01.restype = C.c_double
        L.orc_uniform01.argtypes = [u64, u64]
        L.orc_key_derive.restype = u64
        L.orc_key_derive.argtypes = [u64, u64]
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_gaussian_fill.argtypes = [u64, C.c_int64, C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_param_count_formula.restype = C.c_longlong
        L.orc_pixel_of.restype = C.c_longlong
        L.orc_shift_transfer_total.restype = C.c_longlong
        L.orc_t_of_sigma.restype = C.c_double
        L.orc_t_of_sigma.argtypes = [C.c_double, C.c_double]
        L.orc_init_params_f64.argtypes = [C.c_void_p, u64, C.c_int, C.c_double, C.c_void_p]
        L.orc_init_params_f32.argtypes = [C.c_void_p, u64, C.c_int, C.c_double, C.c_void_p]
        L.orc_forward_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_void_p]
        L.orc_forward_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_int, C.c_void_p]
        L.orc_hidden_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.c_void_p, C.c_void_p]
        L.orc_hidden_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_int, C.c_int,
                                     C.c_void_p, C.c_void_p]
        L.orc_block_window_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_void_p, C.c_void_p]
        L.orc_time_embed_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
        L.orc_backward_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_backward_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_int, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_noise_field_f64.argtypes = [u64, u64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        L.orc_noise_field_f32.argtypes = [u64, u64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        L.orc_solve_gaussian.argtypes = [C.c_double] * 6 + [C.c_int, C.c_double, u64, C.c_void_p, C.c_int64,
                                                            C.c_void_p, C.c_void_p]
        L.orc_solve_affine.argtypes = [C.c_double] * 5 + [C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        fargs = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                 u64, u64, C.c_void_p, C.c_void_p]
        L.orc_forecast_step_f64.argtypes = fargs
        L.orc_solve_net_f64.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int,
                                        C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, u64,
                                        C.c_void_p, C.c_void_p]
        L.orc_forecast_step_f32.argtypes = fargs
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().orc_last_error().decode()
    if rc == 1:
        raise NumericsError(rc, msg)
    if rc == 2:
        raise ConfigError(rc, msg)
    raise OracleError(rc, msg)


# ------------------------------------------------------------------ rng (rng.hpp)
def gaussian(key: int, ctr: int) -> float:
    return lib().orc_gaussian(key, ctr)


def key_derive(key: int, *tags: int) -> int:
    for t in tags:
        key = lib().orc_key_derive(key, t)
    return key


def gaussian_fill(key: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().orc_gaussian_fill(key, n, _p(out))
    return out


def random_field(channels: int, npix: int, key: int) -> np.ndarray:
    """`x.data()[i] = gaussian(key, i)` for a C x N col-major field -> numpy [N][C]."""
    return gaussian_fill(key, channels * npix).reshape(npix, channels)


# ------------------------------------------------------------------ params (model.hpp)
def param_count_formula(cfg: ModelConfig) -> int:
    return lib().orc_param_count_formula(C.byref(_c(cfg)))


def param_shapes(cfg: ModelConfig) -> list[tuple[str, int, int]]:
    c = _c(cfg)
    n = lib().orc_param_arrays(C.byref(c), None, None)
    rows = (C.c_longlong * n)()
    cols = (C.c_longlong * n)()
    lib().orc_param_arrays(C.byref(c), rows, cols)
    out = []
    buf = C.create_string_buffer(128)
    for i in range(n):
        lib().orc_param_name(C.byref(c), i, buf, 128)
        out.append((buf.value.decode(), rows[i], cols[i]))
    return out


def init_params(cfg: ModelConfig, seed: int, random: bool = False, scale: float = 0.25,
                dtype=np.float64) -> np.ndarray:
    """Flat canonical-order parameter vector (init_parameters / init_parameters_random)."""
    n = sum(r * c for _, r, c in param_shapes(cfg))
    out = np.empty(n, dtype)
    fn = lib().orc_init_params_f64 if dtype == np.float64 else lib().orc_init_params_f32
    fn(C.byref(_c(cfg)), seed, int(random), scale, _p(out))
    return out


def split_params(cfg: ModelConfig, flat: np.ndarray) -> list[np.ndarray]:
    """Views of each canonical array in Eigen col-major storage order (flat)."""
    out, off = [], 0
    for _, r, c in param_shapes(cfg):
        out.append(flat[off:off + r * c])
        off += r * c
    return out


# ------------------------------------------------------------------ forward (swin.hpp:327-368)
def forward(cfg: ModelConfig, params: np.ndarray, inp: np.ndarray, t: float, H: int, W: int) -> np.ndarray:
    inp = np.ascontiguousarray(inp, params.dtype)
    out = np.empty((H * W, cfg.out_channels), params.dtype)
    c = _c(cfg)
    if params.dtype == np.float64:
        _check(lib().orc_forward_f64(C.byref(c), _p(params), _p(inp), t, H, W, _p(out)))
    else:
        _check(lib().orc_forward_f32(C.byref(c), _p(params), _p(inp), t, H, W, _p(out)))
    return out


def backward(cfg: ModelConfig, params: np.ndarray, inp: np.ndarray, t: float, H: int, W: int,
             dout: np.ndarray):
    """backward (swin.hpp:419-467): (parameter gradients in canonical flat order, input gradient)."""
    inp = np.ascontiguousarray(inp, params.dtype)
    dout = np.ascontiguousarray(dout, params.dtype)
    g = np.empty_like(params)
    din = np.empty((H * W, cfg.in_channels), params.dtype)
    c = _c(cfg)
    fn = lib().orc_backward_f64 if params.dtype == np.float64 else lib().orc_backward_f32
    _check(fn(C.byref(c), _p(params), _p(inp), t, H, W, _p(dout), _p(g), _p(din)))
    return g, din


def hidden(cfg: ModelConfig, params: np.ndarray, inp: np.ndarray, t: float, H: int, W: int,
           nblocks: int) -> np.ndarray:
    """Residual stream (pixel order [N][h]) after the first `nblocks` blocks."""
    inp = np.ascontiguousarray(inp, params.dtype)
    hid = np.empty((H * W, cfg.hidden_dim), params.dtype)
    out = np.empty((H * W, cfg.out_channels), params.dtype)
    c = _c(cfg)
    fn = lib().orc_hidden_f64 if params.dtype == np.float64 else lib().orc_hidden_f32
    _check(fn(C.byref(c), _p(params), _p(inp), t, H, W, nblocks, _p(hid), _p(out)))
    return hid


def block_window(cfg: ModelConfig, params: np.ndarray, t: float, H: int, W: int, blk: int, wy: int, wx: int,
                 xin: np.ndarray) -> np.ndarray:
    xin = np.ascontiguousarray(xin, np.float32)
    xo = np.empty_like(xin)
    _check(lib().orc_block_window_f32(C.byref(_c(cfg)), _p(params), t, H, W, blk, wy, wx, _p(xin), _p(xo)))
    return xo


def time_embed(cfg: ModelConfig, params: np.ndarray, t: float):
    emb = np.empty(cfg.tdim(), np.float64)
    six = np.empty((cfg.n_blocks(), 6 * cfg.hidden_dim), np.float64)
    lib().orc_time_embed_f64(C.byref(_c(cfg)), _p(params), t, _p(emb), _p(six))
    return emb, six


# ------------------------------------------------------------------ windows (window.hpp)
def pixel_of(H, W, w, shift, wy, wx, r, c) -> int:
    return lib().orc_pixel_of(H, W, w, shift, wy, wx, r, c)


def window_perm(H, W, w, shift) -> np.ndarray:
    perm = np.empty(H * W, np.int64)
    lib().orc_window_perm(H, W, w, shift, _p(perm))
    return perm


def window_gather(H, W, w, shift, tokens: np.ndarray) -> np.ndarray:
    tokens = np.ascontiguousarray(tokens, np.float64)
    out = np.empty_like(tokens)
    lib().orc_window_gather_f64(H, W, w, shift, tokens.shape[1], _p(tokens), _p(out))
    return out


def window_scatter(H, W, w, shift, win_order: np.ndarray) -> np.ndarray:
    win_order = np.ascontiguousarray(win_order, np.float64)
    out = np.zeros_like(win_order)
    lib().orc_window_scatter_f64(H, W, w, shift, win_order.shape[1], _p(win_order), _p(out))
    return out


def seam_mask(H, W, w, shift, wy):
    s = w * w
    m = np.empty((s, s), np.float64)
    return m if lib().orc_seam_mask_f64(H, W, w, shift, wy, _p(m)) else None


def band_of_row(H, W, w, shift, r, sp) -> int:
    return lib().orc_band_of_row(H, W, w, shift, r, sp)


def rope_angles(d, row, col) -> np.ndarray:
    a = np.empty(d // 2, np.float64)
    lib().orc_rope_angles_f64(d, row, col, _p(a))
    return a


def posenc(H, W, C_, dtype=np.float64) -> np.ndarray:
    out = np.empty((H * W, C_), dtype)
    (lib().orc_posenc_f64 if dtype == np.float64 else lib().orc_posenc_f32)(H, W, C_, _p(out))
    return out


def noise_field(run_seed, event, C_, H, W, w, sigma_d=1.0, dtype=np.float64) -> np.ndarray:
    out = np.empty((H * W, C_), dtype)
    fn = lib().orc_noise_field_f64 if dtype == np.float64 else lib().orc_noise_field_f32
    fn(run_seed, event, C_, H, W, w, sigma_d, _p(out))
    return out


# ------------------------------------------------------------------ solver (diffusion.hpp)
def t_of_sigma(sigma, sigma_d=1.0):
    return lib().orc_t_of_sigma(sigma, sigma_d)


def solve_gaussian(x_init, mu=0.0, s0=1.0, sd=1.0, sigma_d=1.0, sigma_min=0.2, sigma_max=500.0, steps=10,
                   churn=0.0, churn_key=0):
    x = np.ascontiguousarray(x_init, np.float64).ravel()
    out = np.empty_like(x)
    fe = C.c_int(0)
    _check(lib().orc_solve_gaussian(mu, s0, sd, sigma_d, sigma_min, sigma_max, steps, churn, churn_key, _p(x),
                                    x.size, _p(out), C.byref(fe)))
    return out, fe.value


def solve_affine(x_init, alpha, beta, steps=10):
    x = np.ascontiguousarray(x_init, np.float64).ravel()
    out = np.empty_like(x)
    _check(lib().orc_solve_affine(alpha, beta, 1.0, 0.2, 500.0, steps, _p(x), x.size, _p(out)))
    return out


def forecast_step(cfg: ModelConfig, params, H, W, x_prev, forc, run_seed, event, st=None, rs=None, fo=None,
                  sigma_d=1.0, sigma_min=0.2, sigma_max=500.0, steps=10, churn=0.0):
    dt = params.dtype
    Cp = cfg.out_channels
    Cf = cfg.in_channels - 2 * Cp
    ident = lambda n: (np.zeros(n, dt), np.ones(n, dt))
    st = st or ident(Cp)
    rs = rs or ident(Cp)
    fo = fo or ident(max(Cf, 1))
    x_prev = np.ascontiguousarray(x_prev, dt)
    forc = np.ascontiguousarray(forc, dt)
    out = np.empty_like(x_prev)
    fe = C.c_int(0)
    fn = lib().orc_forecast_step_f64 if dt == np.float64 else lib().orc_forecast_step_f32
    args = [np.ascontiguousarray(a, dt) for a in (*st, *rs, *fo)]
    _check(fn(C.byref(_c(cfg)), _p(params), sigma_d, sigma_min, sigma_max, steps, churn, H, W, _p(x_prev),
              _p(forc), *[_p(a) for a in args], run_seed, event, _p(out), C.byref(fe)))
    return out, fe.value


def rollout_ensemble(cfg: ModelConfig, params, H, W, x_init, forcings, n_members, n_steps, run_seed, rollout_id,
                     st=None, rs=None, fo=None, **dc):
    """rollout_ensemble (diffusion.hpp:323-339): members x AR steps, out[m][k] = the state after step k of
    member m; step k of member m uses event key_derive(rollout_id, m, k) and forcings[k], and its output
    is the next step's x_prev. Members are independent (their noise streams differ only by the event)."""
    if len(forcings) < n_steps:
        raise ConfigError(2, "rollout: not enough forcing steps")
    x_init = np.ascontiguousarray(x_init, params.dtype)
    out = np.empty((n_members, n_steps) + x_init.shape, params.dtype)
    for m in range(n_members):
        x = x_init
        for k in range(n_steps):
            x, _ = forecast_step(cfg, params, H, W, x, forcings[k], run_seed, key_derive(rollout_id, m, k), st, rs,
                                 fo, **dc)
            out[m, k] = x
    return out


def solve_net(cfg: ModelConfig, params, H, W, x_init, x_prev_std, forc_std, sigma_d=1.0, sigma_min=0.2,
              sigma_max=500.0, steps=10, churn=0.0, churn_key=0):
    """solve_pf_ode with the forecast_step net lambda on given standardized conditioning (f64)."""
    a = [np.ascontiguousarray(v, np.float64) for v in (x_init, x_prev_std, forc_std)]
    out = np.empty_like(a[0])
    fe = C.c_int(0)
    _check(lib().orc_solve_net_f64(C.byref(_c(cfg)), _p(params), sigma_d, sigma_min, sigma_max, steps, churn, H, W,
                                   _p(a[0]), _p(a[1]), _p(a[2]), churn_key, _p(out), C.byref(fe)))
    return out, fe.value


# ------------------------------------------------------------------ training loss (diffusion.hpp:111-192)
def latitude_weights(H: int) -> np.ndarray:
    """grid.hpp:17-82: cos(latitude of each row centre), scaled to unit mean."""
    d = 180.0 / H
    w = np.cos((90.0 - d * (np.arange(H) + 0.5)) * np.pi / 180.0)
    return w * (H / w.sum())


def noise_draw_from_u(u: float, sigma_d=1.0, sigma_min=0.2, sigma_max=500.0) -> float:
    """noise_draw_from_u (diffusion.hpp:76-82): tau log-uniform in [log sigma_min, log sigma_max]."""
    tau = (1.0 - u) * np.log(sigma_min) + u * np.log(sigma_max)
    return float(np.arctan(np.exp(tau) / sigma_d))


def noise_draw_t(t_key: int, sigma_d=1.0, sigma_min=0.2, sigma_max=500.0) -> float:
    """sample_noise_draw (diffusion.hpp:84-86): u = uniform01(t_key, 0)."""
    return noise_draw_from_u(lib().orc_uniform01(t_key, 0), sigma_d, sigma_min, sigma_max)


def weighted_sq_loss(err, alpha_row, kappa, W):
    """weighted_sq_loss (diffusion.hpp:111-123) and its gradient (:125-133); err is [N][C]."""
    N = err.shape[0]
    alpha = np.repeat(np.asarray(alpha_row, err.dtype), W)[:, None]
    kap = np.asarray(kappa, err.dtype)[None, :]
    if kap.shape[1] != err.shape[1]:
        raise ValueError("loss: kappa size does not match channels")
    loss = float((alpha * kap * err * err).sum() / N)
    return loss, (2.0 * alpha / N) * kap * err


def loss_sample(cfg: ModelConfig, params, H, W, x_prev, x0, forc, alpha_row, kappa, t_key, z, sigma_d=1.0,
                sigma_min=0.2, sigma_max=500.0):
    """diffusion_loss_sample (diffusion.hpp:168-192) over the oracle forward / backward: fields are
    [N][C] numpy arrays; returns (loss, parameter gradients in canonical order)."""
    dt = params.dtype
    t = noise_draw_t(t_key, sigma_d, sigma_min, sigma_max)
    t = dt.type(t)
    c, s = (1.0, 0.0) if t == 0 else (np.cos(t), np.sin(t))
    x0 = np.asarray(x0, dt)
    z = np.asarray(z, dt)
    xt = c * x0 + s * z
    v = c * z - s * x0
    inp = np.concatenate([xt / dt.type(sigma_d), np.asarray(x_prev, dt), np.asarray(forc, dt)], axis=1)
    inp = inp + posenc(H, W, cfg.in_channels, dt)
    f = forward(cfg, params, inp, float(t), H, W)
    err = dt.type(sigma_d) * f - v
    loss, gerr = weighted_sq_loss(err, alpha_row, kappa, W)
    dout = dt.type(sigma_d) * gerr
    g, _ = backward(cfg, params, inp, float(t), H, W, dout)
    return loss, g


def fnv1a64(data: bytes, h: int = 0xcbf29ce484222325) -> int:
    """src/chunked_file.cpp:33-41"""
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def save_named_arrays(base: str, cfg: ModelConfig, flat: np.ndarray):
    """save_params / save_named_arrays (checkpoint.hpp:29-47, 78-81): `dtype f32|f64` line, then
    `name RxC offset fnv1a64` per canonical array; the .bin holds the arrays back to back."""
    dt = "f64" if flat.dtype == np.float64 else "f32"
    off = 0
    with open(base + ".bin", "wb") as fb, open(base + ".manifest", "w") as fm:
        fm.write(f"dtype {dt}\n")
        for (name, r, c), a in zip(param_shapes(cfg), split_params(cfg, flat)):
            raw = np.ascontiguousarray(a).tobytes()
            fm.write(f"{name} {r}x{c} {off} {fnv1a64(raw)}\n")
            fb.write(raw)
            off += len(raw)


# ---- chunked field container (chunked_file.hpp:5-13, src/chunked_file.cpp:44-188), numpy restatement
CHUNK_MAGIC = b"SWCHNK01"


def write_chunked_np(path: str, field: np.ndarray, H: int, W: int, ch: int, cw: int):
    """write_chunked (chunked_file.cpp:44-99): field [H*W][C] float32; header of u64s, offset and
    fnv1a64 tables, then each clipped chunk as (c, y, x) row-major."""
    C_ = field.shape[1]
    f = field.reshape(H, W, C_).astype(np.float32)
    ny, nx = -(-H // ch), -(-W // cw)
    chunks = []
    for cy in range(ny):
        for cx in range(nx):
            tile = f[cy * ch:min(H, cy * ch + ch), cx * cw:min(W, cx * cw + cw), :]
            chunks.append(np.ascontiguousarray(tile.transpose(2, 0, 1)).tobytes())
    pos = 8 + 6 * 8 + 2 * 8 * len(chunks)
    offs = []
    for b in chunks:
        offs.append(pos)
        pos += len(b)
    with open(path, "wb") as fo:
        fo.write(CHUNK_MAGIC)
        fo.write(np.array([1, C_, H, W, ch, cw], "<u8").tobytes())
        fo.write(np.array(offs, "<u8").tobytes())
        fo.write(np.array([fnv1a64(b) for b in chunks], "<u8").tobytes())
        for b in chunks:
            fo.write(b)


def read_chunked_np(path: str, y0: int, x0: int, h: int, w: int):
    """ChunkedReader::read_window_slice (chunked_file.cpp:156-188) -> ([h*w][C] float32, chunks read).
    Raises IndexError for a rect outside the grid (std::out_of_range) and ValueError on a checksum
    mismatch (IntegrityError)."""
    raw = open(path, "rb").read()
    if raw[:8] != CHUNK_MAGIC:
        raise ValueError("bad container magic")
    ver, C_, H, W, ch, cw = (int(v) for v in np.frombuffer(raw[8:56], "<u8"))
    if ver != 1:
        raise ValueError("unsupported container version")
    ny, nx = -(-H // ch), -(-W // cw)
    n = ny * nx
    offs = np.frombuffer(raw[56:56 + 8 * n], "<u8")
    sums = np.frombuffer(raw[56 + 8 * n:56 + 16 * n], "<u8")
    if h <= 0 or w <= 0 or y0 < 0 or x0 < 0 or y0 + h > H or x0 + w > W:
        raise IndexError("window rect outside grid")
    out = np.zeros((h, w, C_), np.float32)
    reads = 0
    for cy in range(y0 // ch, (y0 + h - 1) // ch + 1):
        for cx in range(x0 // cw, (x0 + w - 1) // cw + 1):
            idx = cy * nx + cx
            hh, ww = min(ch, H - cy * ch), min(cw, W - cx * cw)
            b = raw[int(offs[idx]):int(offs[idx]) + 4 * C_ * hh * ww]
            if fnv1a64(b) != int(sums[idx]):
                raise ValueError(f"checksum mismatch in chunk {idx}")
            reads += 1
            tile = np.frombuffer(b, np.float32).reshape(C_, hh, ww).transpose(1, 2, 0)
            ys, ye = max(y0, cy * ch), min(y0 + h, cy * ch + hh)
            xs, xe = max(x0, cx * cw), min(x0 + w, cx * cw + ww)
            out[ys - y0:ye - y0, xs - x0:xe - x0] = tile[ys - cy * ch:ye - cy * ch, xs - cx * cw:xe - cx * cw]
    return out.reshape(h * w, C_), reads


def window_owner(wy, wx, a, b):
    oa, ob = C.c_int(), C.c_int()
    lib().orc_window_owner(wy, wx, a, b, C.byref(oa), C.byref(ob))
    return oa.value, ob.value


def shift_transfer_total(H, W, w, s_from, s_to, a, b, sp=1):
    per = (C.c_longlong * (a * b))()
    tot = lib().orc_shift_transfer_total(H, W, w, s_from, s_to, a, b, sp, per)
    return tot, list(per)


def num_threads() -> int:
    return lib().orc_num_threads()


def use_all_cores() -> int:
    """OpenMP threads = the host cores this process may run on (torchrun sets OMP_NUM_THREADS=1)."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    lib().orc_set_num_threads(n)
    return num_threads()
