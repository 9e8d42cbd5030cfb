"""PILC CPU oracle -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference `pixelcodec` pipeline
(/root/reference/pkg/src/pixelcodec), with the bit-level coder lanes and the
predictor in plain C (oracle/pilc_oracle.c, loaded via ctypes). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / `--impl reference` leg
import this module, and only as the checker or the timed CPU baseline. The
product package never imports it.

Parity of this restatement with the reference is pinned by
tests/test_oracle.py against fixtures the reference itself produced
(tests/golden/make_golden.py): table digests, lane bytes, residuals,
whole containers, encoder latents / indices / (mu, s).

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import subprocess
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

# --------------------------------------------------------------------------
# C helpers


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "pilc_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.oracle_encode_lane.restype = I64
        L.oracle_encode_lane.argtypes = [P, P, I64, I64, P, P, I64, ctypes.c_int, P, P]
        L.oracle_decode_lane.restype = I64
        L.oracle_decode_lane.argtypes = [I64, P, I64, P, I64, I64, P, P, P, ctypes.c_int, P, P]
        L.oracle_twar_forward.restype = None
        L.oracle_twar_forward.argtypes = [P, I64, ctypes.c_int, ctypes.c_int, P, P, P]
        L.oracle_twar_decode.restype = None
        L.oracle_twar_decode.argtypes = [P, P, I64, ctypes.c_int, ctypes.c_int, P, P, P]
        L.oracle_encode_batch.restype = None
        L.oracle_encode_batch.argtypes = [P, P, I64, I64, I64, P, P, I64, ctypes.c_int, P, I64, P, P]
        C = ctypes.c_int
        L.oracle_conv_fma.restype = ctypes.c_int
        L.oracle_conv_fma.argtypes = [P, C, C, C, P, P, C, C, C, P]
        L.oracle_expf_np_array.restype = None
        L.oracle_expf_np_array.argtypes = [P, P, I64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(Exception):
    """Raised with the reference's exception class name as .kind."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# pmf.py:65-116 quantize_pmf


def quantize_pmf(masses, M: int) -> np.ndarray:
    m = np.asarray(masses, dtype=np.float64)
    X = m.size
    ideal = m / float(m.sum()) * float(1 << M)
    P = np.floor(ideal).astype(np.int64)
    frac = ideal - P
    short = (1 << M) - int(P.sum())
    # largest remainder first, ties to the smaller index
    order = sorted(range(X), key=lambda i: (-frac[i], i))
    for i in order[:short]:
        P[i] += 1
    for x in range(X):
        if P[x] == 0:
            donor = int(np.argmax(P))
            P[donor] -= 1
            P[x] = 1
    cap = (1 << (M - 1)) - 1
    if (P > cap).any():
        excess = int((P[P > cap] - cap).sum())
        P[P > cap] = cap
        recv = [i for i in range(X) if P[i] < cap]
        if recv:
            w = P[recv].astype(np.float64)
            share = excess * w / w.sum()
            add = np.floor(share).astype(np.int64)
            left = excess - int(add.sum())
            rk = sorted(range(len(recv)), key=lambda j: (-(share[j] - add[j]), recv[j]))
            for j in rk[:left]:
                add[j] += 1
            for j, i in enumerate(recv):
                P[i] += add[j]
    return P


# --------------------------------------------------------------------------
# logistic.py:93-99 default_grid; :25-33 sigmoid; :120-144 masses


def default_grid(D: int = 8) -> np.ndarray:
    if D == 1:
        return np.array([0.5 * 2.0 ** 3.5])
    return 0.5 * 2.0 ** (7.0 * np.arange(D) / (D - 1))


def grid_bytes(g: np.ndarray) -> bytes:
    return struct.pack("<H", g.size) + np.asarray(g, "<f8").tobytes()


def _sig(z):
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    e = np.exp(z[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def logistic_masses(mu: float, s: float) -> np.ndarray:
    v = np.arange(256, dtype=np.float64)
    hi = _sig((v + 0.5 - mu) / s)
    lo = _sig((v - 0.5 - mu) / s)
    m = hi - lo
    m[0] = hi[0]
    m[-1] = 1.0 - lo[-1]
    return m


def residual_pmfs(grid: np.ndarray, M: int) -> np.ndarray:
    return np.stack([quantize_pmf(logistic_masses(128.0, s), M) for s in grid])


def scales_to_d(s, grid: np.ndarray) -> np.ndarray:
    """logistic.py:109-114: log2-space argmin, ties to the smaller index."""
    s = np.asarray(s, dtype=np.float64)
    return np.argmin(np.abs(np.log2(s)[..., None] - np.log2(grid)), axis=-1).astype(np.uint16)


def round_half_away(x):
    """logistic.py:36-40."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5)).astype(np.int64)


# --------------------------------------------------------------------------
# tables.py:71-142 build_tables


def build_tables(P: np.ndarray, M: int):
    """P: (D, X) integer masses. Returns (delta, phi, symbol, pop, next)."""
    P = np.asarray(P, dtype=np.int64)
    D, X = P.shape
    C = np.zeros_like(P)
    C[:, 1:] = np.cumsum(P[:, :-1], axis=1)
    # k: P << k lands in [2^M, 2^(M+1))
    k = np.zeros_like(P)
    for d in range(D):
        for x in range(X):
            kk = 0
            while (P[d, x] << kk) < (1 << M):
                kk += 1
            k[d, x] = kk
    delta = ((k << M) - (P << k)).astype(np.uint16)
    phi = ((1 << M) - P + C).astype(np.uint16)
    T = 1 << M
    symbol = np.zeros((D, T), np.uint8)
    pop = np.zeros((D, T), np.uint8)
    nxt = np.zeros((D, T), np.uint16)
    t = np.arange(T, dtype=np.int64)
    for d in range(D):
        x = np.searchsorted(C[d], t, side="right") - 1
        mid = t - C[d, x] + P[d, x]
        b = np.zeros_like(mid)
        while (mid << b < T).any():
            b = np.where(mid << b < T, b + 1, b)
        symbol[d], pop[d], nxt[d] = x, b, mid << b
    return delta, phi, symbol, pop, nxt


# --------------------------------------------------------------------------
# bits.py:66-87 wire form; tables.py:202-274 lane framing over the C lanes


def encode_lanes(syms: np.ndarray, ds: np.ndarray, L: int, delta, phi, M: int):
    """-> (list of lane wire blobs, list of final states)."""
    syms = np.ascontiguousarray(syms, np.uint8)
    ds = np.ascontiguousarray(ds, np.uint16)
    delta = np.ascontiguousarray(delta, np.uint16)
    phi = np.ascontiguousarray(phi, np.uint16)
    n = syms.size
    blobs, states = [], []
    for lane in range(L):
        cnt = len(range(lane, n, L))
        buf = np.zeros((cnt * (M + 1) + 7) // 8 + 8, np.uint8)
        nb = np.zeros(1, np.int64)
        st = lib().oracle_encode_lane(
            _p(syms[lane:]) if cnt else _p(buf), _p(ds[lane:]) if cnt else _p(buf),
            cnt, L, _p(delta), _p(phi), delta.shape[1], M, _p(buf), _p(nb))
        nbits = int(nb[0])
        payload = bytearray(buf[: (nbits + 7) >> 3].tobytes())
        blobs.append(struct.pack("<Q", nbits) + bytes(payload))
        states.append(int(st))
    return blobs, states


def decode_lanes(blobs, states, count: int, ds: np.ndarray, symbol, pop, nxt, M: int):
    ds = np.ascontiguousarray(ds, np.uint16)
    symbol, pop, nxt = (np.ascontiguousarray(a) for a in (symbol, pop, nxt))
    L = len(blobs)
    out = np.zeros(count, np.uint8)
    s0 = 1 << M
    for lane in range(L):
        cnt = len(range(lane, count, L))
        nbits = struct.unpack_from("<Q", blobs[lane], 0)[0]
        payload = np.frombuffer(blobs[lane][8:], np.uint8).copy()
        if payload.size == 0:
            payload = np.zeros(1, np.uint8)
        st = states[lane]
        if not s0 <= st < 2 * s0:
            raise OracleError("CorruptStreamError", f"lane {lane} initial state out of range")
        lane_out = np.zeros(max(cnt, 1), np.uint8)
        rem = np.zeros(1, np.int64)
        dsl = np.ascontiguousarray(ds[lane::L]) if cnt else np.zeros(1, np.uint16)
        end = lib().oracle_decode_lane(st, _p(payload), nbits, _p(dsl), cnt, 1, _p(symbol),
                                       _p(pop), _p(nxt), M, _p(lane_out), _p(rem))
        if end < 0:
            raise OracleError("CorruptStreamError", f"lane {lane} bit stream underflow")
        if end != s0 or rem[0] != 0:
            raise OracleError("CorruptStreamError", f"lane {lane} did not return to the initial coder state")
        out[lane::L] = lane_out[:cnt]
    return out


# --------------------------------------------------------------------------
# predictor.py:45-92 params; forward/inverse via the C restatement


DEFAULT_W = np.array([[-1, 1, 1], [1, -1, 1], [1, -1, 1]], np.float32)
DEFAULT_B = np.zeros(3, np.float32)


def params_bytes(w, b) -> bytes:
    out = b""
    for c in range(3):
        out += struct.pack("<3f", *np.asarray(w, np.float32)[c]) + struct.pack("<f", np.float32(b[c]))
    return out


def params_hash8(w, b) -> bytes:
    return hashlib.sha256(params_bytes(w, b)).digest()[:8]


def twar_forward(img: np.ndarray, w=DEFAULT_W, b=DEFAULT_B) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8)
    x = img if img.ndim == 4 else img[None]
    out = np.empty_like(x)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    lib().oracle_twar_forward(_p(x), x.shape[0], x.shape[1], x.shape[2], _p(w), _p(b), _p(out))
    return out if img.ndim == 4 else out[0]


def twar_decode(res: np.ndarray, w=DEFAULT_W, b=DEFAULT_B, shift=None) -> np.ndarray:
    res = np.ascontiguousarray(res, np.uint8)
    x = res if res.ndim == 4 else res[None]
    out = np.empty_like(x)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    sp = None
    if shift is not None:
        sh = np.ascontiguousarray(np.asarray(shift) & 0xFF, np.uint8)
        sh = sh if sh.ndim == 4 else sh[None]
        sp = _p(sh)
    lib().oracle_twar_decode(_p(x), sp, x.shape[0], x.shape[1], x.shape[2], _p(w), _p(b), _p(out))
    return out if res.ndim == 4 else out[0]


# --------------------------------------------------------------------------
# weights.py:46-69 tensor order, :106-160 PILW, :175-193 random_weights


def tensor_shapes(K, Dc, C, B):
    s = {}

    def conv(n, co, ci, k):
        s[n + ".w"] = (co, ci, k, k)
        s[n + ".b"] = (co,)

    conv("enc.stem", C, 3, 3)
    conv("enc.down", C, C, 3)
    for i in range(B):
        conv(f"enc.block{i}.conv1", C, C, 3)
        conv(f"enc.block{i}.conv2", C, C, 3)
    conv("enc.proj", Dc, C, 1)
    s["codebook"] = (K, Dc)
    conv("dec.proj", C, Dc, 1)
    for i in range(B):
        conv(f"dec.block{i}.conv1", C, C, 3)
        conv(f"dec.block{i}.conv2", C, C, 3)
    conv("dec.up", 4 * C, C, 3)
    conv("dec.mu", 3, C, 3)
    conv("dec.s", 3, C, 3)
    return s


class Model:
    def __init__(self, cfg, tensors, hist=None, w=DEFAULT_W, b=DEFAULT_B):
        self.K, self.Dc, self.C, self.B = cfg
        self.t = tensors
        self.hist = np.zeros(self.K, np.uint64) if hist is None else np.asarray(hist, np.uint64)
        self.w, self.b = np.asarray(w, np.float32), np.asarray(b, np.float32)
        self._bytes = None

    def to_bytes(self) -> bytes:
        if self._bytes is None:
            out = bytearray(b"PILW" + struct.pack("<B4I", 1, self.K, self.Dc, self.C, self.B))
            names = list(tensor_shapes(self.K, self.Dc, self.C, self.B)) if self.t else []
            out += struct.pack("<I", len(names))
            for nm in names:
                a = np.asarray(self.t[nm], np.float32)
                out += struct.pack("<I", len(nm)) + nm.encode() + struct.pack("<I", a.ndim)
                out += struct.pack(f"<{a.ndim}I", *a.shape) + a.astype("<f4").tobytes()
            out += self.hist.astype("<u8").tobytes() + params_bytes(self.w, self.b)
            out += hashlib.sha256(bytes(out)).digest()[:8]
            self._bytes = bytes(out)
        return self._bytes

    def hash8(self) -> bytes:
        return self.to_bytes()[-8:]

    @classmethod
    def from_bytes(cls, data: bytes) -> "Model":
        K, Dc, C, B = struct.unpack_from("<4I", data, 5)
        (cnt,) = struct.unpack_from("<I", data, 21)
        off, t = 25, {}
        for _ in range(cnt):
            (nl,) = struct.unpack_from("<I", data, off)
            nm = data[off + 4: off + 4 + nl].decode()
            off += 4 + nl
            (r,) = struct.unpack_from("<I", data, off)
            dims = struct.unpack_from(f"<{r}I", data, off + 4)
            off += 4 + 4 * r
            n = int(np.prod(dims))
            t[nm] = np.frombuffer(data, "<f4", n, off).reshape(dims).astype(np.float32)
            off += 4 * n
        hist = np.frombuffer(data, "<u8", K, off).copy()
        off += 8 * K
        vals = struct.unpack_from("<12f", data, off)
        w = np.array([vals[0:3], vals[4:7], vals[8:11]], np.float32)
        b = np.array([vals[3], vals[7], vals[11]], np.float32)
        return cls((K, Dc, C, B), t, hist, w, b)


def random_model(K=256, Dc=32, C=32, B=4, seed=0, scale=1.0) -> Model:
    rng = np.random.default_rng(seed)
    t = {}
    for nm, shp in tensor_shapes(K, Dc, C, B).items():
        if nm.endswith(".b"):
            t[nm] = np.zeros(shp, np.float32)
        elif nm == "codebook":
            t[nm] = rng.normal(0, 1, shp).astype(np.float32)
        else:
            t[nm] = rng.normal(0, scale * np.sqrt(2.0 / int(np.prod(shp[1:]))), shp).astype(np.float32)
    return Model((K, Dc, C, B), t)


# --------------------------------------------------------------------------
# nn.py:15-67 and vqvae.py:33-119 (same numpy op sequence as the reference)


def conv2d(x, w, b, stride=1):
    ci, H, W = x.shape
    co, _, kh, kw = w.shape
    ph, pw = kh // 2, kw // 2
    if ph or pw:
        x = np.pad(x, ((0, 0), (ph, ph), (pw, pw)), mode="edge")
    Ho = (H + 2 * ph - kh) // stride + 1
    Wo = (W + 2 * pw - kw) // stride + 1
    out = np.zeros((co, Ho, Wo), np.float32)
    for i in range(kh):
        for j in range(kw):
            tap = x[:, i: i + (Ho - 1) * stride + 1: stride, j: j + (Wo - 1) * stride + 1: stride]
            out += np.tensordot(w[:, :, i, j], tap, axes=(1, 0))
    return out + b[:, None, None].astype(np.float32)


def relu(x):
    return np.maximum(x, np.float32(0))


def sigmoid32(x):
    x = np.asarray(x, np.float32)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def pixel_shuffle(x, r=2):
    crr, h, w = x.shape
    c = crr // (r * r)
    return x.reshape(c, r, r, h, w).transpose(0, 3, 1, 4, 2).reshape(c, h * r, w * r)


def resblock(x, w1, b1, w2, b2):
    return relu(x + conv2d(relu(conv2d(x, w1, b1)), w2, b2))


def encoder_latents(img: np.ndarray, m: Model) -> np.ndarray:
    """vqvae.py:51-65 -> z as (gh, gw, Dc) float32."""
    t = m.t
    ph, pw = img.shape[0] & 1, img.shape[1] & 1
    if ph or pw:
        img = np.pad(img, ((0, ph), (0, pw), (0, 0)), mode="edge")
    x = np.ascontiguousarray((img.astype(np.float32) / np.float32(127.5) - np.float32(1.0)).transpose(2, 0, 1))
    h = relu(conv2d(x, t["enc.stem.w"], t["enc.stem.b"]))
    h = relu(conv2d(h, t["enc.down.w"], t["enc.down.b"], 2))
    for i in range(m.B):
        h = resblock(h, t[f"enc.block{i}.conv1.w"], t[f"enc.block{i}.conv1.b"],
                     t[f"enc.block{i}.conv2.w"], t[f"enc.block{i}.conv2.b"])
    z = conv2d(h, t["enc.proj.w"], t["enc.proj.b"])
    return np.ascontiguousarray(z.transpose(1, 2, 0))


def argmin_codebook(z: np.ndarray, codebook: np.ndarray) -> np.ndarray:
    """vqvae.py:66-76: f64 squared distance accumulated per component in
    order, first minimum wins. z: (..., Dc)."""
    shp = z.shape[:-1]
    zf = z.reshape(-1, z.shape[-1]).astype(np.float64)
    cb = codebook.astype(np.float64)
    dist = np.zeros((zf.shape[0], cb.shape[0]))
    for c in range(zf.shape[1]):
        diff = zf[:, c, None] - cb[None, :, c]
        dist += diff * diff
    return np.argmin(dist, axis=1).reshape(shp).astype(np.uint8)


def encode_indices(img, m: Model):
    return argmin_codebook(encoder_latents(img, m), m.t["codebook"])


LOG_S_MIN = np.float32(np.log(0.5))
LOG_S_MAX = np.float32(np.log(64.0))


def decode_params(idx: np.ndarray, m: Model, H: int, W: int):
    """vqvae.py:79-113 -> (mu, s) float32 (H, W, 3)."""
    t = m.t
    h = np.ascontiguousarray(t["codebook"][idx.astype(np.int64)].transpose(2, 0, 1))
    h = relu(conv2d(h, t["dec.proj.w"], t["dec.proj.b"]))
    for i in range(m.B):
        h = resblock(h, t[f"dec.block{i}.conv1.w"], t[f"dec.block{i}.conv1.b"],
                     t[f"dec.block{i}.conv2.w"], t[f"dec.block{i}.conv2.b"])
    u = relu(pixel_shuffle(conv2d(h, t["dec.up.w"], t["dec.up.b"])))
    a = np.clip(conv2d(u, t["dec.mu.w"], t["dec.mu.b"]), np.float32(-15), np.float32(15))
    mu = np.float32(255.0) * sigmoid32(a)
    s = np.exp(np.clip(conv2d(u, t["dec.s.w"], t["dec.s.b"]), LOG_S_MIN, LOG_S_MAX))
    s = np.clip(s, np.float32(0.5), np.float32(64.0))
    return (np.ascontiguousarray(mu[:, :H, :W].transpose(1, 2, 0)),
            np.ascontiguousarray(s[:, :H, :W].transpose(1, 2, 0)))


# --------------------------------------------------------------------------
# The same network with every float operation spelled out (pilc_oracle.c
# oracle_conv_fma / oracle_expf_np): the statement of the reference's
# arithmetic that the GPU "exact" network follows. Pinned bit for bit against
# the reference's own z, mu, s by tests/test_oracle.py.


def conv2d_fma(x, w, b, stride=1):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    ci, H, W = x.shape
    co, _, k, _ = w.shape
    p = k // 2
    Ho, Wo = (H + 2 * p - k) // stride + 1, (W + 2 * p - k) // stride + 1
    out = np.empty((co, Ho, Wo), np.float32)
    if lib().oracle_conv_fma(_p(x), ci, H, W, _p(w), _p(b), co, k, stride, _p(out)):
        raise NotImplementedError("no modelled BLAS order for this shape")
    return out


def exp_np(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    lib().oracle_expf_np_array(_p(x), _p(y), x.size)
    return y


def sigmoid_exact(x):
    x = np.asarray(x, np.float32)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = np.float32(1.0) / (np.float32(1.0) + exp_np(-x[pos]))
    e = exp_np(x[~pos])
    out[~pos] = e / (np.float32(1.0) + e)
    return out


def encoder_latents_exact(img: np.ndarray, m: Model) -> np.ndarray:
    t = m.t
    ph, pw = img.shape[0] & 1, img.shape[1] & 1
    if ph or pw:
        img = np.pad(img, ((0, ph), (0, pw), (0, 0)), mode="edge")
    x = np.ascontiguousarray((img.astype(np.float32) / np.float32(127.5) - np.float32(1.0)).transpose(2, 0, 1))
    h = relu(conv2d_fma(x, t["enc.stem.w"], t["enc.stem.b"]))
    h = relu(conv2d_fma(h, t["enc.down.w"], t["enc.down.b"], 2))
    for i in range(m.B):
        r = relu(conv2d_fma(h, t[f"enc.block{i}.conv1.w"], t[f"enc.block{i}.conv1.b"]))
        h = relu(h + conv2d_fma(r, t[f"enc.block{i}.conv2.w"], t[f"enc.block{i}.conv2.b"]))
    z = conv2d_fma(h, t["enc.proj.w"], t["enc.proj.b"])
    return np.ascontiguousarray(z.transpose(1, 2, 0))


def decode_params_exact(idx: np.ndarray, m: Model, H: int, W: int):
    t = m.t
    h = np.ascontiguousarray(t["codebook"][idx.astype(np.int64)].transpose(2, 0, 1))
    h = relu(conv2d_fma(h, t["dec.proj.w"], t["dec.proj.b"]))
    for i in range(m.B):
        r = relu(conv2d_fma(h, t[f"dec.block{i}.conv1.w"], t[f"dec.block{i}.conv1.b"]))
        h = relu(h + conv2d_fma(r, t[f"dec.block{i}.conv2.w"], t[f"dec.block{i}.conv2.b"]))
    u = relu(pixel_shuffle(conv2d_fma(h, t["dec.up.w"], t["dec.up.b"])))
    a = np.clip(conv2d_fma(u, t["dec.mu.w"], t["dec.mu.b"]), np.float32(-15), np.float32(15))
    mu = np.float32(255.0) * sigmoid_exact(a)
    s = exp_np(np.clip(conv2d_fma(u, t["dec.s.w"], t["dec.s.b"]), LOG_S_MIN, LOG_S_MAX))
    s = np.clip(s, np.float32(0.5), np.float32(64.0))
    return (np.ascontiguousarray(mu[:, :H, :W].transpose(1, 2, 0)),
            np.ascontiguousarray(s[:, :H, :W].transpose(1, 2, 0)))


# --------------------------------------------------------------------------
# container.py:128-335


_TAB_CACHE: dict = {}


def _tables(P: np.ndarray, M: int):
    key = (P.tobytes(), M)
    if key not in _TAB_CACHE:
        _TAB_CACHE[key] = build_tables(P, M)
    return _TAB_CACHE[key]


def _stream_table(blobs, states) -> bytes:
    return (struct.pack("<I", sum(len(b) for b in blobs))
            + struct.pack(f"<{len(blobs)}I", *(len(b) for b in blobs))
            + struct.pack(f"<{len(states)}H", *states))


def compress(img: np.ndarray, model: Model | None = None, backend: str = "twar-static",
             M: int = 12, L: int = 1, grid=None, debug_sched: bool = False) -> bytes:
    grid = default_grid() if grid is None else np.asarray(grid, np.float64)
    H, W = img.shape[:2]
    w, b = (model.w, model.b) if model is not None else (DEFAULT_W, DEFAULT_B)
    t = twar_forward(img, w, b)
    delta, phi, _, _, _ = _tables(residual_pmfs(grid, M), M)
    static_d = 0
    iblobs, istates = [], []
    if backend == "twar-vqvae":
        idx = encode_indices(img, model)
        mu, s = decode_params(idx, model, H, W)
        coded = ((t.astype(np.int64) - round_half_away(mu) + 128) & 0xFF).astype(np.uint8)
        dsched = scales_to_d(s, grid).ravel()
        ip = quantize_pmf(model.hist.astype(np.float64) + 1.0, M)[None]
        idelta, iphi, _, _, _ = _tables(ip, M)
        iblobs, istates = encode_lanes(idx.ravel(), np.zeros(idx.size, np.uint16), L, idelta, iphi, M)
    else:
        coded = t
        mad = float(np.mean(np.abs(t.astype(np.float64) - 128.0)))
        s_est = mad / np.log(4.0)
        static_d = int(np.argmin(np.abs(np.log2(float(s_est)) - np.log2(grid)))) if s_est > 0 else 0
        dsched = np.full(coded.size, static_d, np.uint16)
    rblobs, rstates = encode_lanes(coded.ravel(), dsched, L, delta, phi, M)
    flags = 1 if debug_sched else 0
    out = bytearray(b"PILC" + struct.pack("<BBBBB", 1, 1 if backend == "twar-vqvae" else 0, M, 0, flags))
    out += struct.pack("<IIHH", W, H, L, static_d) + grid_bytes(grid) + params_hash8(w, b)
    if backend == "twar-vqvae":
        out += model.hash8() + _stream_table(iblobs, istates)
    out += _stream_table(rblobs, rstates)
    if debug_sched:
        out += struct.pack("<I", zlib.crc32(dsched.astype("<u2").tobytes()))
    for x in iblobs + rblobs:
        out += x
    out += struct.pack("<I", zlib.crc32(bytes(out)))
    return bytes(out)


def decompress(blob: bytes, model: Model | None = None) -> np.ndarray:
    """container.py:195-335 (structure checks abbreviated to the ones the
    batch decoder reproduces); raises OracleError(kind, msg)."""
    if len(blob) < 8 or blob[:4] != b"PILC" or blob[4] != 1:
        raise OracleError("FormatError", "bad magic/version/length")
    if zlib.crc32(blob[:-4]) != struct.unpack_from("<I", blob, len(blob) - 4)[0]:
        raise OracleError("CorruptStreamError", "container checksum mismatch")
    backend, M, pad, flags = blob[5], blob[6], blob[7], blob[8]
    if flags & ~1:  # container.py:223-224
        raise OracleError("FormatError", f"unknown header flags {flags:#x}")
    W, H, L, static_d = struct.unpack_from("<IIHH", blob, 9)
    (D,) = struct.unpack_from("<H", blob, 21)
    grid = np.frombuffer(blob, "<f8", D, 23).copy()
    off = 23 + 8 * D
    ph = blob[off: off + 8]
    off += 8
    w, b = (model.w, model.b) if model is not None else (DEFAULT_W, DEFAULT_B)
    if params_hash8(w, b) != ph:
        raise OracleError("ModelError", "predictor parameters do not match the container")

    def table(off):
        (tot,) = struct.unpack_from("<I", blob, off)
        lens = struct.unpack_from(f"<{L}I", blob, off + 4)
        sts = struct.unpack_from(f"<{L}H", blob, off + 4 + 4 * L)
        return lens, sts, off + 4 + 6 * L

    ilens, ists = (), ()
    if backend == 1:
        mh = blob[off: off + 8]
        off += 8
        ilens, ists, off = table(off)
    rlens, rsts, off = table(off)
    sched_crc = None
    if flags & 1:
        (sched_crc,) = struct.unpack_from("<I", blob, off)
        off += 4
    _, _, sym, pop, nxt = _tables(residual_pmfs(grid, M), M)

    def lanes(off, lens):
        out = []
        for n in lens:
            out.append(blob[off: off + n])
            off += n
        return out, off

    iblobs, off2 = lanes(off, ilens)
    rblobs, _ = lanes(off2, rlens)
    shift = None
    if backend == 1:
        if model is None or model.hash8() != mh:
            raise OracleError("ModelError", "model hash mismatch")
        gh, gw = (H + 1) // 2, (W + 1) // 2
        ip = quantize_pmf(model.hist.astype(np.float64) + 1.0, M)[None]
        _, _, isym, ipop, inxt = _tables(ip, M)
        idx = decode_lanes(iblobs, ists, gh * gw, np.zeros(gh * gw, np.uint16), isym, ipop, inxt, M)
        mu, s = decode_params(idx.reshape(gh, gw), model, H, W)
        dsched = scales_to_d(s, grid).ravel()
        shift = round_half_away(mu)
    else:
        dsched = np.full(H * W * 3, static_d, np.uint16)
    if sched_crc is not None and zlib.crc32(dsched.astype("<u2").tobytes()) != sched_crc:
        raise OracleError("CorruptStreamError", "decoder-side distribution schedule disagrees with the encoder")
    coded = decode_lanes(rblobs, rsts, H * W * 3, dsched, sym, pop, nxt, M).reshape(H, W, 3)
    return twar_decode(coded, w, b, shift=None if shift is None else (shift & 0xFF).astype(np.uint8))
