"""Table-driven semi-dynamic rANS ("ANS-AI"): tables on the host, lanes on
the GPU. Semantics of `pixelcodec/tables.py`.

Tables (tables.py:71-142), built once per distribution set and cached:
    encode  delta[d,x] = k*2^M - P*2^k  (P*2^k in [2^M, 2^(M+1)))
            phi[d,x]   = 2^M - P + C
    decode  for t in [0, 2^M): symbol x, pop count b (minimal with
            (t - C_x + P_x) << b >= 2^M) and next base (t - C_x + P_x) << b
Device layout: one uint32 per entry, encode delta | phi<<16 (D*X words),
decode symbol | b<<8 | next<<16 (D*2^M words).

`interleaved_encode` / `interleaved_decode` keep the reference signatures
(tables.py:202-274) and run the lanes on the GPU (csrc/rans.cu).
"""

from __future__ import annotations

import functools
import hashlib
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .bits import BitStack
from .device import CACHE, ptr, require_device, sptr
from .errors import CoderContractError, CorruptStreamError, TableError
from .pmf import QuantizedPmf


@dataclass(frozen=True)
class EncodeTables:
    M: int
    delta: np.ndarray  # (D, X) uint16
    phi: np.ndarray  # (D, X) uint16

    @property
    def D(self) -> int:
        return int(self.delta.shape[0])

    @property
    def X(self) -> int:
        return int(self.delta.shape[1])

    @property
    def footprint_bytes(self) -> int:
        return self.delta.nbytes + self.phi.nbytes

    @functools.cached_property
    def key(self) -> bytes:
        return hashlib.sha256(self.delta.tobytes() + self.phi.tobytes() + bytes([self.M])).digest()[:16]

    def device_words(self, dev) -> torch.Tensor:
        def make():
            w = self.delta.astype(np.uint32) | (self.phi.astype(np.uint32) << 16)
            return torch.from_numpy(w.view(np.int32).copy()).to(dev)
        return CACHE.get(("enc", self.key), dev, make)


@dataclass(frozen=True)
class DecodeTables:
    M: int
    symbol: np.ndarray  # (D, 2^M) uint8
    pop_count: np.ndarray  # (D, 2^M) uint8
    next_base: np.ndarray  # (D, 2^M) uint16

    @property
    def D(self) -> int:
        return int(self.symbol.shape[0])

    @property
    def footprint_bytes(self) -> int:
        return self.symbol.nbytes + self.pop_count.nbytes + self.next_base.nbytes

    @functools.cached_property
    def key(self) -> bytes:
        return hashlib.sha256(self.symbol.tobytes() + self.pop_count.tobytes()
                              + self.next_base.tobytes() + bytes([self.M])).digest()[:16]

    def device_words(self, dev) -> torch.Tensor:
        def make():
            w = (self.symbol.astype(np.uint32) | (self.pop_count.astype(np.uint32) << 8)
                 | (self.next_base.astype(np.uint32) << 16))
            return torch.from_numpy(w.view(np.int32).copy()).to(dev)
        return CACHE.get(("dec", self.key), dev, make)


def _build(P_rows: tuple, M: int) -> tuple[EncodeTables, DecodeTables]:
    P = np.array(P_rows, dtype=np.int64)
    D, X = P.shape
    T = 1 << M
    C = np.zeros_like(P)
    C[:, 1:] = np.cumsum(P[:, :-1], axis=1)
    # k = number of doublings that lift P into [2^M, 2^(M+1))
    k = M - np.floor(np.log2(P)).astype(np.int64)
    k = np.where((P << k) >= 2 * T, k - 1, k)
    k = np.where((P << k) < T, k + 1, k)
    dval = (k << M) - (P << k)
    pval = T - P + C
    if dval.min() < 0 or dval.max() >= (1 << 16) or pval.max() >= (1 << 16):
        raise TableError("table entry does not fit unsigned 16 bits")
    t = np.arange(T, dtype=np.int64)
    sym = np.empty((D, T), np.int64)
    for d in range(D):
        sym[d] = np.searchsorted(C[d], t, side="right") - 1
    mid = t[None, :] - np.take_along_axis(C, sym, 1) + np.take_along_axis(P, sym, 1)
    # minimal b with mid << b >= 2^M: b = M - floor(log2 mid), mid in [1, 2^M)
    b = M - (np.floor(np.log2(mid)).astype(np.int64))
    b = np.where((mid << b) >= 2 * T, b - 1, b)
    b = np.where((mid << b) < T, b + 1, b)
    b = np.where(mid >= T, 0, b)
    enc = EncodeTables(M, dval.astype(np.uint16), pval.astype(np.uint16))
    dec = DecodeTables(M, sym.astype(np.uint8), b.astype(np.uint8), (mid << b).astype(np.uint16))
    return enc, dec


@functools.lru_cache(maxsize=128)
def _build_cached(P_rows: tuple, M: int):
    return _build(P_rows, M)


_BY_BYTES: dict = {}


def build_tables(dists: Sequence[QuantizedPmf], M: int, verify: bool = False):
    """(EncodeTables, DecodeTables) for a distribution set; cached by content."""
    if M > 12:
        raise TableError(f"M={M}: delta is only guaranteed to fit unsigned 16 bits for M <= 12")
    if not dists:
        raise TableError("need at least one distribution")
    # cache hit: the masses' bytes (and M) name the tables; a hit was
    # validated when it was built (hashing bytes keeps per-call host time
    # in the microseconds, this runs on every compress / decompress)
    key = (M, tuple((p.M, p.P.dtype.str, p.P.tobytes()) for p in dists))
    hit = _BY_BYTES.get(key)
    if hit is not None:
        if verify:
            verify_encode_tables(hit[0], dists)
        return hit
    X = dists[0].X
    if X > 256:
        raise TableError("symbol table is uint8; alphabet must be <= 256")
    cap = (1 << (M - 1)) - 1
    for d, pmf in enumerate(dists):
        if pmf.M != M:
            raise TableError(f"distribution {d} quantized at M={pmf.M}, expected {M}")
        if pmf.X != X:
            raise TableError("all distributions must share one alphabet")
        if int(pmf.P.min()) < 1 or int(pmf.P.max()) > cap:
            raise CoderContractError(f"distribution {d} has masses outside [1, {cap}]")
    rows = tuple(tuple(int(v) for v in p.P) for p in dists)
    enc, dec = _build_cached(rows, M)
    if len(_BY_BYTES) < 256:
        _BY_BYTES[key] = (enc, dec)
    if verify:
        verify_encode_tables(enc, dists)
    return enc, dec


def verify_encode_tables(enc: EncodeTables, dists: Sequence[QuantizedPmf]) -> None:
    """S >> ((delta + S) >> M) must land in [P, 2P) for every (d, x, S)."""
    M = enc.M
    S = np.arange(1 << M, 1 << (M + 1), dtype=np.int64)
    for d, pmf in enumerate(dists):
        P = pmf.P.astype(np.int64)
        sh = (enc.delta[d].astype(np.int64)[:, None] + S[None, :]) >> M
        r = S[None, :] >> sh
        bad = (r < P[:, None]) | (r >= 2 * P[:, None])
        if bad.any():
            xi, si = np.argwhere(bad)[0]
            raise TableError(f"renormalization violated at d={d}, x={xi}, S={(1 << M) + si}")
        if not np.array_equal(enc.phi[d].astype(np.int64), (1 << M) - P + pmf.C.astype(np.int64)):
            raise TableError(f"phi table mismatch for distribution {d}")


# --- single-symbol path (tables.py:169-183; host, for API parity) ----------


def fast_encode(state: int, tables: EncodeTables, d: int, x: int, stream: BitStack) -> int:
    b = (int(tables.delta[d, x]) + state) >> tables.M
    stream.push_bits(state, b)
    return (state >> b) + int(tables.phi[d, x])


def fast_decode(state: int, tables: DecodeTables, d: int, stream: BitStack) -> tuple[int, int]:
    idx = state - (1 << tables.M)
    if not 0 <= idx < (1 << tables.M):
        raise CorruptStreamError(f"decoder state {state} left the resting range")
    x = int(tables.symbol[d, idx])
    return x, int(tables.next_base[d, idx]) + stream.pop_bits(int(tables.pop_count[d, idx]))


# --- lanes -------------------------------------------------------------------


@dataclass
class LaneSet:
    """Independent per-lane coder sessions; symbol i belongs to lane i mod L."""

    states: list
    streams: list

    @property
    def L(self) -> int:
        return len(self.states)


def lane_cap_words(n_sym: int, lanes: int, M: int) -> int:
    per = -(-n_sym // lanes)
    return (per * M + 31) // 32 + 1


def encode_lanes_device(syms: torch.Tensor, n_img: int, n_sym: int, lanes: int, tables: EncodeTables,
                        dev, stream, shift=None, dsched=None, d_img=None):
    """GPU lanes for a batch: returns (scratch, cap, nbits, states) tensors."""
    cap = lane_cap_words(n_sym, lanes, tables.M)
    scratch = torch.empty(n_img * lanes * cap + 4, dtype=torch.int32, device=dev)  # +16 B read slack
    nbits = torch.empty(max(n_img * lanes, 1), dtype=torch.int32, device=dev)
    states = torch.empty(max(n_img * lanes, 1), dtype=torch.int16, device=dev)
    _lib.call("pilc_rans_encode", ptr(syms), ptr(shift), ptr(dsched), ptr(d_img), n_img, n_sym, lanes,
              ptr(tables.device_words(dev)), tables.D, tables.X, tables.M, ptr(scratch), cap,
              ptr(nbits), ptr(states), sptr(stream))
    return scratch, cap, nbits, states


def interleaved_encode(symbols, d_schedule, lanes: int, tables: EncodeTables) -> LaneSet:
    """Encode symbols across `lanes` independent streams (GPU lanes)."""
    if lanes < 1:
        raise CoderContractError("need at least one lane")
    symbols = np.ascontiguousarray(symbols, dtype=np.uint8).ravel()
    d_schedule = np.ascontiguousarray(d_schedule, dtype=np.uint16).ravel()
    if d_schedule.shape != symbols.shape:
        raise CoderContractError("need one distribution index per symbol")
    if symbols.size and (int(d_schedule.max()) >= tables.D or int(symbols.max()) >= tables.X):
        raise CoderContractError("symbol or distribution index outside the tables")
    if tables.D > 256:
        raise CoderContractError("GPU lanes take distribution indices < 256")
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    n = symbols.size
    syms_d = torch.from_numpy(symbols.copy()).to(dev) if n else torch.zeros(1, dtype=torch.uint8, device=dev)
    ds_d = torch.from_numpy(d_schedule.astype(np.uint8)).to(dev) if n else torch.zeros(1, dtype=torch.uint8, device=dev)
    scratch, cap, nbits, states = encode_lanes_device(syms_d, 1, n, lanes, tables, dev, stream, dsched=ds_d)
    scr = scratch.cpu().numpy().view(np.uint32).reshape(-1)
    nb = nbits.cpu().numpy().view(np.uint32)[:lanes]
    st = states.cpu().numpy().view(np.uint16)[:lanes]
    streams = []
    for l in range(lanes):
        words = scr[l * cap:(l + 1) * cap]
        streams.append(BitStack.from_packed(words.view(np.uint8), int(nb[l])))
    return LaneSet([int(s) for s in st], streams)


def interleaved_decode(lane_set: LaneSet, count: int, d_schedule, tables: DecodeTables, workers: int = 1) -> np.ndarray:
    """Exact inverse of interleaved_encode (GPU lanes). `workers` is accepted
    for signature parity; lanes always run concurrently on the GPU."""
    L = lane_set.L
    d_schedule = np.ascontiguousarray(d_schedule, dtype=np.uint16)
    if d_schedule.shape != (count,):
        raise CoderContractError("need one distribution index per symbol")
    if count and int(d_schedule.max()) >= tables.D:
        raise CoderContractError("distribution index outside the tables")
    s0 = 1 << tables.M
    for lane, st in enumerate(lane_set.states):
        if not s0 <= st < 2 * s0:
            raise CorruptStreamError(f"lane {lane} initial state out of range")
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    payloads = [s.to_bytes()[8:] for s in lane_set.streams]
    offs = np.zeros(L, np.uint64)
    pos = 0
    for l, p in enumerate(payloads):
        offs[l] = pos
        pos += len(p)
    buf = np.zeros(pos + 16, np.uint8)
    buf[:pos] = np.frombuffer(b"".join(payloads), np.uint8)
    buf_d = torch.from_numpy(buf).to(dev)
    out = torch.zeros(max(count, 1), dtype=torch.uint8, device=dev)
    lane_status = torch.zeros(L, dtype=torch.uint8, device=dev)
    nbits = np.array([len(s) for s in lane_set.streams], np.uint32)
    states = np.array(lane_set.states, np.uint16)
    ds_d = torch.from_numpy(d_schedule.astype(np.uint8)).to(dev) if count else torch.zeros(1, dtype=torch.uint8, device=dev)
    t_off = torch.from_numpy(offs.view(np.int64)).to(dev)
    t_nb = torch.from_numpy(nbits.view(np.int32)).to(dev)
    t_st = torch.from_numpy(states.view(np.int16)).to(dev)
    _lib.call("pilc_rans_decode", ptr(buf_d), ptr(t_off), ptr(t_nb), ptr(t_st), ptr(ds_d), None, 1, count, L,
              ptr(tables.device_words(dev)), tables.D, tables.M, None, ptr(out), ptr(lane_status), sptr(stream))
    status = lane_status.cpu().numpy()
    for lane in range(L):
        if status[lane] == 24:
            raise CorruptStreamError(f"lane {lane} bit stream underflow")
        if status[lane] == 25:
            raise CorruptStreamError(f"lane {lane} did not return to the initial coder state")
    return out.cpu().numpy()[:count].copy()


def encode_message(symbols, d_schedule, tables: EncodeTables):
    ls = interleaved_encode(symbols, d_schedule, 1, tables)
    return ls.states[0], ls.streams[0]
