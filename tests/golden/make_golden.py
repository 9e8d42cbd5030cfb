"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the reference only exists there):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports `pixelcodec` from /root/reference/pkg/src (read-only; no
__pycache__ is written thanks to the env vars above) and records its outputs
on seeded inputs. Nothing at test time reads /root/reference; the fixtures
are committed. Every array here is what the reference itself produced:

  tables.npz      quantized PMFs (logistic.residual_distributions) and the
                  five coder tables (tables.build_tables) for M = 10, 11, 12
  lanes.npz       tables.interleaved_encode lane blobs on report._bench_symbols
  twar.npz        predictor.forward_residual on random images + params
  static.npz      whole twar-static containers (container.compress)
  vqvae_*.npz     encoder latents z, indices, (mu, s), and twar-vqvae blobs
  small.pilw      random_weights(ModelConfig(32, 8, 8, 1), seed=42) file
  meta.json       hashes / scalars (model hash8, params hash8, table digests)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from pixelcodec import container, logistic, nn, predictor, tables, vqvae  # noqa: E402
from pixelcodec.weights import ModelConfig, random_weights  # noqa: E402

from paper_2206_05279_b200.synth import noise_images, smooth_images  # noqa: E402

SMALL = ModelConfig(K=32, Dc=8, channels=8, blocks=1)


def pack_blobs(blobs):
    sizes = np.array([len(b) for b in blobs], dtype=np.int64)
    offs = np.zeros(len(blobs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offs[1:])
    buf = np.frombuffer(b"".join(blobs), dtype=np.uint8)
    return buf, offs


def table_digest(enc, dec):
    h = hashlib.sha256()
    for a in (enc.delta, enc.phi, dec.symbol, dec.pop_count, dec.next_base):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def encoder_latents(image, w):
    """Replays vqvae.encode_to_indices up to the projection (vqvae.py:57-65)
    with the reference's own nn functions, so z is the reference's z."""
    t = w.tensors
    x = vqvae._normalize(vqvae._even_pad(image))
    h = nn.relu(nn.conv2d(x, t["enc.stem.w"], t["enc.stem.b"]))
    h = nn.relu(nn.conv2d(h, t["enc.down.w"], t["enc.down.b"], stride=2))
    for i in range(w.config.blocks):
        h = nn.residual_block(h, t[f"enc.block{i}.conv1.w"], t[f"enc.block{i}.conv1.b"],
                              t[f"enc.block{i}.conv2.w"], t[f"enc.block{i}.conv2.b"])
    z = nn.conv2d(h, t["enc.proj.w"], t["enc.proj.b"])
    return np.ascontiguousarray(z.transpose(1, 2, 0))  # (gh, gw, Dc)


def main():
    meta = {}
    grid = logistic.default_grid()

    # --- tables -----------------------------------------------------------
    tab = {}
    for M in (10, 11, 12):
        pmfs = logistic.residual_distributions(grid, M)
        enc, dec = tables.build_tables(pmfs, M, verify=True)
        tab[f"P_M{M}"] = np.stack([p.P.astype(np.int64) for p in pmfs])
        tab[f"delta_M{M}"] = enc.delta
        tab[f"phi_M{M}"] = enc.phi
        tab[f"symbol_M{M}"] = dec.symbol
        tab[f"pop_M{M}"] = dec.pop_count
        tab[f"next_M{M}"] = dec.next_base
        meta[f"table_digest_M{M}"] = table_digest(enc, dec)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tab)

    # --- coder lanes on the paper's Table-6 generator (report.py:34-44) ----
    from pixelcodec.pmf import quantize_pmf  # noqa: F401  (import check)
    rng = np.random.default_rng(0)
    M = 12
    pmfs = logistic.residual_distributions(grid, M)
    n = 30000
    d = rng.integers(0, grid.D, n).astype(np.uint16)
    syms = np.empty(n, dtype=np.uint8)
    for i, pmf in enumerate(pmfs):
        sel = d == i
        p = pmf.P.astype(np.float64) / (1 << M)
        syms[sel] = rng.choice(256, int(sel.sum()), p=p)
    enc, dec = tables.build_tables(pmfs, M)
    lanes = {"syms": syms, "d": d}
    for L in (1, 3, 16, 64):
        ls = tables.interleaved_encode(syms, d, L, enc)
        buf, offs = pack_blobs([s.to_bytes() for s in ls.streams])
        lanes[f"L{L}_buf"] = buf
        lanes[f"L{L}_offs"] = offs
        lanes[f"L{L}_states"] = np.array(ls.states, dtype=np.int64)
        back = tables.interleaved_decode(ls, n, d, dec)
        assert np.array_equal(back, syms)
    np.savez_compressed(os.path.join(HERE, "lanes.npz"), **lanes)

    # --- TWAR forward residual -------------------------------------------
    rng = np.random.default_rng(1234)
    tw = {}
    shapes = [(1, 1), (1, 7), (7, 1), (31, 33), (32, 32), (97, 61)]
    for k, (h, w) in enumerate(shapes):
        img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        wts = rng.normal(0, 2, (3, 3)).astype(np.float32)
        bias = rng.normal(0, 20, 3).astype(np.float32)
        p = predictor.PredictorParams(wts, bias)
        tw[f"img{k}"] = img
        tw[f"w{k}"] = wts
        tw[f"b{k}"] = bias
        tw[f"res{k}"] = predictor.forward_residual(img, p)
        tw[f"resdef{k}"] = predictor.forward_residual(img)
        assert np.array_equal(predictor.decode_parallel(tw[f"res{k}"], p), img)
    tw["n"] = np.array(len(shapes))
    np.savez_compressed(os.path.join(HERE, "twar.npz"), **tw)
    meta["default_params_hash8"] = predictor.default_params().hash8().hex()

    # --- twar-static containers ------------------------------------------
    rng = np.random.default_rng(99)
    blobs, imgs, cfgs = [], [], []
    cases = []
    for (h, w) in [(1, 1), (1, 7), (7, 1), (31, 33), (32, 32), (64, 64), (97, 61)]:
        for kind in ("noise", "smooth", "const"):
            if kind == "noise":
                img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
            elif kind == "smooth":
                img = smooth_images(1, h, w, seed=len(cases))[0]
            else:
                img = np.full((h, w, 3), 200, dtype=np.uint8)
            cases.append(img)
    for ci, img in enumerate(cases):
        for (L, M, dbg) in [(1, 12, False), (4, 12, False), (1, 10, False), (3, 11, True)]:
            cfg = container.CodecConfig(lanes=L, M=M, debug_schedule_check=dbg)
            blob = container.compress(img, None, cfg)
            assert np.array_equal(container.decompress(blob), img)
            blobs.append(blob)
            imgs.append(ci)
            cfgs.append((L, M, int(dbg)))
    buf, offs = pack_blobs(blobs)
    st = {"buf": buf, "offs": offs, "img_index": np.array(imgs), "cfg": np.array(cfgs)}
    for ci, img in enumerate(cases):
        st[f"img{ci}"] = img
    st["n_img"] = np.array(len(cases))
    # a fitted-params (params-only model) container: random predictor params
    wts = np.random.default_rng(5).normal(0, 2, (3, 3)).astype(np.float32)
    bias = np.random.default_rng(6).normal(0, 20, 3).astype(np.float32)
    from pixelcodec.weights import ModelWeights
    pm = ModelWeights(ModelConfig(), {}, predictor_params=predictor.PredictorParams(wts, bias))
    st["fit_w"], st["fit_b"] = wts, bias
    st["fit_blob"] = np.frombuffer(container.compress(cases[9], pm), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "static.npz"), **st)

    # --- twar-vqvae: small (test) model and the full default model --------
    small = random_weights(SMALL, seed=42)
    small.save(os.path.join(HERE, "small.pilw"))
    meta["small_hash8"] = small.hash8().hex()
    full = random_weights(ModelConfig(), seed=1)
    meta["full_seed1_hash8"] = full.hash8().hex()
    for tag, model, shapes_ in (
        ("small", small, [(32, 32), (31, 33), (1, 1), (7, 1), (14, 10), (64, 64)]),
        ("full", full, [(32, 32), (32, 32), (17, 13), (64, 64)]),
    ):
        out = {}
        blobs = []
        for k, (h, w) in enumerate(shapes_):
            img = (smooth_images(1, h, w, seed=100 + k)[0] if k % 2 == 0
                   else np.random.default_rng(k).integers(0, 256, (h, w, 3), dtype=np.uint8))
            z = encoder_latents(img, model)
            idx = vqvae.encode_to_indices(img, model)
            mu, s = vqvae.decode_to_params(idx, model, (h, w))
            out[f"img{k}"] = img
            out[f"z{k}"] = z
            out[f"idx{k}"] = idx
            out[f"mu{k}"] = mu
            out[f"s{k}"] = s
            cfg = container.CodecConfig(backend="twar-vqvae", lanes=1 + (k % 3))
            blob = container.compress(img, model, cfg)
            assert np.array_equal(container.decompress(blob, model), img)
            blobs.append(blob)
        buf, offs = pack_blobs(blobs)
        out["buf"], out["offs"] = buf, offs
        out["n"] = np.array(len(shapes_))
        np.savez_compressed(os.path.join(HERE, f"vqvae_{tag}.npz"), **out)

    meta["bits_golden"] = list(b"\x04\x00\x00\x00\x00\x00\x00\x00\x0d")
    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
