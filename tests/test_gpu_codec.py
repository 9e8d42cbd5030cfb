"""GPU parity tests: the sm_100a path (through libpilc_sm100a.so) against the
reference's golden fixtures and the CPU oracle on the same seeded inputs.

Integer/byte work is checked bit-exactly; the VQ-VAE float path is checked
for exact codebook indices (given identical latents z the argmin is
bit-exact; end to end z differs from numpy/BLAS only by summation order),
lossless round trips and bpd within 0.5% of the reference.
"""

import os
import struct
import zlib

import numpy as np
import torch
import pytest

import paper_2206_05279_b200 as pc
import paper_2206_05279_b200.logistic  # noqa: F401
from oracle import oracle as O
from paper_2206_05279_b200 import container as ct
from paper_2206_05279_b200 import predictor, tables, vqvae
from paper_2206_05279_b200.errors import CodecError, CorruptStreamError, FormatError, ModelError
from paper_2206_05279_b200.logistic import default_grid, residual_distributions
from paper_2206_05279_b200.synth import smooth_images

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SMALL = pc.ModelConfig(K=32, Dc=8, channels=8, blocks=1)


def _blobs(z):
    return [z["buf"][z["offs"][i]: z["offs"][i + 1]].tobytes() for i in range(len(z["offs"]) - 1)]


@pytest.fixture(scope="module")
def small_model():
    return pc.ModelWeights.load(os.path.join(GOLDEN, "small.pilw"))


@pytest.fixture(scope="module")
def full_model():
    return pc.random_weights(seed=1)


# --- TWAR ---------------------------------------------------------------------


def test_twar_forward_matches_reference(golden):
    z = golden("twar.npz")
    for k in range(int(z["n"])):
        p = predictor.PredictorParams(z[f"w{k}"], z[f"b{k}"])
        res = predictor.forward_residual(z[f"img{k}"], p)
        assert np.array_equal(res, z[f"res{k}"])
        assert np.array_equal(predictor.forward_residual(z[f"img{k}"]), z[f"resdef{k}"])
        assert np.array_equal(predictor.decode_parallel(res, p), z[f"img{k}"])


@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (5, 37), (33, 31), (64, 64), (130, 70)])
def test_twar_random_params_vs_oracle(shape):
    rng = np.random.default_rng(sum(shape))
    imgs = rng.integers(0, 256, (6, *shape, 3), dtype=np.uint8)
    w = rng.normal(0, 2, (3, 3)).astype(np.float32)
    b = rng.normal(0, 20, 3).astype(np.float32)
    p = predictor.PredictorParams(w, b)
    res = predictor.forward_residual_batch(imgs, p)
    assert np.array_equal(res, O.twar_forward(imgs, w, b))
    assert np.array_equal(predictor.decode_parallel_batch(res, p), imgs)


@pytest.mark.parametrize("bias", [4194303.5, 4194304.0, -4194304.5, 1.5e7, 3.0e9, -2.5e10])
def test_twar_large_accumulators_vs_oracle(bias):
    """round_mod256 takes a float32 path below |acc| = 2^22 and the float64
    one above; both must agree with the reference rounding at the switch."""
    rng = np.random.default_rng(7)
    imgs = rng.integers(0, 256, (4, 9, 11, 3), dtype=np.uint8)
    w = np.array([[0.5, -1, 1], [1, -1, 0.25], [1, -0.5, 1]], np.float32)
    b = np.array([bias, -bias, bias / 3], np.float32)
    p = predictor.PredictorParams(w, b)
    res = predictor.forward_residual_batch(imgs, p)
    assert np.array_equal(res, O.twar_forward(imgs, w, b))
    assert np.array_equal(predictor.decode_parallel_batch(res, p), imgs)


def test_twar_exhaustive_2x2_sample():
    # acceptance 6 style: many 2x2 images with 4-value alphabets
    rng = np.random.default_rng(7)
    vals = np.array([0, 1, 128, 255], np.uint8)
    imgs = vals[rng.integers(0, 4, (20000, 2, 2, 3))]
    for p in (pc.default_params(), predictor.PredictorParams(rng.normal(0, 2, (3, 3)), rng.normal(0, 20, 3))):
        res = predictor.forward_residual_batch(imgs, p)
        assert np.array_equal(res, O.twar_forward(imgs, p.weights, p.bias))
        assert np.array_equal(predictor.decode_parallel_batch(res, p), imgs)


@pytest.mark.parametrize("shape,n", [((32, 32), 13), ((16, 48), 9), ((64, 64), 3), ((24, 40), 5), ((100, 128), 2),
                                     ((5, 37), 4), ((8, 8), 300)])
@pytest.mark.parametrize("kind", ["default", "integral", "float"])
def test_twar_forward_paths_vs_oracle(shape, n, kind):
    """Every forward-residual kernel (whole images through shared memory for
    W = 16 m up to 12 KB, 8-pixel runs for W = 8 m, the per-pixel kernel
    otherwise) with each predictor arithmetic (the default predictor's
    byte-lane path, integer weights, float weights) against the oracle,
    partial image groups included."""
    rng = np.random.default_rng(n * 31 + shape[1])
    imgs = rng.integers(0, 256, (n, *shape, 3), dtype=np.uint8)
    if kind == "default":
        p = pc.default_params()
    elif kind == "integral":
        p = predictor.PredictorParams(np.array([[1, 0, -2], [2, -1, 1], [0, 3, -1]], np.float32),
                                      np.array([5, -7, 300], np.float32))
    else:
        p = predictor.PredictorParams(rng.normal(0, 2, (3, 3)).astype(np.float32), rng.normal(0, 20, 3).astype(np.float32))
    res = predictor.forward_residual_batch(imgs, p)
    assert np.array_equal(res, O.twar_forward(imgs, p.weights, p.bias))
    assert np.array_equal(predictor.decode_parallel_batch(res, p), imgs)


# --- coder lanes --------------------------------------------------------------


@pytest.mark.parametrize("L", [1, 3, 16, 64])
def test_lanes_byte_identical_to_reference(golden, L):
    z = golden("lanes.npz")
    enc, dec = tables.build_tables(residual_distributions(default_grid(), 12), 12)
    ls = tables.interleaved_encode(z["syms"], z["d"], L, enc)
    ref = [z[f"L{L}_buf"][z[f"L{L}_offs"][i]: z[f"L{L}_offs"][i + 1]].tobytes() for i in range(L)]
    assert [s.to_bytes() for s in ls.streams] == ref
    assert ls.states == list(z[f"L{L}_states"])
    assert np.array_equal(tables.interleaved_decode(ls, z["syms"].size, z["d"], dec), z["syms"])


def test_lanes_random_vs_oracle():
    rng = np.random.default_rng(3)
    enc, dec = tables.build_tables(residual_distributions(default_grid(), 11), 11)
    for n, L in [(0, 1), (1, 1), (5, 7), (1000, 1), (4097, 5), (20000, 33)]:
        syms = rng.integers(0, 256, n).astype(np.uint8)
        ds = rng.integers(0, 8, n).astype(np.uint16)
        ls = tables.interleaved_encode(syms, ds, L, enc)
        blobs, states = O.encode_lanes(syms, ds, L, enc.delta, enc.phi, 11)
        assert [s.to_bytes() for s in ls.streams] == blobs and ls.states == states
        assert np.array_equal(tables.interleaved_decode(ls, n, ds, dec), syms)


def test_lane_underflow_and_end_state_detected():
    enc, dec = tables.build_tables(residual_distributions(default_grid(), 12), 12)
    syms = np.arange(300, dtype=np.uint8)
    ds = np.full(300, 3, np.uint16)
    ls = tables.interleaved_encode(syms, ds, 1, enc)
    short = pc.container.BitStack if hasattr(pc.container, "BitStack") else None
    from paper_2206_05279_b200.bits import BitStack
    raw = ls.streams[0].to_bytes()
    nb = struct.unpack_from("<Q", raw)[0]
    trunc = BitStack.from_packed(np.frombuffer(raw[8:], np.uint8), nb - 40)
    with pytest.raises(CorruptStreamError):
        tables.interleaved_decode(tables.LaneSet(ls.states, [trunc]), 300, ds, dec)
    with pytest.raises(CorruptStreamError):  # recorded state outside [2^M, 2^(M+1))
        tables.interleaved_decode(tables.LaneSet([(1 << 12) - 1], ls.streams), 300, ds, dec)
    # an extra leading bit is left unconsumed -> end-state check
    extra = BitStack.from_packed(np.frombuffer(raw[8:] + b"\x00", np.uint8), nb + 1)
    with pytest.raises(CorruptStreamError, match="initial coder state|underflow"):
        tables.interleaved_decode(tables.LaneSet(ls.states, [extra]), 300, ds, dec)
    del short


# --- twar-static containers: byte-identical to the reference -----------------


def test_static_containers_byte_identical(golden):
    z = golden("static.npz")
    blobs = _blobs(z)
    for blob, ci, (L, M, dbg) in zip(blobs, z["img_index"], z["cfg"]):
        img = z[f"img{ci}"]
        cfg = pc.CodecConfig(lanes=int(L), M=int(M), debug_schedule_check=bool(dbg))
        assert pc.compress(img, None, cfg) == blob
        assert np.array_equal(pc.decompress(blob), img)


def test_static_batch_equals_single(golden):
    imgs = smooth_images(37, 32, 32, seed=11)
    buf, off = pc.compress_batch(imgs)
    for i in range(0, 37, 6):
        assert buf[off[i]:off[i + 1]].tobytes() == O.compress(imgs[i])
    out = pc.decompress_batch(buf, off)
    assert np.array_equal(out, imgs)


def test_fitted_params_container(golden):
    z = golden("static.npz")
    m = pc.ModelWeights(pc.ModelConfig(), {}, predictor_params=predictor.PredictorParams(z["fit_w"], z["fit_b"]))
    assert pc.compress(z["img9"], m) == z["fit_blob"].tobytes()
    assert np.array_equal(pc.decompress(z["fit_blob"].tobytes(), m), z["img9"])
    with pytest.raises(ModelError):
        pc.decompress(z["fit_blob"].tobytes())


def test_mixed_shape_batch():
    rng = np.random.default_rng(5)
    imgs = [rng.integers(0, 256, (h, w, 3), dtype=np.uint8) for h, w in [(1, 1), (7, 1), (1, 7), (31, 33), (8, 8), (7, 1)]]
    buf, off = pc.compress_batch(imgs)
    for i, im in enumerate(imgs):
        assert buf[off[i]:off[i + 1]].tobytes() == O.compress(im)
    out = pc.decompress_batch(buf, off)
    assert all(np.array_equal(a, b) for a, b in zip(out, imgs))


# --- twar-vqvae ---------------------------------------------------------------


@pytest.mark.parametrize("tag", ["small", "full"])
def test_argmin_bit_exact_given_z(golden, tag, small_model, full_model):
    z = golden(f"vqvae_{tag}.npz")
    m = small_model if tag == "small" else full_model
    for k in range(int(z["n"])):
        assert np.array_equal(vqvae.argmin_codebook(z[f"z{k}"], m), z[f"idx{k}"])


EXACT = pc.CodecConfig(backend="twar-vqvae")
FAST = pc.CodecConfig(backend="twar-vqvae", numerics="fast")


@pytest.mark.parametrize("tag", ["small", "full"])
def test_exact_network_bit_identical_to_reference(golden, tag, small_model, full_model):
    """The exact network (pilc_vq_*_exact) reproduces the reference's float
    arithmetic: z, indices, mu and s equal pixelcodec's bit for bit, odd
    shapes and the 1 x 1 image (single-pixel convs: OpenBLAS sgemv order)
    included."""
    z = golden(f"vqvae_{tag}.npz")
    m = small_model if tag == "small" else full_model
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        assert np.array_equal(vqvae.encoder_latents(img, m).view(np.uint32), z[f"z{k}"].view(np.uint32)), k
        assert np.array_equal(vqvae.encode_to_indices(img, m), z[f"idx{k}"])
        mu, s = vqvae.decode_to_params(z[f"idx{k}"], m, img.shape[:2])
        assert np.array_equal(mu.view(np.uint32), z[f"mu{k}"].view(np.uint32)), k
        assert np.array_equal(s.view(np.uint32), z[f"s{k}"].view(np.uint32)), k


@pytest.mark.parametrize("tag", ["small", "full"])
def test_exact_vqvae_containers_byte_identical_to_reference(golden, tag, small_model, full_model):
    """numerics="exact" (the default): twar-vqvae containers are byte-identical
    to pixelcodec.compress, and pixelcodec's own containers decode exactly."""
    z = golden(f"vqvae_{tag}.npz")
    m = small_model if tag == "small" else full_model
    ref = _blobs(z)
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        assert pc.compress(img, m, pc.CodecConfig(backend="twar-vqvae", lanes=1 + (k % 3))) == ref[k], k
        assert np.array_equal(pc.decompress(ref[k], m), img)
    out = pc.decompress_batch(z["buf"], z["offs"].astype(np.uint64), m)
    assert all(np.array_equal(out[k], z[f"img{k}"]) for k in range(int(z["n"])))


def _exact_shapes():
    # latent / hi-res rasters whose pixel count leaves 1..8 pixels after the
    # last multiple of 16 (OpenBLAS m-tail order, Ci >= 32), single-pixel
    # latents (sgemv order), and plain shapes
    return [(6, 11), (2, 2), (1, 2), (3, 3), (5, 9), (9, 7), (34, 3), (20, 20), (17, 13)]


@pytest.mark.parametrize("shape", _exact_shapes())
def test_exact_network_vs_oracle_statement(shape, full_model, small_model):
    """Exact network against the oracle's explicit statement of the
    reference arithmetic (oracle_conv_fma: FMA chains, sgemv and m-tail
    orders, numpy's exp), which tests/test_oracle.py pins to the reference;
    z / mu / s bit-identical."""
    rng = np.random.default_rng(sum(shape))
    for m in (full_model, small_model):
        om = O.Model.from_bytes(m.to_bytes())
        img = rng.integers(0, 256, (*shape, 3), dtype=np.uint8)
        z = vqvae.encoder_latents(img, m)
        assert np.array_equal(z.view(np.uint32), O.encoder_latents_exact(img, om).view(np.uint32))
        idx = vqvae.encode_to_indices(img, m)
        assert np.array_equal(idx, O.argmin_codebook(z, om.t["codebook"]))
        mu, s = vqvae.decode_to_params(idx, m, shape)
        mu_o, s_o = O.decode_params_exact(idx, om, *shape)
        assert np.array_equal(mu.view(np.uint32), mu_o.view(np.uint32))
        assert np.array_equal(s.view(np.uint32), s_o.view(np.uint32))


@pytest.mark.parametrize("exact", [True, False])
def test_decoder_shift_and_d_follow_mu_and_s(full_model, exact):
    """The decoder emits (shift, d) directly; they must be exactly
    round_half_away(mu) and scales_to_distributions(s) (logistic.py:36-40,
    109-114) of the same kernel's mu and s, for both decoders."""
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    grid = default_grid()
    for H, W in ((32, 32), (17, 13), (64, 64)):
        gh, gw = vqvae.latent_shape(H, W)
        idx = torch.from_numpy(np.random.default_rng(H * W).integers(0, 256, (16, gh, gw), dtype=np.uint8)).to(dev)
        sh, d, mu, s = (t.cpu().numpy() for t in vqvae.decode_head_device(idx, full_model, H, W, grid, dev, st,
                                                                         want_params=True, exact=exact))
        assert np.array_equal(sh, pc.logistic.round_half_away(mu))
        assert np.array_equal(d, pc.logistic.scales_to_distributions(s, grid))


def test_fast_encoder_vs_exact(golden, full_model):
    """The fast encoder of the default model (tcgen05, 3-product fp16 split
    with per-image power-of-two scales, csrc/tc_conv.cu) is fp32-class: z
    within 2e-5 max|z| of the exact z, and the same codebook indices."""
    z = golden("vqvae_full.npz")
    imgs = [z[f"img{k}"] for k in range(int(z["n"]))] + list(smooth_images(24, 32, 32, seed=77))
    for img in imgs:
        zt = vqvae.encoder_latents(img, full_model, exact=False)
        zf = vqvae.encoder_latents(img, full_model)
        scale = np.abs(zf).max()
        assert np.abs(zt - zf).max() <= 2e-5 * scale, np.abs(zt - zf).max() / scale
        assert np.array_equal(vqvae.encode_to_indices(img, full_model, exact=False),
                              vqvae.encode_to_indices(img, full_model))


def test_fast_decoder_vs_exact(golden, full_model):
    """The fast decoder (tcgen05 bf16) against the exact one: mu within a few
    grey levels, s within 20%; most shifts and nearly all scale indices
    agree. bpd parity is checked end to end below."""
    z = golden("vqvae_full.npz")
    for k in range(int(z["n"])):
        H, W = z[f"img{k}"].shape[:2]
        mu_t, s_t = vqvae.decode_to_params(z[f"idx{k}"], full_model, (H, W), exact=False)
        mu_f, s_f = vqvae.decode_to_params(z[f"idx{k}"], full_model, (H, W))
        assert np.isfinite(mu_t).all() and np.isfinite(s_t).all()
        assert np.abs(mu_t - mu_f).max() < 16.0 and np.abs(mu_t - mu_f).mean() < 1.0
        assert np.abs(np.log(s_t / s_f)).max() < 0.2
        d_t = pc.logistic.scales_to_distributions(s_t, default_grid())
        d_f = pc.logistic.scales_to_distributions(s_f, default_grid())
        assert (d_t == d_f).mean() > 0.95


def test_fast_containers_flagged_and_rejected_by_reference(small_model, full_model):
    """Fast-decoder containers carry header flag 0x80: the reference rejects
    them ("unknown header flags", container.py:223-224, restated by the
    oracle) instead of decoding with other numerics; this package decodes
    them with the fast decoder. Models / shapes the fast decoder does not run
    (C != 32) write unflagged, reference-identical containers."""
    img = smooth_images(1, 32, 32, seed=3)[0]
    blob = pc.compress(img, full_model, FAST)
    assert blob[8] & ct.FLAG_FAST_DECODER and ct.inspect(blob)["numerics"] == "fast"
    assert np.array_equal(pc.decompress(blob, full_model), img)
    with pytest.raises(O.OracleError, match="unknown header flags"):
        O.decompress(blob, O.Model.from_bytes(full_model.to_bytes()))
    blob_s = pc.compress(img, small_model, FAST)
    assert blob_s[8] == 0 and blob_s == pc.compress(img, small_model, EXACT)
    # a static container with the flag is malformed
    st = bytearray(pc.compress(img)[:-4])
    st[8] |= ct.FLAG_FAST_DECODER
    st += struct.pack("<I", zlib.crc32(bytes(st)))
    with pytest.raises(FormatError, match="flags"):
        pc.decompress(bytes(st))


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (31, 33), (32, 32), (97, 61)])
def test_vqvae_round_trip(shape, small_model, full_model):
    rng = np.random.default_rng(sum(shape))
    img = rng.integers(0, 256, (*shape, 3), dtype=np.uint8)
    for m in (small_model, full_model):
        for lanes in (1, 4):
            for num in ("exact", "fast"):
                blob = pc.compress(img, m, pc.CodecConfig(backend="twar-vqvae", lanes=lanes, numerics=num))
                assert np.array_equal(pc.decompress(blob, m), img)


def test_fast_bpd_within_half_percent_of_reference(golden, small_model, full_model):
    for tag, m in (("small", small_model), ("full", full_model)):
        z = golden(f"vqvae_{tag}.npz")
        ref = _blobs(z)
        for k in range(int(z["n"])):
            img = z[f"img{k}"]
            blob = pc.compress(img, m, pc.CodecConfig(backend="twar-vqvae", lanes=1 + (k % 3), numerics="fast"))
            assert abs(len(blob) - len(ref[k])) / len(ref[k]) <= 0.005, (tag, k, len(blob), len(ref[k]))
            assert np.array_equal(pc.decompress(blob, m), img)
            assert ct.parse_header(blob)[0].model_hash == ct.parse_header(ref[k])[0].model_hash


@pytest.mark.parametrize("cfg", [EXACT, FAST], ids=["exact", "fast"])
def test_vqvae_batch_independent_of_batch_size(full_model, cfg):
    imgs = smooth_images(19, 32, 32, seed=2)
    buf, off = pc.compress_batch(imgs, full_model, cfg)
    for i in (0, 7, 18):
        assert pc.compress(imgs[i], full_model, cfg) == buf[off[i]:off[i + 1]].tobytes()
    assert np.array_equal(pc.decompress_batch(buf, off, full_model), imgs)


def test_vqvae_other_precisions_and_schedule_check(small_model):
    rng = np.random.default_rng(9)
    img = rng.integers(0, 256, (17, 13, 3), dtype=np.uint8)
    for M in (10, 11, 12):
        blob = pc.compress(img, small_model, pc.CodecConfig(backend="twar-vqvae", M=M, debug_schedule_check=True))
        assert ct.inspect(blob)["M"] == M
        assert ct.parse_header(blob)[0].schedule_checksum is not None
        assert np.array_equal(pc.decompress(blob, small_model), img)


# --- error handling (reference test_container.py:96-178) -----------------------


def test_bad_magic_version_truncation():
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (8, 8, 3), dtype=np.uint8)
    blob = pc.compress(img)
    with pytest.raises(FormatError):
        pc.decompress(b"JUNK" + blob[4:])
    v = bytearray(blob)
    v[4] = 9
    with pytest.raises(FormatError):
        pc.decompress(bytes(v))
    with pytest.raises(FormatError):
        pc.decompress(b"PIL")
    with pytest.raises(CodecError):
        pc.decompress(blob[: len(blob) // 2])
    bad = bytearray(blob)
    bad[-20] ^= 0x10
    with pytest.raises(CorruptStreamError):
        pc.decompress(bytes(bad))


def test_vqvae_needs_model(small_model):
    img = np.random.default_rng(2).integers(0, 256, (8, 8, 3), dtype=np.uint8)
    blob = pc.compress(img, small_model, pc.CodecConfig(backend="twar-vqvae"))
    with pytest.raises(ModelError):
        pc.decompress(blob)
    with pytest.raises(ModelError):
        pc.decompress(blob, pc.random_weights(SMALL, seed=7))
    with pytest.raises(ModelError):
        pc.compress(img, None, pc.CodecConfig(backend="twar-vqvae"))


def test_schedule_checksum_catches_divergence():
    img = np.random.default_rng(3).integers(0, 256, (12, 10, 3), dtype=np.uint8)
    blob = pc.compress(img, None, pc.CodecConfig(debug_schedule_check=True))
    h, _ = ct.parse_header(blob)
    doctored = bytearray(blob[:-4])
    struct.pack_into("<H", doctored, 19, (h.static_d + 1) % h.grid.D)
    doctored += struct.pack("<I", zlib.crc32(bytes(doctored)))
    with pytest.raises(CorruptStreamError, match="schedule"):
        pc.decompress(bytes(doctored))


def test_single_byte_flips_all_detected():
    # acceptance 10 (test_acceptance.py:337-363), a sample of positions
    img = smooth_images(1, 16, 16, seed=4)[0]
    blob = pc.compress(img)
    rng = np.random.default_rng(0)
    flips = []
    for pos in rng.integers(0, len(blob), 200):
        b = bytearray(blob)
        b[pos] ^= 1 << int(rng.integers(0, 8))
        flips.append(bytes(b))
    sizes = np.array([len(b) for b in flips], np.uint64)
    off = np.zeros(len(flips) + 1, np.uint64)
    np.cumsum(sizes, out=off[1:])
    _, errs = pc.decompress_batch(b"".join(flips), off, raise_on_error=False)
    assert len(errs) == len(flips)


def test_batch_status_codes_match_single_errors(small_model):
    rng = np.random.default_rng(4)
    imgs = rng.integers(0, 256, (6, 9, 11, 3), dtype=np.uint8)
    cfg = pc.CodecConfig(backend="twar-vqvae", lanes=2)
    buf, off = pc.compress_batch(imgs, small_model, cfg)
    buf = buf.copy()
    buf[off[2] + 30] ^= 0xFF  # blob 2 crc failure
    out, errs = pc.decompress_batch(buf, off, small_model, raise_on_error=False)
    assert set(errs) == {2} and isinstance(errs[2], CorruptStreamError)
    for i in (0, 1, 3, 4, 5):
        assert np.array_equal(out[i], imgs[i])


def test_large_batch_round_trip(full_model):
    imgs = smooth_images(512, 32, 32, seed=21)
    for cfg in (EXACT, FAST):
        buf, off = pc.compress_batch(imgs, full_model, cfg)
        assert np.array_equal(pc.decompress_batch(buf, off, full_model), imgs)
    bufs, offs = pc.compress_batch(imgs)
    assert np.array_equal(pc.decompress_batch(bufs, offs), imgs)


def test_tcgen05_decoder_deterministic(full_model):
    """Compress and decompress each run the decoder: its (shift, d) planes
    must be bit-identical across calls and batch sizes, or blobs
    would not decode. Batches large enough for every CTA to cycle its
    shared-memory rings several times."""
    from paper_2206_05279_b200.logistic import default_grid

    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 256, (1024, 16, 16), dtype=np.uint8)
    ref = [t.cpu().numpy() for t in vqvae.decode_head_device(torch.from_numpy(idx).to(dev), full_model, 32, 32,
                                                             default_grid(), dev, s, exact=False)]
    for _ in range(2):
        out = [t.cpu().numpy() for t in vqvae.decode_head_device(torch.from_numpy(idx).to(dev), full_model, 32, 32,
                                                                 default_grid(), dev, s, exact=False)]
        assert all(np.array_equal(a, b) for a, b in zip(ref, out))
    sub = [t.cpu().numpy() for t in vqvae.decode_head_device(torch.from_numpy(idx[:3]).to(dev), full_model, 32, 32,
                                                             default_grid(), dev, s, exact=False)]
    assert all(np.array_equal(a[:3], b) for a, b in zip(ref, sub))


def test_frames_as_patch_containers(small_model):
    """BASELINE config 4: frames split into patch containers. Blobs come out
    frame by frame in raster order, byte-identical to compressing the patch
    list, for grids with ragged bottom rows and right columns."""
    from paper_2206_05279_b200 import patches as pt

    cfg = pc.CodecConfig(backend="twar-vqvae")
    for (H, W), (ph, pw) in (((100, 70), (32, 32)), ((64, 128), (64, 64))):
        frames = smooth_images(2, H, W, seed=H + W)
        buf, off = pt.compress_frames(frames, small_model, cfg, ph, pw)
        plist = [p for f in frames for p in pt.split_frame(f, ph, pw)]
        rbuf, roff = pc.compress_batch(plist, small_model, cfg)
        assert np.array_equal(off, roff) and np.array_equal(buf, rbuf)
        out = pt.decompress_frames(buf, off, 2, H, W, small_model, ph, pw)
        assert np.array_equal(out, frames)


def test_indices_equal_reference_on_sample(full_model):
    """Codebook indices of the fast (tcgen05) encoder equal the reference's
    -- the oracle's numpy/BLAS restatement, bit-identical to pixelcodec on
    the same BLAS -- on 192 synthetic images (49152 latents);
    tools/index_parity.py runs larger samples."""
    om = O.Model.from_bytes(full_model.to_bytes())
    imgs = smooth_images(192, 32, 32, seed=123)
    gpu = np.stack([vqvae.encode_to_indices(im, full_model, exact=False) for im in imgs])
    ref = np.stack([O.encode_indices(im, om) for im in imgs])
    assert int((gpu != ref).sum()) == 0


def test_speculative_decode_misses_are_redone(small_model):
    """decompress_batch queues the decode of a batch that looks like the last
    one before its summary is read; a batch of another shape / config, or one
    with a corrupt blob, must still decode exactly / raise exactly."""
    cfg = pc.CodecConfig(backend="twar-vqvae")
    a = smooth_images(24, 32, 32, seed=1)
    b = smooth_images(24, 16, 48, seed=2)
    ba, oa = pc.compress_batch(a, small_model, cfg)
    bb, ob = pc.compress_batch(b, small_model, cfg)
    bs, os_ = pc.compress_batch(a)  # static backend, same shape and count
    for _ in range(2):
        assert np.array_equal(pc.decompress_batch(ba, oa, small_model), a)
        assert np.array_equal(pc.decompress_batch(bb, ob, small_model), b)
        assert np.array_equal(pc.decompress_batch(bs, os_, small_model), a)
    bad = np.array(ba, copy=True)
    bad[int(oa[5]) + 150] ^= 0x04
    with pytest.raises(pc.CodecError):
        pc.decompress_batch(bad, oa, small_model)
    assert np.array_equal(pc.decompress_batch(ba, oa, small_model), a)


def test_trained_model_round_trip_and_vs_oracle():
    """tests/golden/trained.pilw (trainer port, one-code index histogram):
    indices equal the oracle's, containers within 0.5% of the oracle's size,
    batch and single paths lossless -- including odd shapes."""
    m = pc.ModelWeights.load(os.path.join(GOLDEN, "trained.pilw"))
    om = O.Model.from_bytes(m.to_bytes())
    cfg = pc.CodecConfig(backend="twar-vqvae")
    imgs = smooth_images(64, 32, 32, seed=321)
    buf, off = pc.compress_batch(imgs, m, cfg)
    assert np.array_equal(pc.decompress_batch(buf, off, m), imgs)
    for k in range(0, 64, 8):
        assert np.array_equal(vqvae.encode_to_indices(imgs[k], m), O.encode_indices(imgs[k], om))
        ref = O.compress(imgs[k], om, backend="twar-vqvae")
        n = int(off[k + 1] - off[k])
        assert abs(n - len(ref)) / len(ref) <= 0.005, (k, n, len(ref))
    for shape in ((17, 33), (1, 1), (64, 8)):
        img = smooth_images(1, *shape, seed=7)[0]
        blob = pc.compress(img, m, cfg)
        assert np.array_equal(pc.decompress(blob, m), img)


@pytest.mark.parametrize("shape,n", [((32, 32), 301), ((30, 18), 7), ((1, 1), 3), ((17, 33), 5), ((34, 34), 150),
                                     ((33, 2), 9), ((64, 64), 2)])
def test_fused_encoder_blocks_bit_identical(full_model, shape, n):
    """enc_trunk_kernel (every block + the projection, activations in shared
    memory, two images in flight per CTA), tc3_block_kernel (conv1 + conv2 of
    a block, T in shared memory) and two separate tc3 launches per block give
    exactly the same z and indices. n = 301 / 150 leave the CTAs uneven image
    counts (odd and even per-CTA sequences through the two operand buffers)."""
    from paper_2206_05279_b200 import _lib
    from paper_2206_05279_b200.device import as_device_u8, require_device

    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    imgs = smooth_images(n, *shape, seed=606)
    gh, gw = vqvae.latent_shape(*shape)
    img_d = as_device_u8(imgs, dev, stream)
    out = []
    for trunk, fused in ((1, 1), (0, 1), (0, 0)):
        prev_t = _lib.set_tuning(_lib.TUNE_ENC_TRUNK, trunk)
        prev = _lib.set_tuning(_lib.TUNE_BLOCK_FUSION, fused)
        try:
            z = torch.empty((n, gh, gw, 32), dtype=torch.float32, device=dev)
            idx = vqvae.encode_indices_device(img_d, full_model, dev, stream, z_out=z, exact=False)
            out.append((z.cpu().numpy(), idx.cpu().numpy()))
        finally:
            _lib.set_tuning(_lib.TUNE_BLOCK_FUSION, prev)
            _lib.set_tuning(_lib.TUNE_ENC_TRUNK, prev_t)
    z0 = out[0][0]
    assert np.isfinite(z0).all() and np.abs(z0).max() > 0 and len(np.unique(z0)) > z0.size // 4  # a live z
    for o in out[1:]:
        assert np.array_equal(z0.view(np.uint32), o[0].view(np.uint32))
        assert np.array_equal(out[0][1], o[1])


@pytest.mark.parametrize("shape,n", [((32, 32), 301), ((30, 18), 7), ((1, 1), 3), ((17, 33), 5), ((64, 64), 3),
                                     ((34, 34), 10), ((3, 250), 4), ((250, 3), 2)])
def test_decoder_trunk_kernel_bit_identical(full_model, shape, n):
    """dec_trunk2_kernel (activations in pixel pairs, N=64 MMAs with
    zero-weight K chunks) and dec_trunk_kernel (one pixel per MMA row), both
    gather + all block convs with the activations in shared memory, give
    exactly the mu / s / shift / scale index of the per-layer tcgen05 decoder
    -- partial last groups, odd padded widths (an extra even-width column),
    one-pixel-wide grids and the G = 1 (64 x 64) case included."""
    from paper_2206_05279_b200 import _lib
    from paper_2206_05279_b200.device import require_device

    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    H, W = shape
    gh, gw = vqvae.latent_shape(H, W)
    rng = np.random.default_rng(5)
    idx = torch.from_numpy(rng.integers(0, 256, (n, gh, gw), dtype=np.uint8)).to(dev)
    grid = default_grid()
    out = []
    for on in (2, 1, 0):
        prev = _lib.set_tuning(_lib.TUNE_DEC_TRUNK, on)
        try:
            r = vqvae.decode_head_device(idx, full_model, H, W, grid, dev, stream, want_params=True, exact=False)
            out.append([t.cpu().numpy() for t in r])
        finally:
            _lib.set_tuning(_lib.TUNE_DEC_TRUNK, prev)
    assert len(np.unique(out[0][2])) > min(out[0][2].size // 8, 50)  # a live decoder (mu)
    for o in out[1:]:
        for a, b in zip(out[0], o):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("shape,n,D", [((32, 32), 301, 8), ((30, 18), 7, 8), ((1, 1), 3, 8), ((17, 33), 5, 8),
                                       ((34, 34), 150, 8), ((33, 2), 9, 8), ((2, 200), 4, 8), ((64, 64), 2, 8),
                                       ((32, 32), 40, 20), ((18, 30), 6, 1)])
def test_decoder_output_stage_bit_identical(full_model, shape, n, D):
    """dec_uphead_kernel (up conv + pixel shuffle + head of one image per CTA
    iteration, the hi-res activations in shared memory) gives exactly the mu /
    s / shift / scale index of the two launches through HBM (up conv, then
    the pair head); 64 x 64 does not fit its tiles and takes the two launches
    either way. n = 301 / 150 leave the CTAs uneven image counts."""
    from paper_2206_05279_b200 import _lib
    from paper_2206_05279_b200.device import require_device

    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    H, W = shape
    gh, gw = vqvae.latent_shape(H, W)
    rng = np.random.default_rng(11)
    idx = torch.from_numpy(rng.integers(0, 256, (n, gh, gw), dtype=np.uint8)).to(dev)
    grid = default_grid(D)  # D > 9: the head epilogue's threshold loop in shared memory
    out = []
    for on in (1, 0):
        prev = _lib.set_tuning(_lib.TUNE_DEC_UPHEAD, on)
        try:
            r = vqvae.decode_head_device(idx, full_model, H, W, grid, dev, stream, want_params=True, exact=False)
            out.append([t.cpu().numpy() for t in r])
        finally:
            _lib.set_tuning(_lib.TUNE_DEC_UPHEAD, prev)
    mu = out[0][2] if len(out[0]) > 2 else None
    if mu is not None:
        assert np.isfinite(mu).all() and len(np.unique(mu)) > min(mu.size // 8, 50)  # a live decoder
    for a, b in zip(*out):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("K,B", [(97, 2), (256, 1), (13, 3)])
def test_decoder_kernels_other_model_sizes(K, B):
    """The pair decoder trunk (its weight-chunk ring over 2B layers, the
    K-row table) and the output stage on models with other codebook sizes
    and block counts: exactly the per-layer decoder's mu / s / shift / d."""
    from paper_2206_05279_b200 import _lib
    from paper_2206_05279_b200.device import require_device

    model = pc.random_weights(pc.ModelConfig(K=K, Dc=32, channels=32, blocks=B), seed=K + B)
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(K)
    idx = torch.from_numpy(rng.integers(0, K, (50, 16, 16), dtype=np.uint8)).to(dev)
    out = []
    for trunk, uphead in ((2, 1), (0, 0)):
        p1 = _lib.set_tuning(_lib.TUNE_DEC_TRUNK, trunk)
        p2 = _lib.set_tuning(_lib.TUNE_DEC_UPHEAD, uphead)
        try:
            r = vqvae.decode_head_device(idx, model, 32, 32, default_grid(), dev, stream, want_params=True,
                                         exact=False)
            out.append([t.cpu().numpy() for t in r])
        finally:
            _lib.set_tuning(_lib.TUNE_DEC_TRUNK, p1)
            _lib.set_tuning(_lib.TUNE_DEC_UPHEAD, p2)
    for a, b in zip(*out):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_report_rows_in_reference_format():
    """report.run_bench (report.py:47-104 twin): rows carry the reference's
    keys; the GPU coder rows come from a checked round trip."""
    from paper_2206_05279_b200 import report

    rows = report.run_bench(lane_counts=(1, 8), n_symbols=1 << 14, image_hw=(24, 40), batch=16, reps=2)
    assert [r["phase"] for r in rows[:4]] == ["coder-encode-fast", "coder-decode-fast"] * 2
    assert {r["phase"] for r in rows[4:]} == {"model-inference", "ar-decode-parallel", "roundtrip-batch"}
    for r in rows:
        assert set(r) == {"phase", "lanes", "bytes", "seconds", "mb_per_s"} and r["mb_per_s"] > 0


@pytest.mark.parametrize("shape", [(96, 96), (150, 200), (2, 300), (40, 520), (300, 7)])
def test_vqvae_wide_images_round_trip(full_model, shape):
    """Wide images: tcgen05 kernels shrink their copy rings, and shapes whose
    tiles cannot fit shared memory at all run the exact network (a function
    of the shape only; such fast containers are unflagged). Indices stay
    equal to the oracle's."""
    img = smooth_images(1, *shape, seed=17)[0]
    for cfg in (EXACT, FAST):
        blob = pc.compress(img, full_model, cfg)
        assert np.array_equal(pc.decompress(blob, full_model), img)
        assert bool(blob[8] & ct.FLAG_FAST_DECODER) == (cfg is FAST and ct.fast_decoder(full_model, *shape))
        buf, off = pc.compress_batch(np.stack([img, img[::-1].copy()]), full_model, cfg)
        assert np.array_equal(pc.decompress_batch(buf, off, full_model)[0], img)
    om = O.Model.from_bytes(full_model.to_bytes())
    ref = O.encode_indices(img, om)
    assert np.array_equal(vqvae.encode_to_indices(img, full_model, exact=False), ref)
    assert np.array_equal(vqvae.encode_to_indices(img, full_model), ref)


# --- multi-GPU: one process over a device list, and one process per rank -----


@pytest.mark.parametrize("cfg", [None, FAST], ids=["static", "fast"])
def test_devices_list_matches_one_device(full_model, cfg):
    """compress_batch / decompress_batch with devices=[...] (one host thread
    and stream per device, zero-copy rebased outputs; multi.py) give exactly
    the one-device results. On a one-GPU box the list names device 0 three
    times, which exercises the threading and the offset rebasing."""
    n = torch.cuda.device_count()
    devs = [i % n for i in range(3)]
    imgs = smooth_images(37, 32, 32, seed=8)
    model = full_model if cfg is not None else None
    cfg = cfg or pc.CodecConfig()
    buf1, off1 = pc.compress_batch(imgs, model, cfg)
    buf, off = pc.compress_batch(imgs, model, cfg, devices=devs)
    assert np.array_equal(off, off1) and np.array_equal(buf, buf1)
    out = pc.decompress_batch(buf, off, model, devices=devs)
    assert isinstance(out, np.ndarray) and np.array_equal(out, imgs)
    # mixed shapes and a corrupt blob: per-blob errors keep their batch index
    mixed = [smooth_images(1, 9 + i % 3, 7, seed=i)[0] for i in range(7)]
    mb, mo = pc.compress_batch(mixed, model, cfg, devices=devs)
    mb = np.array(mb, copy=True)
    mb[int(mo[4]) + 12] ^= 0x20
    res, errs = pc.decompress_batch(mb, mo, model, devices=devs, raise_on_error=False)
    assert set(errs) == {4}
    assert all(np.array_equal(res[i], mixed[i]) for i in range(7) if i != 4)


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_05279_b200.shard import compress_sharded, decompress_sharded

        torch.cuda.set_device(rank % torch.cuda.device_count())
        model = pc.random_weights(seed=1)
        cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
        imgs = smooth_images(21, 32, 32, seed=12)
        packed = compress_sharded(imgs, model, cfg, dst=0)
        obj = [packed]
        dist.broadcast_object_list(obj, src=0)
        buf, off = obj[0]
        back = decompress_sharded(buf, off, model, dst=0)
        if rank == 0:
            q.put((buf.tobytes(), off.tolist(), back.tobytes()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_sharded_ranks_on_the_gpu_path(full_model):
    """shard.compress_sharded / decompress_sharded: two ranks (processes),
    each on its GPU (both on device 0 on a one-GPU box), the product GPU
    path per rank, results gathered on rank 0 identical to one batch."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    buf, off, back = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    imgs = smooth_images(21, 32, 32, seed=12)
    rb, ro = pc.compress_batch(imgs, full_model, FAST)
    assert buf == rb.tobytes() and off == ro.tolist()
    assert back == imgs.tobytes()


# --- a sharp trained model (tests/golden/sharp.pilw, make_sharp.py) ----------


@pytest.fixture(scope="module")
def sharp_model():
    return pc.ModelWeights.load(os.path.join(GOLDEN, "sharp.pilw"))


def test_sharp_model_exact_matches_reference(golden, sharp_model):
    """With a model that predicts sharply (bpd ~4.9 vs 5.8 static), the exact
    network still reproduces pixelcodec: mu / s bit for bit, containers
    byte-identical, the reference's containers decode exactly."""
    z = golden("vqvae_sharp.npz")
    ref = _blobs(z)
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        mu, s = vqvae.decode_to_params(z[f"idx{k}"], sharp_model, img.shape[:2])
        assert np.array_equal(mu.view(np.uint32), z[f"mu{k}"].view(np.uint32))
        assert np.array_equal(s.view(np.uint32), z[f"s{k}"].view(np.uint32))
        assert pc.compress(img, sharp_model, pc.CodecConfig(backend="twar-vqvae", lanes=1 + (k % 2))) == ref[k]
        assert np.array_equal(pc.decompress(ref[k], sharp_model), img)


@pytest.mark.parametrize("H,n", [(32, 512), (64, 128)])
def test_sharp_model_fast_bpd_within_half_percent(sharp_model, H, n):
    """north_star's float contract where it is sensitive: with sharp (mu, s)
    a wrong recentring shift costs bits, so the bf16 fast decoder's bits/dim
    is compared with the reference arithmetic's (the exact numerics, whose
    containers equal pixelcodec's) on n images: |delta| / bpd <= 0.5%
    (measured: +0.006%)."""
    imgs = smooth_images(n, H, H, seed=91)
    sizes = {}
    for cfg in (EXACT, FAST):
        buf, off = pc.compress_batch(imgs, sharp_model, cfg)
        assert np.array_equal(pc.decompress_batch(buf, off, sharp_model), imgs)
        sizes[cfg.numerics] = float(off[-1])
    rel = (sizes["fast"] - sizes["exact"]) / sizes["exact"]
    assert abs(rel) <= 0.005, rel
    bpd = 8 * sizes["exact"] / imgs.size
    assert bpd < 5.5  # the model is sharp: well below the static backend (~5.8 / 5.5)


def test_full_hd_frame_as_one_container(full_model):
    """A 1920x1080 frame as a single container (no patches): both numerics
    round trip, and the fast container is flagged exactly when the fast
    decoder takes the shape (its tiles must fit shared memory)."""
    frame = smooth_images(1, 1080, 1920, seed=44)[0]
    blobs = {}
    for cfg in (EXACT, FAST):
        blob = pc.compress(frame, full_model, cfg)
        assert np.array_equal(pc.decompress(blob, full_model), frame)
        blobs[cfg.numerics] = blob
    assert bool(blobs["fast"][8] & ct.FLAG_FAST_DECODER) == ct.fast_decoder(full_model, 1080, 1920)
    assert not blobs["exact"][8] & ct.FLAG_FAST_DECODER


def test_edge_cases_of_the_batch_apis(small_model, full_model):
    """Device lists longer than the batch (empty shares), patch-frame offsets
    that do not match the frame count, the reference suite's odd model
    (C = 6, Dc = 4: single-pixel layers outside the modelled sgemv orders run
    the plain chain) on tiny images, and fast numerics with the schedule
    checksum."""
    from paper_2206_05279_b200 import patches as pt

    n = torch.cuda.device_count()
    two = smooth_images(2, 16, 16, seed=3)
    buf, off = pc.compress_batch(two, full_model, FAST, devices=[i % n for i in range(3)])
    assert np.array_equal(pc.decompress_batch(buf, off, full_model, devices=[i % n for i in range(3)]), two)
    frames = smooth_images(1, 70, 90, seed=5)
    fb, fo = pt.compress_frames(frames, small_model, EXACT, 32, 32)
    with pytest.raises(FormatError):
        pt.decompress_frames(fb, fo[:-1], 1, 70, 90, small_model, 32, 32)
    odd = pc.random_weights(pc.ModelConfig(K=16, Dc=4, channels=6, blocks=2), seed=2)
    for shape in ((1, 1), (2, 2), (1, 5), (3, 2)):
        img = np.random.default_rng(sum(shape)).integers(0, 256, (*shape, 3), dtype=np.uint8)
        for cfg in (EXACT, FAST):
            assert np.array_equal(pc.decompress(pc.compress(img, odd, cfg), odd), img)
    img = smooth_images(1, 24, 40, seed=6)[0]
    cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast", debug_schedule_check=True)
    blob = pc.compress(img, full_model, cfg)
    assert blob[8] == (ct.FLAG_FAST_DECODER | ct.FLAG_SCHEDULE_CHECKSUM)
    assert np.array_equal(pc.decompress(blob, full_model), img)


def test_stream_codec_frames_match_sync_calls(full_model):
    """StreamCodec.compress_frames / decompress_frames (patch containers,
    several requests in flight, two patch sizes with ragged edge groups)
    return exactly what patches.compress_frames / decompress_frames return."""
    from paper_2206_05279_b200 import patches as pt
    from paper_2206_05279_b200.stream import StreamCodec

    reqs = [(smooth_images(2, 150, 200, seed=s), 64) for s in range(3)] + [(smooth_images(3, 70, 90, seed=7), 32)]
    with StreamCodec(full_model, FAST) as codec:
        futs = [codec.compress_frames(fr, p, p) for fr, p in reqs]
        packed = [f.result() for f in futs]
        backs = [codec.decompress_frames(buf, off, len(fr), fr.shape[1], fr.shape[2], p, p)
                 for (fr, p), (buf, off) in zip(reqs, packed)]
        for (fr, p), (buf, off), g in zip(reqs, packed, backs):
            rb, ro = pt.compress_frames(fr, full_model, FAST, p, p)
            assert np.array_equal(off, ro) and buf.tobytes() == rb.tobytes()
            assert np.array_equal(g.result(), fr)
        bad = np.array(packed[0][0], copy=True)
        bad[int(packed[0][1][5]) + 40] ^= 0x10
        with pytest.raises(CorruptStreamError):
            codec.decompress_frames(bad, packed[0][1], 2, 150, 200, 64, 64).result()
        assert np.array_equal(codec.decompress_frames(*packed[1], 2, 150, 200, 64, 64).result(), reqs[1][0])


def test_stream_codec_frames_after_other_layouts(full_model, monkeypatch):
    """Frame decodes right after batches with the same blob count but another
    shape, then another M (a decode speculates on the last layout seen for its
    batch size and StreamCodec writes the patches into the frames before the
    guess is checked): the frames come back exact, the early write redone."""
    from paper_2206_05279_b200 import patches as pt
    from paper_2206_05279_b200.stream import StreamCodec

    misses = []
    verify = pt._verify

    def counting(results):
        try:
            verify(results)
        except ct.SpeculationMiss:
            misses.append(1)
            raise

    monkeypatch.setattr(pt, "_verify", counting)

    frames = smooth_images(3, 64, 128, seed=21)  # 32x32 patches: 8 per frame, one shape group of 24 blobs
    other_shape = smooth_images(24, 24, 40, seed=22)
    other_m = smooth_images(24, 32, 32, seed=23)
    m11 = pc.CodecConfig(backend="twar-vqvae", numerics="fast", M=11)
    with StreamCodec(full_model, FAST) as codec, StreamCodec(full_model, m11) as codec11:
        fb, fo = codec.compress_frames(frames, 32, 32).result()
        b, o = codec.compress(other_shape).result()
        assert np.array_equal(codec.decompress(b, o).result(), other_shape)
        assert np.array_equal(codec.decompress_frames(fb, fo, 3, 64, 128, 32, 32).result(), frames)
        b, o = codec11.compress(other_m).result()
        assert np.array_equal(codec11.decompress(b, o).result(), other_m)
        assert np.array_equal(codec.decompress_frames(fb, fo, 3, 64, 128, 32, 32).result(), frames)
        assert np.array_equal(codec.decompress_frames(fb, fo, 3, 64, 128, 32, 32).result(), frames)
    assert len(misses) >= 2  # both layout changes were caught and redone


def test_stream_codec_matches_sync_calls(full_model):
    """StreamCodec (stream.py): pipelined requests (uploads, kernels and
    downloads on separate streams, results as futures) return exactly what
    compress_batch / decompress_batch return, in order, including a corrupt
    request and a request of another shape in between."""
    from paper_2206_05279_b200.stream import StreamCodec

    batches = [smooth_images(300, 32, 32, seed=s) for s in range(4)] + [smooth_images(7, 17, 29, seed=9)]
    with StreamCodec(full_model, FAST) as codec:
        futs = [codec.compress(b) for b in batches]
        packed = [f.result() for f in futs]
        backs = [codec.decompress(buf, off) for buf, off in packed]
        for b, (buf, off), g in zip(batches, packed, backs):
            rb, ro = pc.compress_batch(b, full_model, FAST)
            assert np.array_equal(off, ro) and buf.tobytes() == rb.tobytes()
            assert np.array_equal(g.result(), b)
        bad = np.array(packed[1][0], copy=True)
        bad[int(packed[1][1][3]) + 30] ^= 0x08
        fbad = codec.decompress(bad, packed[1][1])
        fok = codec.decompress(*packed[2])
        with pytest.raises(CorruptStreamError):
            fbad.result()
        assert np.array_equal(fok.result(), batches[2])


def test_stream_codec_exact_numerics_matches_reference(full_model, golden):
    """StreamCodec with the default numerics (the exact network): the
    containers it makes for the reference's own fixture images are the
    reference's bytes (lanes 1..3 as the fixtures were made), requests of
    several codecs in flight at once, and they decode back exactly."""
    from paper_2206_05279_b200.stream import StreamCodec

    z = golden("vqvae_full.npz")
    n = int(z["n"])
    codecs = [StreamCodec(full_model, pc.CodecConfig(backend="twar-vqvae", lanes=1 + j)) for j in range(3)]
    try:
        futs = [codecs[k % 3].compress(z[f"img{k}"][None]) for k in range(n)]
        packed = [f.result() for f in futs]
        backs = [codecs[k % 3].decompress(*packed[k]) for k in range(n)]
        for k in range(n):
            buf, off = packed[k]
            assert buf[off[0]:off[1]].tobytes() == z["buf"][z["offs"][k]: z["offs"][k + 1]].tobytes()
            assert np.array_equal(backs[k].result()[0], z[f"img{k}"])
    finally:
        for c in codecs:
            c.close()


@pytest.mark.parametrize("seed", range(16))
def test_randomized_configs_round_trip_and_oracle(seed, small_model, full_model):
    """Randomised sweep over the container's parameter space: shapes 1..70 x
    1..70 (odd and one-pixel-wide included), batch sizes, backend, numerics,
    M in 10..12, lanes 1..65535 (more lanes than symbols included), smooth
    and noise images, with and without the schedule check. Every batch round
    trips exactly through compress_batch / decompress_batch, and one
    container per batch is compared with the oracle byte for byte (static and
    exact vqvae) or decoded by it (fast: must be rejected, flag 0x80)."""
    rng = np.random.default_rng(1000 + seed)
    oms = {}
    for case in range(8):
        H, W = int(rng.integers(1, 71)), int(rng.integers(1, 71))
        if case == 0:
            H, W = (1, int(rng.integers(1, 71))) if seed % 2 else (int(rng.integers(1, 71)), 1)
        n = int(rng.integers(1, 13))
        backend = "twar-static" if rng.random() < 0.3 else "twar-vqvae"
        numerics = "fast" if rng.random() < 0.5 else "exact"
        M = int(rng.integers(10, 13))
        L = int(rng.choice([1, 2, 3, 7, 64, 1000, 65535]))
        dbg = bool(rng.random() < 0.3)
        model = full_model if rng.random() < 0.5 else small_model
        imgs = (smooth_images(n, H, W, seed=seed * 100 + case) if rng.random() < 0.6
                else rng.integers(0, 256, (n, H, W, 3), dtype=np.uint8))
        cfg = pc.CodecConfig(backend=backend, M=M, lanes=L, numerics=numerics, debug_schedule_check=dbg)
        m = model if backend == "twar-vqvae" else None
        buf, off = pc.compress_batch(imgs, m, cfg)
        back = pc.decompress_batch(buf, off, m)
        assert np.array_equal(back, imgs), (H, W, n, backend, numerics, M, L)
        k = int(rng.integers(0, n))
        blob = buf[off[k]: off[k + 1]].tobytes()
        key = id(model)
        if key not in oms:
            oms[key] = O.Model.from_bytes(model.to_bytes())
        om = oms[key] if backend == "twar-vqvae" else None
        fast_net = backend == "twar-vqvae" and numerics == "fast" and ct.fast_decoder(model, H, W)
        if fast_net:
            assert blob[8] & ct.FLAG_FAST_DECODER
        elif H <= 2 and W <= 2 and backend == "twar-vqvae":
            pass  # single-pixel layers: outside the oracle's stated BLAS orders
        else:
            assert blob == O.compress(imgs[k], om, backend=backend, M=M, L=L, debug_sched=dbg), \
                (H, W, backend, numerics, M, L)


def test_frame_api_edge_cases(small_model):
    """Frame API arguments: zero frames, patch sizes below 1, patches larger
    than the frame (one ragged group), one-pixel frames -- synchronous and
    through StreamCodec."""
    from paper_2206_05279_b200 import patches as pt
    from paper_2206_05279_b200.errors import ParameterError
    from paper_2206_05279_b200.stream import StreamCodec

    empty = np.zeros((0, 20, 30, 3), np.uint8)
    buf, off = pt.compress_frames(empty, small_model, EXACT, 16, 16)
    assert buf.size == 0 and off.tolist() == [0]
    assert pt.decompress_frames(buf, off, 0, 20, 30, small_model, 16, 16).shape == (0, 20, 30, 3)
    with pytest.raises(ParameterError):
        pt.compress_frames(smooth_images(1, 8, 8, seed=1), small_model, EXACT, 0, 8)
    with pytest.raises(ParameterError):
        pt.decompress_frames(buf, off, 0, 20, 30, small_model, 8, -1)
    for shape, p in (((1, 20, 30), 64), ((2, 1, 1), 8), ((1, 9, 70), 4)):
        fr = smooth_images(shape[0], shape[1], shape[2], seed=shape[2])
        b, o = pt.compress_frames(fr, small_model, EXACT, p, p)
        assert np.array_equal(pt.decompress_frames(b, o, shape[0], shape[1], shape[2], small_model, p, p), fr)
    with StreamCodec(small_model, EXACT) as codec:
        b, o = codec.compress_frames(empty, 16, 16).result()
        assert b.size == 0 and codec.decompress_frames(b, o, 0, 20, 30, 16, 16).result().shape == (0, 20, 30, 3)
        with pytest.raises(ParameterError):
            codec.compress_frames(smooth_images(1, 8, 8, seed=1), 8, 0)


@pytest.mark.parametrize("K", [256, 97])
def test_argmin_near_ties(full_model, K):
    """Both argmins -- the float32-screen kernel and the encoders'
    tensor-core one (3xTF32 screen + proven error radius + exact float64
    rescore) -- against the reference's float64 argmin on adversarial
    latents: duplicated codes (exact ties: the lower code wins), codes one
    ulp apart, latents on the midpoints between code pairs (plus noise well
    inside the screen's error radius), and large-magnitude latents."""
    rng = np.random.default_rng(K)
    cb = rng.normal(0, 1, (K, 32)).astype(np.float32)
    cb[K // 2] = cb[K // 3]                                      # exact duplicate
    cb[K // 4] = cb[K // 5]
    cb[K - 1] = cb[7]
    cb[K - 2] = np.nextafter(cb[11], np.float32(np.inf))         # one ulp apart, every component
    cb[K - 3] = cb[13]
    cb[K - 3, 5] = np.nextafter(cb[13, 5], np.float32(-np.inf))  # one ulp apart, one component
    cfg = pc.ModelConfig(K=K, Dc=32, channels=32, blocks=full_model.config.blocks)
    tensors = dict(full_model.tensors) if K == full_model.config.K else \
        {k: v for k, v in pc.random_weights(cfg, seed=3).tensors.items()}
    tensors["codebook"] = cb
    m = pc.ModelWeights(cfg, tensors)
    a, b = rng.integers(0, K, 6000), rng.integers(0, K, 6000)
    mid = 0.5 * (cb[a].astype(np.float64) + cb[b].astype(np.float64))
    z = [mid.astype(np.float32),                                          # midpoints
         (mid + rng.normal(0, 1e-6, mid.shape)).astype(np.float32),       # near them
         cb[rng.integers(0, K, 2000)],                                    # on codes (duplicates included)
         (cb[rng.integers(0, K, 2000)] + rng.normal(0, 1e-7, (2000, 32))).astype(np.float32),
         (1e3 * rng.normal(0, 1, (2000, 32))).astype(np.float32)]         # far from every code
    z = np.concatenate(z).reshape(-1, 8, 32)
    ref = O.argmin_codebook(z, cb)
    assert np.array_equal(vqvae.argmin_codebook(z, m), ref)
    assert np.array_equal(vqvae.argmin_codebook(z, m, tensor_cores=True), ref)  # the encoders' argmin


def test_concurrent_host_threads_one_device(full_model, small_model):
    """Host threads driving one GPU at once (each on its own stream, with
    different image shapes, models and numerics, so the same kernels launch
    concurrently with different shared-memory sizes): every result equals
    the single-threaded one. (Per-launch shared-memory attributes used to
    race here: one thread's setting undercut another's launch.)"""
    from concurrent.futures import ThreadPoolExecutor

    jobs = []
    for j in range(8):
        shape = [(32, 32), (17, 29), (64, 64), (40, 24)][j % 4]
        m = full_model if j % 3 else small_model
        cfg = EXACT if j % 2 else FAST
        jobs.append((smooth_images(6 + j, *shape, seed=70 + j), m, cfg))
    want = [pc.compress_batch(im, m, cfg) for im, m, cfg in jobs]
    dev = torch.device("cuda", 0)

    def run(job):
        im, m, cfg = job
        with torch.cuda.stream(torch.cuda.Stream(dev)):
            outs = []
            for _ in range(3):
                buf, off = pc.compress_batch(im, m, cfg)
                outs.append((buf.tobytes(), off.copy(), pc.decompress_batch(buf, off, m)))
            return outs

    with ThreadPoolExecutor(max_workers=8) as ex:
        got = list(ex.map(run, jobs))
    for (im, _, _), (wb, wo), outs in zip(jobs, want, got):
        for buf, off, back in outs:
            assert buf == wb.tobytes() and np.array_equal(off, wo)
            assert np.array_equal(back, im)
