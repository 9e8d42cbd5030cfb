"""Pin the CPU oracle to the reference's own outputs (tests/golden/)."""

import hashlib
import json
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLDEN, "meta.json")) as f:
        return json.load(f)


def _blobs(z):
    buf, offs = z["buf"], z["offs"]
    return [buf[offs[i]: offs[i + 1]].tobytes() for i in range(len(offs) - 1)]


@pytest.mark.parametrize("M", [10, 11, 12])
def test_tables_match_reference(golden, meta, M):
    t = golden("tables.npz")
    P = O.residual_pmfs(O.default_grid(), M)
    assert np.array_equal(P, t[f"P_M{M}"])
    delta, phi, sym, pop, nxt = O.build_tables(P, M)
    for a, k in ((delta, "delta"), (phi, "phi"), (sym, "symbol"), (pop, "pop"), (nxt, "next")):
        assert np.array_equal(a, t[f"{k}_M{M}"]), k
    h = hashlib.sha256()
    for a in (delta, phi, sym, pop, nxt):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest()[:16] == meta[f"table_digest_M{M}"]


def test_golden_pmf_center_masses(golden):
    # P[128] at M=12 for d=0..7
    P = golden("tables.npz")["P_M12"]
    assert list(P[:, 128]) == [1647, 788, 415, 213, 111, 59, 32, 16]


@pytest.mark.parametrize("L", [1, 3, 16, 64])
def test_lanes_byte_identical(golden, L):
    z = golden("lanes.npz")
    t = golden("tables.npz")
    delta, phi = t["delta_M12"], t["phi_M12"]
    blobs, states = O.encode_lanes(z["syms"], z["d"], L, delta, phi, 12)
    ref = [z[f"L{L}_buf"][z[f"L{L}_offs"][i]: z[f"L{L}_offs"][i + 1]].tobytes() for i in range(L)]
    assert blobs == ref
    assert states == list(z[f"L{L}_states"])
    back = O.decode_lanes(blobs, states, z["syms"].size, z["d"], t["symbol_M12"], t["pop_M12"], t["next_M12"], 12)
    assert np.array_equal(back, z["syms"])


def test_twar_matches_reference(golden):
    z = golden("twar.npz")
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        res = O.twar_forward(img, z[f"w{k}"], z[f"b{k}"])
        assert np.array_equal(res, z[f"res{k}"])
        assert np.array_equal(O.twar_forward(img), z[f"resdef{k}"])
        assert np.array_equal(O.twar_decode(res, z[f"w{k}"], z[f"b{k}"]), img)


def test_params_hash(meta):
    assert O.params_hash8(O.DEFAULT_W, O.DEFAULT_B).hex() == meta["default_params_hash8"] == "0e27be90fd4a910b"


def test_static_containers_byte_identical(golden):
    z = golden("static.npz")
    blobs = _blobs(z)
    for blob, ci, (L, M, dbg) in zip(blobs, z["img_index"], z["cfg"]):
        img = z[f"img{ci}"]
        mine = O.compress(img, None, "twar-static", int(M), int(L), None, bool(dbg))
        assert mine == blob
        assert np.array_equal(O.decompress(blob), img)


def test_fitted_params_container(golden):
    z = golden("static.npz")
    m = O.Model((256, 32, 32, 4), {}, None, z["fit_w"], z["fit_b"])
    blob = z["fit_blob"].tobytes()
    assert O.compress(z["img9"], m) == blob
    assert np.array_equal(O.decompress(blob, m), z["img9"])


def test_model_files(golden, meta):
    small = O.Model.from_bytes(golden("small.pilw"))
    assert small.hash8().hex() == meta["small_hash8"]
    assert small.to_bytes() == golden("small.pilw")
    assert O.random_model(32, 8, 8, 1, seed=42).to_bytes() == golden("small.pilw")
    assert O.random_model(seed=1).hash8().hex() == meta["full_seed1_hash8"] == "7c4b307f421f97a8"


@pytest.mark.parametrize("tag", ["small", "full"])
def test_vqvae_matches_reference(golden, tag):
    z = golden(f"vqvae_{tag}.npz")
    m = O.Model.from_bytes(golden("small.pilw")) if tag == "small" else O.random_model(seed=1)
    blobs = _blobs(z)
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        lat = O.encoder_latents(img, m)
        np.testing.assert_allclose(lat, z[f"z{k}"], rtol=0, atol=1e-5)
        assert np.array_equal(O.argmin_codebook(z[f"z{k}"], m.t["codebook"]), z[f"idx{k}"])
        idx = O.encode_indices(img, m)
        assert np.array_equal(idx, z[f"idx{k}"])
        mu, s = O.decode_params(idx, m, *img.shape[:2])
        assert np.array_equal(mu, z[f"mu{k}"]) and np.array_equal(s, z[f"s{k}"])
        L = 1 + (k % 3)
        assert O.compress(img, m, "twar-vqvae", 12, L) == blobs[k]
        assert np.array_equal(O.decompress(blobs[k], m), img)


def test_bits_golden(meta):
    # bits.py wire form: push 1,0,1,1 -> 4-bit count + 0x0D (test_bits.py:31-36)
    blob = struct.pack("<Q", 4) + bytes([0b1101])
    assert list(blob) == meta["bits_golden"]


def test_corruption_detected(golden):
    z = golden("static.npz")
    blob = bytearray(_blobs(z)[12])
    blob[-20] ^= 0x10
    with pytest.raises(O.OracleError) as e:
        O.decompress(bytes(blob))
    assert e.value.kind == "CorruptStreamError"


# --- the explicit statement of the reference's float arithmetic ---------------
# (oracle_conv_fma / oracle_expf_np: what the GPU exact network implements)


@pytest.mark.parametrize("tag", ["small", "full"])
def test_fma_statement_reproduces_reference_network(golden, tag):
    """The reference's own z, mu, s (tests/golden, made by pixelcodec) equal
    the explicit FMA-chain / sgemv / m-tail / numpy-exp statement bit for bit."""
    import paper_2206_05279_b200 as pc

    z = golden(f"vqvae_{tag}.npz")
    if tag == "small":
        m = O.Model.from_bytes(golden("small.pilw"))
    else:
        m = O.Model.from_bytes(pc.random_weights(pc.ModelConfig(), seed=1).to_bytes())
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        H, W = img.shape[:2]
        assert np.array_equal(O.encoder_latents_exact(img, m).view(np.uint32), z[f"z{k}"].view(np.uint32))
        mu, s = O.decode_params_exact(z[f"idx{k}"], m, H, W)
        assert np.array_equal(mu.view(np.uint32), z[f"mu{k}"].view(np.uint32))
        assert np.array_equal(s.view(np.uint32), z[f"s{k}"].view(np.uint32))


def test_conv_statement_matches_numpy_blas():
    """oracle_conv_fma against the reference's nn.conv2d arithmetic (numpy +
    OpenBLAS, restated op for op by O.conv2d) on random layers of every shape
    class: plain, m-tail (1..8 leftover pixels, Ci >= 32), single pixel."""
    rng = np.random.default_rng(5)
    checked = 0
    for ci, co in ((3, 32), (8, 8), (32, 32), (32, 128), (32, 3), (8, 3), (40, 16)):
        for H, W in ((1, 1), (1, 2), (2, 2), (1, 7), (3, 3), (4, 5), (6, 11), (9, 7), (16, 17), (2, 14)):
            for ks, st in ((3, 1), (3, 2), (1, 1)):
                x = rng.standard_normal((ci, H, W)).astype(np.float32)
                w = rng.standard_normal((co, ci, ks, ks)).astype(np.float32)
                b = rng.standard_normal(co).astype(np.float32)
                try:
                    got = O.conv2d_fma(x, w, b, st)
                except NotImplementedError:
                    continue
                assert np.array_equal(got.view(np.uint32), O.conv2d(x, w, b, st).view(np.uint32)), (ci, co, H, W, ks, st)
                checked += 1
    assert checked > 150


@pytest.mark.parametrize("lo,hi", [(-15.0, 15.0), (float(np.float32(np.log(0.5))), float(np.float32(np.log(64.0))))])
def test_exp_statement_matches_numpy(lo, hi):
    """oracle_expf_np equals np.exp (float32) on the head's input ranges:
    every float32 in [lo, hi] at a stride of 61 bit patterns (~3.5e7 values)."""
    def f32_range(a, b):
        # float32 bit patterns of [a, b] (sign-magnitude: handle each sign)
        out = []
        a32, b32 = np.float32(a), np.float32(b)
        if a32 < 0:
            top = np.array([-a32], np.float32).view(np.uint32)[0]
            lo_b = np.array([max(0.0, -b32)], np.float32).view(np.uint32)[0] if b32 < 0 else 0
            out.append((np.arange(lo_b, top + 1, 61, dtype=np.uint32) | np.uint32(0x80000000)).view(np.float32))
        if b32 >= 0:
            lo_b = np.array([max(0.0, a32)], np.float32).view(np.uint32)[0]
            top = np.array([b32], np.float32).view(np.uint32)[0]
            out.append(np.arange(lo_b, top + 1, 61, dtype=np.uint32).view(np.float32))
        return np.concatenate(out)

    x = f32_range(lo, hi)
    assert np.array_equal(O.exp_np(x).view(np.uint32), np.exp(x).view(np.uint32))


def test_fma_statement_reproduces_reference_sharp_model(golden):
    """The same pin on the trained sharp model (tests/golden/sharp.pilw):
    the reference's mu and s equal the explicit statement bit for bit."""
    m = O.Model.from_bytes(golden("sharp.pilw"))
    z = golden("vqvae_sharp.npz")
    for k in range(int(z["n"])):
        img = z[f"img{k}"]
        H, W = img.shape[:2]
        assert np.array_equal(O.encode_indices(img, m), z[f"idx{k}"])
        mu, s = O.decode_params_exact(z[f"idx{k}"], m, H, W)
        assert np.array_equal(mu.view(np.uint32), z[f"mu{k}"].view(np.uint32))
        assert np.array_equal(s.view(np.uint32), z[f"s{k}"].view(np.uint32))
