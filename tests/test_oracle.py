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
