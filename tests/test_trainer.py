"""Trainer port (paper_2206_05279_b200/trainer.py <- pkg/trainer/src): its
graph is the codec's graph (checked against the oracle's inference network),
its loss is the codec's bin convention, and what it exports is a PILW file
the codec and the oracle read unchanged."""

import hashlib
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2206_05279_b200 import trainer as T
from paper_2206_05279_b200.synth import smooth_images
from paper_2206_05279_b200.weights import ModelConfig, ModelWeights, random_weights

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _params(w: ModelWeights):
    return {k: torch.tensor(v, dtype=torch.float64) for k, v in w.tensors.items()}


@pytest.mark.parametrize("shape", [(16, 16), (15, 9)])
def test_trainer_graph_equals_codec_graph(shape):
    """encode/quantize/decode of the trainer == oracle encoder_latents /
    argmin_codebook / decode_params (vqvae.py:51-113), odd sizes included."""
    H, W = shape
    w = random_weights(ModelConfig(32, 8, 8, 2), seed=3, scale=0.5)
    om = O.Model.from_bytes(w.to_bytes())
    imgs = smooth_images(2, H, W, seed=11)
    p = _params(w)
    x = torch.tensor(imgs, dtype=torch.float64).permute(0, 3, 1, 2)
    z = T.encode(x, p, 2)
    idx, zq, zst = T.quantize(z, p["codebook"])
    mu, s = T.decode(zst, p, 2, H, W)
    for n in range(2):
        z_ref = O.encoder_latents(imgs[n], om)
        np.testing.assert_allclose(z[n].permute(1, 2, 0).numpy(), z_ref, rtol=1e-4, atol=1e-4)
        idx_ref = O.argmin_codebook(z_ref, om.t["codebook"])
        assert (idx[n].numpy() == idx_ref).mean() > 0.99
        mu_ref, s_ref = O.decode_params(idx[n].numpy(), om, H, W)
        np.testing.assert_allclose(mu[n].permute(1, 2, 0).numpy(), mu_ref, rtol=1e-4, atol=1e-3)
        np.testing.assert_allclose(s[n].permute(1, 2, 0).numpy(), s_ref, rtol=1e-4, atol=1e-4)
    # straight-through: forward value is zq, gradient flows to z
    np.testing.assert_allclose(zst.detach().numpy(), zq.detach().numpy(), atol=1e-12)


def test_nll_bits_uses_codec_bins():
    """losses.ts:18-32 == -log2 of the codec's logistic bin masses
    (logistic.py, tail bins at 0 and 255)."""
    rng = np.random.default_rng(0)
    t = np.concatenate([[0, 255, 0, 255], rng.integers(0, 256, 60)]).astype(np.float64)
    mu = rng.uniform(0, 255, t.size)
    s = rng.uniform(0.5, 64, t.size)
    got = T.nll_bits(torch.tensor(t), torch.tensor(mu), torch.tensor(s)).item()
    ref = np.mean([-np.log2(max(O.logistic_masses(m, sc)[int(v)], 1e-12)) for v, m, sc in zip(t, mu, s)])
    assert abs(got - ref) < 1e-9 * max(1.0, ref)


def test_vq_loss_gradients_are_split():
    """codebook term trains zq only, commitment term (x beta) trains z only."""
    z = torch.randn(2, 4, 3, 3, dtype=torch.float64, requires_grad=True)
    zq = torch.randn(2, 4, 3, 3, dtype=torch.float64, requires_grad=True)
    T.vq_loss(z, zq, 0.25).backward()
    n = z.numel()
    torch.testing.assert_close(z.grad, 0.25 * 2 * (z - zq).detach() / n)
    torch.testing.assert_close(zq.grad, 2 * (zq - z).detach() / n)


def test_short_training_run_exports_a_working_model():
    cfg = ModelConfig(16, 8, 8, 1)
    torch.manual_seed(0)
    w, losses = T.train(cfg, steps=40, batch=4, dataset=24, size=16, init_scale=0.3, device="cpu",
                        residual_fn=O.twar_forward)
    assert len(losses) == 40 and all(np.isfinite(losses))
    assert np.mean(losses[-5:]) < np.mean(losses[:5])
    assert int(w.histogram.sum()) == 24 * 8 * 8  # one full pass, every latent counted
    back = ModelWeights.from_bytes(w.to_bytes())
    assert back.hash8() == w.hash8() and back.config == cfg
    om = O.Model.from_bytes(w.to_bytes())
    for img in smooth_images(2, 16, 16, seed=99):
        blob = O.compress(img, om, backend="twar-vqvae")
        np.testing.assert_array_equal(O.decompress(blob, om), img)


def test_batch_picks_follow_reference_rng():
    """train.ts:61-64 picks floor(rng(seed+1)() * n); mulberry32 data.ts:17-25."""
    from paper_2206_05279_b200.synth import mulberry32

    def ref_rng(seed):
        a = seed & 0xFFFFFFFF
        while True:
            a = (a + 0x6D2B79F5) & 0xFFFFFFFF
            t = ((a ^ (a >> 15)) * (1 | a)) & 0xFFFFFFFF
            t = ((t + (((t ^ (t >> 7)) * (61 | t)) & 0xFFFFFFFF)) & 0xFFFFFFFF) ^ t
            yield ((t ^ (t >> 14)) & 0xFFFFFFFF) / 4294967296

    g = ref_rng(1)
    ref = [int(next(g) * 1000) for _ in range(50)]
    got = np.floor(mulberry32(1, 0, 50) * 1000).astype(int).tolist()
    assert got == ref


def test_trained_fixture():
    """tests/golden/trained.pilw (make_trained.py): full config, a one-code
    index histogram (the collapse the reference objective shows)."""
    data = open(os.path.join(GOLDEN, "trained.pilw"), "rb").read()
    w = ModelWeights.from_bytes(data)
    assert w.config == ModelConfig()
    assert hashlib.sha256(data[:-8]).digest()[:8] == data[-8:]
    assert int((w.histogram > 0).sum()) == 1
    assert int(w.histogram.sum()) == 1000 * 16 * 16
