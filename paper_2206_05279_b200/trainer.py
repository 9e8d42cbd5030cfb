"""Briefly train a PILC model on synthetic data and export it as PILW.

PyTorch port of the reference trainer's objective and loop
(`pkg/trainer/src/{model,losses,train}.ts`, tfjs in the reference; SURVEY
§8f rank 4): the same graph as the codec's inference network (edge-replicate
padded 3x3 convolutions, one stride-2 stage, residual blocks, pixel shuffle
with channel order c*4 + dy*2 + dx, mu = 255 sigmoid(clip(a, +-15)),
s = clip(exp(clip(b, ln 0.5, ln 64)), 0.5, 64)), trained on

    nll_bits(t; mu, s) + alpha * (||sg(z) - zq||^2 + beta ||z - sg(zq)||^2)

with a straight-through quantizer (losses.ts:18-48, model.ts:130-150), where
t is the fixed-predictor residual of the image (predictor.forward_residual)
and the logistic bins have tail-absorbing edges at 0 and 255. Adam, the
reference's defaults (config.ts: alpha 125, beta 0.25, lr 1e-3). The index
histogram over one full pass goes into the PILW file (train.ts:96-112), so
the codec's index stream PMF matches the trained model.

This is offline tooling, not the codec's hot path: the network runs in
torch (cuDNN where available). The exported file is the contract; the codec
and the oracle read it unchanged.

    python -m paper_2206_05279_b200.trainer --steps 400 --batch 32 --out model.pilw
"""

from __future__ import annotations

import argparse
import math

import numpy as np
import torch
import torch.nn.functional as F

from .predictor import default_params, forward_residual
from .synth import mulberry32, smooth_images
from .weights import ModelConfig, ModelWeights, random_weights, tensor_shapes

MU_LOGIT_LIMIT = 15.0
LOG_S_MIN = float(np.float32(math.log(0.5)))
LOG_S_MAX = float(np.float32(math.log(64.0)))
LOG2E = 1.0 / math.log(2.0)


def _conv(x, p, name, stride=1):
    w, b = p[f"{name}.w"], p[f"{name}.b"]
    if w.shape[-1] == 3:
        x = F.pad(x, (1, 1, 1, 1), mode="replicate")  # nn.py edge padding
    return F.conv2d(x, w, b, stride=stride)


def _block(x, p, name):
    h = F.relu(_conv(x, p, f"{name}.conv1"))
    return F.relu(x + _conv(h, p, f"{name}.conv2"))


def encode(images: torch.Tensor, p: dict, blocks: int) -> torch.Tensor:
    """(B, 3, H, W) pixel values -> latent (B, Dc, ceil(H/2), ceil(W/2))."""
    x = images / 127.5 - 1.0
    H, W = x.shape[-2:]
    if H % 2 or W % 2:  # _even_pad
        x = F.pad(x, (0, W % 2, 0, H % 2), mode="replicate")
    h = F.relu(_conv(x, p, "enc.stem"))
    h = F.relu(_conv(h, p, "enc.down", stride=2))
    for i in range(blocks):
        h = _block(h, p, f"enc.block{i}")
    return _conv(h, p, "enc.proj")


def quantize(z: torch.Tensor, codebook: torch.Tensor):
    """Nearest code per latent (indices detached), zq and the straight-through latent."""
    B, Dc, h, w = z.shape
    flat = z.permute(0, 2, 3, 1).reshape(-1, Dc)
    with torch.no_grad():
        d = (flat * flat).sum(1, keepdim=True) + (codebook * codebook).sum(1)[None] - 2 * flat @ codebook.T
        idx = d.argmin(1)
    zq = codebook[idx].reshape(B, h, w, Dc).permute(0, 3, 1, 2)
    return idx.reshape(B, h, w), zq, z + (zq - z).detach()


def decode(z: torch.Tensor, p: dict, blocks: int, H: int, W: int):
    h = F.relu(_conv(z, p, "dec.proj"))
    for i in range(blocks):
        h = _block(h, p, f"dec.block{i}")
    u = F.relu(F.pixel_shuffle(_conv(h, p, "dec.up"), 2))  # channel c*4 + dy*2 + dx -> (dy, dx)
    a = torch.clamp(_conv(u, p, "dec.mu"), -MU_LOGIT_LIMIT, MU_LOGIT_LIMIT)
    mu = 255.0 * torch.sigmoid(a)
    s = torch.clamp(torch.exp(torch.clamp(_conv(u, p, "dec.s"), LOG_S_MIN, LOG_S_MAX)), 0.5, 64.0)
    return mu[..., :H, :W], s[..., :H, :W]


def nll_bits(t: torch.Tensor, mu: torch.Tensor, s: torch.Tensor) -> torch.Tensor:
    """Mean bits per value of integer targets t under logistic(mu, s) with unit
    bins and tail-absorbing edges at 0 and 255 (losses.ts:18-32)."""
    z_up = (t + 0.5 - mu) / s
    z_lo = (t - 0.5 - mu) / s
    mass = torch.sigmoid(z_up) - torch.sigmoid(z_lo)
    mass = torch.where(t == 0, torch.sigmoid(z_up), mass)
    mass = torch.where(t == 255, torch.sigmoid(-z_lo), mass)
    return -LOG2E * torch.log(torch.clamp(mass, min=1e-12)).mean()


def vq_loss(z: torch.Tensor, zq: torch.Tensor, beta: float) -> torch.Tensor:
    return ((z.detach() - zq) ** 2).mean() + beta * ((z - zq.detach()) ** 2).mean()


def train(config: ModelConfig = ModelConfig(), steps: int = 200, batch: int = 8, dataset: int = 1000,
          size: int = 32, lr: float = 1e-3, alpha: float = 125.0, beta: float = 0.25, seed: int = 0,
          device=None, log_every: int = 0, residual_fn=None,
          init_scale: float = 1.0, restart_every: int = 0, data_init: bool = False) -> tuple[ModelWeights, list]:
    """Train on `dataset` synthetic smooth images of size x size; returns the
    weights (with the index histogram of one full pass) and the loss curve.

    `residual_fn(images (N, H, W, 3) uint8) -> (N, H, W, 3) uint8` makes the
    targets; default: the codec's own GPU predictor kernel. `init_scale`
    multiplies the He-normal std of the convolutions (1.0 = model.ts:75-80).

    Against codebook collapse (the reference trainer's failure mode at these
    settings: every latent maps to one code) two standard VQ-VAE remedies,
    off by default so the default run is the reference's: `data_init` sets
    the codebook to encoder outputs of the first batch, and every
    `restart_every` steps codes unused since the last restart are moved onto
    randomly chosen current encoder outputs (dead-code restart)."""
    dev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    init = random_weights(config, seed=seed, scale=init_scale)
    p = {k: torch.tensor(v, device=dev, requires_grad=True) for k, v in init.tensors.items()}
    imgs = smooth_images(dataset, size, size, seed=seed)
    res = np.asarray((residual_fn or (lambda x: forward_residual(x, default_params())))(imgs), np.uint8)
    x_all = torch.tensor(imgs, dtype=torch.float32, device=dev).permute(0, 3, 1, 2)
    t_all = torch.tensor(res, dtype=torch.float32, device=dev).permute(0, 3, 1, 2)
    opt = torch.optim.Adam(list(p.values()), lr=lr)
    # train.ts:61-64: batch picks floor(rng(seed + 1)() * n), drawn in order
    picks = np.floor(mulberry32(seed + 1, 0, steps * batch) * dataset).astype(np.int64).reshape(steps, batch)
    B = config.blocks
    losses = []
    gen = torch.Generator(device="cpu").manual_seed(seed + 2)
    used = torch.zeros(config.K, dtype=torch.bool, device=dev)

    def sample_latents(z, k):
        flat = z.detach().permute(0, 2, 3, 1).reshape(-1, z.shape[1])
        sel = torch.randint(0, flat.shape[0], (k,), generator=gen).to(dev)
        return flat[sel]

    for step in range(steps):
        pick = torch.from_numpy(picks[step]).to(dev)
        x, t = x_all[pick], t_all[pick]
        z = encode(x, p, B)
        if data_init and step == 0:
            with torch.no_grad():
                p["codebook"].copy_(sample_latents(z, config.K))
        idx, zq, zst = quantize(z, p["codebook"])
        if restart_every:
            used[idx.reshape(-1).unique()] = True
            if step % restart_every == restart_every - 1:
                dead = (~used).nonzero().reshape(-1)
                if dead.numel():
                    with torch.no_grad():
                        p["codebook"][dead] = sample_latents(z, dead.numel())
                    opt.state.pop(p["codebook"], None)  # fresh Adam moments for the moved codes
                used.zero_()
        mu, s = decode(zst, p, B, size, size)
        loss = nll_bits(t, mu, s) + alpha * vq_loss(z, zq, beta)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        v = float(loss.detach())
        if not math.isfinite(v):
            raise RuntimeError(f"training diverged at step {step}")
        losses.append(v)
        if log_every and step % log_every == 0:
            print(f"step {step:5d}  loss {v:.4f}")
    hist = np.zeros(config.K, np.uint64)
    with torch.no_grad():
        for i in range(0, dataset, 256):
            idx, _, _ = quantize(encode(x_all[i:i + 256], p, B), p["codebook"])
            hist += np.bincount(idx.reshape(-1).cpu().numpy(), minlength=config.K).astype(np.uint64)
    tensors = {k: p[k].detach().cpu().numpy().astype(np.float32).reshape(shape)
               for k, shape in tensor_shapes(config).items()}
    return ModelWeights(config, tensors, histogram=hist), losses


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--dataset", type=int, default=1000)
    ap.add_argument("--size", type=int, default=32)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--alpha", type=float, default=125.0)
    ap.add_argument("--beta", type=float, default=0.25)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--restart-every", type=int, default=0, help="dead-code restart period (0: off)")
    ap.add_argument("--data-init", action="store_true", help="codebook from the first batch's latents")
    ap.add_argument("--init-scale", type=float, default=1.0)
    ap.add_argument("--out", default="model.pilw")
    ap.add_argument("--log-every", type=int, default=50)
    a = ap.parse_args(argv)
    w, losses = train(steps=a.steps, batch=a.batch, dataset=a.dataset, size=a.size, lr=a.lr, alpha=a.alpha,
                      beta=a.beta, seed=a.seed, log_every=a.log_every, restart_every=a.restart_every,
                      data_init=a.data_init, init_scale=a.init_scale)
    w.save(a.out)
    print(f"saved {a.out}: final loss {losses[-1]:.4f}, hash8 {w.hash8().hex()}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
