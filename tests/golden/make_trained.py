"""Generate tests/golden/trained.pilw: the full model (K256 Dc32 C32 B4)
briefly trained by paper_2206_05279_b200.trainer (the port of the reference's
pkg/trainer) on 1000 synthetic 32x32 smooth images.

    python tests/golden/make_trained.py

Targets come from the oracle's predictor (bit-identical to the codec's GPU
predictor, so this runs on a CPU-only box). Settings: the reference defaults
(alpha 125, beta 0.25, lr 1e-3, batch 8, seed 0) except steps=600 and
init_scale=0.3 -- with model.ts's He-normal init at full scale the mu/s heads
start saturated past their clips (zero gradient) and the model never leaves
s = 64. Like the reference trainer at these settings, the codebook collapses
onto a single code, so the file also pins the codec on a one-symbol index
histogram.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2206_05279_b200 import trainer  # noqa: E402

if __name__ == "__main__":
    torch.set_num_threads(1)
    torch.manual_seed(0)
    w, losses = trainer.train(steps=600, batch=8, init_scale=0.3, device="cpu",
                              residual_fn=oracle.twar_forward, log_every=100)
    out = os.path.join(HERE, "trained.pilw")
    w.save(out)
    print(f"{out}: final loss {losses[-1]:.4f}, codes used {(w.histogram > 0).sum()}, hash8 {w.hash8().hex()}")
