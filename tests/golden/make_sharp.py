"""Generate tests/golden/sharp.pilw: the full model (K256 Dc32 C32 B4)
trained by paper_2206_05279_b200.trainer long enough to make sharp (mu, s)
predictions, with the codebook kept alive (data init + dead-code restarts;
the reference trainer's settings collapse onto one code, see
make_trained.py). It is the model that stresses the fast decoder's bits/dim
against the reference's arithmetic (tests/test_gpu_codec.py).

    python tests/golden/make_sharp.py [out.pilw]     (on a GPU box; ~minutes)

Settings: the reference defaults (alpha 125, beta 0.25, lr 1e-3, seed 0)
with batch 64, 4000 steps, init_scale 0.3, data_init, restart_every 100, on
4000 synthetic 32x32 smooth images; targets from the codec's own GPU TWAR
predictor.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_05279_b200 import trainer  # noqa: E402

if __name__ == "__main__":
    torch.manual_seed(0)
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "sharp.pilw")
    w, losses = trainer.train(steps=4000, batch=64, dataset=4000, init_scale=0.3, data_init=True,
                              restart_every=100, log_every=500)
    w.save(out)
    used = int((w.histogram > 0).sum())
    print(f"{out}: final loss {np.mean(losses[-100:]):.4f} bits (+vq), codes used {used}, hash8 {w.hash8().hex()}")
