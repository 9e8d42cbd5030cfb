"""Quick numerical check of the tcgen05 decoder against the fp32 SIMT decoder."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.synth import smooth_images
m = pc.random_weights(seed=1)
rng = np.random.default_rng(0)
for (H, W) in [(32, 32), (17, 13), (64, 64), (1, 1)]:
    idx = rng.integers(0, 256, ((H + 1) // 2, (W + 1) // 2)).astype(np.uint8)
    t0 = time.time()
    mu_t, s_t = vqvae.decode_to_params(idx, m, (H, W))
    torch.cuda.synchronize()
    mu_f, s_f = vqvae.decode_to_params(idx, m, (H, W), precise=True)
    print(H, W, "max|dmu|", float(np.abs(mu_t - mu_f).max()), "mean|dmu|", float(np.abs(mu_t - mu_f).mean()),
          "max|dlog s|", float(np.abs(np.log(s_t / s_f)).max()), "t", round(time.time() - t0, 3), flush=True)
