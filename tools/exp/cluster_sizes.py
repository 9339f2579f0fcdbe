"""Cluster-size distribution of the bench's K-Means (DeepSeek shape, 64 -> 16 per layer): what the merge's
stage packing sees.  Experiment, run on a GPU box."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2508_19078_b200 import synthetic  # noqa: E402
from paper_2508_19078_b200.driver import cluster_model, expert_features_model  # noqa: E402

cfg = synth.CONFIGS["deepseek_moe"]
m = synthetic.master_weights(cfg)
feats, _, _ = expert_features_model(m)
hist = torch.randint(1, 1000, (cfg.n_layers, cfg.n_experts), dtype=torch.int64, device="cuda")
cl = cluster_model(feats, hist, 16).cpu().numpy()
sizes = collections.Counter()
for l in range(cl.shape[0]):
    sizes.update(np.bincount(cl[l], minlength=16).tolist())
print("cluster size -> count over all layers:", dict(sorted(sizes.items())))
# stages used per chunk index by chunk-aligned packing (ceil(m/4) per cluster) vs packed (64/4 = 16)
aligned = sum(c * -(-s // 4) if s else c for s, c in sizes.items()) / cl.shape[0]
print(f"stages per chunk index: chunk-aligned {aligned:.1f}, packed {cfg.n_experts / 4:.1f}")
