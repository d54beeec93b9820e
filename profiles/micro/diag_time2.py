"""Wall time of one diagnostics call at 2M / B = 1024: pageable vs page-locked host features."""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2203_15565_b200 as p  # noqa: E402

C_, K, D, B = 2000000, 8, 512, 1024
cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(), lr=0.1)
sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
sh.init_center_shards(1)
rng = np.random.default_rng(0)
X = rng.standard_normal((D, B))
lab = rng.integers(0, C_, B)
Xp = torch.empty(D, B, dtype=torch.float64, pin_memory=True).numpy()
Xp[:] = X
for name, x in (("pageable", X), ("pinned", Xp), ("pageable", X), ("pinned", Xp)):
    sh.diagnostics(x, lab)
    t0 = time.perf_counter()
    for _ in range(5):
        sh.diagnostics(x, lab)
    print(name, (time.perf_counter() - t0) / 5 * 1e3, "ms")
t0 = time.perf_counter()
for _ in range(20):
    np.isfinite(X).all()
print("numpy isfinite scan", (time.perf_counter() - t0) / 20 * 1e3, "ms")
