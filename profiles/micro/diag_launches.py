"""One diagnostics call at 2M / B = 1024 (for an ncu launch list of its kernels)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2203_15565_b200 as p  # noqa: E402

C_, K, D, B = 2000000, 8, 512, 1024
cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(), lr=0.1)
sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
sh.init_center_shards(1)
rng = np.random.default_rng(0)
X = rng.standard_normal((D, B))
lab = rng.integers(0, C_, B)
for _ in range(2):
    d = sh.diagnostics(X, lab)
print(d)
