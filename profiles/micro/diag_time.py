"""Time the diagnostics call at the bench configuration (2M classes, K=8 on one GPU, B=1024,
d=512).  Run plainly for wall time, or under ncu for the per-kernel launch list."""
import time

import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2203_15565_b200 as p  # noqa: E402

C_, K, D, B = 2_000_000, 8, 512, 1024
sh = p.CenterShards(p.ShardLayout(C_, K), D, p.StepConfig(), max_batch=B)
sh.init_center_shards(1)
rng = np.random.default_rng(0)
X = rng.standard_normal((D, B))
labels = rng.integers(0, C_, B)
for i in range(3):
    t0 = time.perf_counter()
    d = sh.diagnostics(X, labels)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.2f} ms  apcs={d.apcs:.6f} amncs={d.amncs:.6f}")
