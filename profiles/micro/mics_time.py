"""mics (metrics.hpp:150-164) at Glint360K scale on one GPU: C=360k, d=512 -> a 2 C^2 d =
1.33e14 flop screening GEMM + exact re-evaluation."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2203_15565_b200 as p  # noqa: E402

C_, K, D = 360_000, 8, 512
sh = p.CenterShards(p.ShardLayout(C_, K), D, p.StepConfig(), max_batch=8)
sh.init_center_shards(1)
sh.mics()  # warm-up (allocations)
t0 = time.perf_counter()
m = sh.mics()
dt = time.perf_counter() - t0
flop = 2.0 * C_ * C_ * D
print(f"mics C={C_}: {dt:.3f} s  ({flop / dt / 1e12:.0f} TFLOP/s effective)  mean={m.mean():.6f} max={m.max():.6f}")
