"""Checkpoint section throughput (write then read back) at Glint360K scale: C=360k, K=8, d=512
on one GPU (W + momentum = 2 x 737 MB fp32 -> a 2.95 GB fp64 section in the reference encoding)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2203_15565_b200 as p  # noqa: E402

C_, K, D = 360_000, 8, 512
sh = p.CenterShards(p.ShardLayout(C_, K), D, p.StepConfig(), max_batch=64)
sh.init_center_shards(1)
path = "/tmp/pfc_ckpt_bench.bin"
t0 = time.perf_counter()
sh.write_shards(path)
tw = time.perf_counter() - t0
size = os.path.getsize(path)
t0 = time.perf_counter()
end = sh.read_shards(path, 0)
tr = time.perf_counter() - t0
assert end == size
print(f"section {size / 1e9:.2f} GB: write {tw:.2f} s ({size / tw / 1e9:.2f} GB/s), "
      f"read {tr:.2f} s ({size / tr / 1e9:.2f} GB/s)")
os.remove(path)
