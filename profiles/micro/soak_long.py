"""Long soak of the north-star configuration (2M classes, K = 8, B = 1024, d = 512, bf16): STEPS
graph-replayed device steps with per-step inputs, seeds and a decaying lr, run twice in fresh
contexts.  Checks: every step's status (loss finite, no device error); the sampled buffers of
every CHECK-th step bit-exact against the oracle's build_buffers on the same labels; the two runs
bitwise identical (losses, final centres and momentum of shard 3, last dX).
  python profiles/micro/soak_long.py [STEPS] [CHECK]"""
import hashlib
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2203_15565_b200 as p  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

C_, K, B, D = 2_000_000, 8, 1024, 512
STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
CHECK = int(sys.argv[2]) if len(sys.argv) > 2 else 250
port = Oracle("port")


def run(check):
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(64.0, 0.5), lr=0.1)
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
    sh.init_center_shards(11)
    x = torch.empty(B, D, device="cuda")
    lab = torch.empty(B, dtype=torch.int64, device="cuda")
    dx = torch.empty(B, D, device="cuda")
    losses, checked = [], 0
    t0 = time.perf_counter()
    for step in range(STEPS):
        sh.bench_inputs(5, step, B, x.data_ptr(), lab.data_ptr())
        cfg.lr = 0.1 * (1.0 - step / STEPS)
        cfg.step_index = step
        stream = p.make_stream("iteration", step)
        out = sh.step_device(x.data_ptr(), lab.data_ptr(), B, dx.data_ptr(), cfg,
                             p.SeededRng(5, stream))
        assert np.isfinite(out.loss), step
        losses.append(out.loss)
        if check and step % CHECK == 0:
            want, npos = port.build_buffers(C_, K, lab.cpu().numpy(), 0.1, 5, stream)
            for k, b in enumerate(sh.buffers()):
                assert np.array_equal(b.class_indices, want[k]) and b.num_positives == npos[k], (step, k)
            checked += 1
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    w, m = sh.get_shard(3)
    dxh = dx.cpu().numpy()
    sh.close()
    return np.array(losses), w, m, dxh, checked, secs


a = run(True)
b = run(False)
same = (np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        and np.array_equal(a[3], b[3]))
h = hashlib.sha256(a[1].tobytes() + a[2].tobytes()).hexdigest()[:16]
print(f"steps {STEPS} x 2 runs at 2M/K=8/B=1024 bf16: all losses finite; buffers bit-exact vs "
      f"oracle at {a[4]} checked steps; runs bitwise identical: {same}; loss first/last "
      f"{a[0][0]:.6f} / {a[0][-1]:.6f}; shard-3 W+mom sha256 {h}; wall {a[5]:.1f} s / {b[5]:.1f} s")
assert same
