"""GPU: a long run of the device path at Glint360K scale (360k classes, K = 8, B = 1024, d = 512):
300 graph-replayed steps with per-step seeds and a changing lr, every step's status checked, run
twice in fresh contexts.  The final centres, momentum and loss must be bitwise identical (the
step has no floating-point atomics and a fixed reduction order), and every loss finite."""
import numpy as np
import pytest

import paper_2203_15565_b200 as p

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

C_, K, B, D, STEPS = 360_000, 8, 1024, 512, 300


def _run():
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(64.0, 0.5), lr=0.1)
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
    sh.init_center_shards(7)
    x = torch.empty(B, D, device="cuda")
    lab = torch.empty(B, dtype=torch.int64, device="cuda")
    dx = torch.empty(B, D, device="cuda")
    losses = []
    for step in range(STEPS):
        sh.bench_inputs(3, step, B, x.data_ptr(), lab.data_ptr())
        cfg.lr = 0.1 * (1.0 - step / STEPS)
        cfg.step_index = step
        out = sh.step_device(x.data_ptr(), lab.data_ptr(), B, dx.data_ptr(), cfg,
                             p.SeededRng(3, p.make_stream("iteration", step)))
        losses.append(out.loss)
    w, m = sh.get_shard(5)
    dxh = dx.cpu().numpy()
    sh.close()
    return np.array(losses), w, m, dxh


def test_soak_300_steps_deterministic():
    l1, w1, m1, d1 = _run()
    l2, w2, m2, d2 = _run()
    assert np.isfinite(l1).all()
    assert np.array_equal(l1, l2)
    assert np.array_equal(w1, w2) and np.array_equal(m1, m2) and np.array_equal(d1, d2)
    assert np.isfinite(w1).all() and np.isfinite(m1).all()
    # the run did update the centres: momentum is non-zero on sampled rows
    assert np.abs(m1).max() > 0
