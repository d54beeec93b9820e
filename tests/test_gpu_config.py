"""GPU parity of the reference's per-call StepConfig and of batches past the old 8192 cap.

* The reference takes its StepConfig on every call (shardsim.hpp:166-168): one set of device
  shards steps through configs whose r (capacity grows and shrinks), margin kind and scale
  (per-row offsets at s = 128), filter, momentum and weight decay change from step to step, each
  step checked against the oracle stepping the same state with the same config.
* The bitmap sampler has no batch-size limit of its own: a 16384-row batch (labels drawn from
  a subset of the classes, so the capacity holds) is bit-exact in the sampled buffers and within
  the contract in values.
"""
import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg
from tests.helpers import device_rows, make_shards, rel_fro, rel_max
from oracle.oracle import shards_to_rows

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TOL = {  # loss rel, dX fro, W' max/max (tests/test_gpu_step.py contract)
    p.PRECISION_FP32: (1e-6, 1e-5, 1e-6),
    p.PRECISION_BF16: (1e-4, 1e-2, 1e-3),
}
MK = {"cosface": p.ADDITIVE_COSINE, "arcface": p.ADDITIVE_ANGULAR}

# r, margin, s, m, tau, momentum, weight decay
SCHEDULE = [
    (0.1, "arcface", 64.0, 0.5, None, 0.9, 5e-4),
    (0.2, "cosface", 64.0, 0.4, None, 0.5, 5e-4),
    (0.05, "cosface", 64.0, 0.4, 0.1, 0.9, 0.0),
    (0.3, "cosface", 128.0, 0.35, None, 0.9, 5e-4),
    (0.1, "arcface", 64.0, 0.5, None, 0.9, 5e-4),
]


@pytest.mark.parametrize("precision", [p.PRECISION_FP32, p.PRECISION_BF16], ids=["fp32", "bf16"])
def test_step_config_changes_between_calls(precision, port):
    C_, K, D, B = 20000, 4, 256, 96
    W = port.init_centers(C_, K, D, 3)
    M = np.zeros_like(W)
    r0, mk0, s0, m0, tau0, mu0, wd0 = SCHEDULE[0]
    cfg0 = p.StepConfig(r=r0, margin=p.MarginConfig(MK[mk0], s0, m0), filter_threshold=tau0,
                        momentum=mu0, weight_decay=wd0)
    sh = make_shards(W, M, C_, K, D, cfg0, B, precision)
    tl, tdx, tw = TOL[precision]
    fw = 1.0
    for step, (r, mk, s, m, tau, mu, wd) in enumerate(SCHEDULE):
        if precision == p.PRECISION_BF16:
            tau = None  # bf16 + filter has its own contract (test_gpu_edges.py)
        cfg = p.StepConfig(r=r, margin=p.MarginConfig(MK[mk], s, m), filter_threshold=tau,
                           momentum=mu, weight_decay=wd, lr=0.1)
        ocfg = OracleCfg(r=r, margin=mk, scale=s, m=m, filter_threshold=tau, lr=0.1,
                         momentum=mu, weight_decay=wd)
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        stream = port.make_stream("iteration", step)
        res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
        ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream)
        assert sh.capacity == ref["buffers"].shape[1]
        for k, buf in enumerate(res.buffers):
            assert np.array_equal(buf.class_indices, ref["buffers"][k]), step
        # value bounds scale with s (tests/test_gpu_edges.py); W and momentum carry every earlier
        # step's error forward, so the largest scale seen so far sets the bound
        f = max(1.0, s / 64.0)
        fw = max(fw, f)
        Wd, _ = device_rows(sh, C_, K, D)
        Wr = shards_to_rows(W, C_, K, D)
        rows = np.unique(ref["buffers"].ravel())
        assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= tl * f, step
        assert rel_fro(res.d_features, ref["dX"]) <= tdx * f, step
        assert rel_max(Wd[rows], Wr[rows]) <= tw * fw * fw, step
    sh.close()


def test_batch_beyond_8192(port):
    C_, K, D, B = 20000, 2, 64, 16384
    W = port.init_centers(C_, K, D, 1)
    M = np.zeros_like(W)
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(), lr=0.1)
    ocfg = OracleCfg(r=0.1, margin="arcface", scale=64.0, m=0.5, lr=0.1)
    sh = make_shards(W, M, C_, K, D, cfg, B, p.PRECISION_BF16)
    X, _ = port.bench_inputs(C_, D, B, 1, 0)
    rng = np.random.default_rng(5)
    # 1200 distinct classes spread over both shards (capacity 1000 per shard)
    pool = np.concatenate([rng.choice(10000, 600, replace=False),
                           10000 + rng.choice(10000, 600, replace=False)])
    labels = pool[rng.integers(0, pool.size, B)].astype(np.int64)
    stream = port.make_stream("iteration", 0)
    res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
    ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream)
    for k, buf in enumerate(res.buffers):
        assert np.array_equal(buf.class_indices, ref["buffers"][k])
    tl, tdx, tw = TOL[p.PRECISION_BF16]
    assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= tl
    assert rel_fro(res.d_features, ref["dX"]) <= tdx
    Wd, _ = device_rows(sh, C_, K, D)
    rows = np.unique(ref["buffers"].ravel())
    assert rel_max(Wd[rows], shards_to_rows(W, C_, K, D)[rows]) <= tw
    sh.close()
