"""Out-of-bounds write check of every kernel path (SURVEY §5 race / memory checking).

compute-sanitizer is not available on this pool (it has left GPUs needing a reset), so the
library's own guard mode stands in for memcheck's write checks: with PFC_FLAG_GUARD every device
buffer of a context sits between two 4 KB regions filled with a pattern, and
pfc_gpu_check_guards compares them after the work.  Each case also checks its values against the
oracle, so a kernel that reads outside its buffer (the guards hold 0xA5 bytes, not zeros) shows
up as a parity failure.

Paths covered: bf16 tcgen05 engine (graph and eager; D = 512 CTA-pair update, D = 200 single-CTA
update with a ragged last dim block), fp32 validation engine, per-row offsets (MaxEpi pass),
filter mask, full sampling (r = 1), host drop-in with page-locked copies inside the graph,
device FeatureBatch, ragged and tiny batches, repeated labels, diagnostics / mics, checkpoint
write + read, and the 2-rank loopback path (host and device entries).
"""
import os
import tempfile

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shard_bounds

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

MK = {"cosface": p.ADDITIVE_COSINE, "arcface": p.ADDITIVE_ANGULAR}


def build(port, C_, K, D, B, precision, flags, margin="arcface", s=64.0, m=0.5, r=0.1, tau=None,
          **kw):
    cfg = p.StepConfig(r=r, margin=p.MarginConfig(MK[margin], s, m), filter_threshold=tau, lr=0.1)
    ocfg = OracleCfg(r=r, margin=margin, scale=s, m=m, filter_threshold=tau, lr=0.1)
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=precision,
                        flags=flags | p.FLAG_GUARD, **kw)
    W = port.init_centers(C_, K, D, 1)
    off = 0
    for k, (lo, hi) in enumerate(shard_bounds(C_, K)):
        n = D * (hi - lo)
        if k in sh.local_shards:
            sh.set_shard(k, W[off:off + n].reshape(D, hi - lo))
        off += n
    return sh, cfg, ocfg, W


def check_steps(port, sh, cfg, ocfg, W, C_, K, D, B, steps=2, labels_fn=None, pin=False):
    M = np.zeros_like(W)
    # a sanity bound on the values (the parity contract itself lives in test_gpu_step.py; a
    # single-row bf16 batch has no averaging over rows, hence 1e-3 here)
    tol = 1e-6 if sh.precision == p.PRECISION_FP32 else 1e-3
    for i in range(steps):
        X, labels = port.bench_inputs(C_, D, B, 1, i)
        if labels_fn is not None:
            labels = labels_fn(labels)
        out = None
        if pin:
            xh = torch.empty(D, B, dtype=torch.float64, pin_memory=True).numpy()
            lh = torch.empty(B, dtype=torch.int64, pin_memory=True).numpy()
            out = torch.empty(D, B, dtype=torch.float64, pin_memory=True).numpy()
            xh[:] = X
            lh[:] = labels
            X, labels = xh, lh
        stream = p.make_stream("iteration", i)
        res = sh.step_host(X, labels, cfg, p.SeededRng(1, stream), out=out)
        ref = port.step(ocfg, C_, K, D, W, M, np.asarray(X), np.asarray(labels), 1, stream)
        assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= tol, (res.loss, ref["loss"])
    assert sh.check_guards() == 0


CASES = [  # name, C, K, D, B, precision, flags, extra
    ("bf16_d512_graph", 20000, 2, 512, 256, p.PRECISION_BF16, 0, {}),
    ("bf16_d512_eager", 20000, 2, 512, 256, p.PRECISION_BF16, p.FLAG_NO_GRAPH, {}),
    ("bf16_d200_ragged", 7001, 3, 200, 77, p.PRECISION_BF16, 0, {}),
    ("bf16_b1", 5000, 2, 128, 1, p.PRECISION_BF16, 0, {}),
    ("bf16_exact_s128", 20000, 2, 512, 128, p.PRECISION_BF16, 0,
     {"margin": "cosface", "s": 128.0, "m": 0.4}),
    ("bf16_filter", 10000, 2, 256, 192, p.PRECISION_BF16, 0,
     {"margin": "cosface", "m": 0.4, "r": 0.3, "tau": 0.1}),
    ("bf16_full_fc", 6000, 4, 128, 96, p.PRECISION_BF16, 0, {"margin": "cosface", "m": 0.4, "r": 1.0}),
    ("tf32_d512_graph", 20000, 2, 512, 256, p.PRECISION_TF32, 0, {}),
    ("bf16_d768_nc3", 8000, 2, 768, 128, p.PRECISION_BF16, 0, {}),
    ("tf32_d1000_nc4_eager", 6000, 3, 1000, 96, p.PRECISION_TF32, p.FLAG_NO_GRAPH, {}),
    ("fp32_graph", 9000, 3, 256, 96, p.PRECISION_FP32, 0, {}),
    ("fp32_eager_d200", 7001, 3, 200, 77, p.PRECISION_FP32, p.FLAG_NO_GRAPH, {}),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_guards_intact(case, port):
    name, C_, K, D, B, prec, flags, extra = case
    sh, cfg, ocfg, W = build(port, C_, K, D, B, prec, flags, **extra)
    check_steps(port, sh, cfg, ocfg, W, C_, K, D, B)
    sh.close()


def test_guards_pinned_host_and_repeated_labels(port):
    C_, K, D, B = 16, 1, 512, 2048
    sh, cfg, ocfg, W = build(port, C_, K, D, B, p.PRECISION_BF16, 0, margin="cosface", m=0.4, r=1.0)
    check_steps(port, sh, cfg, ocfg, W, C_, K, D, B, pin=True,
                labels_fn=lambda lab: np.where(np.arange(B) < 700, 3, lab))
    sh.close()


def test_guards_device_featurebatch_diag_mics_checkpoint(port):
    C_, K, D, B = 12000, 3, 256, 128
    sh, cfg, ocfg, W = build(port, C_, K, D, B, p.PRECISION_BF16, 0)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    xd = torch.from_numpy(X).cuda()
    ld = torch.from_numpy(labels).cuda()
    sh.step_features(xd, ld, cfg, p.SeededRng(1, p.make_stream("iteration", 0)))
    sh.diagnostics(X, labels)
    sh.mics()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "shards.bin")
        sh.write_shards(path)
        sh.read_shards(path)
    torch.cuda.synchronize()
    assert sh.check_guards() == 0
    sh.close()


@pytest.mark.parametrize("precision", [p.PRECISION_BF16, p.PRECISION_FP32], ids=["bf16", "fp32"])
def test_guards_loopback_two_ranks(precision, port):
    from tests.test_gpu_multirank import run_ranks
    C_, K, D, B, R = 12000, 4, 256, 128, 2
    lid = p.loopback_id()
    X, labels = port.bench_inputs(C_, D, B, 1, 0)

    def rank(rk):
        sh, cfg, _, _ = build(port, C_, K, D, B, precision, 0, rank=rk, world_size=R, nccl_id=lid)
        st = sh.step_host(X, labels, cfg, p.SeededRng(1, p.make_stream("iteration", 0)))
        bl = B // R
        xl = torch.from_numpy(np.ascontiguousarray(X[:, rk * bl:(rk + 1) * bl].T)).float().cuda()
        ll = torch.from_numpy(labels[rk * bl:(rk + 1) * bl].copy()).cuda()
        dx = torch.empty(bl, D, device="cuda")
        torch.cuda.synchronize()
        sh.step_device(xl.data_ptr(), ll.data_ptr(), bl, dx.data_ptr(), cfg,
                       p.SeededRng(1, p.make_stream("iteration", 1)))
        n = sh.check_guards()
        sh.close()
        return st.loss, n
    out = run_ranks(R, rank)
    assert all(o[1] == 0 for o in out)
    assert out[0][0] == out[1][0]
