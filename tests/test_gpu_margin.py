"""The combined (m1, m2, m3) margin -- an extension beyond the reference (the north
star names "ArcFace/CosFace combined margin"; the reference has only plain / CosFace / ArcFace,
margin.hpp:11).  z_pos = s (cos(m1 theta + m2) - m3), theta = acos of the cosine clamped like
ArcFace (margin.hpp:50-51), derivative s m1 sin(m1 theta + m2) / sqrt(1 - c^2), zero in the clamp.

Parity pins, strongest first:
  * (1, m, 0) runs the reference's ArcFace arithmetic operation for operation: the device step is
    bit-identical to the ArcFace step on the same state and inputs (fp32 and bf16 engines);
  * general (m1, m2, m3) against the oracle's restatement (pfc_oracle.c MK_COMB, itself pinned to
    the reference through the same identities in tests/test_oracle.py), under the step contract
    of tests/test_gpu_step.py for each precision.
"""
import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shards_to_rows
from tests.helpers import device_rows, make_shards, rel_fro, rel_max
from tests.test_gpu_step import TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("precision", [p.PRECISION_FP32, p.PRECISION_BF16], ids=["fp32", "bf16"])
def test_combined_arcface_point_is_bit_identical(precision, port):
    C_, K, D, B = 12000, 2, 256, 128
    W = port.init_centers(C_, K, D, 2)
    M = np.zeros_like(W)
    arc = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(64.0, 0.5), lr=0.1)
    comb = p.StepConfig(r=0.1, margin=p.MarginConfig.combined(64.0, 1.0, 0.5, 0.0), lr=0.1)
    sa = make_shards(W, M, C_, K, D, arc, B, precision)
    sc = make_shards(W, M, C_, K, D, comb, B, precision)
    for step in range(2):
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        rng = p.SeededRng(1, port.make_stream("iteration", step))
        ra = p.distributed_partial_step(sa, X, labels, arc, rng)
        rc = p.distributed_partial_step(sc, X, labels, comb, rng)
        assert ra.loss == rc.loss
        assert np.array_equal(ra.d_features, rc.d_features)
    wa, ma = device_rows(sa, C_, K, D)
    wc, mc = device_rows(sc, C_, K, D)
    assert np.array_equal(wa, wc) and np.array_equal(ma, mc)
    sa.close()
    sc.close()


# s, m1, m2, m3
COMBOS = [(64.0, 1.0, 0.3, 0.2), (64.0, 0.9, 0.4, 0.15), (32.0, 1.0, 0.0, 0.35)]


@pytest.mark.parametrize("precision", [p.PRECISION_FP32, p.PRECISION_BF16, p.PRECISION_TF32],
                         ids=["fp32", "bf16", "tf32"])
@pytest.mark.parametrize("combo", COMBOS, ids=["m1_1.0", "m1_0.9", "cos_like"])
def test_combined_matches_oracle(combo, precision, port):
    s, m1, m2, m3 = combo
    C_, K, D, B = 20000, 4, 512, 256
    tl, tdf, tdm, tw = TOL[precision]
    W = port.init_centers(C_, K, D, 1)
    M = np.zeros_like(W)
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.combined(s, m1, m2, m3), lr=0.1)
    ocfg = OracleCfg(r=0.1, margin="combined", scale=s, m=m2, m1=m1, m3=m3, lr=0.1)
    sh = make_shards(W, M, C_, K, D, cfg, B, precision)
    for step in range(2):
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        stream = port.make_stream("iteration", step)
        res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
        ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream)
        for k, buf in enumerate(res.buffers):
            assert np.array_equal(buf.class_indices, ref["buffers"][k])
        Wd, _ = device_rows(sh, C_, K, D)
        rows = np.unique(ref["buffers"].ravel())
        assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= tl, (res.loss, ref["loss"])
        assert rel_fro(res.d_features, ref["dX"]) <= tdf
        assert rel_max(res.d_features, ref["dX"]) <= tdm
        assert rel_max(Wd[rows], shards_to_rows(W, C_, K, D)[rows]) <= tw
    sh.close()


def test_combined_config_errors_and_per_call_switch(port):
    C_, K, D, B = 8000, 2, 128, 64
    with pytest.raises(p.ConfigError, match=r"m1 must be in \(0, 2\]"):
        p.CenterShards(p.ShardLayout(C_, K), D,
                       p.StepConfig(margin=p.MarginConfig.combined(64.0, 0.0, 0.3, 0.2)))
    with pytest.raises(p.ConfigError, match=r"m3 must be in \[0, 1\)"):
        p.CenterShards(p.ShardLayout(C_, K), D,
                       p.StepConfig(margin=p.MarginConfig.combined(64.0, 1.0, 0.3, 1.0)))
    # a context created with CosFace switches to the combined margin per call (set_step_config)
    W = port.init_centers(C_, K, D, 1)
    M = np.zeros_like(W)
    cos = p.StepConfig(r=0.1, margin=p.MarginConfig.cosface_style(), lr=0.1)
    comb = p.StepConfig(r=0.1, margin=p.MarginConfig.combined(64.0, 1.0, 0.3, 0.2), lr=0.1)
    sh = make_shards(W, M, C_, K, D, cos, B, p.PRECISION_FP32)
    for step, (cfg, ocfg) in enumerate([
            (cos, OracleCfg(r=0.1, margin="cosface", scale=64.0, m=0.4, lr=0.1)),
            (comb, OracleCfg(r=0.1, margin="combined", scale=64.0, m=0.3, m1=1.0, m3=0.2, lr=0.1))]):
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        stream = port.make_stream("iteration", step)
        res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
        ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream)
        assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= 1e-6
        assert rel_fro(res.d_features, ref["dX"]) <= 1e-5
    sh.close()
