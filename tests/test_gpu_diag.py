"""GPU parity of the step's diagnostics (pfc_gpu_diagnostics; metrics.hpp:56-146, reported by
the reference step with with_diagnostics, shardsim.hpp:401-410).

Contract: apcs and amncs (and the conflicted / hard split) are EXACT up to the fp32 storage of
W and X: |delta| <= 1e-6 against the reference's fp64 values (golden, init state), and <= 1e-9
against the oracle evaluated on the device's own fp32 state.  amncs is exact because the bf16
GEMM only screens: every class within the bf16 error band of the running maximum is
re-evaluated in fp64 (diag.cuh)."""
import json
import os

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from tests.helpers import device_rows  # noqa: F401  (shared fixtures live in conftest)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PREC = [p.PRECISION_BF16, p.PRECISION_FP32]


def identities(C_, labels):
    # tests/golden/make_golden.py: diag_identities
    ci = np.arange(C_, dtype=np.int64) // 3
    si = labels // 3
    si = np.where(np.arange(len(labels)) % 5 == 0, si + 1, si)
    return ci, si


def device_state(sh, C_, K, D):
    """The device's fp32 W in the reference's shard-concatenated D x owned layout (fp64)."""
    return np.concatenate([sh.get_shard(k)[0].ravel() for k in range(K)])


def close(a, b, tol):
    return (a is None and b is None) or (a is not None and b is not None and abs(a - b) <= tol)


@pytest.mark.parametrize("precision", PREC, ids=["bf16", "fp32"])
def test_diagnostics_match_reference_golden(precision, port):
    with open(os.path.join(GOLDEN, "diag.json")) as f:
        cases = json.load(f)
    for cs in cases:
        C_, K, D, B = cs["C"], cs["K"], cs["D"], cs["B"]
        sh = p.CenterShards(p.ShardLayout(C_, K), D, p.StepConfig(), max_batch=B, precision=precision)
        sh.init_center_shards(1)
        X, labels = port.bench_inputs(C_, D, B, 1, 0)
        ci, si = identities(C_, labels)
        plain = sh.diagnostics(X, labels)
        split = sh.diagnostics(X, labels, p.ConflictInfo(ci, si))
        g = cs["plain"]
        assert abs(plain.apcs - g["apcs"]) <= 1e-6 and abs(plain.amncs - g["amncs"]) <= 1e-6, cs["name"]
        assert plain.amncs_hard is None and plain.amncs_conflicted is None
        g = cs["split"]
        assert abs(split.apcs - g["apcs"]) <= 1e-6 and abs(split.amncs - g["amncs"]) <= 1e-6, cs["name"]
        assert close(split.amncs_hard, g["amncs_hard"], 1e-6), cs["name"]
        assert close(split.amncs_conflicted, g["amncs_conflicted"], 1e-6), cs["name"]
        sh.close()


@pytest.mark.parametrize("precision", PREC, ids=["bf16", "fp32"])
def test_diagnostics_exact_after_steps(precision, port):
    """After training steps (W moved), the device diagnostics equal the oracle evaluated on
    the device's own state to 1e-9: the bf16 screening never loses the true maximum."""
    C_, K, D, B = 50000, 4, 256, 64
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style())
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=precision)
    sh.init_center_shards(2)
    for step in range(2):
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, p.make_stream("iteration", step)))
    X, labels = port.bench_inputs(C_, D, B, 1, 7)
    # a conflict structure with many siblings: identities in groups of 2 classes
    ci = np.arange(C_, dtype=np.int64) // 2
    si = labels // 2
    W = device_state(sh, C_, K, D)
    want = port.diagnostics(C_, K, D, W, X, labels, ci, si)
    got = sh.diagnostics(X, labels, p.ConflictInfo(ci, si))
    assert abs(got.apcs - want["apcs"]) <= 1e-9
    assert abs(got.amncs - want["amncs"]) <= 1e-9
    assert close(got.amncs_hard, want["amncs_hard"], 1e-9)
    assert close(got.amncs_conflicted, want["amncs_conflicted"], 1e-9)
    sh.close()


def test_step_with_diagnostics_reports_pre_update_state(port):
    C_, K, D, B = 4000, 4, 512, 64
    cfg = p.StepConfig(r=0.2, margin=p.MarginConfig.arcface_style())
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
    sh.init_center_shards(1)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    before = sh.diagnostics(X, labels)
    cfg.with_diagnostics = True
    cfg.step_index = 11
    res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, 5))
    assert res.diagnostics is not None and res.diagnostics.iteration == 11
    assert res.diagnostics.apcs == before.apcs and res.diagnostics.amncs == before.amncs
    after = sh.diagnostics(X, labels)
    assert after.apcs != before.apcs  # the step moved the centres afterwards
    with pytest.raises(p.ContractError, match="build_buffers: label 4000 outside"):
        bad = labels.copy()
        bad[3] = 4000
        p.distributed_partial_step(sh, X, bad, cfg, p.SeededRng(1, 6))
    with pytest.raises(p.ContractError, match="apcs: label 4000 owned by no shard"):
        sh.diagnostics(X, bad)
    Xn = X.copy()
    Xn[2, 5] = np.nan
    with pytest.raises(p.NumericalError, match="l2_normalize_columns: non-finite entry in 512x64 result"):
        sh.diagnostics(Xn, labels)
    sh.close()


@pytest.mark.parametrize("precision", PREC, ids=["bf16", "fp32"])
def test_mics_matches_reference_and_oracle(precision, port):
    """mics (metrics.hpp:150-164): within 1e-6 of the reference golden values at init, and
    within 1e-9 of the oracle on the device's own state (exact, not bf16)."""
    with open(os.path.join(GOLDEN, "mics.json")) as f:
        cases = json.load(f)
    for cs in cases:
        C_, K, D = cs["C"], cs["K"], cs["D"]
        sh = p.CenterShards(p.ShardLayout(C_, K), D, p.StepConfig(), max_batch=8, precision=precision)
        sh.init_center_shards(cs["seed"])
        got = sh.mics()
        assert np.max(np.abs(got - np.array(cs["mics"]))) <= 1e-6, cs["name"]
        want = port.mics(C_, K, D, device_state(sh, C_, K, D))
        assert np.max(np.abs(got - want)) <= 1e-9, cs["name"]
        sh.close()
    # a larger case with trained (moved) centres
    C_, K, D, B = 20000, 2, 128, 64
    cfg = p.StepConfig(r=0.2, margin=p.MarginConfig.arcface_style())
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=precision)
    sh.init_center_shards(3)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, 1))
    want = port.mics(C_, K, D, device_state(sh, C_, K, D))
    assert np.max(np.abs(sh.mics() - want)) <= 1e-9
    sh.close()
