"""GPU parity on the reference-legal edges of distributed_partial_step:

  * a label repeated far more than 256 times in one batch (every row feeds dwt,
    shardsim.hpp:349-376);
  * margin scales where a fixed softmax offset cannot hold (the reference's max-subtracted
    softmax is exact for any s > 0, shardsim.hpp:270-318; margin.hpp:22-28): per-row offsets;
  * rows whose every logit lies far below the fixed offset at s = 64 (rerun with per-row
    offsets);
  * the filter mask in bf16 (decided on bf16-operand cosines): mask flips only within 2^-7 of
    tau, and identical values once the oracle replays the GPU's own mask;
  * the logits themselves (debug export), against the oracle's within SURVEY §8(c)'s bound
    max|dz|/s <= 1e-3 (bf16) / 1e-5 (fp32).

Tolerances are the contract of tests/test_gpu_step.py.
"""
import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shards_to_rows
from tests.helpers import device_rows, make_shards, rel_fro, rel_max

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TOL = {  # loss rel, dX fro, dX max/max, W' max/max
    p.PRECISION_FP32: (1e-6, 1e-5, 3e-5, 1e-6),
    p.PRECISION_BF16: (1e-4, 1e-2, 1e-2, 1e-3),
}
ZTOL = {p.PRECISION_FP32: 1e-5, p.PRECISION_BF16: 1e-3}  # max |z - z_ref| / s
PREC = [p.PRECISION_FP32, p.PRECISION_BF16]
PREC_IDS = ["fp32", "bf16"]
MK = {"cosface": p.ADDITIVE_COSINE, "arcface": p.ADDITIVE_ANGULAR, "plain": p.PLAIN}


def cfgs(margin, s, m, r, tau=None, lr=0.1):
    mc = p.MarginConfig(MK[margin], s, m)
    return (p.StepConfig(r=r, margin=mc, filter_threshold=tau, lr=lr),
            OracleCfg(r=r, margin=margin, scale=s, m=m, filter_threshold=tau, lr=lr))


def run_and_compare(port, C_, K, D, X, labels, W, M, margin, s, m, r, precision, tau=None,
                    flags=0, check_logits=True, mask_from_gpu=False):
    """One step on the GPU (host drop-in) and on the oracle from the same state; asserts the
    contract and returns the GPU result and the oracle's."""
    B = len(labels)
    scfg, ocfg = cfgs(margin, s, m, r, tau)
    sh = make_shards(W, M, C_, K, D, scfg, B, precision, flags=flags | p.FLAG_DEBUG_LOGITS)
    W0, M0 = W.copy(), M.copy()
    stream = port.make_stream("iteration", 0)
    res = p.distributed_partial_step(sh, X, labels, scfg, p.SeededRng(1, stream))
    z = sh.debug_logits(B).transpose(1, 0, 2)  # [K][B][cap]
    ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream, want_extra=True)
    for k, buf in enumerate(res.buffers):
        assert np.array_equal(buf.class_indices, ref["buffers"][k])
    cos = ref["cos"]
    gmask = np.isneginf(z)
    info = {}
    if tau is not None:
        pos = np.zeros_like(gmask)
        cap = cos.shape[2]
        for b, y in enumerate(labels):
            k = y // ((C_ + K - 1) // K)
            j = np.searchsorted(ref["buffers"][k][:ref["npos"][k]], y)
            pos[k, b, j] = True
        omask = (cos > tau) & ~pos
        flips = gmask != omask
        info["mask_flips"] = int(flips.sum())
        info["masked"] = int(omask.sum())
        if precision == p.PRECISION_FP32:
            assert not flips.any()
        else:  # decided on bf16-operand cosines: only within 2^-7 of tau
            assert np.all(np.abs(cos[flips] - tau) < 2.0 ** -7), np.abs(cos[flips] - tau).max()
        if mask_from_gpu and flips.any():
            # replay the GPU's own decisions in the oracle: values must then meet the contract
            W, M = W0.copy(), M0.copy()
            ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream, want_extra=True,
                            mask=gmask)
    if check_logits:
        # z_ref = s cos (negatives) / margin(cos) on the positive, unmasked entries only
        zr = s * cos
        for b, y in enumerate(labels):
            k = y // ((C_ + K - 1) // K)
            j = np.searchsorted(ref["buffers"][k][:ref["npos"][k]], y)
            zr[k, b, j] = port._apply_margin(cos[k, b, j], 1, MK[margin], s, m)
        live = ~gmask & ~np.isneginf(zr)
        if tau is not None:
            live &= ~((cos > tau) & (zr == s * cos))  # oracle-masked negatives carry no logit
        dz = np.abs(z[live] - zr[live]).max() / s
        info["logit_max_abs_over_s"] = float(dz)
        assert dz <= ZTOL[precision], dz
    # the cosine's own rounding (bf16 operands ~2^-9 / sqrt(D), fp32 ~1e-7) reaches the logits
    # multiplied by s: the value bounds, calibrated at the BASELINE s = 64, scale with s above it
    # (the logit bound max|dz|/s above does not).  Loss and dX are compared relative to their own
    # size, which grows with s, so their bounds scale by f = s / 64.  W' is compared relative to
    # W (unit rows, independent of s) while its error is lr times the dW error, whose absolute
    # size grows as s (the gradient's scale) times s dcos (the probability error): f^2.
    f = max(1.0, s / 64.0)
    tl, tdf, tdm, tw = (t * f for t in TOL[precision])
    tw *= f
    Wd, Md = device_rows(sh, C_, K, D)
    Wr = shards_to_rows(W, C_, K, D)
    rows = np.unique(ref["buffers"].ravel())
    info.update(loss=res.loss, loss_ref=ref["loss"],
                loss_rel=abs(res.loss - ref["loss"]) / abs(ref["loss"]),
                dX_fro=rel_fro(res.d_features, ref["dX"]), dX_max=rel_max(res.d_features, ref["dX"]),
                W_max=rel_max(Wd[rows], Wr[rows]))
    assert info["loss_rel"] <= tl, info
    assert info["dX_fro"] <= tdf and info["dX_max"] <= tdm, info
    assert info["W_max"] <= tw, info
    sh.close()
    return res, ref, info


def unit_rows_state(port, C_, K, D, seed=1):
    W = port.init_centers(C_, K, D, seed)
    return W, np.zeros_like(W)


@pytest.mark.parametrize("precision", PREC, ids=PREC_IDS)
@pytest.mark.parametrize("margin,m", [("cosface", 0.4), ("arcface", 0.5)])
def test_label_repeated_thousands_of_times(precision, margin, m, port):
    """C = 16, K = 1, r = 1.0, B = 4096: every class is a positive of ~256 rows and the full
    buffer is sampled; every row's correction reaches dW."""
    C_, K, D, B = 16, 1, 512, 4096
    W, M = unit_rows_state(port, C_, K, D)
    X, _ = port.bench_inputs(C_, D, B, 1, 0)
    labels = np.random.default_rng(3).integers(0, C_, B)
    labels[:1500] = 7  # one class repeated 1500+ times
    run_and_compare(port, C_, K, D, X, labels, W, M, margin, 64.0, m, 1.0, precision)


@pytest.mark.parametrize("precision", PREC, ids=PREC_IDS)
def test_all_labels_equal(precision, port):
    C_, K, D, B = 10000, 2, 512, 1024
    W, M = unit_rows_state(port, C_, K, D)
    X, _ = port.bench_inputs(C_, D, B, 1, 1)
    labels = np.full(B, 6789)
    run_and_compare(port, C_, K, D, X, labels, W, M, "arcface", 64.0, 0.5, 0.1, precision)


@pytest.mark.parametrize("precision,scale", [(p.PRECISION_FP32, 128.0), (p.PRECISION_FP32, 256.0),
                                             (p.PRECISION_FP32, 1000.0), (p.PRECISION_BF16, 128.0),
                                             (p.PRECISION_BF16, 256.0)],
                         ids=["fp32-128", "fp32-256", "fp32-1000", "bf16-128", "bf16-256"])
def test_large_margin_scale(scale, precision, port):
    """CosFace at s = 128 / 256 / 1000: per-row offsets (exact for any s > 0); the value
    contract scales by s / 64 (logit rounding times s), the logit bound holds as is."""
    C_, K, D, B = 20000, 2, 512, 256
    W, M = unit_rows_state(port, C_, K, D)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    run_and_compare(port, C_, K, D, X, labels, W, M, "cosface", scale, 0.4, 0.1, precision)


@pytest.mark.parametrize("precision", PREC, ids=PREC_IDS)
def test_forced_per_row_offsets_at_s64(precision, port):
    """FLAG_EXACT_SOFTMAX at the BASELINE margin: same contract as the fixed offset."""
    C_, K, D, B = 20000, 2, 512, 256
    W, M = unit_rows_state(port, C_, K, D)
    X, labels = port.bench_inputs(C_, D, B, 1, 2)
    run_and_compare(port, C_, K, D, X, labels, W, M, "arcface", 64.0, 0.5, 0.1, precision,
                    flags=p.FLAG_EXACT_SOFTMAX)


@pytest.mark.parametrize("precision", PREC, ids=PREC_IDS)
def test_fixed_offset_underflow_reruns_per_row(precision, port):
    """Every centre almost parallel to u and every feature almost -u: all cosines ~ -1, so at
    s = 64 every logit sits ~88 below the fixed offset 24 and exp underflows.  The reference is
    exact here; the host drop-in reruns the step with per-row offsets and matches it."""
    C_, K, D, B = 3000, 2, 128, 64
    rng = np.random.default_rng(11)
    u = rng.standard_normal(D)
    u /= np.linalg.norm(u)
    rows = u[None, :] + 0.02 * rng.standard_normal((C_, D))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    from oracle.oracle import rows_to_shards
    W = rows_to_shards(rows, C_, K, D)
    M = np.zeros_like(W)
    X = (-u[:, None] + 0.02 * rng.standard_normal((D, B))) * 3.0
    labels = rng.integers(0, C_, B)
    _, ref, _ = run_and_compare(port, C_, K, D, X, labels, W, M, "cosface", 64.0, 0.4, 0.1,
                                precision, check_logits=False)
    assert np.isfinite(ref["loss"])


@pytest.mark.parametrize("tau", [0.1, 0.05])
def test_bf16_filter_contract(tau, port):
    """bf16 + filter at d = 512: the mask is decided on the bf16-operand cosine, so it may flip
    only where |cos - tau| < 2^-7; with the oracle replaying the GPU's mask, loss / dX / W'
    meet the bf16 contract and the logits the 1e-3 bound."""
    C_, K, D, B = 10000, 2, 512, 256
    W, M = unit_rows_state(port, C_, K, D)
    X, labels = port.bench_inputs(C_, D, B, 1, 3)
    _, _, info = run_and_compare(port, C_, K, D, X, labels, W, M, "cosface", 64.0, 0.4, 0.3,
                                 p.PRECISION_BF16, tau=tau, mask_from_gpu=True)
    assert info["masked"] > 0


@pytest.mark.parametrize("precision", PREC, ids=PREC_IDS)
@pytest.mark.parametrize("margin,m,tau", [("arcface", 0.5, None), ("cosface", 0.4, None),
                                          ("plain", 0.0, None), ("cosface", 0.4, 0.08)])
def test_logits_match_oracle(margin, m, tau, precision, port):
    """Direct check of z = margin(s cos) (max|dz|/s <= 1e-3 bf16, 1e-5 fp32)."""
    C_, K, D, B = 12000, 3, 512, 192
    s = 1.0 if margin == "plain" else 64.0
    W, M = unit_rows_state(port, C_, K, D)
    X, labels = port.bench_inputs(C_, D, B, 1, 4)
    run_and_compare(port, C_, K, D, X, labels, W, M, margin, s, m, 0.2, precision, tau=tau,
                    mask_from_gpu=True)
