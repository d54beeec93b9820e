"""Seeded schedules of per-call StepConfig changes (pfc_gpu_set_step_config; the reference takes
a StepConfig per call, shardsim.hpp:166-168) against the oracle stepping the same state: each
schedule runs 6 steps on one context, every step drawing r (capacity grows and shrinks: column
buffers reallocated, graphs recaptured), the margin kind and scale (s > 64: per-row offsets),
the filter, momentum and weight decay; fp32 mode (filter decisions exact up to a cosine within
rounding of tau, replayed if one flips), buffers bit-exact, values within the fp32 contract.
PFC_CFG_FUZZ_SCHEDULES / PFC_CFG_FUZZ_SEED widen it for a one-off run."""
import os

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shards_to_rows
from tests.helpers import device_rows, make_shards, rel_fro, rel_max

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

MK = {"cosface": p.ADDITIVE_COSINE, "arcface": p.ADDITIVE_ANGULAR}


def _schedules(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        steps = []
        for _ in range(6):
            mk = str(rng.choice(["cosface", "arcface"]))
            s = float(rng.choice([32.0, 64.0, 96.0, 128.0]))
            m = 0.4 if mk == "cosface" else 0.5
            steps.append((float(rng.choice([0.05, 0.1, 0.2, 0.35])), mk, s, m,
                          0.1 if rng.random() < 0.3 else None, float(rng.choice([0.0, 0.5, 0.9])),
                          float(rng.choice([0.0, 5e-4]))))
        out.append((f"sched{i:02d}", int(rng.integers(6000, 20000)), int(rng.choice([1, 2, 4])),
                    int(rng.choice([128, 256])), int(rng.integers(40, 160)), steps))
    return out


SCHED = _schedules(int(os.environ.get("PFC_CFG_FUZZ_SCHEDULES", "3")),
                   int(os.environ.get("PFC_CFG_FUZZ_SEED", "5")))


@pytest.mark.parametrize("sched", SCHED, ids=[s[0] for s in SCHED])
def test_config_schedule(sched, port):
    name, C_, K, D, B, steps = sched
    W = port.init_centers(C_, K, D, 2)
    M = np.zeros_like(W)
    r0, mk0, s0, m0, tau0, mu0, wd0 = steps[0]
    cfg0 = p.StepConfig(r=r0, margin=p.MarginConfig(MK[mk0], s0, m0), filter_threshold=tau0,
                        momentum=mu0, weight_decay=wd0)
    sh = make_shards(W, M, C_, K, D, cfg0, B, p.PRECISION_FP32, flags=p.FLAG_DEBUG_LOGITS)
    fw = 1.0
    for step, (r, mk, s, m, tau, mu, wd) in enumerate(steps):
        cfg = p.StepConfig(r=r, margin=p.MarginConfig(MK[mk], s, m), filter_threshold=tau,
                           momentum=mu, weight_decay=wd, lr=0.1)
        ocfg = OracleCfg(r=r, margin=mk, scale=s, m=m, filter_threshold=tau, lr=0.1, momentum=mu,
                         weight_decay=wd)
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        cap = -(-int(np.ceil(C_ * r - 1e-9)) // K)  # buffer_capacity, sampler.hpp:50-57
        blk = -(-C_ // K)
        if np.bincount(np.unique(labels) // blk, minlength=K).max() > cap:
            continue  # a CapacityError draw: the reference throws before touching the state
        stream = port.make_stream("iteration", step)
        W0, M0 = W.copy(), M.copy()
        res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
        ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream, want_extra=tau is not None)
        assert sh.capacity == ref["buffers"].shape[1], (name, step)
        for k, buf in enumerate(res.buffers):
            assert np.array_equal(buf.class_indices, ref["buffers"][k]), (name, step, k)
        if tau is not None:
            z = sh.debug_logits(B).transpose(1, 0, 2)
            gmask = np.isneginf(z)
            pos = np.zeros_like(gmask)
            for b, y in enumerate(labels):
                k = y // blk
                pos[k, b, np.searchsorted(ref["buffers"][k][:ref["npos"][k]], y)] = True
            flips = gmask != ((ref["cos"] > tau) & ~pos)
            if flips.any():
                assert np.all(np.abs(ref["cos"][flips] - tau) < 1e-5), (name, step)
                W, M = W0.copy(), M0.copy()
                ref = port.step(ocfg, C_, K, D, W, M, X, labels, 1, stream, mask=gmask)
        f = max(1.0, s / 64.0)
        fw = max(fw, f)
        Wd, _ = device_rows(sh, C_, K, D)
        rows = np.unique(ref["buffers"].ravel())
        assert abs(res.loss - ref["loss"]) / abs(ref["loss"]) <= 1e-6 * f, (name, step)
        assert rel_fro(res.d_features, ref["dX"]) <= 1e-5 * f, (name, step)
        assert rel_max(Wd[rows], shards_to_rows(W, C_, K, D)[rows]) <= 1e-6 * fw * fw, (name, step)
    sh.close()
