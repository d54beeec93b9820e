"""GPU: a seeded sweep of step configurations against the oracle (same contract as
test_gpu_step.py), two steps each (the second update carries momentum).  The 16 cases are drawn once from a fixed generator, so every run tests the
same ones; they cover the paths the hand-picked cases may miss:
  * class counts that leave a ragged last tile and a short last shard;
  * batches that are not multiples of 32 (the logits epilogue's fragment path: a warp's 32 rows
    straddle the batch end);
  * D not a multiple of 64;
  * K = 1..7, r up to 1.0 (full sampling), CosFace / ArcFace / plain margins, the filter.
bf16 and tf32 are checked where their contracts apply (128 <= D <= 1024, no filter: the tensor-core
paths flip the filter's mask decisions within their rounding of tau, and tiny D is a smoke bound
only; D > 1024 must be refused with ConfigError); fp32 everywhere.
"""
import json
import math
import os

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleError, shards_to_rows
from tests.helpers import device_rows, make_shards, oracle_cfg, rel_fro, rel_max, step_cfg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TOL = {p.PRECISION_FP32: (1e-6, 1e-5, 3e-5, 1e-6), p.PRECISION_BF16: (1e-4, 1e-2, 1e-2, 1e-3),
       p.PRECISION_TF32: (2e-5, 1e-3, 2.5e-3, 2e-4)}
PREC_NAME = {p.PRECISION_FP32: "fp32", p.PRECISION_BF16: "bf16", p.PRECISION_TF32: "tf32"}
RESULTS = os.path.join(os.path.dirname(os.path.dirname(__file__)), "gpurun_out", "fuzz.jsonl")


def _cases(n=16, seed=2203):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        K = int(rng.integers(1, 8))
        C_ = int(rng.integers(800, 24000))
        B = int(rng.integers(17, 520))
        D = int(rng.choice([72, 128, 200, 256, 328, 384, 520]))
        margin = str(rng.choice(["cosface", "arcface", "plain"]))
        m = {"cosface": 0.4, "arcface": 0.5, "plain": 0.0}[margin]
        tau = 0.2 if i % 4 == 3 else None
        # enough capacity for ~B/K distinct positives per shard (+ slack), else full sampling
        r_min = min(1.0, math.ceil((2.5 * B / C_ + 0.02) * 100) / 100)
        r = float(min(1.0, max(r_min, round(float(rng.uniform(0.05, 0.6)), 2))))
        if rng.random() < 0.15:
            r = 1.0
        out.append((f"fuzz{i:02d}_C{C_}_K{K}_B{B}_D{D}_{margin}_r{r}" + ("_tau" if tau else ""),
                    C_, K, B, D, r, margin, m, tau))
    return out


# PFC_FUZZ_CASES / PFC_FUZZ_SEED widen the sweep for a one-off run (profiles/r2/fuzz_wide.txt)
CASES = _cases(int(os.environ.get("PFC_FUZZ_CASES", "16")), int(os.environ.get("PFC_FUZZ_SEED", "2203")))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fuzz_step_matches_oracle(case, port):
    name, C_, K, B, D, r, mg, m, tau = case
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    stream = port.make_stream("iteration", 0)
    # a draw the reference rejects (a shard with more positives than capacity, or owning fewer
    # classes than capacity): the library must raise CapacityError with the reference's text
    cap = math.ceil(math.ceil(C_ * r - 1e-9) / K)
    blk = -(-C_ // K)
    per = np.bincount(np.unique(labels) // blk, minlength=K)
    owned = [min((k + 1) * blk, C_) - min(k * blk, C_) for k in range(K)]
    if per.max() > cap or min(owned) < cap:
        W0 = port.init_centers(C_, K, D, 1)
        with pytest.raises(OracleError) as ref_err:
            port.step(oracle_cfg(mg, m, r, tau), C_, K, D, W0.copy(), np.zeros_like(W0), X,
                      labels, 1, stream)
        sh = make_shards(W0, np.zeros_like(W0), C_, K, D, step_cfg(mg, m, r, tau), B,
                         p.PRECISION_FP32)
        with pytest.raises(p.CapacityError) as err:
            p.distributed_partial_step(sh, X, labels, step_cfg(mg, m, r, tau), p.SeededRng(1, stream))
        assert ref_err.value.kind == "CapacityError" and str(err.value) == ref_err.value.msg, (
            str(err.value), ref_err.value.msg)
        sh.close()
        return
    W0 = port.init_centers(C_, K, D, 1)
    # two steps (the second update carries momentum, mu * m != 0); the second only when its
    # labels also fit the shards' capacity
    W, M = W0.copy(), np.zeros_like(W0)
    refs = []
    for step in range(2):
        Xs, ls = (X, labels) if step == 0 else port.bench_inputs(C_, D, B, 1, step)
        if step > 0 and np.bincount(np.unique(ls) // blk, minlength=K).max() > cap:
            break
        st = port.make_stream("iteration", step)
        ref = port.step(oracle_cfg(mg, m, r, tau), C_, K, D, W, M, Xs, ls, 1, st)
        refs.append((Xs, ls, st, ref, shards_to_rows(W, C_, K, D), shards_to_rows(M, C_, K, D)))
    precisions = [p.PRECISION_FP32]
    if D > 1024:  # the tensor-core paths refuse it (dW clusters cover four 256-dim blocks)
        with pytest.raises(p.ConfigError, match="dim <= 1024"):
            make_shards(W0, np.zeros_like(W0), C_, K, D, step_cfg(mg, m, r, tau), B,
                        p.PRECISION_BF16)
    elif D >= 128 and tau is None:
        precisions += [p.PRECISION_BF16, p.PRECISION_TF32]
    for precision in precisions:
        tl, tdf, tdm, tw = TOL[precision]
        if precision != p.PRECISION_FP32 and D < 512:
            # the tensor-core contract is stated at D >= 512; a cosine of unit vectors whose
            # D elements are rounded independently errs as 1 / sqrt(D), so below 512 every bound
            # scales by sqrt(512 / D) (the 120-case sweep, profiles/r2/fuzz_wide.txt)
            f = math.sqrt(512.0 / D)
            tl, tdf, tdm, tw = tl * f, tdf * f, tdm * f, tw * f
        if precision != p.PRECISION_FP32 and B < 64:
            # W' is compared as max/max of the whole centres; its error is the operands'
            # rounding times the UPDATE, which grows as 1 / B (two steps with momentum)
            tw *= 64.0 / B
        sh = make_shards(W0, np.zeros_like(W0), C_, K, D, step_cfg(mg, m, r, tau), B, precision)
        for step, (Xs, ls, st, ref, Wr, Mr) in enumerate(refs):
            rows = np.unique(ref["buffers"].ravel())
            untouched = np.setdiff1d(np.arange(C_), rows)
            Wd0, Md0 = device_rows(sh, C_, K, D)
            res = p.distributed_partial_step(sh, Xs, ls, step_cfg(mg, m, r, tau), p.SeededRng(1, st))
            for k, buf in enumerate(res.buffers):
                assert np.array_equal(buf.class_indices, ref["buffers"][k]), (name, step, k)
                assert buf.num_positives == ref["npos"][k]
            Wd, Md = device_rows(sh, C_, K, D)
            rec = {"case": name, "precision": PREC_NAME[precision], "step": step,
                   "loss_rel": abs(res.loss - ref["loss"]) / abs(ref["loss"]),
                   "dX_fro": rel_fro(res.d_features, ref["dX"]),
                   "dX_maxmax": rel_max(res.d_features, ref["dX"]),
                   "W_maxmax": rel_max(Wd[rows], Wr[rows]), "mom_maxmax": rel_max(Md[rows], Mr[rows])}
            os.makedirs(os.path.dirname(RESULTS), exist_ok=True)
            with open(RESULTS, "a") as f:
                f.write(json.dumps(rec) + "\n")
            assert rec["loss_rel"] <= tl, rec
            assert rec["dX_fro"] <= tdf, rec
            assert rec["dX_maxmax"] <= tdm, rec
            assert rec["W_maxmax"] <= tw, rec
            if precision == p.PRECISION_FP32:
                assert rec["mom_maxmax"] <= 3e-5, rec
            assert np.array_equal(Wd[untouched], Wd0[untouched])
            assert np.array_equal(Md[untouched], Md0[untouched])
        sh.close()
