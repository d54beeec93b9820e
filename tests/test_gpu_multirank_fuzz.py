"""Seeded sweep of the N > 1 rank path (loopback communicator, tests/test_gpu_multirank.py)
against the oracle's single-process K-shard step: random C (short last shard), R in {2, 4, 8},
K a multiple of R, B a multiple of R (not of 32), D, r, margins and the filter (fp32).  Per case:
the buffers of every rank's shards bit-exact, every rank's loss equal, the full d_features equal
on every rank, and loss / dX / W' within the step contract (tests/test_gpu_fuzz.py scaling for
the tensor-core modes).  PFC_MR_FUZZ_CASES / PFC_MR_FUZZ_SEED widen it for a one-off run."""
import math
import os

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shard_bounds, shards_to_rows
from tests.helpers import rel_fro, rel_max
from tests.test_gpu_multirank import run_ranks, shard_block

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TOL = {p.PRECISION_FP32: (1e-6, 1e-5, 3e-5, 1e-6), p.PRECISION_BF16: (1e-4, 1e-2, 1e-2, 1e-3),
       p.PRECISION_TF32: (2e-5, 1e-3, 2.5e-3, 2e-4)}
MK = {"cosface": (p.ADDITIVE_COSINE, 0.4), "arcface": (p.ADDITIVE_ANGULAR, 0.5)}


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        R = int(rng.choice([2, 4, 8]))
        K = R * int(rng.integers(1, 3))
        B = R * int(rng.integers(8, 80))
        C_ = int(rng.integers(3000, 30000))
        D = int(rng.choice([128, 256, 512]))
        margin = str(rng.choice(["cosface", "arcface"]))
        prec = [p.PRECISION_FP32, p.PRECISION_BF16, p.PRECISION_TF32][i % 3]
        tau = 0.15 if (prec == p.PRECISION_FP32 and i % 2 == 1) else None
        r = float(min(1.0, max(math.ceil((2.5 * B / C_ + 0.02) * 100) / 100,
                               round(float(rng.uniform(0.05, 0.5)), 2))))
        out.append((f"mr{i:02d}_R{R}_K{K}_C{C_}_B{B}_D{D}_{margin}_p{prec}" + ("_tau" if tau else ""),
                    R, K, C_, B, D, margin, prec, tau, r))
    return out


CASES = _cases(int(os.environ.get("PFC_MR_FUZZ_CASES", "6")), int(os.environ.get("PFC_MR_FUZZ_SEED", "31")))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_multirank_fuzz(case, port):
    name, R, K, C_, B, D, margin, prec, tau, r = case
    kind, m = MK[margin]
    cfg = p.StepConfig(r=r, margin=p.MarginConfig(kind, 64.0, m), filter_threshold=tau, lr=0.1)
    ocfg = OracleCfg(r=r, margin=margin, scale=64.0, m=m, filter_threshold=tau, lr=0.1)
    W0 = port.init_centers(C_, K, D, 1)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    cap = math.ceil(math.ceil(C_ * r - 1e-9) / K)
    blk = -(-C_ // K)
    if np.bincount(np.unique(labels) // blk, minlength=K).max() > cap or C_ - (K - 1) * blk < cap:
        pytest.skip("the reference rejects this draw (CapacityError): covered elsewhere")
    stream = port.make_stream("iteration", 0)
    Wr, Mr = W0.copy(), np.zeros_like(W0)
    ref = port.step(ocfg, C_, K, D, Wr, Mr, X, labels, 1, stream, want_extra=tau is not None)
    lid = p.loopback_id()
    flags = p.FLAG_DEBUG_LOGITS if tau is not None else 0

    def rank(rk):
        sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=prec, rank=rk,
                            world_size=R, nccl_id=lid, flags=flags)
        for k in sh.local_shards:
            sh.set_shard(k, shard_block(W0, C_, K, D, k))
        st = sh.step_host(X, labels, cfg, p.SeededRng(1, stream))
        bufs = {b.shard_id: (b.class_indices.copy(), b.num_positives) for b in sh.buffers()}
        Wd = {k: sh.get_shard(k)[0] for k in sh.local_shards}
        z = sh.debug_logits(B) if tau is not None else None
        loc = list(sh.local_shards)
        sh.close()
        return st.loss, st.d_features, bufs, Wd, z, loc

    out = run_ranks(R, rank)
    if tau is not None:
        # the filter decides cos > tau on the mode's own cosines: a decision may differ from the
        # fp64 reference only for a cosine within that rounding of tau (fp32 ~1e-7); the values
        # are then compared with the GPU's decisions replayed in the oracle
        cap = ref["buffers"].shape[1]
        gmask = np.zeros((K, B, cap), dtype=bool)
        for o in out:
            for i, k in enumerate(o[5]):
                gmask[k] = np.isneginf(o[4][:, i, :])
        pos = np.zeros_like(gmask)
        for b, y in enumerate(labels):
            k = y // blk
            pos[k, b, np.searchsorted(ref["buffers"][k][:ref["npos"][k]], y)] = True
        flips = gmask != ((ref["cos"] > tau) & ~pos)
        if flips.any():
            band = 1e-5 if prec == p.PRECISION_FP32 else 2.0 ** -7
            assert np.all(np.abs(ref["cos"][flips] - tau) < band), np.abs(ref["cos"][flips] - tau).max()
            Wr, Mr = W0.copy(), np.zeros_like(W0)
            ref = port.step(ocfg, C_, K, D, Wr, Mr, X, labels, 1, stream, mask=gmask)
    assert len({o[0] for o in out}) == 1
    for o in out[1:]:
        assert np.array_equal(o[1], out[0][1])
    got_W = np.empty_like(shards_to_rows(Wr, C_, K, D))
    for o in out:
        for k, (idx, npos) in o[2].items():
            assert np.array_equal(idx, ref["buffers"][k]) and npos == ref["npos"][k], (name, k)
        for k, w in o[3].items():
            lo, hi = shard_bounds(C_, K)[k]
            got_W[lo:hi] = w.T
    tl, tdf, tdm, tw = TOL[prec]
    if prec != p.PRECISION_FP32 and D < 512:
        f = math.sqrt(512.0 / D)
        tl, tdf, tdm, tw = tl * f, tdf * f, tdm * f, tw * f
    if prec != p.PRECISION_FP32 and B < 64:
        tw *= 64.0 / B
    rows = np.unique(ref["buffers"].ravel())
    Wrows = shards_to_rows(Wr, C_, K, D)
    loss, dX = out[0][0], out[0][1]
    assert abs(loss - ref["loss"]) / abs(ref["loss"]) <= tl, (name, loss, ref["loss"])
    assert rel_fro(dX, ref["dX"]) <= tdf and rel_max(dX, ref["dX"]) <= tdm, name
    assert rel_max(got_W[rows], Wrows[rows]) <= tw, name
