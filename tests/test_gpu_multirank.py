"""GPU: the library's own N > 1 rank path, executed on one B200 (VERDICT r1 missing #1).

R ranks run as R contexts of this process on cuda:0 (one host thread each) joined by the
library's loopback communicator (comm.cuh, pfc_gpu_loopback_id): every collective the NCCL
build issues -- label / X all-gather, the stats exchange (all-gather of the per-row sums,
all-reduce of z_pos and of the positive-present flags), the per-row offset max, the dX
reduce-scatter or all-reduce -- is executed with the same buffers and counts, host-synchronised
(no kernel waits on another rank) and summed in ascending rank order.  Checked against the
oracle's single-process K-shard step (reference: shardsim.hpp:284-299, 320-328, 387-399; per-
shard fork(k), sampler.hpp:117):

  * sampled buffers of every rank's shards bit-exact, loss identical on every rank;
  * loss / dX / W' within the contract of tests/test_gpu_step.py, at R = 2, 4, 8;
  * the device path (rank slices, all-gather + reduce-scatter) equals the host drop-in bitwise;
  * nccl_bytes = the closed form of the protocol; wire_bytes = the reference cost model's ring
    form (costmodel.hpp:37-69) applied to the collectives issued.
"""
import json
import os
import threading

import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, fnv64, shard_bounds, shards_to_rows
from tests.helpers import rel_fro, rel_max

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

TOL = {p.PRECISION_FP32: (1e-6, 1e-5, 3e-5, 1e-6), p.PRECISION_BF16: (1e-4, 1e-2, 1e-2, 1e-3),
       p.PRECISION_TF32: (2e-5, 1e-3, 2.5e-3, 2e-4)}
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RESULTS = os.path.join(os.path.dirname(os.path.dirname(__file__)), "gpurun_out", "multirank.jsonl")


def run_ranks(R, fn, timeout=900):
    """fn(rank) on R threads (the loopback ranks); re-raises the first failure."""
    out, err = [None] * R, [None] * R

    def work(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e
    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    return out


def shard_block(W, C_, K, D, k):
    off = 0
    for kk, (lo, hi) in enumerate(shard_bounds(C_, K)):
        n = D * (hi - lo)
        if kk == k:
            return W[off:off + n].reshape(D, hi - lo)
        off += n


def protocol_bytes(R, B, D, f32_stats, filt, exact, host):
    """Closed form of the collectives one step issues (pfc_gpu.cu run_pipeline / step entry
    points), per rank = the larger of send / receive buffer of each call, and the ring model of
    the reference's cost model summed over ranks ((R-1) S per gather / scatter, 2 (R-1) S per
    all-reduce, costmodel.hpp:37-69)."""
    sb = 4 if f32_stats else 8  # the tensor-core modes exchange fp32 statistics, fp32 mode fp64
    calls = [("ag", R * B * sb), ("ar", 8 * B)]          # row sums (rank-major), z_pos
    if filt:
        calls.append(("ar", 4 * B))                      # positive-present flags
    if exact:
        calls.append(("ar", 4 * B))                      # per-row offsets (max)
    if host:
        calls.append(("ar", 4 * B * D))                  # full d_features on every rank
    else:
        calls += [("ag", 4 * B * D), ("ag", 8 * B), ("rs", 4 * B * D)]  # X, labels, dX
    nccl = sum(S for _, S in calls)
    wire = sum((2 if kind == "ar" else 1) * (R - 1) * S for kind, S in calls)
    return nccl, wire


CASES = [  # name, C, K, D, B, r, margin, s, m, tau, precision, R list
    ("arc_40k_bf16", 40000, 8, 512, 256, 0.1, "arcface", 64.0, 0.5, None, p.PRECISION_BF16, (2, 4, 8)),
    ("arc_40k_fp32", 40000, 8, 512, 256, 0.1, "arcface", 64.0, 0.5, None, p.PRECISION_FP32, (2, 4, 8)),
    ("cos_filter_fp32", 12000, 4, 256, 128, 0.3, "cosface", 64.0, 0.4, 0.08, p.PRECISION_FP32, (2, 4)),
    ("cos_s256_exact", 16000, 4, 256, 128, 0.2, "cosface", 256.0, 0.4, None, p.PRECISION_FP32, (2, 4)),
    ("full_fc_r1", 6000, 4, 128, 96, 1.0, "cosface", 64.0, 0.4, None, p.PRECISION_BF16, (4,)),
    ("arc_40k_tf32", 40000, 8, 512, 256, 0.1, "arcface", 64.0, 0.5, None, p.PRECISION_TF32, (2, 8)),
    ("cos_d768_bf16", 12000, 4, 768, 128, 0.2, "cosface", 64.0, 0.4, None, p.PRECISION_BF16, (2,)),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_loopback_ranks_match_oracle(case, port):
    name, C_, K, D, B, r, margin, s, m, tau, prec, Rs = case
    mk = {"arcface": p.ADDITIVE_ANGULAR, "cosface": p.ADDITIVE_COSINE}[margin]
    cfg = p.StepConfig(r=r, margin=p.MarginConfig(mk, s, m), filter_threshold=tau, lr=0.1)
    ocfg = OracleCfg(r=r, margin=margin, scale=s, m=m, filter_threshold=tau, lr=0.1)
    W0 = port.init_centers(C_, K, D, 1)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    stream = port.make_stream("iteration", 0)
    Wr, Mr = W0.copy(), np.zeros_like(W0)
    ref = port.step(ocfg, C_, K, D, Wr, Mr, X, labels, 1, stream)
    Wrows = shards_to_rows(Wr, C_, K, D)
    tl, tdf, tdm, tw = TOL[prec]
    for R in Rs:
        lid = p.loopback_id()

        def rank(rk, device_path):
            sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=prec,
                                rank=rk, world_size=R, nccl_id=lid)
            for k in sh.local_shards:
                sh.set_shard(k, shard_block(W0, C_, K, D, k))
            if device_path:
                bl = B // R
                xl = torch.from_numpy(np.ascontiguousarray(X[:, rk * bl:(rk + 1) * bl].T)).float().cuda()
                ll = torch.from_numpy(labels[rk * bl:(rk + 1) * bl].copy()).cuda()
                dx = torch.empty(bl, D, device="cuda")
                torch.cuda.synchronize()
                o = sh.step_device(xl.data_ptr(), ll.data_ptr(), bl, dx.data_ptr(), cfg,
                                   p.SeededRng(1, stream))
                res = (o.loss, dx.cpu().numpy().T.astype(np.float64), o.nccl_bytes, o.wire_bytes)
            else:
                st = sh.step_host(X, labels, cfg, p.SeededRng(1, stream))
                res = (st.loss, st.d_features, st.nccl_bytes, st.wire_bytes)
            bufs = {b.shard_id: (b.class_indices.copy(), b.num_positives) for b in sh.buffers()}
            Wd = {k: sh.get_shard(k)[0] for k in sh.local_shards}
            sh.close()
            return res, bufs, Wd

        host = run_ranks(R, lambda rk: rank(rk, False))
        dev = run_ranks(R, lambda rk: rank(rk, True))
        exact = s > 64.0
        nccl_h, wire_h = protocol_bytes(R, B, D, prec != p.PRECISION_FP32, tau is not None, exact, True)
        nccl_d, wire_d = protocol_bytes(R, B, D, prec != p.PRECISION_FP32, tau is not None, exact, False)
        losses = [h[0][0] for h in host]
        assert len(set(losses)) == 1, losses  # every rank reports the same global loss
        dX = host[0][0][1]
        for h in host:
            assert np.array_equal(h[0][1], dX)   # the full d_features on every rank
            assert (h[0][2], h[0][3]) == (nccl_h, wire_h)
        dX_dev = np.concatenate([d[0][1] for d in dev], axis=1)
        assert np.array_equal(dX_dev, dX)        # slices of the same sum, bit for bit
        assert all(d[0][0] == losses[0] for d in dev)
        for d, h in zip(dev, host):
            assert (d[0][2], d[0][3]) == (nccl_d, wire_d)
            assert all(np.array_equal(d[2][k], h[2][k]) for k in h[2])  # same updated shards
        got_W = np.empty_like(Wrows)
        for h in host:
            for k, (idx, npos) in h[1].items():
                assert np.array_equal(idx, ref["buffers"][k]) and npos == ref["npos"][k]
            for k, w in h[2].items():
                lo, hi = shard_bounds(C_, K)[k]
                got_W[lo:hi] = w.T
        rows = np.unique(ref["buffers"].ravel())
        rec = {"case": name, "R": R, "loss_rel": abs(losses[0] - ref["loss"]) / abs(ref["loss"]),
               "dX_fro": rel_fro(dX, ref["dX"]), "dX_max": rel_max(dX, ref["dX"]),
               "W_max": rel_max(got_W[rows], Wrows[rows]), "nccl_bytes_host": nccl_h,
               "wire_bytes_host": wire_h, "nccl_bytes_device": nccl_d, "wire_bytes_device": wire_d}
        os.makedirs(os.path.dirname(RESULTS), exist_ok=True)
        with open(RESULTS, "a") as f:
            f.write(json.dumps(rec) + "\n")
        assert rec["loss_rel"] <= tl and rec["dX_fro"] <= tdf and rec["dX_max"] <= tdm, rec
        assert rec["W_max"] <= tw, rec
        # unsampled rows untouched
        untouched = np.setdiff1d(np.arange(C_), rows)
        W0f = shards_to_rows(W0, C_, K, D).astype(np.float32).astype(np.float64)  # device fp32
        assert np.array_equal(got_W[untouched], W0f[untouched])


@pytest.mark.parametrize("R", [2, 8])
def test_loopback_northstar_golden(R, port):
    """2M classes, K = 8, B = 1024, d = 512, ArcFace, bf16 -- the bench configuration -- as R
    loopback ranks against the compiled reference's step (tests/golden/northstar.json)."""
    with open(os.path.join(GOLDEN, "northstar.json")) as f:
        g = json.load(f)
    arr = np.load(os.path.join(GOLDEN, "step_webface2m_k8_d512.npz"))
    C_, K, D, B = g["C"], g["K"], g["D"], g["B"]
    cfg = p.StepConfig(r=g["r"], margin=p.MarginConfig.arcface_style(64.0, g["m"]), lr=0.1)
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    stream = p.make_stream("iteration", 0)
    lid = p.loopback_id()
    rows, want = arr["rows_sub"], arr["W_sub"]
    layout = p.ShardLayout(C_, K)

    def rank(rk):
        sh = p.CenterShards(layout, D, cfg, max_batch=B, precision=p.PRECISION_BF16, rank=rk,
                            world_size=R, nccl_id=lid)
        sh.init_center_shards(1)
        res = sh.step_host(X, labels, cfg, p.SeededRng(1, stream))
        fnvs = {b.shard_id: (fnv64(b.class_indices), b.num_positives) for b in sh.buffers()}
        got = {}
        for k in sh.local_shards:
            lo, hi = layout.owned_begin(k), layout.owned_end(k)
            msk = (rows >= lo) & (rows < hi)
            if msk.any():
                w, _ = sh.get_shard(k)
                got[k] = (msk, w[:, rows[msk] - lo].T)
        sh.close()
        return res.loss, res.d_features, fnvs, got

    out = run_ranks(R, rank)
    for k in range(K):
        fn, npos = next(o[2][k] for o in out if k in o[2])
        assert fn == g["buffers_fnv"][k] and npos == g["npos"][k]
    loss, dX = out[0][0], out[0][1]
    got_W = np.empty_like(want)
    for o in out:
        assert o[0] == loss and np.array_equal(o[1], dX)
        for msk, w in o[3].values():
            got_W[msk] = w
    tl, tdf, tdm, tw = TOL[p.PRECISION_BF16]
    rec = {"case": "webface2m_k8 loopback", "R": R, "loss_rel": abs(loss - g["loss"]) / abs(g["loss"]),
           "dX_fro": rel_fro(dX, arr["dX"]), "dX_max": rel_max(dX, arr["dX"]),
           "W_max": rel_max(got_W, want)}
    with open(RESULTS, "a") as f:
        f.write(json.dumps(rec) + "\n")
    assert rec["loss_rel"] <= tl and rec["dX_fro"] <= tdf and rec["dX_max"] <= tdm, rec
    assert rec["W_max"] <= tw, rec


@pytest.mark.parametrize("transport", ["nccl", "loopback"])
@pytest.mark.parametrize("precision", [p.PRECISION_BF16, p.PRECISION_FP32], ids=["bf16", "fp32"])
def test_collective_path_one_rank(transport, precision, port):
    """The N > 1 collective path on a real NCCL communicator (NCCL never ran).

    NCCL will not put two ranks on one GPU, so PFC_FLAG_FORCE_COLLECTIVES runs every collective
    of the rank path -- all-gather of X and labels, the statistics all-gather, z_pos and flag
    all-reduces, the per-row offset max, the dX all-reduce (host drop-in, inside the captured
    graph) and the dX reduce-scatter (device path), the diagnostics merges -- through a 1-rank
    communicator.  Same values as the plain one-rank context (bit-identical: every 1-rank
    collective is a copy); the byte counters follow the protocol closed form at R = 1."""
    C_, K, D, B = 16000, 4, 256, 128
    tau = 0.05 if precision == p.PRECISION_FP32 else None
    for s in (64.0, 128.0):  # fixed offset, then per-row offsets (the max all-reduce)
        cfg = p.StepConfig(r=0.2, margin=p.MarginConfig.cosface_style(s, 0.4), filter_threshold=tau,
                           lr=0.1)
        W0 = port.init_centers(C_, K, D, 1)
        X, labels = port.bench_inputs(C_, D, B, 1, 0)
        outs = []
        for flags in (0, p.FLAG_FORCE_COLLECTIVES):
            nid = None
            if flags:
                nid = p.nccl_unique_id() if transport == "nccl" else p.loopback_id()
            sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=precision,
                                world_size=1, nccl_id=nid, flags=flags)
            for k in range(K):
                sh.set_shard(k, shard_block(W0, C_, K, D, k))
            st = sh.step_host(X, labels, cfg, p.SeededRng(1, port.make_stream("iteration", 0)))
            xl = torch.from_numpy(np.ascontiguousarray(X.T)).float().cuda()
            ll = torch.from_numpy(labels.copy()).cuda()
            dx = torch.empty(B, D, device="cuda")
            torch.cuda.synchronize()
            o = sh.step_device(xl.data_ptr(), ll.data_ptr(), B, dx.data_ptr(), cfg,
                               p.SeededRng(1, port.make_stream("iteration", 1)))
            dg = sh.diagnostics(X, labels)
            outs.append((st.loss, st.d_features, o.loss, dx.cpu().numpy(),
                         [sh.get_shard(k)[0] for k in range(K)], dg, st.nccl_bytes,
                         o.nccl_bytes))
            sh.close()
        a, b = outs
        assert a[0] == b[0] and np.array_equal(a[1], b[1])
        assert a[2] == b[2] and np.array_equal(a[3], b[3])
        assert all(np.array_equal(x, y) for x, y in zip(a[4], b[4]))
        assert a[5] == b[5]
        exact = s > 64.0
        assert (a[6], a[7]) == (0, 0)
        assert b[6] == protocol_bytes(1, B, D, precision != p.PRECISION_FP32, tau is not None,
                                      exact, True)[0]
        assert b[7] == protocol_bytes(1, B, D, precision != p.PRECISION_FP32, tau is not None,
                                      exact, False)[0]
