"""CPU, world_size 2 (gloo): the N-rank decomposition of the step that libpfc_gpu.so runs over
NCCL / the loopback communicator (pfc_gpu.cu: run_pipeline, pfc_gpu_step_device), emulated rank by
rank in fp64 numpy with exactly its exchanges and its softmax formulation, against the oracle's
single-process K-shard step:

  rank r owns reference shards [r*K/R, (r+1)*K/R) and rows [r*B/R, (r+1)*B/R) of the batch
  1. all-gather X_local, labels_local (rank-major = all_gather_features, shardsim.hpp:86-115)
  2. rank-local sampling of its own shards (fork(k) with the GLOBAL k, sampler.hpp:117)
  3. softmax offset o_b: fixed max(0, s - 40) for s <= 64, else the rank-local max over
     unmasked logits all-reduced with MAX (collective 1, shardsim.hpp:284-299)
  4. rank-local sums of E = exp(z - o) all-gathered [R][B] and summed in ascending rank order,
     z_pos all-reduced (SUM: only the owner contributes), with a filter the positive-present
     flags all-reduced (collective 2, shardsim.hpp:320-338); loss = log S + o - z_pos
  5. G = diag(s / (B S)) E + the positive correction delta_b (epilogues.cuh header): dX partial
     with the rank's own feat_proj share, dW^T = E^T (rowscale x^) + delta x^, fused update
  6. reduce-scatter of the dX partials (collective 3, shardsim.hpp:387-399)
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _margin(c, pos, kind, s, m):
    if kind == "cosface":
        return s * (c - m) if pos else s * c
    if not pos:
        return s * c
    cc = min(max(c, -1 + 1e-7), 1 - 1e-7)
    return s * np.cos(np.arccos(cc) + m)


def _dmargin(c, pos, kind, s, m):
    if kind == "cosface" or not pos:
        return s
    if c <= -1 + 1e-7 or c >= 1 - 1e-7:
        return 0.0
    return s * np.sin(np.arccos(c) + m) / np.sqrt(1 - c * c)


CASES = [  # C, K, B, D, r, kind, s, m, tau
    (400, 4, 32, 16, 0.5, "arcface", 64.0, 0.5, None),   # fixed offset
    (400, 4, 32, 16, 0.5, "cosface", 160.0, 0.4, None),  # per-row offsets (s > 64)
    (300, 2, 24, 16, 1.0, "cosface", 64.0, 0.4, 0.05),   # filter: hasval exchange
]


def _rank_step(o, rank, world, case):
    from oracle.oracle import OracleCfg, shard_bounds, shards_to_rows
    C_, K, B, D, r, kind, s, m, tau = case
    lr, mu, wd = 0.1, 0.9, 5e-4
    X, labels = o.bench_inputs(C_, D, B, 1, 0)  # D x B, the global batch
    stream = o.make_stream("iteration", 0)
    W0 = o.init_centers(C_, K, D, 1)
    Wrows = shards_to_rows(W0, C_, K, D)        # class rows, fp64
    Mrows = np.zeros_like(Wrows)
    bl = B // world
    # -- 1. rank-local inputs, all-gathered rank-major
    x_local = torch.from_numpy(np.ascontiguousarray(X[:, rank * bl:(rank + 1) * bl].T))
    l_local = torch.from_numpy(labels[rank * bl:(rank + 1) * bl].copy())
    xg = [torch.zeros_like(x_local) for _ in range(world)]
    lg = [torch.zeros_like(l_local) for _ in range(world)]
    dist.all_gather(xg, x_local)
    dist.all_gather(lg, l_local)
    Xg = torch.cat(xg).numpy()                  # [B][D]
    Lg = torch.cat(lg).numpy()
    assert np.array_equal(Xg, X.T) and np.array_equal(Lg, labels)
    # -- 2. rank-local sampling of shards [k0, k0+nk)
    nk = K // world
    k0 = rank * nk
    bufs, npos = o.build_buffers(C_, K, Lg, r, 1, stream)
    cols = bufs[k0:k0 + nk].ravel()              # local concatenated buffer (global ids)
    blk = (C_ + K - 1) // K
    pos_col = np.full(B, -1)
    for b, y in enumerate(Lg):
        ks = y // blk
        if k0 <= ks < k0 + nk:
            row = bufs[ks, :npos[ks]]
            pos_col[b] = (ks - k0) * bufs.shape[1] + int(np.searchsorted(row, y))
    xn = np.linalg.norm(Xg, axis=1)
    xh = Xg / np.maximum(xn, 1e-12)[:, None]
    wsel = Wrows[cols]
    wn = np.linalg.norm(wsel, axis=1)
    wh = wsel / np.maximum(wn, 1e-12)[:, None]
    cos = xh @ wh.T                               # [B][ncols]
    z = s * cos
    zpos = np.zeros(B)
    pos = np.zeros_like(cos, dtype=bool)
    for b in range(B):
        if pos_col[b] >= 0:
            z[b, pos_col[b]] = _margin(cos[b, pos_col[b]], True, kind, s, m)
            zpos[b] = z[b, pos_col[b]]
            pos[b, pos_col[b]] = True
    masked = (cos > tau) & ~pos if tau is not None else np.zeros_like(pos)
    # -- 3. softmax offset
    if s <= 64.0:
        off = np.full(B, max(0.0, s - 40.0))
    else:
        lm = np.where(masked, -np.inf, z).max(axis=1)
        om = torch.from_numpy(np.where(np.isfinite(lm), lm, -1e30))
        dist.all_reduce(om, op=dist.ReduceOp.MAX)
        off = om.numpy()
    # -- 4. rank-local sums of E, exchanged; z_pos and hasval all-reduced
    E = np.where(masked, 0.0, np.exp(z - off[:, None]))
    ls = E.sum(axis=1)
    LS = [torch.zeros(B, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(LS, torch.from_numpy(ls))
    zp = torch.from_numpy(zpos)
    dist.all_reduce(zp)
    if tau is not None:
        hv = torch.from_numpy((~masked).any(axis=1).astype(np.int32))
        dist.all_reduce(hv)
        assert (hv.numpy() > 0).all()
    S = np.zeros(B)
    for rr in range(world):                       # ascending rank order
        S += LS[rr].numpy()
    zpos = zp.numpy()
    loss = float(np.mean(np.log(S) + off - zpos))
    # -- 5. G = diag(rowscale) E + positive correction
    rowscale = s / (B * S)
    delta = np.zeros(B)
    for b in range(B):
        if pos_col[b] >= 0:
            c = cos[b, pos_col[b]]
            pp = np.exp(zpos[b] - off[b]) / S[b]
            delta[b] = (pp - 1.0) / B * _dmargin(c, True, kind, s, m) - rowscale[b] * E[b, pos_col[b]]
    racc = rowscale[:, None] * (E @ wh)           # sum_j g_bj w^_j over negatives ...
    for b in range(B):
        if pos_col[b] >= 0:
            racc[b] += delta[b] * wh[pos_col[b]]    # ... plus the positive's exact gradient
    fproj = np.sum(racc * xh, axis=1)              # feat_proj = x^ . r (c = x^ . w^)
    dx_part = (racc - fproj[:, None] * xh) / np.maximum(xn, 1e-12)[:, None]
    dwt = E.T @ (rowscale[:, None] * xh)
    for b in range(B):
        if pos_col[b] >= 0:
            dwt[pos_col[b]] += delta[b] * xh[b]
    cproj = np.sum(dwt * wh, axis=1)               # center_proj = w^ . dwt
    dW = (dwt - cproj[:, None] * wh) / np.maximum(wn, 1e-12)[:, None]
    gg = dW + wd * wsel
    v = mu * Mrows[cols] + gg
    Wnew = wsel - lr * v
    # -- 6. reduce-scatter of dX (gloo: all-reduce + owner slice)
    dxt = torch.from_numpy(np.ascontiguousarray(dx_part))
    dist.all_reduce(dxt)
    dx_mine = dxt.numpy()[rank * bl:(rank + 1) * bl]
    # -- compare with the single-process K-shard oracle step
    Wref, Mref = W0.copy(), np.zeros_like(W0)
    ref = o.step(OracleCfg(r=r, margin=kind, scale=s, m=m, filter_threshold=tau, lr=lr,
                           momentum=mu, weight_decay=wd), C_, K, D, Wref, Mref, X, labels, 1,
                 stream)
    Wref_rows = shards_to_rows(Wref, C_, K, D)
    return {
        "case": list(case), "rank": rank,
        "loss_rel": abs(loss - ref["loss"]) / abs(ref["loss"]),
        "dx_rel": float(np.abs(dx_mine - ref["dX"].T[rank * bl:(rank + 1) * bl]).max()
                        / np.abs(ref["dX"]).max()),
        "w_rel": float(np.abs(Wnew - Wref_rows[cols]).max() / np.abs(Wref_rows).max()),
        "buffers_local": bool(np.array_equal(bufs[k0:k0 + nk], ref["buffers"][k0:k0 + nk])),
        "owned": [shard_bounds(C_, K)[k] for k in range(k0, k0 + nk)],
    }


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from oracle.oracle import Oracle
        o = Oracle("port")
        q.put([_rank_step(o, rank, world, case) for case in CASES])
    finally:
        dist.destroy_process_group()


def test_two_rank_decomposition_equals_oracle():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    outs = [r for _ in procs for r in q.get(timeout=180)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for r in outs:
        assert r["buffers_local"]
        assert r["loss_rel"] < 1e-12, r
        assert r["dx_rel"] < 1e-10, r
        assert r["w_rel"] < 1e-12, r
    assert sorted(o["rank"] for o in outs) == sorted([0, 1] * len(CASES))
