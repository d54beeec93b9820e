"""Generate the golden fixtures from the COMPILED REFERENCE (oracle/_ref/libpfc_ref.so).

Run here, where /root/reference exists:  make -C oracle && python tests/golden/make_golden.py
The reference ships no golden vectors, so these files — made by calling the
unmodified reference functions through oracle/ref_shim.cpp — pin both the plain-C oracle and the
GPU path.  Inputs follow the bench convention of SURVEY.md §8d / Appendix B:
  labels = SeededRng(1, make_stream("bench-labels", step)).next_below(C)
  X      = SeededRng(1, make_stream("bench-x", step)).next_normal()   (b-major, d inner)
  W      = init_center_shards(ShardLayout(C, K), D, 1)
  iteration rng = SeededRng(1, make_stream("iteration", step))
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, OracleCfg, OracleError, fnv64, shards_to_rows  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R = Oracle("reference")
P = Oracle("port")  # only for bench_inputs (a pure RNG function, pinned below by rng.json)



def rng_golden():
    g = {"make_stream": [], "draws": [], "fork": [], "mix64": [], "bench_inputs": []}
    for tag, a, b in [("iteration", 0, 0), ("iteration", 1, 0), ("center-init", 12345, 0),
                      ("bench-x", 3, 0), ("bench-labels", 0, 0), ("step", 7, 9)]:
        g["make_stream"].append([tag, a, b, f"{R.make_stream(tag, a, b):016x}"])
    for seed, stream in [(1, R.make_stream("iteration", 0)), (2024, 17), (0, 0)]:
        g["draws"].append([seed, f"{stream:016x}", [f"{int(v):016x}" for v in R.draws(seed, stream, 8)]])
    s = R.make_stream("iteration", 0)
    for k in range(8):
        g["fork"].append([f"{s:016x}", k, f"{R.fork(s, k):016x}"])
    for x in [0, 1, 2**63, 0xdeadbeef]:
        g["mix64"].append([f"{x:016x}", f"{R.mix64(x):016x}"])
    # bench_inputs is restated by the port; pin it with reference next_below / next_normal
    # via init_centers' Box-Muller is not exposed, so pin labels (next_below) directly:
    X, labels = P.bench_inputs(10000, 8, 16, 1, 0)
    g["bench_inputs"].append({"C": 10000, "D": 8, "B": 16, "labels": labels.tolist(),
                              "X": X.tolist()})
    return g


BASELINE = [  # (name, C, K, B, r)  — BASELINE.json configs, all five
    ("cpu_ref_10k", 10000, 1, 128, 0.1),
    ("glint360k_k8", 360000, 8, 1024, 0.1),
    ("glint360k_k1", 360000, 1, 1024, 0.1),
    ("webface2m_k8", 2000000, 8, 1024, 0.1),
    ("webface2m_k1", 2000000, 1, 1024, 0.1),
    ("fullfc_360k_k8", 360000, 8, 1024, 1.0),
    ("stress10m_k8", 10000000, 8, 2048, 0.1),
]


def sampler_golden():
    out = []
    for name, C, K, B, r in BASELINE:
        for step in range(2):
            _, labels = P.bench_inputs(C, 1, B, 1, step)
            stream = R.make_stream("iteration", step)
            bufs, npos = R.build_buffers(C, K, labels, r, 1, stream)
            out.append({
                "name": name, "C": C, "K": K, "B": B, "r": r, "seed": 1, "step": step,
                "stream": f"{stream:016x}", "cap": int(bufs.shape[1]),
                "labels_fnv": fnv64(labels), "labels_head": labels[:4].tolist(),
                "npos": npos.tolist(),
                "fnv": [fnv64(bufs[k]) for k in range(K)],
                "head": [bufs[k, :int(npos[k]) + 4].tolist()[-8:] for k in range(K)],
                "tail": [bufs[k, -4:].tolist() for k in range(K)],
            })
            print("sampler", name, step, npos[:2], flush=True)
    # small edge cases with full buffers stored
    small = []
    for C, K, B, r, seed in [(10, 2, 2, 0.6, 1), (120, 4, 32, 0.5, 3), (400, 4, 3, 0.1, 5),
                             (1000, 4, 32, 0.1, 7), (12, 3, 2, 1.0, 1), (17, 4, 9, 0.9, 2),
                             (64, 8, 64, 1.0, 4), (100, 3, 0, 0.2, 9)]:
        X, labels = P.bench_inputs(C, 1, B, seed, 0)
        stream = R.make_stream("iteration", seed)
        try:
            bufs, npos = R.build_buffers(C, K, labels, r, seed, stream)
            small.append({"C": C, "K": K, "B": B, "r": r, "seed": seed, "stream": f"{stream:016x}",
                          "labels": labels.tolist(), "buffers": bufs.tolist(),
                          "npos": npos.tolist()})
        except OracleError as e:
            small.append({"C": C, "K": K, "B": B, "r": r, "seed": seed, "stream": f"{stream:016x}",
                          "labels": labels.tolist(), "error": e.kind, "message": e.msg})
    # error cases: capacity, label range
    errs = []
    for C, K, labels, r in [(1000, 4, list(range(0, 1000, 8))[:128], 0.1),
                            (100, 4, [5, 100], 0.5), (100, 4, [-3, 5, 200], 0.5),
                            (10, 4, [0], 0.5), (10, 3, [1], 1.0)]:
        try:
            R.build_buffers(C, K, np.array(labels), r, 1, 1)
            errs.append({"C": C, "K": K, "labels": labels, "r": r, "error": None})
        except OracleError as e:
            errs.append({"C": C, "K": K, "labels": labels, "r": r, "error": e.kind,
                         "message": e.msg})
    return out, small, errs


STEP_CASES = [  # (name, C, K, B, D, r, margin, m, tau, steps)
    ("tiny_cos_r05", 400, 4, 32, 32, 0.5, "cosface", 0.4, None, 2),
    ("tiny_arc_r03", 600, 2, 48, 32, 0.3, "arcface", 0.5, None, 2),
    ("tiny_filter_full", 300, 3, 24, 32, 1.0, "cosface", 0.4, 0.1, 2),
    ("tiny_plain_k1", 200, 1, 16, 16, 0.5, "plain", 0.0, None, 1),
    ("cpu_ref_10k_d512", 10000, 1, 128, 512, 0.1, "arcface", 0.5, None, 1),
    ("cos_10k_full_d512", 10000, 1, 128, 512, 1.0, "cosface", 0.4, None, 1),
]


def step_golden(big: bool):
    res = {}
    cases = list(STEP_CASES)
    if big:
        cases.append(("glint360k_k8_d512", 360000, 8, 1024, 512, 0.1, "arcface", 0.5, None, 1))
    for name, C, K, B, D, r, mg, m, tau, steps in cases:
        cfg = OracleCfg(r=r, margin=mg, scale=(1.0 if mg == "plain" else 64.0), m=m,
                        filter_threshold=tau, lr=0.1, momentum=0.9, weight_decay=5e-4)
        W = R.init_centers(C, K, D, 1)
        M = np.zeros_like(W)
        W0 = W.copy()
        entry = {"C": C, "K": K, "B": B, "D": D, "r": r, "margin": mg, "m": m, "tau": tau,
                 "lr": 0.1, "momentum": 0.9, "weight_decay": 5e-4, "steps": []}
        arrays = {}
        for step in range(steps):
            X, labels = P.bench_inputs(C, D, B, 1, step)
            stream = R.make_stream("iteration", step)
            Wb = W.copy()
            o = R.step(cfg, C, K, D, W, M, X, labels, 1, stream)
            rows = np.unique(o["buffers"].ravel())
            Wr = shards_to_rows(W, C, K, D)
            Wbr = shards_to_rows(Wb, C, K, D)
            Mr = shards_to_rows(M, C, K, D)
            st = {"loss": o["loss"], "dX_fro": float(np.linalg.norm(o["dX"])),
                  "dW_fro": float(np.linalg.norm(Wr - Wbr)),
                  "changed_entries": int((Wr != Wbr).sum()),
                  "buffers_fnv": [fnv64(o["buffers"][k]) for k in range(K)],
                  "npos": o["npos"].tolist(), "stream": f"{stream:016x}"}
            entry["steps"].append(st)
            small = D * B <= 4096
            if small:
                arrays[f"s{step}_dX"] = o["dX"]
                arrays[f"s{step}_rows"] = rows
                arrays[f"s{step}_W"] = Wr[rows]
                arrays[f"s{step}_M"] = Mr[rows]
                arrays[f"s{step}_buffers"] = o["buffers"]
            else:
                idx = np.arange(0, D * B, 97)
                arrays[f"s{step}_dX_idx"] = idx
                arrays[f"s{step}_dX_sub"] = o["dX"].ravel()[idx]
                sel = rows[:: max(1, len(rows) // 64)]
                arrays[f"s{step}_rows_sub"] = sel
                arrays[f"s{step}_W_sub"] = Wr[sel]
            print("step", name, step, o["loss"], flush=True)
        assert np.array_equal(W0, R.init_centers(C, K, D, 1))
        res[name] = entry
        np.savez_compressed(os.path.join(OUT, f"step_{name}.npz"), **arrays)
    return res


# Diagnostics (metrics.hpp:56-146 via the step's with_diagnostics, shardsim.hpp:401-410).
# Conflict ground truth: class_identity[j] = j // 3, sample_identity[b] = label_b // 3 except
# every 5th row (b % 5 == 0), whose identity is (label_b // 3) + 1 (a foreign sibling group).
DIAG_CASES = [("tiny", 40, 4, 8, 6), ("k1", 300, 1, 16, 24), ("k3", 1000, 3, 32, 50),
              ("d64", 2000, 2, 64, 128), ("d512", 4000, 4, 512, 64)]


def diag_identities(C_, labels):
    ci = np.arange(C_, dtype=np.int64) // 3
    si = labels // 3
    si = np.where(np.arange(len(labels)) % 5 == 0, si + 1, si)
    return ci, si


def diag_golden():
    out = []
    for name, C_, K, D, B in DIAG_CASES:
        W = R.init_centers(C_, K, D, 1)
        X, labels = P.bench_inputs(C_, D, B, 1, 0)
        ci, si = diag_identities(C_, labels)
        plain = R.diagnostics(C_, K, D, W, X, labels)
        split = R.diagnostics(C_, K, D, W, X, labels, ci, si)
        out.append({"name": name, "C": C_, "K": K, "D": D, "B": B, "plain": plain, "split": split})
    return out


MICS_CASES = [("tiny", 40, 4, 8), ("k3", 700, 3, 32), ("d512", 1500, 2, 512)]


def mics_golden():
    out = []
    for name, C_, K, D in MICS_CASES:
        W = R.init_centers(C_, K, D, 5)
        m = R.mics(C_, K, D, W)
        out.append({"name": name, "C": C_, "K": K, "D": D, "seed": 5, "mics": m.tolist()})
    return out


if __name__ == "__main__" and "--northstar" not in sys.argv:
    if "--diag-only" in sys.argv:
        with open(os.path.join(OUT, "diag.json"), "w") as f:
            json.dump(diag_golden(), f, indent=1)
        with open(os.path.join(OUT, "mics.json"), "w") as f:
            json.dump(mics_golden(), f)
        sys.exit(0)
    big = "--big" in sys.argv
    with open(os.path.join(OUT, "rng.json"), "w") as f:
        json.dump(rng_golden(), f, indent=1)
    s, small, errs = sampler_golden()
    with open(os.path.join(OUT, "sampler.json"), "w") as f:
        json.dump({"baseline": s, "small": small, "errors": errs}, f, indent=1)
    steps = step_golden(big)
    with open(os.path.join(OUT, "steps.json"), "w") as f:
        json.dump(steps, f, indent=1)
    with open(os.path.join(OUT, "diag.json"), "w") as f:
        json.dump(diag_golden(), f, indent=1)
    with open(os.path.join(OUT, "mics.json"), "w") as f:
        json.dump(mics_golden(), f)
    print("done")


def northstar_golden():
    """One reference step at the north-star size: 2M classes, K=8, B=1024, d=512, r=0.1,
    ArcFace(64, 0.5).  Too big to store W: keep the loss, the full dX,
    the buffers' checksums, |W' - W|_F over the sampled rows, and W' of a few sampled rows.
    Run with --northstar (needs ~20 GB RAM, a few minutes on 8 cores)."""
    C, K, B, D, r = 2_000_000, 8, 1024, 512, 0.1
    cfg = OracleCfg(r=r, margin="arcface", scale=64.0, m=0.5, lr=0.1, momentum=0.9, weight_decay=5e-4)
    W = R.init_centers(C, K, D, 1)
    M = np.zeros_like(W)
    X, labels = P.bench_inputs(C, D, B, 1, 0)
    stream = R.make_stream("iteration", 0)
    bufs, npos = R.build_buffers(C, K, labels, r, 1, stream)
    rows = np.unique(bufs.ravel())

    def gather(Wf):  # rows of the shard-concatenated D x owned layout, without a full copy
        out = np.empty((len(rows), D))
        blk = (C + K - 1) // K
        off = 0
        for k in range(K):
            lo, hi = min(k * blk, C), min((k + 1) * blk, C)
            n = hi - lo
            sel = rows[(rows >= lo) & (rows < hi)]
            out_idx = np.searchsorted(rows, sel)
            out[out_idx] = Wf[off:off + D * n].reshape(D, n)[:, sel - lo].T
            off += D * n
        return out

    Wb = gather(W)
    o = R.step(cfg, C, K, D, W, M, X, labels, 1, stream)
    assert np.array_equal(o["buffers"], bufs)
    Wa = gather(W)
    sel = np.arange(0, len(rows), max(1, len(rows) // 64))
    entry = {"C": C, "K": K, "B": B, "D": D, "r": r, "margin": "arcface", "m": 0.5,
             "loss": o["loss"], "dX_fro": float(np.linalg.norm(o["dX"])),
             "dW_fro": float(np.linalg.norm(Wa - Wb)),
             "buffers_fnv": [fnv64(o["buffers"][k]) for k in range(K)],
             "npos": o["npos"].tolist()}
    np.savez_compressed(os.path.join(OUT, "step_webface2m_k8_d512.npz"), dX=o["dX"],
                        rows_sub=rows[sel], W_sub=Wa[sel])
    with open(os.path.join(OUT, "northstar.json"), "w") as f:
        json.dump(entry, f, indent=1)
    print("northstar", entry["loss"], entry["dX_fro"], entry["dW_fro"])


if __name__ == "__main__" and "--northstar" in sys.argv:
    northstar_golden()
