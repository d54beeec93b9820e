"""compute-sanitizer driver (SURVEY §5 race / memory checking): a few steps of the hot path on
small configurations, in both precisions, through the captured CUDA graph and eagerly
(PFC_FLAG_NO_GRAPH), plus one per-row-offset step (the max-only GEMM pass) and one loopback
2-rank step.  Checked against the oracle so a run that "passes" the sanitizer with wrong
values is caught too.

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python profiles/sanitize_step.py [case]
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2203_15565_b200 as p  # noqa: E402
from oracle.oracle import Oracle, OracleCfg, shard_bounds  # noqa: E402


def shards(o, C_, K, D, cfg, B, precision, flags=0, **kw):
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B, precision=precision,
                        flags=flags, **kw)
    W = o.init_centers(C_, K, D, 1)
    off = 0
    for k, (lo, hi) in enumerate(shard_bounds(C_, K)):
        if k in sh.local_shards:
            n = D * (hi - lo)
            sh.set_shard(k, W[off:off + n].reshape(D, hi - lo))
        off += D * (hi - lo)
    return sh, W


def one(o, precision, flags, C_=6000, K=2, D=256, B=96, steps=2, scale=64.0):
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.cosface_style(scale, 0.4), lr=0.1)
    sh, W = shards(o, C_, K, D, cfg, B, precision, flags)
    M = np.zeros_like(W)
    for i in range(steps):
        X, labels = o.bench_inputs(C_, D, B, 1, i)
        stream = p.make_stream("iteration", i)
        res = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, stream))
        ref = o.step(OracleCfg(r=0.1, margin="cosface", scale=scale, m=0.4), C_, K, D, W, M, X,
                     labels, 1, stream)
        rel = abs(res.loss - ref["loss"]) / abs(ref["loss"])
        assert rel < 1e-3, rel
    sh.close()
    print(f"precision={precision} flags={flags} s={scale}: {steps} steps ok", flush=True)


def loopback(o, precision, R=2, C_=6000, K=2, D=256, B=96):
    cfg = p.StepConfig(r=0.1, margin=p.MarginConfig.arcface_style(), lr=0.1)
    lid = p.loopback_id()
    X, labels = o.bench_inputs(C_, D, B, 1, 0)
    out = [None] * R

    def rank(r):
        sh, _ = shards(o, C_, K, D, cfg, B, precision, rank=r, world_size=R, nccl_id=lid)
        res = sh.step_host(X, labels, cfg, p.SeededRng(1, p.make_stream("iteration", 0)))
        out[r] = res.loss
        sh.close()
    ts = [threading.Thread(target=rank, args=(r,)) for r in range(R)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out[0] is not None and out[0] == out[1], out
    print(f"loopback R={R} precision={precision}: ok", flush=True)


def main():
    o = Oracle("port")
    case = sys.argv[1] if len(sys.argv) > 1 else "all"
    if case in ("all", "bf16"):
        one(o, p.PRECISION_BF16, 0)
        one(o, p.PRECISION_BF16, p.FLAG_NO_GRAPH)
        one(o, p.PRECISION_BF16, p.FLAG_NO_GRAPH, scale=128.0)  # per-row offsets (MaxEpi pass)
    if case in ("all", "fp32"):
        one(o, p.PRECISION_FP32, 0)
        one(o, p.PRECISION_FP32, p.FLAG_NO_GRAPH)
    if case in ("all", "loopback"):
        loopback(o, p.PRECISION_BF16)


if __name__ == "__main__":
    main()
