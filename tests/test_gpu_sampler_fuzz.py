"""Seeded fuzz of the bitmap sampler (sampler.cu) against the oracle's build_buffers
(sampler.hpp:63-126): random C (edge sizes around the 32-bit words and 32-word chunks of the
label bitmap included), K, r, batch sizes and label multisets (heavy repeats, classes at the
shard and chunk boundaries, C - 1), in both bitmap chunk geometries (32 words; 1024 words as
past 16.7M classes, PFC_FLAG_WIDE_SAMPLER_CHUNKS).  Buffers must be bit-exact, order included;
an input the reference rejects must raise the same error text."""
import numpy as np
import pytest

import paper_2203_15565_b200 as p
from oracle.oracle import OracleError

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def cases(n=160, seed=11):
    rng = np.random.default_rng(seed)
    edge_c = [1, 2, 31, 32, 33, 63, 64, 65, 1023, 1024, 1025, 32767, 32768, 32769, 65537]
    out = []
    for i in range(n):
        C_ = int(edge_c[i]) if i < len(edge_c) else int(rng.integers(2, 300000))
        K = int(rng.integers(1, 9))
        r = float(rng.choice([0.05, 0.1, 0.3, 0.5, 1.0]))
        B = int(rng.integers(1, 600))
        kind = i % 4
        if kind == 0:    # uniform labels
            lab = rng.integers(0, C_, B)
        elif kind == 1:  # a few classes repeated many times
            pool = rng.integers(0, C_, max(1, min(C_, 5)))
            lab = pool[rng.integers(0, pool.size, B)]
        elif kind == 2:  # shard / word / chunk boundaries and the last class
            blk = -(-C_ // K)
            cand = {0, C_ - 1}
            for k in range(K + 1):
                for d in (-1, 0, 1):
                    cand.add(k * blk + d)
            for w in range(0, C_, 1024):
                for d in (-1, 0, 31, 32):
                    cand.add(w + d)
            cand = np.array(sorted(c for c in cand if 0 <= c < C_))
            lab = cand[rng.integers(0, cand.size, B)]
        else:            # dense block of consecutive classes
            lo = int(rng.integers(0, C_))
            lab = (lo + rng.integers(0, 200, B)) % C_
        out.append((C_, K, r, np.asarray(lab, dtype=np.int64), int(rng.integers(1, 1 << 30))))
    return out


@pytest.mark.parametrize("flags", [0, p.FLAG_WIDE_SAMPLER_CHUNKS], ids=["chunk32", "chunk1024"])
def test_sampler_fuzz(flags, port):
    for C_, K, r, lab, seed in cases():
        stream = port.make_stream("fuzz", seed)
        try:
            want, npos = port.build_buffers(C_, K, lab, r, seed, stream)
            err = None
        except OracleError as e:
            want, err = None, e
        sh = p.CenterShards(p.ShardLayout(C_, K), 8, p.StepConfig(r=r), max_batch=max(len(lab), 1),
                            flags=flags)
        X = np.random.default_rng(0).standard_normal((8, len(lab)))
        if err is not None:
            with pytest.raises(p.Error) as got:
                p.distributed_partial_step(sh, X, lab, p.StepConfig(r=r, lr=0.0),
                                           p.SeededRng(seed, stream))
            assert type(got.value).__name__ == err.kind and str(got.value) == err.msg, (C_, K, r)
        else:
            p.distributed_partial_step(sh, X, lab, p.StepConfig(r=r, lr=0.0), p.SeededRng(seed, stream))
            for k, b in enumerate(sh.buffers()):
                assert np.array_equal(b.class_indices, want[k]), (C_, K, r, len(lab), k)
                assert b.num_positives == npos[k]
        sh.close()


@pytest.mark.parametrize("flags", [0, p.FLAG_WIDE_SAMPLER_CHUNKS], ids=["chunk32", "chunk1024"])
def test_sampler_positives_beyond_shared_staging(flags, port):
    """More distinct positives across the local shards (10000) than the chain walk stages in
    shared memory (kWalkPositives = 8192): the walk's complement lookups fall back to the
    positives in global memory; buffers still bit-exact."""
    C_, K, B, r = 400000, 2, 16384, 0.1
    rng = np.random.default_rng(3)
    pool = np.concatenate([rng.choice(200000, 5000, replace=False),
                           200000 + rng.choice(200000, 5000, replace=False)])
    lab = pool[rng.integers(0, pool.size, B)].astype(np.int64)
    lab[:pool.size] = pool  # every pool class present
    stream = port.make_stream("fuzz", 99)
    want, npos = port.build_buffers(C_, K, lab, r, 5, stream)
    assert npos.sum() == 10000
    sh = p.CenterShards(p.ShardLayout(C_, K), 8, p.StepConfig(r=r), max_batch=B, flags=flags)
    X = np.random.default_rng(0).standard_normal((8, B))
    p.distributed_partial_step(sh, X, lab, p.StepConfig(r=r, lr=0.0), p.SeededRng(5, stream))
    for k, b in enumerate(sh.buffers()):
        assert np.array_equal(b.class_indices, want[k]) and b.num_positives == npos[k]
    sh.close()
