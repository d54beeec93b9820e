"""Checkpoint shard sections: the reference's on-disk encoding
(trainer.hpp:235-338 save/load_checkpoint, io.hpp:18-91 put_matrix) written from and read into
the device state.  Resume must be bit-identical (acceptance criterion 9)."""
import os
import struct

import numpy as np
import pytest

import paper_2203_15565_b200 as p

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def parse_section(buf, off):
    """The reference reader (load_checkpoint's shard loop + BinaryReader::get_matrix)."""
    (count,) = struct.unpack_from("<q", buf, off)
    off += 8
    shards = []
    for _ in range(count):
        k, lo, hi = struct.unpack_from("<qqq", buf, off)
        off += 24
        mats = []
        for _ in range(2):
            rows, cols = struct.unpack_from("<qq", buf, off)
            off += 16
            mats.append(np.frombuffer(buf, dtype="<f8", count=rows * cols, offset=off).reshape(rows, cols))
            off += 8 * rows * cols
        shards.append((k, lo, hi, mats[0], mats[1]))
    return shards, off


def test_checkpoint_roundtrip_and_resume(tmp_path, port):
    C_, K, D, B = 3000, 3, 64, 96
    cfg = p.StepConfig(r=0.2, margin=p.MarginConfig.arcface_style())

    def steps(sh, lo, hi):
        out = []
        for step in range(lo, hi):
            X, labels = port.bench_inputs(C_, D, B, 1, step)
            r = p.distributed_partial_step(sh, X, labels, cfg, p.SeededRng(1, p.make_stream("iteration", step)))
            out.append((r.loss, r.d_features.copy()))
        return out

    a = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
    a.init_center_shards(4)
    steps(a, 0, 2)
    path = str(tmp_path / "ckpt.bin")
    header = b"PFCDCKPT-header-written-by-the-caller"
    with open(path, "wb") as f:
        f.write(header)
    a.write_shards(path, append=True)
    buf = open(path, "rb").read()
    shards, end = parse_section(buf, len(header))
    assert end == len(buf) and len(shards) == K
    layout = p.ShardLayout(C_, K)
    for k, (sid, lo, hi, W, M) in enumerate(shards):
        assert (sid, lo, hi) == (k, layout.owned_begin(k), layout.owned_end(k))
        w, m = a.get_shard(k)
        assert np.array_equal(W, w) and np.array_equal(M, m)
    # resume into a fresh context: bit-identical state and continuation
    b = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=B)
    assert b.read_shards(path, len(header)) == len(buf)
    for k in range(K):
        assert all(np.array_equal(x, y) for x, y in zip(a.get_shard(k), b.get_shard(k)))
    ra, rb = steps(a, 2, 4), steps(b, 2, 4)
    for (la, da), (lb, db) in zip(ra, rb):
        assert la == lb and np.array_equal(da, db)
    for k in range(K):
        assert all(np.array_equal(x, y) for x, y in zip(a.get_shard(k), b.get_shard(k)))
    # errors: truncated file, foreign layout
    open(str(tmp_path / "short.bin"), "wb").write(buf[:len(buf) // 2])
    with pytest.raises(p.DataError, match="truncated checkpoint"):
        b.read_shards(str(tmp_path / "short.bin"), len(header))
    c = p.CenterShards(p.ShardLayout(C_ + 1, K), D, cfg, max_batch=B)
    with pytest.raises(p.ContractError, match="does not match the contiguous equal partition"):
        c.read_shards(path, len(header))
    with pytest.raises(p.DataError, match="cannot open"):
        b.read_shards(str(tmp_path / "missing.bin"))
    for s in (a, b, c):
        s.close()
