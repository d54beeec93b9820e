"""CPU: the C-ABI library loads and exports every entry point of include/pfc_gpu.h; the host
mirror of rng.hpp / sampler.hpp agrees with the oracle.  No compute calls (no GPU here)."""
import ctypes
import os

import numpy as np
import pytest

import paper_2203_15565_b200 as p


def test_library_exports_every_header_symbol():
    if not os.path.exists(p.LIB_PATH):
        pytest.skip("libpfc_gpu.so not built (run __graft_entry__.build())")
    lib = p.load_library()
    names = p.header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert b"sm_100a" in lib.pfc_gpu_version()


def test_library_is_sm100a_tcgen05():
    import subprocess
    if not os.path.exists(p.LIB_PATH):
        pytest.skip("not built")
    sass = subprocess.run(["cuobjdump", "-sass", p.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA + TMEM
    import re
    assert not re.search(r"\s HMMA", sass)  # no legacy mma.sync path (only UTCHMMA)


def test_create_without_gpu_fails_loudly():
    if not os.path.exists(p.LIB_PATH):
        pytest.skip("not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(p.Error):
        p.CenterShards(p.ShardLayout(100, 1), 8, p.StepConfig(r=0.5), max_batch=8)


def test_create_validates_before_touching_a_device():
    """pfc_gpu_create checks the descriptor before any CUDA call (the reference's error types,
    and the tensor-core paths' dim limit) -- runnable without a GPU."""
    if not os.path.exists(p.LIB_PATH):
        pytest.skip("not built")
    cfg = p.StepConfig(r=0.1)
    for prec in (p.PRECISION_BF16, p.PRECISION_TF32):
        with pytest.raises(p.ConfigError, match="dim <= 1024"):
            p.CenterShards(p.ShardLayout(1000, 2), 1028, cfg, max_batch=8, precision=prec)
        with pytest.raises(p.ConfigError, match="dim % 4 == 0"):
            p.CenterShards(p.ShardLayout(1000, 2), 130, cfg, max_batch=8, precision=prec)
    with pytest.raises(p.ConfigError, match="unknown precision"):
        p.CenterShards(p.ShardLayout(1000, 2), 128, cfg, max_batch=8, precision=7)
    with pytest.raises(p.ContractError, match="max_batch"):
        p.CenterShards(p.ShardLayout(1000, 2), 128, cfg, max_batch=(1 << 20) + 1)
    with pytest.raises(p.ContractError, match="sampling ratio"):
        p.CenterShards(p.ShardLayout(1000, 2), 128, p.StepConfig(r=1.5), max_batch=8)
    # the combined-margin extension's parameters (checked by the library itself, not only by
    # MarginConfig.validate)
    for m1, m3, msg in ((0.0, 0.2, r"m1 must be in \(0, 2\]"), (1.0, 1.0, r"m3 must be in \[0, 1\)")):
        d = p.Desc(1000, 128, 2, 8, 0.1, p.COMBINED, 64.0, 0.3, 0, 0.0, 0.9, 5e-4,
                   p.PRECISION_BF16, 0, 0, 1, None, 0, m1, m3)
        h = ctypes.c_void_p()
        lib = p.load_library()
        assert lib.pfc_gpu_create(ctypes.byref(d), ctypes.byref(h)) == 4  # PFC_ERR_CONFIG
        import re
        assert re.search(msg, lib.pfc_gpu_last_error(None).decode())


def test_rng_mirror_matches_oracle(port):
    for tag, a, b in [("iteration", 0, 0), ("center-init", 77, 0), ("x", 3, 9)]:
        assert p.make_stream(tag, a, b) == port.make_stream(tag, a, b)
    s = p.make_stream("iteration", 4)
    for k in range(5):
        assert p.SeededRng(1, s).fork(k).stream_id == port.fork(s, k)


def test_layout_and_capacity_mirror(port):
    for C_, K, r in [(600000, 8, 0.1), (1000, 4, 1.0), (10, 2, 0.6), (2000000, 8, 0.1), (17, 4, 0.9)]:
        assert p.buffer_capacity(p.ShardLayout(C_, K), r) == port.capacity(C_, K, r)
    lay = p.ShardLayout(10, 4)
    assert [lay.owned_begin(k) for k in range(4)] == [0, 3, 6, 9]
    assert lay.owned_end(3) == 10 and lay.owner(9) == 3
    with pytest.raises(p.ContractError):
        p.buffer_capacity(lay, 0.0)
    with pytest.raises(p.ConfigError):
        p.MarginConfig(p.PLAIN, 64.0, 0.0).validate()


def test_header_structs_match_ctypes_layout():
    # offsets of the C structs must match the ctypes mirrors (plain C, no padding surprises)
    assert ctypes.sizeof(p.StepArgs) == 32
    assert ctypes.sizeof(p.StepOut) == 72
    assert p.Desc.flags.offset > p.Desc.nccl_id.offset


def test_header_structs_match_c_compiler(tmp_path):
    """sizeof / offsetof of every struct in include/pfc_gpu.h, as gcc lays them out, against the
    ctypes mirrors the Python package and INTEGRATION.md's bindings use."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    mirrors = {"pfc_gpu_desc": p.Desc, "pfc_gpu_step_config": p.StepConfigC,
               "pfc_gpu_step_args": p.StepArgs, "pfc_gpu_step_out": p.StepOut}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "pfc_gpu.h"', 'int main(void) {']
    for cname, py in mirrors.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ['  return 0;', '}']
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "abi"
    subprocess.check_call(["gcc", "-std=c11", "-I", inc, str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    got = {}
    for line in out:
        if line:
            c, f, v = line.split()
            got[(c, f)] = int(v)
    for cname, py in mirrors.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
