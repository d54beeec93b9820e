"""GPU: the C++ drop-in (include/pfc/gpu_step.hpp) against the reference's own
pfc::distributed_partial_step, both called from one C++ program built against the reference
headers (oracle/_ref/adapter_parity, made by `make -C oracle` where /root/reference exists)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/adapter_parity not built")
def test_cpp_dropin_matches_reference_step():
    from tests.helpers import assert_fresh_binary
    assert_fresh_binary(EXE)
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "adapter_parity.jsonl"), "w") as f:
        f.write(p.stdout)
    assert lines, p.stderr
    bad = [l for l in lines if not l["pass"]]
    assert p.returncode == 0 and not bad, bad or p.stderr
    assert all(l.get("buffers_bit_exact", True) for l in lines)
