"""GPU: the trainer integration (include/pfc/gpu_trainer.hpp over pfc_gpu_trainer_*, SURVEY §8f
row 3) against the reference's own pfc::train, both called from one C++ program built against
the reference headers (oracle/_ref/trainer_parity, made by `make -C oracle` where
/root/reference exists): multi-epoch end results in fp32 and bf16, with and without conflict
splits; GPU checkpoint/resume bit-identical to an uninterrupted run; checkpoints exchanged
with the reference in both directions."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "trainer_parity")


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/trainer_parity not built")
def test_gpu_train_matches_reference_train():
    from tests.helpers import assert_fresh_binary
    assert_fresh_binary(EXE)
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "trainer_parity.jsonl"), "w") as f:
        f.write(p.stdout)
    assert lines, p.stderr
    cases = {l["case"] for l in lines}
    assert {"train_fp32", "train_fp32_conflict", "train_bf16", "resume_bit_exact",
            "checkpoint_cross"} <= cases, (cases, p.stderr)
    bad = [l for l in lines if not l["pass"]]
    assert p.returncode == 0 and not bad, bad or p.stderr
