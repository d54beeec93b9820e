"""Shared test helpers: build device shards from oracle state and compare per the tolerance
contract of SURVEY.md §8(c) / DESIGN.md."""
import hashlib
import os

import numpy as np

import paper_2203_15565_b200 as p
from oracle.oracle import OracleCfg, shard_bounds, shards_to_rows

MARGINS = {"cosface": p.MarginConfig.cosface_style, "arcface": p.MarginConfig.arcface_style,
           "plain": p.MarginConfig.plain}


def step_cfg(margin: str, m: float, r: float, tau=None, lr=0.1):
    mc = p.MarginConfig.plain() if margin == "plain" else MARGINS[margin](64.0, m)
    return p.StepConfig(r=r, margin=mc, filter_threshold=tau, lr=lr)


def oracle_cfg(margin: str, m: float, r: float, tau=None, lr=0.1):
    return OracleCfg(r=r, margin=margin, scale=1.0 if margin == "plain" else 64.0,
                     m=0.0 if margin == "plain" else m, filter_threshold=tau, lr=lr)


def make_shards(W, M, C_, K, D, cfg, max_batch, precision, flags=0):
    sh = p.CenterShards(p.ShardLayout(C_, K), D, cfg, max_batch=max_batch, precision=precision,
                        flags=flags)
    off = 0
    for k, (lo, hi) in enumerate(shard_bounds(C_, K)):
        n = D * (hi - lo)
        sh.set_shard(k, W[off:off + n].reshape(D, hi - lo), M[off:off + n].reshape(D, hi - lo))
        off += n
    return sh


def device_rows(sh, C_, K, D):
    Ws, Ms = [], []
    for k in range(K):
        w, m = sh.get_shard(k)
        Ws.append(w.ravel())
        Ms.append(m.ravel())
    return shards_to_rows(np.concatenate(Ws), C_, K, D), shards_to_rows(np.concatenate(Ms), C_, K, D)


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the sources each prebuilt parity program embeds a hash of (oracle/Makefile *_SRCS, same order)
PARITY_SOURCES = {
    "adapter_parity": ["oracle/adapter_parity.cpp", "include/pfc/gpu_step.hpp", "include/pfc_gpu.h"],
    "trainer_parity": ["oracle/trainer_parity.cpp", "include/pfc/gpu_trainer.hpp",
                       "include/pfc/gpu_step.hpp", "include/pfc_gpu.h"],
    "trainer_bench": ["oracle/trainer_bench.cpp", "include/pfc/gpu_trainer.hpp",
                      "include/pfc/gpu_step.hpp", "include/pfc_gpu.h"],
}


def source_hash(name: str) -> str:
    h = hashlib.sha256()
    for f in PARITY_SOURCES[name]:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def assert_fresh_binary(exe: str) -> None:
    """A prebuilt parity program must come from the current sources (it cannot be rebuilt on a
    box without the reference headers)."""
    import subprocess
    name = os.path.basename(exe)
    got = subprocess.run([exe, "--source-hash"], capture_output=True, text=True, timeout=60).stdout.strip()
    assert got == source_hash(name), (f"{exe} is stale (built from sources {got}, current "
                                      f"{source_hash(name)}): rebuild with make -C oracle")
