"""CPU: pin the plain-C oracle (oracle/pfc_oracle.c) against the golden vectors made by the
compiled reference (tests/golden/make_golden.py) and SURVEY.md Appendix B.
Mirrors the reference's own [rng], [sampler], [loss] and [shardsim] test tags."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleCfg, OracleError, fnv64, ref_available, shards_to_rows


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def test_rng_known_answers(port, golden_dir):
    g = load(golden_dir, "rng.json")
    for tag, a, b, want in g["make_stream"]:
        assert f"{port.make_stream(tag, a, b):016x}" == want
    for seed, stream, want in g["draws"]:
        got = [f"{int(v):016x}" for v in port.draws(seed, int(stream, 16), len(want))]
        assert got == want
    for s, k, want in g["fork"]:
        assert f"{port.fork(int(s, 16), k):016x}" == want
    for x, want in g["mix64"]:
        assert f"{port.mix64(int(x, 16)):016x}" == want


def test_rng_appendix_b(port):
    # SURVEY.md Appendix B (generated from the compiled reference)
    s = port.make_stream("iteration", 0)
    assert s == 0xe3da8f7cae11d6ba
    assert port.fnv1a("iteration") == 0xf1cc065d080f9fcc
    assert port.mix64(1) == 0xb456bcfc34c2cb2c and port.mix64(0) == 0
    assert port.fork(s, 0) == 0x680dfa7350cba7e6 and port.fork(s, 7) == 0xe931d2aa9a5d8eda
    assert int(port.draws(1, port.fork(s, 0), 1)[0]) == 0x4a0a0c0cda14d279


def test_capacity_formula(port):
    # tests/test_sampler.cpp:9-15
    assert port.capacity(600000, 8, 0.1) == 7500
    assert port.capacity(1000, 4, 1.0) == 250
    assert port.capacity(10, 2, 0.6) == 3
    assert port.capacity(10, 2, 0.0) == -1 and port.capacity(10, 2, 1.5) == -1


def test_sampler_baseline_configs(port, golden_dir):
    g = load(golden_dir, "sampler.json")
    for e in g["baseline"]:
        if e["C"] > 2_000_000 or (e["C"] >= 2_000_000 and e["K"] == 1):
            continue  # 10M / 2M-K1 pools: covered on the GPU; keep the CPU suite fast
        _, labels = port.bench_inputs(e["C"], 1, e["B"], e["seed"], e["step"])
        assert fnv64(labels) == e["labels_fnv"]
        bufs, npos = port.build_buffers(e["C"], e["K"], labels, e["r"], e["seed"],
                                        int(e["stream"], 16))
        assert npos.tolist() == e["npos"]
        assert [fnv64(bufs[k]) for k in range(e["K"])] == e["fnv"], e["name"]


def test_sampler_small_and_errors(port, golden_dir):
    g = load(golden_dir, "sampler.json")
    for e in g["small"]:
        if "error" in e:
            with pytest.raises(OracleError) as ei:
                port.build_buffers(e["C"], e["K"], e["labels"], e["r"], e["seed"],
                                   int(e["stream"], 16))
            assert ei.value.kind == e["error"] and ei.value.msg == e["message"]
            continue
        bufs, npos = port.build_buffers(e["C"], e["K"], e["labels"], e["r"], e["seed"],
                                        int(e["stream"], 16))
        assert bufs.tolist() == e["buffers"] and npos.tolist() == e["npos"]
    for e in g["errors"]:
        if e["error"] is None:
            port.build_buffers(e["C"], e["K"], e["labels"], e["r"], 1, 1)
            continue
        with pytest.raises(OracleError) as ei:
            port.build_buffers(e["C"], e["K"], e["labels"], e["r"], 1, 1)
        assert ei.value.kind == e["error"] and ei.value.msg == e["message"]


def test_margin_closed_forms(port):
    # tests/test_loss.cpp:37-51
    assert port._apply_margin(0.5, 1, 1, 64.0, 0.4) == pytest.approx(64 * 0.1)
    assert port._apply_margin(0.3, 0, 1, 64.0, 0.4) == pytest.approx(19.2)
    assert port._apply_margin(0.4, 0, 2, 64.0, 0.5) == pytest.approx(25.6)
    c = 1 - 1e-7
    assert port._apply_margin(1.0, 1, 2, 64.0, 0.5) == pytest.approx(64 * np.cos(np.arccos(c) + 0.5))
    assert port._margin_derivative(1.0, 1, 2, 64.0, 0.5) == 0.0
    assert port._margin_derivative(0.2, 0, 2, 64.0, 0.5) == 64.0


STEP_FAST = ["tiny_cos_r05", "tiny_arc_r03", "tiny_filter_full", "tiny_plain_k1",
             "cpu_ref_10k_d512", "cos_10k_full_d512"]


@pytest.mark.parametrize("name", STEP_FAST)
def test_step_matches_reference_golden(port, golden_dir, name):
    e = load(golden_dir, "steps.json")[name]
    arr = np.load(os.path.join(golden_dir, f"step_{name}.npz"))
    C_, K, B, D = e["C"], e["K"], e["B"], e["D"]
    cfg = OracleCfg(r=e["r"], margin=e["margin"], scale=1.0 if e["margin"] == "plain" else 64.0,
                    m=e["m"], filter_threshold=e["tau"], lr=e["lr"], momentum=e["momentum"],
                    weight_decay=e["weight_decay"])
    W = port.init_centers(C_, K, D, 1)
    M = np.zeros_like(W)
    for step, st in enumerate(e["steps"]):
        X, labels = port.bench_inputs(C_, D, B, 1, step)
        Wb = shards_to_rows(W, C_, K, D)
        o = port.step(cfg, C_, K, D, W, M, X, labels, 1, int(st["stream"], 16))
        # the restatement follows the reference's op order: bit-identical
        assert o["loss"] == st["loss"]
        assert [fnv64(o["buffers"][k]) for k in range(K)] == st["buffers_fnv"]
        Wr = shards_to_rows(W, C_, K, D)
        assert int((Wr != Wb).sum()) == st["changed_entries"]
        if f"s{step}_dX" in arr:
            assert np.array_equal(o["dX"], arr[f"s{step}_dX"])
            rows = arr[f"s{step}_rows"]
            assert np.array_equal(Wr[rows], arr[f"s{step}_W"])
            assert np.array_equal(shards_to_rows(M, C_, K, D)[rows], arr[f"s{step}_M"])
        else:
            idx = arr[f"s{step}_dX_idx"]
            assert np.array_equal(o["dX"].ravel()[idx], arr[f"s{step}_dX_sub"])
            assert np.array_equal(Wr[arr[f"s{step}_rows_sub"]], arr[f"s{step}_W_sub"])


def test_appendix_b_step_values(port):
    # SURVEY.md Appendix B, 10k/K=1/B=128/r=0.1 ArcFace(64,0.5)
    C_, K, D, B = 10000, 1, 512, 128
    W = port.init_centers(C_, K, D, 1)
    assert W.reshape(D, C_)[0, 0] == -0.023853608029664498
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    assert X[0, 0] == 0.18561977740519164
    cfg = OracleCfg(r=0.1, margin="arcface", m=0.5)
    o = port.step(cfg, C_, K, D, W, np.zeros_like(W), X, labels, 1, port.make_stream("iteration", 0))
    assert o["loss"] == 41.598627063948094
    assert float(np.linalg.norm(o["dX"])) == pytest.approx(2.347419215188e-01, rel=1e-12)


def test_step_errors(port):
    cfg = OracleCfg(r=0.1)
    W = port.init_centers(1000, 4, 8, 1)
    labels = np.arange(0, 1000, 8)[:128]
    X = np.ones((8, len(labels)))
    with pytest.raises(OracleError) as ei:
        port.step(cfg, 1000, 4, 8, W, np.zeros_like(W), X, labels, 1, 1)
    assert ei.value.kind == "CapacityError"
    assert "shard 0 received 32 distinct positives but capacity is 25" in ei.value.msg
    bad = OracleCfg(r=0.5, margin="plain", scale=64.0, m=0.0)
    with pytest.raises(OracleError) as ei:
        port.step(bad, 1000, 4, 8, W, np.zeros_like(W), np.ascontiguousarray(X[:, :4]), [1, 2, 3, 4], 1, 1)
    assert ei.value.kind == "ConfigError"


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_port_equals_compiled_reference_random():
    from oracle.oracle import Oracle
    P, R = Oracle("port"), Oracle("reference")
    rng = np.random.default_rng(0)
    for trial in range(6):
        K = int(rng.integers(1, 5))
        C_ = int(rng.integers(50, 400))
        B = int(rng.integers(1, 24))
        D = int(rng.integers(2, 20))
        r = float(rng.choice([0.3, 0.5, 1.0]))
        tau = None if trial % 2 else 0.3
        cfg = OracleCfg(r=r, margin=["cosface", "arcface", "cosface"][trial % 3], m=0.3,
                        filter_threshold=tau)
        labels = rng.integers(0, C_, B)
        X = rng.standard_normal((D, B))
        W1 = P.init_centers(C_, K, D, trial)
        W2 = W1.copy()
        M1, M2 = np.zeros_like(W1), np.zeros_like(W1)
        try:
            o1 = P.step(cfg, C_, K, D, W1, M1, X, labels, 3, 77)
        except OracleError as e1:
            with pytest.raises(OracleError) as e2:
                R.step(cfg, C_, K, D, W2, M2, X, labels, 3, 77)
            assert e1.kind == e2.value.kind and e1.msg == e2.value.msg
            continue
        o2 = R.step(cfg, C_, K, D, W2, M2, X, labels, 3, 77)
        assert o1["loss"] == o2["loss"]
        assert np.array_equal(o1["dX"], o2["dX"]) and np.array_equal(W1, W2)


def _diag_identities(C_, labels):
    # tests/golden/make_golden.py: diag_identities
    ci = np.arange(C_, dtype=np.int64) // 3
    si = labels // 3
    si = np.where(np.arange(len(labels)) % 5 == 0, si + 1, si)
    return ci, si


def test_diagnostics_match_reference_golden(port, golden_dir):
    """apcs / amncs (+ conflicted / hard split): the C restatement of metrics.hpp:56-146 is
    bit-identical to the compiled reference on every golden case."""
    with open(os.path.join(golden_dir, "diag.json")) as f:
        cases = json.load(f)
    for cs in cases:
        C_, K, D, B = cs["C"], cs["K"], cs["D"], cs["B"]
        W = port.init_centers(C_, K, D, 1)
        X, labels = port.bench_inputs(C_, D, B, 1, 0)
        ci, si = _diag_identities(C_, labels)
        assert port.diagnostics(C_, K, D, W, X, labels) == cs["plain"], cs["name"]
        assert port.diagnostics(C_, K, D, W, X, labels, ci, si) == cs["split"], cs["name"]


def test_diagnostics_errors(port):
    W = port.init_centers(30, 2, 8, 1)
    X = np.ones((8, 3))
    with pytest.raises(OracleError, match="apcs: label 30 owned by no shard"):
        port.diagnostics(30, 2, 8, W, X, np.array([0, 1, 30]))
    with pytest.raises(OracleError, match="amncs: needs at least two classes"):
        port.diagnostics(1, 1, 8, port.init_centers(1, 1, 8, 1), X, np.array([0, 0, 0]))


def test_mics_matches_reference_golden(port, golden_dir):
    """metrics.hpp:150-164: the C restatement is bit-identical to the compiled reference."""
    with open(os.path.join(golden_dir, "mics.json")) as f:
        cases = json.load(f)
    for cs in cases:
        W = port.init_centers(cs["C"], cs["K"], cs["D"], cs["seed"])
        assert port.mics(cs["C"], cs["K"], cs["D"], W).tolist() == cs["mics"], cs["name"]
    with pytest.raises(OracleError, match="mics: needs at least two classes"):
        port.mics(1, 1, 4, port.init_centers(1, 1, 4, 1))


def test_combined_margin_identities(port):
    """The combined-margin extension (pfc_oracle.c MK_COMB) is pinned to the reference's own
    margins through its identities: (1, m, 0) is ArcFace operation for operation (bit-equal,
    clamp region included) and (1, 0, m) is CosFace up to the ArcFace clamp of the cosine."""
    for c in (-1.0, -0.999999995, -0.7, -0.1, 0.0, 0.2, 0.55, 0.9999, 1.0):
        for is_pos in (0, 1):
            assert port._apply_margin_combined(c, is_pos, 64.0, 1.0, 0.5, 0.0) == \
                port._apply_margin(c, is_pos, 2, 64.0, 0.5)
            assert port._margin_derivative_combined(c, is_pos, 64.0, 1.0, 0.5) == \
                port._margin_derivative(c, is_pos, 2, 64.0, 0.5)
            if abs(c) < 1.0 - 1e-7:
                assert port._apply_margin_combined(c, is_pos, 64.0, 1.0, 0.0, 0.4) == \
                    pytest.approx(port._apply_margin(c, is_pos, 1, 64.0, 0.4), abs=1e-12)
    # m1 scales the angle: d/dc of s (cos(m1 acos c + m2) - m3) by central differences
    for c in (-0.6, 0.1, 0.7):
        h = 1e-6
        num = (port._apply_margin_combined(c + h, 1, 64.0, 0.9, 0.4, 0.15) -
               port._apply_margin_combined(c - h, 1, 64.0, 0.9, 0.4, 0.15)) / (2 * h)
        assert port._margin_derivative_combined(c, 1, 64.0, 0.9, 0.4) == pytest.approx(num, rel=1e-6)


def test_combined_margin_step_arcface_point(port):
    """A whole oracle step with combined (1, 0.5, 0) equals the ArcFace step bit for bit."""
    from oracle.oracle import OracleCfg
    C_, K, D, B = 600, 2, 16, 32
    X, labels = port.bench_inputs(C_, D, B, 1, 0)
    out = []
    for cfg in (OracleCfg(r=0.3, margin="arcface", scale=64.0, m=0.5),
                OracleCfg(r=0.3, margin="combined", scale=64.0, m=0.5, m1=1.0, m3=0.0)):
        W = port.init_centers(C_, K, D, 1)
        M = np.zeros_like(W)
        ref = port.step(cfg, C_, K, D, W, M, X, labels, 1, 7)
        out.append((ref["loss"], ref["dX"], W))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
