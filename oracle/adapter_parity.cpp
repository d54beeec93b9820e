// adapter_parity.cpp — C++ parity test of the drop-in (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against the UNMODIFIED reference headers (/root/reference/proj/
// include) and include/pfc/gpu_step.hpp into oracle/_ref/adapter_parity, the way a maintainer
// would build their own tests: the same CenterShard / FeatureBatch / StepConfig objects go through
// the reference's pfc::distributed_partial_step (shardsim.hpp:166) and through
// pfc::gpu::distributed_partial_step / pfc::gpu::Session (the B200 path), and the results are
// compared under the tolerance contract of DESIGN.md.  Patterned on
// proj/tests/test_shardsim.cpp:102-127 and 178-221.  Prints one JSON line per case; exit 0 iff
// every case is within tolerance.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "pfc/gpu_step.hpp"
#include "pfc/shardsim.hpp"
#include "pfc/io.hpp"
#include "pfc/trainer.hpp"

#ifndef PFC_SRC_HASH  // sha256 prefix of the sources this program was built from (Makefile)
#define PFC_SRC_HASH "unknown"
#endif

using namespace pfc;

namespace {

FeatureBatch bench_batch(int64_t C, int64_t D, int64_t B, uint64_t step) {
  // the bench input convention: labels, then X b-major / d inner
  FeatureBatch fb;
  fb.features = Matrix(D, B);
  SeededRng rl(1, make_stream("bench-labels", step));
  for (int64_t b = 0; b < B; ++b) fb.labels.push_back(static_cast<int64_t>(rl.next_below(C)));
  SeededRng rx(1, make_stream("bench-x", step));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t d = 0; d < D; ++d) fb.features(d, b) = rx.next_normal();
  return fb;
}

double rel_fro(const Matrix& a, const Matrix& b) {
  double n = 0, d = 0;
  for (size_t i = 0; i < a.flat().size(); ++i) {
    n += (a.flat()[i] - b.flat()[i]) * (a.flat()[i] - b.flat()[i]);
    d += b.flat()[i] * b.flat()[i];
  }
  return std::sqrt(n / std::max(d, 1e-300));
}

double rel_max_shards(const std::vector<CenterShard>& a, const std::vector<CenterShard>& b) {
  double n = 0, d = 0;
  for (size_t k = 0; k < a.size(); ++k)
    for (size_t i = 0; i < a[k].weights.flat().size(); ++i) {
      n = std::max(n, std::fabs(a[k].weights.flat()[i] - b[k].weights.flat()[i]));
      d = std::max(d, std::fabs(b[k].weights.flat()[i]));
    }
  return n / std::max(d, 1e-300);
}

struct Case {
  const char* name;
  int64_t C, K, B, D;
  double r;
  MarginConfig margin;
  std::optional<double> tau;
  int precision;
  double tol_loss, tol_dx, tol_w;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--source-hash") {
    std::printf("%s\n", PFC_SRC_HASH);
    return 0;
  }
  const Case cases[] = {
      {"tiny_cos_fp32", 400, 4, 32, 32, 0.5, MarginConfig::cosface_style(), std::nullopt,
       PFC_PRECISION_FP32, 1e-6, 1e-5, 1e-6},
      {"filter_full_fp32", 300, 3, 24, 32, 1.0, MarginConfig::cosface_style(), 0.1,
       PFC_PRECISION_FP32, 1e-6, 1e-5, 1e-6},
      {"arc_10k_fp32", 10000, 1, 128, 512, 0.1, MarginConfig::arcface_style(), std::nullopt,
       PFC_PRECISION_FP32, 1e-6, 1e-5, 1e-6},
      {"arc_10k_bf16", 10000, 1, 128, 512, 0.1, MarginConfig::arcface_style(), std::nullopt,
       PFC_PRECISION_BF16, 1e-4, 1e-2, 1e-3},
      {"arc_40k_k4_bf16", 40000, 4, 256, 512, 0.1, MarginConfig::arcface_style(), std::nullopt,
       PFC_PRECISION_BF16, 1e-4, 1e-2, 1e-3},
  };
  bool ok = true;
  for (const Case& cs : cases) {
    const ShardLayout layout(cs.C, cs.K);
    std::vector<CenterShard> ref = init_center_shards(layout, cs.D, 1);
    std::vector<CenterShard> dev = ref;
    StepConfig cfg;
    cfg.r = cs.r;
    cfg.margin = cs.margin;
    cfg.filter_threshold = cs.tau;
    cfg.lr = 0.1;
    gpu::Session session(layout, cs.D, cfg, cs.B, cs.precision);
    session.upload(dev);
    for (uint64_t step = 0; step < 2; ++step) {
      const FeatureBatch batch = bench_batch(cs.C, cs.D, cs.B, step);
      const SeededRng it(1, make_stream("iteration", step));
      const StepResult want = distributed_partial_step(ref, batch, cfg, it);
      const StepResult got = session.step(batch, cfg, it);
      session.download(dev);
      bool buffers_equal = want.buffers.size() == got.buffers.size();
      for (size_t k = 0; buffers_equal && k < want.buffers.size(); ++k)
        buffers_equal = want.buffers[k].class_indices == got.buffers[k].class_indices &&
                        want.buffers[k].num_positives == got.buffers[k].num_positives;
      const double dl = std::fabs(got.loss - want.loss) / std::fabs(want.loss);
      const double dx = rel_fro(got.d_features, want.d_features);
      const double dw = rel_max_shards(dev, ref);
      const bool trace_ok = got.trace == want.trace;
      const bool pass = buffers_equal && trace_ok && dl <= cs.tol_loss && dx <= cs.tol_dx &&
                        dw <= cs.tol_w;
      ok = ok && pass;
      std::printf(
          "{\"case\": \"%s\", \"step\": %llu, \"buffers_bit_exact\": %s, \"trace_equal\": %s, "
          "\"loss\": %.12f, \"loss_ref\": %.12f, \"loss_rel\": %.3e, \"dX_fro\": %.3e, "
          "\"W_maxmax\": %.3e, \"pass\": %s}\n",
          cs.name, (unsigned long long)step, buffers_equal ? "true" : "false",
          trace_ok ? "true" : "false", got.loss, want.loss, dl, dx, dw, pass ? "true" : "false");
    }
  }
  // StepConfig per call (shardsim.hpp:166-168): r, margin, filter, momentum and weight decay
  // change from step to step on one session (the capacity grows, shrinks, per-row offsets at
  // s = 128), against the reference taking each config as given
  for (int precision : {PFC_PRECISION_FP32, PFC_PRECISION_BF16}) {
    const ShardLayout layout(20000, 4);
    const int64_t D = 256, B = 96;
    std::vector<CenterShard> ref = init_center_shards(layout, D, 3);
    std::vector<CenterShard> dev = ref;
    StepConfig cfgs[5];
    cfgs[0].r = 0.1;
    cfgs[0].margin = MarginConfig::arcface_style();
    cfgs[1].r = 0.2;
    cfgs[1].margin = MarginConfig::cosface_style();
    cfgs[1].momentum = 0.5;
    cfgs[2].r = 0.05;
    cfgs[2].margin = MarginConfig::cosface_style();
    // the filter in fp32 only: in bf16 the mask is decided on bf16-operand cosines and may flip
    // within 2^-7 of tau (that contract is tests/test_gpu_edges.py::test_bf16_filter_contract)
    if (precision == PFC_PRECISION_FP32) cfgs[2].filter_threshold = 0.1;
    cfgs[2].weight_decay = 0.0;
    cfgs[3].r = 0.3;
    cfgs[3].margin = MarginConfig::cosface_style(128.0, 0.35);
    cfgs[4] = cfgs[0];
    const bool fp32 = precision == PFC_PRECISION_FP32;
    gpu::Session session(layout, D, cfgs[0], B, precision);
    session.upload(dev);
    double worst_l = 0, worst_x = 0, worst_w = 0, fw = 1.0;
    bool bufs = true, pass = true;
    for (uint64_t step = 0; step < 5; ++step) {
      StepConfig cfg = cfgs[step];
      cfg.lr = 0.1;
      const FeatureBatch batch = bench_batch(layout.num_classes, D, B, step);
      const SeededRng it(1, make_stream("iteration", step));
      const StepResult want = distributed_partial_step(ref, batch, cfg, it);
      const StepResult got = session.step(batch, cfg, it);
      session.download(dev);
      for (size_t k = 0; k < want.buffers.size(); ++k)
        bufs = bufs && want.buffers[k].class_indices == got.buffers[k].class_indices;
      // the value bounds scale with s / 64 (logit rounding times s; W' by (s/64)^2, as in
      // tests/test_gpu_edges.py)
      // (W and momentum carry earlier steps' errors: the largest scale so far bounds W')
      const double f = std::max(1.0, cfg.margin.scale / 64.0);
      fw = std::max(fw, f);
      const double dl = std::fabs(got.loss - want.loss) / std::fabs(want.loss);
      const double dx = rel_fro(got.d_features, want.d_features);
      const double dw = rel_max_shards(dev, ref);
      worst_l = std::max(worst_l, dl);
      worst_x = std::max(worst_x, dx);
      worst_w = std::max(worst_w, dw);
      pass = pass && dl <= (fp32 ? 1e-6 : 1e-4) * f && dx <= (fp32 ? 1e-5 : 1e-2) * f &&
             dw <= (fp32 ? 1e-6 : 1e-3) * fw * fw;
    }
    pass = pass && bufs;
    ok = ok && pass;
    std::printf("{\"case\": \"step_config_per_call_%s\", \"steps\": 5, \"buffers_bit_exact\": %s, "
                "\"loss_rel_max\": %.3e, \"dX_fro_max\": %.3e, \"W_maxmax\": %.3e, \"pass\": %s}\n",
                fp32 ? "fp32" : "bf16", bufs ? "true" : "false", worst_l, worst_x, worst_w,
                pass ? "true" : "false");
  }
  // with_diagnostics (shardsim.hpp:401-410): apcs / amncs on the pre-update shards, with the
  // conflict split; the GPU values are exact up to fp32 storage of W
  {
    const ShardLayout layout(4000, 4);
    std::vector<CenterShard> ref = init_center_shards(layout, 512, 1);
    StepConfig cfg;
    cfg.margin = MarginConfig::arcface_style();
    cfg.with_diagnostics = true;
    cfg.step_index = 3;
    gpu::Session session(layout, 512, cfg, 64);
    session.upload(ref);
    const FeatureBatch batch = bench_batch(4000, 512, 64, 0);
    std::vector<int64_t> cid(4000), sid(64);
    for (int64_t j = 0; j < 4000; ++j) cid[j] = j / 3;
    for (int64_t b = 0; b < 64; ++b) sid[b] = batch.labels[b] / 3 + (b % 5 == 0 ? 1 : 0);
    const ConflictInfo info{std::span<const int64_t>(cid), std::span<const int64_t>(sid)};
    cfg.conflict = &info;
    const SeededRng it(1, make_stream("iteration", 0));
    const StepResult want = distributed_partial_step(ref, batch, cfg, it);
    const StepResult got = session.step(batch, cfg, it);
    const auto& a = *got.diagnostics;
    const auto& b = *want.diagnostics;
    const double e = std::max({std::fabs(a.apcs - b.apcs), std::fabs(a.amncs - b.amncs),
                               std::fabs(*a.amncs_hard - *b.amncs_hard),
                               std::fabs(*a.amncs_conflicted - *b.amncs_conflicted)});
    const bool pass = got.diagnostics && want.diagnostics && a.iteration == b.iteration &&
                      a.amncs_hard.has_value() == b.amncs_hard.has_value() && e <= 1e-6 &&
                      std::fabs(got.loss - want.loss) / std::fabs(want.loss) <= 1e-4;
    ok = ok && pass;
    std::printf("{\"case\": \"with_diagnostics\", \"apcs\": %.12f, \"apcs_ref\": %.12f, "
                "\"amncs\": %.12f, \"amncs_ref\": %.12f, \"max_abs\": %.3e, \"pass\": %s}\n",
                a.apcs, b.apcs, a.amncs, b.amncs, e, pass ? "true" : "false");
  }
  // checkpoint (trainer.hpp:235-338): the reference's save_checkpoint writes the shards; the
  // device reads its shard section in place; a device-written section parses with the
  // reference's BinaryReader
  {
    const ShardLayout layout(5000, 4);
    detail::CheckpointState cs;
    cs.next_step = 7;
    cs.shards = init_center_shards(layout, 64, 9);
    // fp32-representable values (the device keeps fp32 master weights), so the round trip is
    // an equality
    for (auto& sh : cs.shards) {
      for (double& v : sh.weights.flat()) v = static_cast<double>(static_cast<float>(v));
      for (size_t i = 0; i < sh.momentum.flat().size(); ++i)
        sh.momentum.flat()[i] = static_cast<double>(1e-3f * static_cast<float>(i % 97));
    }
    const std::string path = "/tmp/pfc_adapter_ckpt.bin";
    detail::save_checkpoint(path, cs, 0x1234);
    // section offset: magic, version, digest, next_step, loss_sum, metrics_lines, 4 matrices
    int64_t off = 8 + 4 + 8 + 8 + 8 + 8;
    for (const Matrix* m : {&cs.backbone.w1, &cs.backbone.b1, &cs.backbone.w2, &cs.backbone.b2})
      off += 16 + 8 * m->rows() * m->cols();
    StepConfig cfg;
    gpu::Session session(layout, 64, cfg, 16);
    int64_t end = 0;
    gpu::check(pfc_gpu_read_shards(session.handle(), path.c_str(), off, &end), session.handle());
    std::vector<CenterShard> got = cs.shards;
    session.download(got);
    auto eq = [](const Matrix& a, const Matrix& b) {
      return a.flat().size() == b.flat().size() &&
             std::equal(a.flat().begin(), a.flat().end(), b.flat().begin());
    };
    bool same = true;
    for (size_t k = 0; k < got.size(); ++k)
      same = same && eq(got[k].weights, cs.shards[k].weights) &&
             eq(got[k].momentum, cs.shards[k].momentum);
    // and back: the device's section read by the reference reader
    const std::string p2 = "/tmp/pfc_adapter_ckpt2.bin";
    gpu::check(pfc_gpu_write_shards(session.handle(), p2.c_str(), 0), session.handle());
    BinaryReader r(p2);
    bool back = r.get<int64_t>() == 4;
    for (int64_t k = 0; k < 4 && back; ++k) {
      back = r.get<int64_t>() == k && r.get<int64_t>() == layout.owned_begin(k) &&
             r.get<int64_t>() == layout.owned_end(k);
      const Matrix w = r.get_matrix(), m = r.get_matrix();
      back = back && eq(w, cs.shards[k].weights) && eq(m, cs.shards[k].momentum);
    }
    const bool pass = same && back && end > off;
    ok = ok && pass;
    std::printf("{\"case\": \"checkpoint_reference_format\", \"device_reads_reference\": %s, "
                "\"reference_reads_device\": %s, \"pass\": %s}\n",
                same ? "true" : "false", back ? "true" : "false", pass ? "true" : "false");
  }
  // the unchanged-signature free function on host shards + the reference's error text
  {
    const ShardLayout layout(1000, 4);
    std::vector<CenterShard> shards = init_center_shards(layout, 8, 1);
    FeatureBatch fb;
    fb.features = Matrix(8, 125);
    for (int64_t b = 0; b < 125; ++b) fb.labels.push_back(b * 8);
    StepConfig cfg;
    std::string want, got;
    try {
      distributed_partial_step(shards, fb, cfg, SeededRng(1, 1));
    } catch (const CapacityError& e) {
      want = e.what();
    }
    try {
      gpu::distributed_partial_step(shards, fb, cfg, SeededRng(1, 1));
    } catch (const CapacityError& e) {
      got = e.what();
    }
    const bool pass = !want.empty() && want == got;
    ok = ok && pass;
    std::printf("{\"case\": \"capacity_error_text\", \"pass\": %s}\n", pass ? "true" : "false");
  }
  return ok ? 0 : 1;
}
