// trainer_parity.cpp — parity test of the trainer integration (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against the UNMODIFIED reference headers and
// include/pfc/gpu_trainer.hpp into oracle/_ref/trainer_parity.  The same SyntheticDataset and
// TrainConfig go through the reference's pfc::train (trainer.hpp:362-581, fp64 on the CPU) and
// pfc::gpu::train (backbone, step, diagnostics on the GPU; X / dX resident in HBM), patterned on
// proj/tests/test_trainer.cpp.  Cases:
//   train_<precision>[_conflict]  end results of a multi-epoch run (losses, diagnostics records,
//                                  mics, accuracy, verification, backbone) within tolerance
//   resume_bit_exact               GPU stop_after_step + checkpoint + resume == uninterrupted GPU
//   checkpoint_cross               the GPU resumes the reference's checkpoint and the reference
//                                  resumes the GPU's (byte-compatible containers)
// Prints one JSON line per case; exit 0 iff every case passes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "pfc/gpu_trainer.hpp"
#include "pfc/trainer.hpp"

#ifndef PFC_SRC_HASH  // sha256 prefix of the sources this program was built from (Makefile)
#define PFC_SRC_HASH "unknown"
#endif

using namespace pfc;

namespace {

SyntheticDataset make_dataset(bool conflicts) {
  SynthConfig sc;
  sc.num_identities = 300;
  sc.samples_min = 6;
  sc.samples_max = 10;
  sc.dim = 32;
  sc.seed = 5;
  SyntheticDataset ds = generate(sc);
  if (conflicts) {
    SeededRng rng(7, make_stream("parity-split"));
    ds = conflict_split(ds, 20, 20, rng);
  }
  return ds;
}

TrainConfig make_config() {
  TrainConfig c;
  c.r = 0.25;
  c.shards = 2;
  c.batch = 48;
  c.epochs = 2;
  c.eval_every = 20;
  c.hidden_dim = 48;
  c.embed_dim = 64;
  c.margin = MarginConfig::arcface_style();
  c.warmup_epochs = 0.5;
  return c;
}

double rel(double a, double b) { return std::fabs(a - b) / std::max(std::fabs(b), 1e-300); }

double rel_max(const Matrix& a, const Matrix& b) {
  double n = 0, d = 0;
  for (size_t i = 0; i < a.flat().size(); ++i) {
    n = std::max(n, std::fabs(a.flat()[i] - b.flat()[i]));
    d = std::max(d, std::fabs(b.flat()[i]));
  }
  return n / std::max(d, 1e-300);
}

double rel_fro(const Matrix& a, const Matrix& b, double& num, double& den) {
  for (size_t i = 0; i < a.flat().size(); ++i) {
    num += (a.flat()[i] - b.flat()[i]) * (a.flat()[i] - b.flat()[i]);
    den += b.flat()[i] * b.flat()[i];
  }
  return std::sqrt(num / std::max(den, 1e-300));
}

struct Cmp {
  double loss_mean, loss_final, diag, mics, acc, tar, backbone, centers;
  double backbone_fro, centers_fro;  // norm-wise (the bf16 contract is norm-wise)
  bool same_records;
};

Cmp compare(const TrainResult& g, const TrainResult& r) {
  Cmp c{};
  c.loss_mean = rel(g.mean_loss, r.mean_loss);
  c.loss_final = rel(g.final_loss, r.final_loss);
  c.same_records = g.diagnostics.size() == r.diagnostics.size() && g.steps_run == r.steps_run &&
                   g.stopped_early == r.stopped_early &&
                   g.verification.has_value() == r.verification.has_value();
  for (size_t i = 0; c.same_records && i < g.diagnostics.size(); ++i) {
    const auto &a = g.diagnostics[i], &b = r.diagnostics[i];
    c.same_records = a.iteration == b.iteration &&
                     a.amncs_hard.has_value() == b.amncs_hard.has_value() &&
                     a.amncs_conflicted.has_value() == b.amncs_conflicted.has_value();
    c.diag = std::max({c.diag, std::fabs(a.apcs - b.apcs), std::fabs(a.amncs - b.amncs)});
    if (a.amncs_hard && b.amncs_hard) c.diag = std::max(c.diag, std::fabs(*a.amncs_hard - *b.amncs_hard));
    if (a.amncs_conflicted && b.amncs_conflicted)
      c.diag = std::max(c.diag, std::fabs(*a.amncs_conflicted - *b.amncs_conflicted));
  }
  c.mics = std::fabs(g.mics_max - r.mics_max);
  c.acc = std::fabs(g.train_accuracy - r.train_accuracy);
  c.tar = g.verification && r.verification ? std::fabs(g.verification->tar - r.verification->tar) : 0.0;
  c.backbone = std::max(rel_max(g.backbone.w1, r.backbone.w1), rel_max(g.backbone.w2, r.backbone.w2));
  double n = 0, d = 0;
  rel_fro(g.backbone.w1, r.backbone.w1, n, d);
  c.backbone_fro = rel_fro(g.backbone.w2, r.backbone.w2, n, d);
  n = d = 0;
  for (size_t k = 0; k < g.shards.size() && k < r.shards.size(); ++k) {
    c.centers = std::max(c.centers, rel_max(g.shards[k].weights, r.shards[k].weights));
    c.centers_fro = rel_fro(g.shards[k].weights, r.shards[k].weights, n, d);
  }
  return c;
}

bool identical(const TrainResult& a, const TrainResult& b) {
  auto eq = [](const Matrix& x, const Matrix& y) {
    return x.flat().size() == y.flat().size() &&
           std::equal(x.flat().begin(), x.flat().end(), y.flat().begin());
  };
  bool same = a.mean_loss == b.mean_loss && a.final_loss == b.final_loss &&
              a.mics_max == b.mics_max && a.train_accuracy == b.train_accuracy &&
              a.steps_run == b.steps_run && a.diagnostics.size() == b.diagnostics.size() &&
              eq(a.backbone.w1, b.backbone.w1) && eq(a.backbone.w2, b.backbone.w2) &&
              eq(a.backbone.b1, b.backbone.b1) && eq(a.backbone.b2, b.backbone.b2);
  for (size_t i = 0; same && i < a.diagnostics.size(); ++i)
    same = a.diagnostics[i].iteration == b.diagnostics[i].iteration &&
           a.diagnostics[i].apcs == b.diagnostics[i].apcs &&
           a.diagnostics[i].amncs == b.diagnostics[i].amncs;
  for (size_t k = 0; same && k < a.shards.size(); ++k)
    same = eq(a.shards[k].weights, b.shards[k].weights) && eq(a.shards[k].momentum, b.shards[k].momentum);
  return same;
}

struct Lines : TrainSink {
  std::vector<std::string> lines;
  void metrics_line(const std::string& l) override { lines.push_back(l); }
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--source-hash") {
    std::printf("%s\n", PFC_SRC_HASH);
    return 0;
  }
  bool ok = true;
  // ---- end results against the reference (fp32 validation mode and bf16 tensor cores)
  struct Run {
    const char* name;
    bool conflicts;
    int precision;
    double tol_loss, tol_diag, tol_acc, tol_tar, tol_w;
    bool normwise;  // gate the backbone / centres on the relative Frobenius error
  };
  const Run runs[] = {
      {"train_fp32", false, PFC_PRECISION_FP32, 1e-4, 1e-4, 0.01, 0.02, 1e-3, false},
      {"train_fp32_conflict", true, PFC_PRECISION_FP32, 1e-4, 1e-4, 0.01, 0.02, 1e-3, false},
      {"train_bf16", false, PFC_PRECISION_BF16, 2e-2, 2e-2, 0.05, 0.1, 0.1, true},
      {"train_bf16_conflict", true, PFC_PRECISION_BF16, 2e-2, 2e-2, 0.05, 0.1, 0.1, true},
  };
  for (const Run& run : runs) {
    const SyntheticDataset ds = make_dataset(run.conflicts);
    const TrainConfig cfg = make_config();
    Lines ref_lines, gpu_lines;
    double t0 = now_ms();
    const TrainResult want = train(ds, cfg, &ref_lines);
    const double t_ref = now_ms() - t0;
    t0 = now_ms();
    const TrainResult got = gpu::train(ds, cfg, &gpu_lines, run.precision);
    const double t_gpu = now_ms() - t0;
    const Cmp c = compare(got, want);
    const bool pass = c.same_records && gpu_lines.lines.size() == ref_lines.lines.size() &&
                      c.loss_mean <= run.tol_loss && c.diag <= run.tol_diag &&
                      c.mics <= run.tol_diag && c.acc <= run.tol_acc && c.tar <= run.tol_tar &&
                      (run.normwise ? c.backbone_fro : c.backbone) <= run.tol_w &&
                      (run.normwise ? c.centers_fro : c.centers) <= run.tol_w;
    ok = ok && pass;
    std::printf(
        "{\"case\": \"%s\", \"steps\": %lld, \"records\": %zu, \"mean_loss\": %.9f, "
        "\"mean_loss_ref\": %.9f, \"mean_loss_rel\": %.3e, \"final_loss_rel\": %.3e, "
        "\"diag_max_abs\": %.3e, \"mics_abs\": %.3e, \"acc\": %.4f, \"acc_ref\": %.4f, "
        "\"tar_abs\": %.3e, \"backbone_rel\": %.3e, \"centers_rel\": %.3e, "
        "\"backbone_fro\": %.3e, \"centers_fro\": %.3e, \"ms_gpu\": %.1f, \"ms_ref\": %.1f, "
        "\"pass\": %s}\n",
        run.name, (long long)got.steps_run, got.diagnostics.size(), got.mean_loss, want.mean_loss,
        c.loss_mean, c.loss_final, c.diag, c.mics, got.train_accuracy, want.train_accuracy, c.tar,
        c.backbone, c.centers, c.backbone_fro, c.centers_fro, t_gpu, t_ref,
        pass ? "true" : "false");
  }
  // ---- checkpoint / resume on the GPU is bit-identical to the uninterrupted GPU run
  {
    const SyntheticDataset ds = make_dataset(true);
    TrainConfig cfg = make_config();
    const TrainResult full = gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    cfg.checkpoint_path = "/tmp/pfc_trainer_parity_gpu.ckpt";
    cfg.stop_after_step = 37;
    const TrainResult part = gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    cfg.stop_after_step = 0;
    cfg.resume = true;
    const TrainResult resumed = gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    const bool pass = part.stopped_early && part.steps_run == 37 && identical(resumed, full);
    ok = ok && pass;
    std::printf("{\"case\": \"resume_bit_exact\", \"stopped_at\": %lld, \"mean_loss\": %.17g, "
                "\"mean_loss_full\": %.17g, \"pass\": %s}\n",
                (long long)part.steps_run, resumed.mean_loss, full.mean_loss, pass ? "true" : "false");
  }
  // ---- the containers are compatible both ways
  {
    const SyntheticDataset ds = make_dataset(false);
    TrainConfig cfg = make_config();
    const TrainResult ref_full = train(ds, cfg);
    const TrainResult gpu_full = gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    cfg.stop_after_step = 29;
    // reference stops, GPU resumes
    cfg.checkpoint_path = "/tmp/pfc_trainer_parity_ref.ckpt";
    cfg.resume = false;
    train(ds, cfg);
    cfg.resume = true;
    cfg.stop_after_step = 0;
    const TrainResult gpu_resumed = gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    // GPU stops, reference resumes
    cfg.checkpoint_path = "/tmp/pfc_trainer_parity_gpu2.ckpt";
    cfg.resume = false;
    cfg.stop_after_step = 29;
    gpu::train(ds, cfg, nullptr, PFC_PRECISION_FP32);
    cfg.resume = true;
    cfg.stop_after_step = 0;
    const TrainResult ref_resumed = train(ds, cfg);
    const Cmp a = compare(gpu_resumed, ref_full);
    const Cmp b = compare(ref_resumed, gpu_full);
    const bool pass = a.same_records && b.same_records && a.loss_mean <= 1e-4 &&
                      b.loss_mean <= 1e-4 && a.diag <= 1e-4 && b.diag <= 1e-4;
    ok = ok && pass;
    std::printf("{\"case\": \"checkpoint_cross\", \"gpu_resumes_ref_loss_rel\": %.3e, "
                "\"ref_resumes_gpu_loss_rel\": %.3e, \"pass\": %s}\n",
                a.loss_mean, b.loss_mean, pass ? "true" : "false");
  }
  return ok ? 0 : 1;
}
