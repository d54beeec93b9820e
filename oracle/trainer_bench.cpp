// trainer_bench.cpp — trainer throughput, reference vs device (MEASUREMENT, built like the
// parity programs against the unmodified reference headers into oracle/_ref/trainer_bench).
//
// pfc::train (trainer.hpp:362-581, fp64 on the host) and pfc::gpu::train (include/
// pfc/gpu_trainer.hpp: backbone, step and diagnostics on the GPU) run the same SyntheticDataset
// and TrainConfig for `steps` steps (stop_after_step, so the reference's O(N C d) final
// evaluation is not timed).  Prints one JSON line with ms per training step for each.
#include <string>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "pfc/gpu_trainer.hpp"
#include "pfc/trainer.hpp"

#ifndef PFC_SRC_HASH  // sha256 prefix of the sources this program was built from (Makefile)
#define PFC_SRC_HASH "unknown"
#endif

using namespace pfc;

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "--source-hash") {
    std::printf("%s\n", PFC_SRC_HASH);
    return 0;
  }
  const int64_t identities = argc > 1 ? std::atoll(argv[1]) : 20000;
  const int64_t steps = argc > 2 ? std::atoll(argv[2]) : 100;
  SynthConfig sc;
  sc.num_identities = identities;
  sc.samples_min = 8;
  sc.samples_max = 12;
  sc.dim = 64;
  sc.seed = 11;
  const SyntheticDataset ds = generate(sc);
  TrainConfig cfg;
  cfg.r = 0.1;
  cfg.shards = 8;
  cfg.batch = 512;
  cfg.epochs = 3;
  cfg.warmup_epochs = 0.5;
  cfg.eval_every = 50;
  cfg.hidden_dim = 256;
  cfg.embed_dim = 128;
  cfg.margin = MarginConfig::arcface_style();
  cfg.stop_after_step = steps;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  // warm-up of the device (context, module load, graph capture) outside the timing
  {
    TrainConfig w = cfg;
    w.stop_after_step = 2;
    gpu::train(ds, w, nullptr, PFC_PRECISION_BF16);
  }
  auto t0 = now();
  const TrainResult g = gpu::train(ds, cfg, nullptr, PFC_PRECISION_BF16);
  auto t1 = now();
  const TrainResult r = train(ds, cfg);
  auto t2 = now();
  std::printf("{\"bench\": \"trainer\", \"classes\": %lld, \"points\": %lld, \"batch\": %lld, "
              "\"embed_dim\": %lld, \"hidden_dim\": %lld, \"shards\": %lld, \"r\": %.2f, "
              "\"steps\": %lld, \"gpu_ms_per_step\": %.4f, \"ref_ms_per_step\": %.4f, "
              "\"speedup\": %.1f, \"gpu_mean_loss\": %.6f, \"ref_mean_loss\": %.6f, "
              "\"records\": [%zu, %zu]}\n",
              (long long)ds.num_classes(), (long long)ds.num_points(), (long long)cfg.batch,
              (long long)cfg.embed_dim, (long long)cfg.hidden_dim, (long long)cfg.shards, cfg.r,
              (long long)g.steps_run, ms(t0, t1) / (double)g.steps_run,
              ms(t1, t2) / (double)r.steps_run, ms(t1, t2) / ms(t0, t1) * (double)g.steps_run /
                                                    (double)r.steps_run,
              g.mean_loss, r.mean_loss, g.diagnostics.size(), r.diagnostics.size());
  return 0;
}
