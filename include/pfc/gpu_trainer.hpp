// gpu_trainer.hpp — pfc::gpu::train: the reference's training loop (trainer.hpp:362-581) with
// its hot path on the B200 and the step's features / gradients resident in HBM.
//
//   #include "pfc/gpu_trainer.hpp"       // pulls in the host project's pfc/trainer.hpp
//   TrainResult r = pfc::gpu::train(dataset, cfg, sink);     // == pfc::train(dataset, cfg, sink)
//
// What runs where:
//   device  the dataset points, the backbone (forward, apply_gradient), the centre shards, every
//           distributed_partial_step, the with_diagnostics apcs / amncs, mics, the checkpoint's
//           shard section (pfc_gpu_write_shards / pfc_gpu_read_shards).
//   host    the identity split, the epoch shuffles and the lr schedule (the reference's own
//           functions), the checkpoint header / backbone / diagnostics sections, and the final
//           nearest-centre accuracy and verification over downloaded embeddings (evaluation).
// Per step the host sends the batch's point ids (8 B each) and reads back the step status.
//
// Same inputs, same outputs: TrainConfig / SyntheticDataset / TrainSink / TrainResult are the host
// project's types; checkpoints are byte-compatible with pfc::train's in both directions
// (trainer.hpp:235-338).  Numerics: the backbone is fp64 with the reference's summation order;
// the step follows the precision chosen (PFC_PRECISION_BF16 or _FP32).
#pragma once

#include <cstdio>
#include <string>
#include <vector>

#include "pfc/gpu_step.hpp"
#include "pfc/trainer.hpp"

namespace pfc::gpu {

// RAII handle over pfc_gpu_trainer_* (include/pfc_gpu.h)
class DeviceTrainer {
 public:
  DeviceTrainer(Session& session, const SyntheticDataset& ds, const TrainConfig& cfg)
      : ctx_(session.handle()), hidden_(cfg.hidden_dim), embed_(cfg.embed_dim), in_(ds.dim()) {
    void* t = nullptr;
    check(pfc_gpu_trainer_create(ctx_, ds.points.flat().data(), ds.dim(), ds.num_points(),
                                 ds.observed_labels.data(), cfg.hidden_dim, cfg.embed_dim,
                                 cfg.seed, &t),
          ctx_);
    t_ = t;
  }
  ~DeviceTrainer() {
    if (t_) pfc_gpu_trainer_destroy(t_);
  }
  DeviceTrainer(const DeviceTrainer&) = delete;
  DeviceTrainer& operator=(const DeviceTrainer&) = delete;

  void forward(const int64_t* ids, int64_t n) { check(pfc_gpu_trainer_forward(t_, ids, n), ctx_); }
  DiagnosticsSnapshot diagnostics(const ConflictInfo* conflict, int64_t iteration) {
    pfc_gpu_diag_out o{};
    check(pfc_gpu_trainer_diagnostics(t_, conflict ? conflict->class_identity.data() : nullptr,
                                      conflict ? conflict->sample_identity.data() : nullptr, &o),
          ctx_);
    DiagnosticsSnapshot d;
    d.iteration = iteration;
    d.apcs = o.apcs;
    d.amncs = o.amncs;
    if (o.has_conflicted) d.amncs_conflicted = o.amncs_conflicted;
    if (o.has_split) d.amncs_hard = o.amncs_hard;
    return d;
  }
  double step(const SeededRng& rng, double lr, int64_t step_index) {
    pfc_gpu_step_args a{rng.seed(), rng.stream_id(), lr, step_index};
    pfc_gpu_step_out o{};
    check(pfc_gpu_trainer_step(t_, &a, &o), ctx_);
    return o.loss;
  }
  void apply_gradient(double lr) { check(pfc_gpu_trainer_apply_gradient(t_, lr), ctx_); }
  void nearest_center(const std::vector<int64_t>& ids, std::vector<int64_t>& best) {
    check(pfc_gpu_trainer_nearest_center(t_, ids.data(), static_cast<int64_t>(ids.size()),
                                         best.data()),
          ctx_);
  }
  void pair_cosines(const std::vector<int64_t>& ids, std::vector<double>& out) {
    check(pfc_gpu_trainer_pair_cosines(t_, ids.data(), static_cast<int64_t>(ids.size()),
                                       out.data()),
          ctx_);
  }
  Matrix embed(const std::vector<int64_t>& ids) {
    Matrix m(embed_, static_cast<int64_t>(ids.size()));
    if (!ids.empty())
      check(pfc_gpu_trainer_embed(t_, ids.data(), static_cast<int64_t>(ids.size()), m.flat().data()),
            ctx_);
    return m;
  }
  Backbone backbone() const {
    Backbone bb;
    bb.w1 = Matrix(hidden_, in_);
    bb.b1 = Matrix(hidden_, 1);
    bb.w2 = Matrix(embed_, hidden_);
    bb.b2 = Matrix(embed_, 1);
    check(pfc_gpu_trainer_get_backbone(t_, bb.w1.flat().data(), bb.b1.flat().data(),
                                       bb.w2.flat().data(), bb.b2.flat().data()),
          ctx_);
    return bb;
  }
  void set_backbone(const Backbone& bb) {
    if (bb.w1.rows() != hidden_ || bb.w1.cols() != in_ || bb.w2.rows() != embed_ ||
        bb.w2.cols() != hidden_ || bb.b1.rows() != hidden_ || bb.b2.rows() != embed_)
      throw ShapeError("pfc::gpu::train: checkpoint backbone shape differs from the config");
    check(pfc_gpu_trainer_set_backbone(t_, bb.w1.flat().data(), bb.b1.flat().data(),
                                       bb.w2.flat().data(), bb.b2.flat().data()),
          ctx_);
  }

 private:
  void* ctx_;
  void* t_ = nullptr;
  int64_t hidden_, embed_, in_;
};

namespace detail {

// The checkpoint container of trainer.hpp:235-338 (io.hpp encoding: raw little-endian scalars,
// matrices as int64 rows, int64 cols, rows*cols fp64), written and read in sections so that the
// centre shards go straight between the device and the file.
class CkptFile {
 public:
  CkptFile(const std::string& path, const char* mode) : path_(path), f_(std::fopen(path.c_str(), mode)) {
    if (!f_)
      throw DataError((mode[0] == 'r' ? "cannot open: " : "cannot open for writing: ") + path);
  }
  ~CkptFile() {
    if (f_) std::fclose(f_);
  }
  CkptFile(const CkptFile&) = delete;
  CkptFile& operator=(const CkptFile&) = delete;

  template <typename T>
  void put(T v) {
    if (std::fwrite(&v, sizeof(T), 1, f_) != 1) throw DataError("write failed: " + path_);
  }
  void put_matrix(const Matrix& m) {
    put<int64_t>(m.rows());
    put<int64_t>(m.cols());
    const auto fl = m.flat();
    if (!fl.empty() && std::fwrite(fl.data(), sizeof(double), fl.size(), f_) != fl.size())
      throw DataError("write failed: " + path_);
  }
  template <typename T>
  T get() {
    T v{};
    if (std::fread(&v, sizeof(T), 1, f_) != 1) throw DataError("truncated file: " + path_);
    return v;
  }
  Matrix get_matrix() {
    const auto rows = get<int64_t>();
    const auto cols = get<int64_t>();
    if (rows < 0 || cols < 0 || rows * cols > (1ll << 32))
      throw DataError("implausible matrix header in " + path_);
    Matrix m(rows, cols);
    auto fl = m.flat();
    if (!fl.empty() && std::fread(fl.data(), sizeof(double), fl.size(), f_) != fl.size())
      throw DataError("truncated file: " + path_);
    return m;
  }
  int64_t tell() const { return static_cast<int64_t>(std::ftell(f_)); }
  void seek(int64_t off) {
    if (std::fseek(f_, static_cast<long>(off), SEEK_SET) != 0) throw DataError("truncated file: " + path_);
  }
  void close() {
    const bool bad = std::fclose(f_) != 0;
    f_ = nullptr;
    if (bad) throw DataError("write failed: " + path_);
  }

 private:
  std::string path_;
  std::FILE* f_;
};

// save_checkpoint (trainer.hpp:235-275) with the shard section written from the device
inline void save_checkpoint(const std::string& path, Session& session, const DeviceTrainer& tr,
                            int64_t next_step, double loss_sum,
                            const std::vector<DiagnosticsSnapshot>& diags, uint64_t digest) {
  {
    CkptFile w(path, "wb");
    w.put<uint64_t>(pfc::detail::kCheckpointMagic);
    w.put<uint32_t>(pfc::detail::kCheckpointVersion);
    w.put<uint64_t>(digest);
    w.put<int64_t>(next_step);
    w.put<double>(loss_sum);
    w.put<int64_t>(static_cast<int64_t>(diags.size()));  // metrics_lines
    const Backbone bb = tr.backbone();
    w.put_matrix(bb.w1);
    w.put_matrix(bb.b1);
    w.put_matrix(bb.w2);
    w.put_matrix(bb.b2);
    w.close();
  }
  check(pfc_gpu_write_shards(session.handle(), path.c_str(), 1), session.handle());
  CkptFile w(path, "ab");
  w.put<int64_t>(static_cast<int64_t>(diags.size()));
  for (const DiagnosticsSnapshot& d : diags) {
    w.put<int64_t>(d.iteration);
    w.put<double>(d.apcs);
    w.put<double>(d.amncs);
    w.put<uint8_t>(d.amncs_conflicted.has_value());
    w.put<double>(d.amncs_conflicted.value_or(0.0));
    w.put<uint8_t>(d.amncs_hard.has_value());
    w.put<double>(d.amncs_hard.value_or(0.0));
  }
  w.close();
}

struct Resumed {
  int64_t next_step = 0;
  double loss_sum = 0.0;
  std::vector<DiagnosticsSnapshot> diagnostics;
};

// load_checkpoint (trainer.hpp:296-336) with the shard section read into the device
inline Resumed load_checkpoint(const std::string& path, uint64_t expect_digest, Session& session,
                               DeviceTrainer& tr) {
  Resumed st;
  int64_t shard_offset = 0;
  {
    CkptFile r(path, "rb");
    if (r.get<uint64_t>() != pfc::detail::kCheckpointMagic) throw DataError("not a checkpoint: " + path);
    if (r.get<uint32_t>() != pfc::detail::kCheckpointVersion)
      throw DataError("checkpoint version mismatch: " + path);
    if (r.get<uint64_t>() != expect_digest)
      throw DataError("checkpoint was produced by a different config/dataset: " + path);
    st.next_step = r.get<int64_t>();
    st.loss_sum = r.get<double>();
    r.get<int64_t>();  // metrics_lines
    Backbone bb;
    bb.w1 = r.get_matrix();
    bb.b1 = r.get_matrix();
    bb.w2 = r.get_matrix();
    bb.b2 = r.get_matrix();
    tr.set_backbone(bb);
    shard_offset = r.tell();
  }
  int64_t end = 0;
  check(pfc_gpu_read_shards(session.handle(), path.c_str(), shard_offset, &end), session.handle());
  CkptFile r(path, "rb");
  r.seek(end);
  const auto n = r.get<int64_t>();
  for (int64_t i = 0; i < n; ++i) {
    DiagnosticsSnapshot d;
    d.iteration = r.get<int64_t>();
    d.apcs = r.get<double>();
    d.amncs = r.get<double>();
    const bool has_c = r.get<uint8_t>() != 0;
    const double c = r.get<double>();
    const bool has_h = r.get<uint8_t>() != 0;
    const double h = r.get<double>();
    if (has_c) d.amncs_conflicted = c;
    if (has_h) d.amncs_hard = h;
    st.diagnostics.push_back(d);
  }
  return st;
}

inline std::vector<CenterShard> download_shards(const Session& session, const ShardLayout& layout,
                                                int64_t dim) {
  std::vector<CenterShard> shards;
  for (int64_t k = 0; k < layout.num_shards; ++k) {
    CenterShard s;
    s.shard_id = k;
    s.class_begin = layout.owned_begin(k);
    s.class_end = layout.owned_end(k);
    s.weights = Matrix(dim, s.class_end - s.class_begin);
    s.momentum = Matrix(dim, s.class_end - s.class_begin);
    shards.push_back(std::move(s));
  }
  session.download(shards);
  return shards;
}

}  // namespace detail

// == pfc::train(ds, cfg, sink) (trainer.hpp:362-581) with the step, the backbone and the
// diagnostics on device `device`.  precision: PFC_PRECISION_BF16 (tensor cores) or
// PFC_PRECISION_FP32 (validation).
inline TrainResult train(const SyntheticDataset& ds, const TrainConfig& cfg,
                         TrainSink* sink = nullptr, int precision = PFC_PRECISION_BF16,
                         int device = 0) {
  cfg.validate();
  ds.validate();
  const int64_t classes = ds.num_classes();
  const ShardLayout layout(classes, cfg.shards);

  // the identity-disjoint split and the point lists (trainer.hpp:370-382)
  const auto [train_ids, eval_ids] = split_identities(ds, cfg.eval_fraction, cfg.seed);
  std::vector<uint8_t> held_out(static_cast<size_t>(ds.num_identities()), 0);
  for (int64_t g : eval_ids) held_out[static_cast<size_t>(g)] = 1;
  std::vector<int64_t> train_points, eval_points;
  for (int64_t i = 0; i < ds.num_points(); ++i)
    (held_out[static_cast<size_t>(ds.true_identities[i])] ? eval_points : train_points).push_back(i);
  if (train_points.empty()) throw DataError("train: no training points after the split");

  // schedule (trainer.hpp:384-393)
  const auto n_train = static_cast<int64_t>(train_points.size());
  const int64_t steps_per_epoch = (n_train + cfg.batch - 1) / cfg.batch;
  Schedule schedule;
  schedule.base_lr = cfg.base_lr;
  schedule.total_steps = cfg.epochs * steps_per_epoch;
  schedule.warmup_steps =
      static_cast<int64_t>(cfg.warmup_epochs * static_cast<double>(steps_per_epoch));
  schedule.power = cfg.power;
  schedule.validate();
  const uint64_t digest = pfc::detail::config_digest(cfg, ds);

  // device state: shards (Session), dataset + backbone (DeviceTrainer)
  StepConfig base;
  base.r = cfg.r;
  base.margin = cfg.margin;
  base.filter_threshold = cfg.filter_threshold;
  base.momentum = cfg.momentum;
  base.weight_decay = cfg.weight_decay;
  Session session(layout, cfg.embed_dim, base, cfg.batch, precision, device);
  DeviceTrainer tr(session, ds, cfg);

  TrainResult result;
  double loss_sum = 0.0;
  int64_t start_step = 0;
  if (cfg.resume) {
    detail::Resumed st = detail::load_checkpoint(cfg.checkpoint_path, digest, session, tr);
    result.diagnostics = std::move(st.diagnostics);
    loss_sum = st.loss_sum;
    start_step = st.next_step;
  } else {
    session.init_center_shards(cfg.seed);  // init_center_shards(layout, embed_dim, seed)
  }

  const bool has_conflicts =
      std::any_of(ds.corruption.begin(), ds.corruption.end(),
                  [](const CorruptionRecord& c) { return c.conflict_group >= 0; });

  // epoch order: Fisher-Yates from ("shuffle", epoch) (trainer.hpp:415-424)
  std::vector<int64_t> order;
  int64_t order_epoch = -1;
  auto order_for = [&](int64_t epoch) {
    if (order_epoch == epoch) return;
    order = train_points;
    SeededRng rng(cfg.seed, make_stream("shuffle", static_cast<uint64_t>(epoch)));
    for (int64_t i = n_train - 1; i > 0; --i)
      std::swap(order[static_cast<size_t>(i)],
                order[static_cast<size_t>(rng.next_below(static_cast<uint64_t>(i + 1)))]);
    order_epoch = epoch;
  };
  auto save_state = [&](int64_t next_step) {
    if (cfg.checkpoint_path.empty()) return;
    detail::save_checkpoint(cfg.checkpoint_path, session, tr, next_step, loss_sum,
                            result.diagnostics, digest);
  };
  auto host_state = [&]() {
    result.backbone = tr.backbone();
    result.shards = detail::download_shards(session, layout, cfg.embed_dim);
  };

  const int64_t total_steps = schedule.total_steps;
  std::vector<int64_t> ids(static_cast<size_t>(cfg.batch));
  std::vector<int64_t> batch_identity(static_cast<size_t>(cfg.batch));
  for (int64_t step = start_step; step < total_steps; ++step) {
    const int64_t epoch = step / steps_per_epoch;
    const int64_t slot = step % steps_per_epoch;
    order_for(epoch);
    const int64_t lo = slot * cfg.batch;
    const int64_t bsz = std::min(lo + cfg.batch, n_train) - lo;
    for (int64_t b = 0; b < bsz; ++b) {
      ids[static_cast<size_t>(b)] = order[static_cast<size_t>(lo + b)];
      batch_identity[static_cast<size_t>(b)] = ds.true_identities[ids[static_cast<size_t>(b)]];
    }
    tr.forward(ids.data(), bsz);  // features stay on the device

    const double lr = lr_at(schedule, step);
    const bool with_diag = (step % cfg.eval_every == 0) || step == total_steps - 1;
    const ConflictInfo conflict{ds.class_identity,
                                std::span<const int64_t>(batch_identity.data(), static_cast<size_t>(bsz))};
    std::optional<DiagnosticsSnapshot> diag;
    if (with_diag) diag = tr.diagnostics(has_conflicts ? &conflict : nullptr, step);

    const SeededRng iter_rng(cfg.seed, make_stream("iteration", static_cast<uint64_t>(step)));
    double loss;
    try {
      loss = tr.step(iter_rng, lr, step);
    } catch (const NumericalError& e) {
      if (!cfg.checkpoint_path.empty())
        throw NumericalError(std::string(e.what()) + "; last good checkpoint: " + cfg.checkpoint_path);
      throw;
    }
    loss_sum += loss;
    result.final_loss = loss;
    if (lr > 0.0 && cfg.backbone_lr_scale > 0.0) tr.apply_gradient(lr * cfg.backbone_lr_scale);
    if (diag) {
      result.diagnostics.push_back(*diag);
      if (sink != nullptr) sink->metrics_line(pfc::detail::format_metrics_line(*diag));
    }
    result.steps_run = step + 1;
    if (cfg.stop_after_step > 0 && step + 1 >= cfg.stop_after_step && step + 1 < total_steps) {
      save_state(step + 1);
      result.stopped_early = true;
      result.mean_loss = loss_sum / static_cast<double>(result.steps_run);
      host_state();
      return result;
    }
  }
  result.mean_loss = total_steps > 0 ? loss_sum / static_cast<double>(total_steps) : 0.0;
  save_state(total_steps);

  // final-state diagnostics (trainer.hpp:516-518): mics on the device
  std::vector<double> mics_values(static_cast<size_t>(classes));
  check(pfc_gpu_mics(session.handle(), mics_values.data()), session.handle());
  result.mics_max = *std::max_element(mics_values.begin(), mics_values.end());
  host_state();

  // nearest-centre training accuracy (trainer.hpp:519-547): the O(n C D) scan runs on the
  // device (pfc_gpu_trainer_nearest_center, fp64 in the reference's order)
  {
    std::vector<int64_t> best(static_cast<size_t>(n_train));
    tr.nearest_center(train_points, best);
    int64_t correct = 0;
    for (int64_t b = 0; b < n_train; ++b)
      correct += best[static_cast<size_t>(b)] ==
                 ds.observed_labels[train_points[static_cast<size_t>(b)]];
    result.train_accuracy = static_cast<double>(correct) / static_cast<double>(n_train);
  }

  // open-set verification on the held-out identities (trainer.hpp:548-577): the pair cosines
  // come from the device (pfc_gpu_trainer_pair_cosines); scores are split by identity in the
  // reference's (i, j) order and scored by the host project's own verify_tar_at_far
  if (!eval_points.empty()) {
    const auto n_eval = static_cast<int64_t>(eval_points.size());
    std::vector<double> pair_cos(static_cast<size_t>(n_eval * (n_eval - 1) / 2));
    tr.pair_cosines(eval_points, pair_cos);
    std::vector<double> genuine, impostor;
    size_t at = 0;
    for (int64_t i = 0; i < n_eval; ++i)
      for (int64_t j = i + 1; j < n_eval; ++j, ++at) {
        const bool same = ds.true_identities[eval_points[static_cast<size_t>(i)]] ==
                          ds.true_identities[eval_points[static_cast<size_t>(j)]];
        (same ? genuine : impostor).push_back(pair_cos[at]);
      }
    if (!genuine.empty() && !impostor.empty()) {
      try {
        result.verification = verify_tar_at_far(genuine, impostor, cfg.far_target);
      } catch (const CapacityError&) {
        // too few impostor pairs to resolve far_target (as the reference)
      }
    }
  }
  return result;
}

}  // namespace pfc::gpu
