// gpu_step.hpp — C++ drop-in for pfc::distributed_partial_step over libpfc_gpu.so.
//
// Include this instead of calling the CPU simulator's step:
//
//   #include "pfc/gpu_step.hpp"      // pulls in the host project's pfc/shardsim.hpp types
//   pfc::gpu::Session session(layout, dim, cfg, max_batch);   // device-resident shards
//   session.upload(shards);                                    // or session.init_center_shards(seed)
//   StepResult r = session.step(batch, cfg, iteration_rng);    // == distributed_partial_step
//
// or, for callers that keep host-resident shards, the unchanged signature
//   StepResult pfc::gpu::distributed_partial_step(std::vector<CenterShard>&, const FeatureBatch&,
//                                                 const StepConfig&, const SeededRng&);
// (reference: proj/include/pfc/shardsim.hpp:166-168), which uploads the shards, steps on the
// B200 and downloads the updated shards each call.
//
// The value types are the host project's own (pfc/types.hpp, pfc/sampler.hpp, pfc/margin.hpp,
// pfc/rng.hpp, pfc/shardsim.hpp); failures are rethrown as the matching pfc::*Error with the
// reference's message text (pfc/error.hpp:9-42).
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "pfc/shardsim.hpp"
#include "pfc_gpu.h"

namespace pfc::gpu {

[[noreturn]] inline void throw_status(int rc, const char* msg) {
  const std::string m = msg ? msg : "pfc_gpu error";
  switch (rc) {
    case PFC_ERR_SHAPE: throw ShapeError(m);
    case PFC_ERR_CONTRACT: throw ContractError(m);
    case PFC_ERR_CAPACITY: throw CapacityError(m);
    case PFC_ERR_CONFIG: throw ConfigError(m);
    case PFC_ERR_NUMERICAL: throw NumericalError(m);
    case PFC_ERR_IO: throw DataError(m);
    default: throw Error(m);
  }
}

inline void check(int rc, const void* ctx) {
  if (rc != PFC_OK) throw_status(rc, pfc_gpu_last_error(ctx));
}

// Device-resident replacement of std::vector<CenterShard> for one rank (one GPU).
class Session {
 public:
  Session(const ShardLayout& layout, int64_t dim, const StepConfig& cfg, int64_t max_batch,
          int precision = PFC_PRECISION_BF16, int device = 0, int rank = 0, int world_size = 1,
          const uint8_t* nccl_id = nullptr, int flags = 0)
      : layout_(layout), dim_(dim), cfg_(cfg) {
    cfg.margin.validate();  // margin.hpp:22-28 (ConfigError)
    pfc_gpu_desc d{};
    d.num_classes = layout.num_classes;
    d.dim = dim;
    d.num_shards = layout.num_shards;
    d.max_batch = max_batch;
    d.r = cfg.r;
    d.margin_kind = static_cast<int32_t>(cfg.margin.kind);
    d.margin_scale = cfg.margin.scale;
    d.margin_m = cfg.margin.margin;
    d.has_filter = cfg.filter_threshold ? 1 : 0;
    d.filter_threshold = cfg.filter_threshold.value_or(0.0);
    d.momentum = cfg.momentum;
    d.weight_decay = cfg.weight_decay;
    d.precision = precision;
    d.device = device;
    d.rank = rank;
    d.world_size = world_size;
    d.nccl_id = nccl_id;
    d.flags = flags;
    void* h = nullptr;
    check(pfc_gpu_create(&d, &h), nullptr);
    ctx_ = h;
    pfc_gpu_local_shards(ctx_, &first_, &nlocal_);
  }
  ~Session() {
    if (ctx_) pfc_gpu_destroy(ctx_);
  }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  int64_t capacity() const { return pfc_gpu_capacity(ctx_); }
  bool owns_shard(int64_t k) const { return k >= first_ && k < first_ + nlocal_; }
  void* handle() const { return ctx_; }

  // CenterShard <-> device (types.hpp:29-47 layout: D x owned fp64)
  void upload(const std::vector<CenterShard>& shards) {
    for (const CenterShard& s : shards)
      if (owns_shard(s.shard_id))
        check(pfc_gpu_set_shard(ctx_, s.shard_id, s.weights.flat().data(),
                                s.momentum.flat().data()),
              ctx_);
  }
  void download(std::vector<CenterShard>& shards) const {
    for (CenterShard& s : shards)
      if (owns_shard(s.shard_id))
        check(pfc_gpu_get_shard(ctx_, s.shard_id, s.weights.flat().data(),
                                s.momentum.flat().data()),
              ctx_);
  }
  // init_center_shards (shardsim.hpp:56-82) on the device
  void init_center_shards(uint64_t seed) { check(pfc_gpu_init_shards(ctx_, seed), ctx_); }

  // apcs / amncs (metrics.hpp:56-146) of a batch against the current device shards
  DiagnosticsSnapshot diagnostics(const FeatureBatch& batch,
                                  const ConflictInfo* conflict = nullptr) {
    batch.validate();
    pfc_gpu_diag_out o{};
    check(pfc_gpu_diagnostics(ctx_, batch.features.flat().data(), batch.labels.data(),
                              batch.batch(), conflict ? conflict->class_identity.data() : nullptr,
                              conflict ? conflict->sample_identity.data() : nullptr, &o),
          ctx_);
    DiagnosticsSnapshot d;
    d.apcs = o.apcs;
    d.amncs = o.amncs;
    if (o.has_conflicted) d.amncs_conflicted = o.amncs_conflicted;
    if (o.has_split) d.amncs_hard = o.amncs_hard;
    return d;
  }

  // == distributed_partial_step(shards, batch, cfg, iteration_rng) with the shards on the GPU.
  StepResult step(const FeatureBatch& batch, const StepConfig& cfg,
                  const SeededRng& iteration_rng) {
    batch.validate();        // types.hpp:21-25 (ShapeError)
    cfg.margin.validate();   // margin.hpp:22-28 (ConfigError)
    if (cfg.margin.kind != cfg_.margin.kind || cfg.margin.scale != cfg_.margin.scale ||
        cfg.margin.margin != cfg_.margin.margin || cfg.r != cfg_.r ||
        cfg.filter_threshold != cfg_.filter_threshold || cfg.momentum != cfg_.momentum ||
        cfg.weight_decay != cfg_.weight_decay) {
      // the reference takes its StepConfig per call (shardsim.hpp:166-168)
      pfc_gpu_step_config sc{cfg.r, static_cast<int32_t>(cfg.margin.kind), cfg.margin.scale,
                             cfg.margin.margin, cfg.filter_threshold ? 1 : 0,
                             cfg.filter_threshold.value_or(0.0), cfg.momentum, cfg.weight_decay};
      check(pfc_gpu_set_step_config(ctx_, &sc), ctx_);
      cfg_ = cfg;
    }
    if (batch.dim() != dim_) throw ShapeError("pfc::gpu::Session::step: feature dim mismatch");
    std::optional<DiagnosticsSnapshot> diag;
    if (cfg.with_diagnostics) {
      // the reference reports them for the pre-update shards (shardsim.hpp:401-417), after its
      // own label check (build_buffers): validate first, then measure, then step
      for (int64_t l : batch.labels)
        if (l < 0 || l >= layout_.num_classes)
          throw ContractError("build_buffers: label " + std::to_string(l) + " outside [0, " +
                              std::to_string(layout_.num_classes) + ")");
      diag = diagnostics(batch, cfg.conflict);
      diag->iteration = cfg.step_index;
    }
    pfc_gpu_step_args a{iteration_rng.seed(), iteration_rng.stream_id(), cfg.lr, cfg.step_index};
    pfc_gpu_step_out o{};
    StepResult res;
    res.d_features = Matrix(batch.dim(), batch.batch());
    check(pfc_gpu_step(ctx_, batch.features.flat().data(), batch.labels.data(), batch.batch(), &a,
                       res.d_features.flat().data(), &o),
          ctx_);
    res.diagnostics = diag;
    res.loss = o.loss;
    res.trace.allgather_bytes = o.allgather_bytes;
    res.trace.reduce_scalar_bytes = o.reduce_scalar_bytes;
    res.trace.reduce_grad_bytes = o.reduce_grad_bytes;
    res.trace.reduce_ops = o.reduce_ops;
    const int64_t cap = o.capacity;
    for (int64_t k = first_; k < first_ + nlocal_; ++k) {
      SampleBuffer b;
      b.shard_id = k;
      b.class_indices.resize(static_cast<size_t>(cap));
      check(pfc_gpu_get_buffers(ctx_, k, b.class_indices.data(), &b.num_positives), ctx_);
      res.buffers.push_back(std::move(b));
    }
    return res;
  }

 private:
  ShardLayout layout_;
  int64_t dim_;
  StepConfig cfg_;
  void* ctx_ = nullptr;
  int64_t first_ = 0, nlocal_ = 0;
};

// The reference signature (shardsim.hpp:166-168) for host-resident shards: one GPU, all K
// shards on it; shards are uploaded before and downloaded after the step.
inline StepResult distributed_partial_step(std::vector<CenterShard>& shards,
                                           const FeatureBatch& batch, const StepConfig& cfg,
                                           const SeededRng& iteration_rng) {
  if (shards.empty()) throw ContractError("distributed_partial_step: no shards");
  batch.validate();
  cfg.margin.validate();
  if (!(cfg.lr >= 0.0)) throw ContractError("distributed_partial_step: lr must be >= 0");
  const auto K = static_cast<int64_t>(shards.size());
  const ShardLayout layout(shards.back().class_end, K);
  for (int64_t k = 0; k < K; ++k)
    if (shards[k].class_begin != layout.owned_begin(k) ||
        shards[k].class_end != layout.owned_end(k))
      throw ContractError("distributed_partial_step: shard " + std::to_string(k) +
                          " does not match the contiguous equal partition");
  const int64_t dim = shards.front().weights.rows();
  // one cached session per thread, rebuilt when the shape or the step-invariant config changes
  thread_local std::unique_ptr<Session> cached;
  thread_local std::string key;
  // keyed on the shape; a StepConfig change is applied by Session::step (per-call config)
  const std::string k = std::to_string(layout.num_classes) + "/" + std::to_string(K) + "/" +
                        std::to_string(dim) + "/" + std::to_string(batch.batch());
  if (!cached || key != k) {
    cached.reset();
    cached = std::make_unique<Session>(layout, dim, cfg, std::max<int64_t>(batch.batch(), 1));
    key = k;
  }
  cached->upload(shards);
  StepResult r = cached->step(batch, cfg, iteration_rng);
  cached->download(shards);
  return r;
}

}  // namespace pfc::gpu
