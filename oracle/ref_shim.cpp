// ref_shim.cpp — C ABI over the UNMODIFIED reference headers (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile from /root/reference/proj/include with the reference's
// flags (g++ -std=c++20 -O3 -ffp-contract=off -pthread, proj/CMakeLists.txt:12-13)
// into oracle/_ref/libpfc_ref.so.  It is the executable reference used to
//   * pin the C restatement (oracle/pfc_oracle.c) and generate tests/golden/*,
//   * time the reference CPU path for bench.py's cpu_baseline / --impl reference.
// No reference source is copied here: every computation is a call into the
// reference's own pfc:: functions (rng.hpp, sampler.hpp, shardsim.hpp).
//
// Signatures mirror oracle/pfc_oracle.c (prefix pfcr_ instead of pfco_) so the
// two are interchangeable in tests.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "pfc/metrics.hpp"
#include "pfc/shardsim.hpp"

namespace {

struct StepCfgC {
    double r;
    int32_t margin_kind;
    double margin_scale, margin_m;
    int32_t has_filter;
    double filter_threshold;
    double lr, momentum, weight_decay;
    int64_t step_index;
};

int status_of(const std::exception& e) {
    if (dynamic_cast<const pfc::ShapeError*>(&e)) return 1;
    if (dynamic_cast<const pfc::ContractError*>(&e)) return 2;
    if (dynamic_cast<const pfc::CapacityError*>(&e)) return 3;
    if (dynamic_cast<const pfc::ConfigError*>(&e)) return 4;
    if (dynamic_cast<const pfc::NumericalError*>(&e)) return 5;
    return 8;
}

void set_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) {
        std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
        err[errlen - 1] = 0;
    }
}

pfc::StepConfig to_cfg(const StepCfgC& c) {
    pfc::StepConfig cfg;
    cfg.r = c.r;
    cfg.margin = pfc::MarginConfig{static_cast<pfc::MarginKind>(c.margin_kind), c.margin_scale,
                                   c.margin_m};
    if (c.has_filter) cfg.filter_threshold = c.filter_threshold;
    cfg.lr = c.lr;
    cfg.momentum = c.momentum;
    cfg.weight_decay = c.weight_decay;
    cfg.step_index = c.step_index;
    return cfg;
}

void load_shards(std::vector<pfc::CenterShard>& shards, const double* W, const double* M) {
    size_t off = 0;
    for (auto& s : shards) {
        const size_t n = static_cast<size_t>(s.weights.size());
        std::memcpy(s.weights.flat().data(), W + off, n * sizeof(double));
        if (M) std::memcpy(s.momentum.flat().data(), M + off, n * sizeof(double));
        off += n;
    }
}

void store_shards(const std::vector<pfc::CenterShard>& shards, double* W, double* M) {
    size_t off = 0;
    for (const auto& s : shards) {
        const size_t n = static_cast<size_t>(s.weights.size());
        if (W) std::memcpy(W + off, s.weights.flat().data(), n * sizeof(double));
        if (M) std::memcpy(M + off, s.momentum.flat().data(), n * sizeof(double));
        off += n;
    }
}

pfc::FeatureBatch make_batch(const double* X, const int64_t* labels, int64_t D, int64_t B) {
    pfc::FeatureBatch batch;
    batch.features = pfc::Matrix(D, B);
    std::memcpy(batch.features.flat().data(), X, static_cast<size_t>(D * B) * sizeof(double));
    batch.labels.assign(labels, labels + B);
    return batch;
}

struct Session {
    int64_t C, K, D;
    std::vector<pfc::CenterShard> shards;
};

}  // namespace

extern "C" {

uint64_t pfcr_mix64(uint64_t x) { return pfc::detail::mix64(x); }
uint64_t pfcr_fnv1a(const char* s, int64_t n, uint64_t h) {
    return pfc::detail::fnv1a(std::string_view(s, static_cast<size_t>(n)), h);
}
uint64_t pfcr_make_stream(const char* tag, int64_t n, uint64_t a, uint64_t b) {
    return pfc::make_stream(std::string_view(tag, static_cast<size_t>(n)), a, b);
}
uint64_t pfcr_fork(uint64_t stream, uint64_t label) {
    return pfc::SeededRng(0, stream).fork(label).stream_id();
}
void pfcr_draw_u64(uint64_t seed, uint64_t stream, int64_t n, uint64_t* out) {
    pfc::SeededRng r(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
int64_t pfcr_capacity(int64_t C, int64_t K, double r) {
    try {
        return pfc::buffer_capacity(pfc::ShardLayout(C, K), r);
    } catch (const std::exception&) {
        return -1;
    }
}

int pfcr_build_buffers(int64_t C, int64_t K, const int64_t* labels, int64_t B, double r,
                       uint64_t seed, uint64_t stream, int64_t* out, int64_t* npos,
                       char* err, int errlen) {
    try {
        const pfc::ShardLayout layout(C, K);
        auto bufs = pfc::build_buffers(layout, std::span<const int64_t>(labels, B), r,
                                       pfc::SeededRng(seed, stream));
        const size_t cap = bufs.front().class_indices.size();
        for (size_t k = 0; k < bufs.size(); ++k) {
            std::memcpy(out + k * cap, bufs[k].class_indices.data(), cap * sizeof(int64_t));
            if (npos) npos[k] = bufs[k].num_positives;
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return status_of(e);
    }
}

void pfcr_init_centers(int64_t C, int64_t K, int64_t D, uint64_t seed, double* W) {
    auto shards = pfc::init_center_shards(pfc::ShardLayout(C, K), D, seed);
    store_shards(shards, W, nullptr);
}

// One distributed_partial_step on caller-provided state (W, M updated in place).
int pfcr_step(const StepCfgC* c, int64_t C, int64_t K, int64_t D, double* W, double* M,
              const double* X, const int64_t* labels, int64_t B, uint64_t seed, uint64_t stream,
              double* loss, double* dX, int64_t* buffers, int64_t* npos, double* /*dcenters*/,
              double* /*cos*/, char* err, int errlen) {
    try {
        const pfc::ShardLayout layout(C, K);
        std::vector<pfc::CenterShard> shards;
        for (int64_t k = 0; k < K; ++k) {
            pfc::CenterShard s;
            s.shard_id = k;
            s.class_begin = layout.owned_begin(k);
            s.class_end = layout.owned_end(k);
            s.weights = pfc::Matrix(D, s.owned());
            s.momentum = pfc::Matrix(D, s.owned());
            shards.push_back(std::move(s));
        }
        load_shards(shards, W, M);
        const pfc::FeatureBatch batch = make_batch(X, labels, D, B);
        pfc::StepResult res =
            pfc::distributed_partial_step(shards, batch, to_cfg(*c), pfc::SeededRng(seed, stream));
        *loss = res.loss;
        std::memcpy(dX, res.d_features.flat().data(), static_cast<size_t>(D * B) * sizeof(double));
        if (buffers) {
            const size_t cap = res.buffers.front().class_indices.size();
            for (size_t k = 0; k < res.buffers.size(); ++k) {
                std::memcpy(buffers + k * cap, res.buffers[k].class_indices.data(),
                            cap * sizeof(int64_t));
                if (npos) npos[k] = res.buffers[k].num_positives;
            }
        }
        store_shards(shards, W, M);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return status_of(e);
    }
}

// apcs / amncs (metrics.hpp:56-146) on caller-provided shards, as the step computes them with
// with_diagnostics (shardsim.hpp:401-410).
int pfcr_diagnostics(int64_t C, int64_t K, int64_t D, const double* W, const double* X,
                     const int64_t* labels, int64_t B, const int64_t* class_identity,
                     const int64_t* sample_identity, double* out, int32_t* flags, char* err,
                     int errlen) {
    try {
        const pfc::ShardLayout layout(C, K);
        std::vector<pfc::CenterShard> shards;
        for (int64_t k = 0; k < K; ++k) {
            pfc::CenterShard s;
            s.shard_id = k;
            s.class_begin = layout.owned_begin(k);
            s.class_end = layout.owned_end(k);
            s.weights = pfc::Matrix(D, s.owned());
            s.momentum = pfc::Matrix(D, s.owned());
            shards.push_back(std::move(s));
        }
        std::vector<double> M(static_cast<size_t>(C * D), 0.0);
        load_shards(shards, W, M.data());
        const pfc::FeatureBatch batch = make_batch(X, labels, D, B);
        out[0] = pfc::apcs(batch, shards);
        pfc::ConflictInfo info;
        const bool split = class_identity && sample_identity;
        if (split) {
            info.class_identity = std::span<const int64_t>(class_identity, static_cast<size_t>(C));
            info.sample_identity = std::span<const int64_t>(sample_identity, static_cast<size_t>(B));
        }
        const pfc::AmncsResult a = pfc::amncs(batch, shards, split ? &info : nullptr);
        out[1] = a.amncs;
        out[2] = a.conflicted.value_or(0.0);
        out[3] = a.hard.value_or(0.0);
        flags[0] = a.conflicted.has_value() ? 1 : 0;
        flags[1] = split ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return status_of(e);
    }
}

// mics (metrics.hpp:150-164) on caller-provided shards
int pfcr_mics(int64_t C, int64_t K, int64_t D, const double* W, double* out, char* err, int errlen) {
    try {
        const pfc::ShardLayout layout(C, K);
        std::vector<pfc::CenterShard> shards;
        for (int64_t k = 0; k < K; ++k) {
            pfc::CenterShard s;
            s.shard_id = k;
            s.class_begin = layout.owned_begin(k);
            s.class_end = layout.owned_end(k);
            s.weights = pfc::Matrix(D, s.owned());
            s.momentum = pfc::Matrix(D, s.owned());
            shards.push_back(std::move(s));
        }
        std::vector<double> M(static_cast<size_t>(C * D), 0.0);
        load_shards(shards, W, M.data());
        const std::vector<double> r = pfc::mics(shards);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return status_of(e);
    }
}

// Persistent session: shards live inside the reference's own types, so timing a
// step measures only pfc::distributed_partial_step (bench.py --impl reference).
void* pfcr_session_create(int64_t C, int64_t K, int64_t D, uint64_t seed) {
    auto* s = new Session{C, K, D, pfc::init_center_shards(pfc::ShardLayout(C, K), D, seed)};
    return s;
}

// The same shards as init_center_shards (shardsim.hpp:56-82) -- every class column drawn from its
// own SeededRng(seed, make_stream("center-init", class)) with the reference's next_normal and
// unit-normalised -- filled by `threads` host threads over contiguous class ranges (the per-class
// streams make the result independent of the split).  Used by the bench's reference arm, whose
// 2M-class init would otherwise take ~80 s single-threaded before the timed steps.
void* pfcr_session_create_par(int64_t C, int64_t K, int64_t D, uint64_t seed, int threads) {
    const pfc::ShardLayout layout(C, K);
    std::vector<pfc::CenterShard> shards(static_cast<size_t>(K));
    for (int64_t k = 0; k < K; ++k) {
        pfc::CenterShard& s = shards[static_cast<size_t>(k)];
        s.shard_id = k;
        s.class_begin = layout.owned_begin(k);
        s.class_end = layout.owned_end(k);
        s.weights = pfc::Matrix(D, s.owned());
        s.momentum = pfc::Matrix(D, s.owned());
    }
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            const int64_t c0 = C * t / threads, c1 = C * (t + 1) / threads;
            for (int64_t c = c0; c < c1; ++c) {
                pfc::CenterShard& s = shards[static_cast<size_t>(layout.owner(c))];
                const int64_t j = c - s.class_begin;
                pfc::SeededRng rng(seed, pfc::make_stream("center-init", static_cast<uint64_t>(c)));
                double norm = 0.0;
                for (int64_t d = 0; d < D; ++d) {
                    const double v = rng.next_normal();
                    s.weights(d, j) = v;
                    norm += v * v;
                }
                const double inv = 1.0 / std::max(std::sqrt(norm), 1e-12);
                for (int64_t d = 0; d < D; ++d) s.weights(d, j) *= inv;
            }
        });
    for (auto& th : pool) th.join();
    return new Session{C, K, D, std::move(shards)};
}

void pfcr_session_destroy(void* h) { delete static_cast<Session*>(h); }

void pfcr_session_get(void* h, double* W, double* M) {
    store_shards(static_cast<Session*>(h)->shards, W, M);
}

int pfcr_session_step(void* h, const StepCfgC* c, const double* X, const int64_t* labels,
                      int64_t B, uint64_t seed, uint64_t stream, double* loss, double* dX,
                      char* err, int errlen) {
    auto* s = static_cast<Session*>(h);
    try {
        const pfc::FeatureBatch batch = make_batch(X, labels, s->D, B);
        pfc::StepResult res = pfc::distributed_partial_step(s->shards, batch, to_cfg(*c),
                                                            pfc::SeededRng(seed, stream));
        *loss = res.loss;
        if (dX)
            std::memcpy(dX, res.d_features.flat().data(),
                        static_cast<size_t>(s->D * B) * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return status_of(e);
    }
}

}  // extern "C"
