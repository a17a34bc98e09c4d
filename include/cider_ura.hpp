// cider_ura.hpp — header-only C++ adapter: the B200 engine behind the reference's own decoder
// types (/root/reference/proj/include/ura). Include it from code that already builds against the
// reference (it needs ura/*.hpp) and link libcider.so. Nothing here does arithmetic: every call
// goes through the C ABI of cider.h.
//
//   cider::GpuStructuredDenoiser : ura::Denoiser          (denoiser.hpp:109-130)
//       drop-in for ura::StructuredDenoiser inside the reference's run_refinement /
//       run_with_remasking / remask_pass (refine.cpp:134-292) — one forward per call.
//   cider::GpuRefiner::run_refinement / run_with_remasking / remask_pass (refine.hpp:60-62, 97-107)
//       the whole T-step loop on the device, batched over bins; RefineTrace filled like the
//       reference's; run_with_remasking takes any ura::ConfidenceScorer (scores on the host between
//       the device passes, the reference's stage loop).
//   cider::make_bin_decoder -> ura::BinDecoder            (protocol.hpp:32-40)
//       for run_protocol_frame (protocol.cpp:73).
//   cider::GpuBp::bp_decode / sic_decode                  (bp.hpp:72-93)
//       the reference's FFT-BP / SIC-BP decoders (WHT backend) on the device, batched over bins;
//   cider::make_sic_bin_decoder -> ura::BinDecoder        SIC-BP per bin for run_protocol_frame.
//
// Errors: status 3 -> std::domain_error, 4 -> std::runtime_error, with the library's message
// (which keeps the reference's prefixes, e.g. "embed_grid: token out of range").
#pragma once

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <future>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include "cider.h"
#include "ura/bp.hpp"
#include "ura/denoiser.hpp"
#include "ura/protocol.hpp"
#include "ura/refine.hpp"

namespace cider {

inline void check(int rc) {
    if (rc == CIDER_OK) return;
    const std::string msg = cider_last_error();
    if (rc == CIDER_EINVAL) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

// ura::DenoiserParams (ref-exact: 1 block, hidden = D, sum-pool Psi) -> cider.h flat weights.
inline std::vector<float> flatten(const ura::DenoiserParams& p) {
    std::vector<float> w;
    auto put = [&](const std::vector<double>& v) {
        for (double x : v) w.push_back(float(x));
    };
    put(p.embed);
    put(p.out_proj);
    put(p.sym_embed);
    for (const ura::TwoLayerMap* t : {&p.gate_a, &p.check_agg, &p.fuse_b}) {
        if (t->hidden != p.gate_a.hidden) throw std::domain_error("cider: maps must share one hidden width");
        put(t->w1);
        put(t->b1);
        put(t->w2);
        put(t->b2);
    }
    return w;
}

inline std::vector<int32_t> edges_of(const ura::ParityCheckMatrix& h) {
    std::vector<int32_t> e;
    for (const ura::ParityEdge& x : h.entries()) e.insert(e.end(), {x.check, x.slot, x.coeff});
    return e;
}

// Owns one device context (weights + Tanner tables resident on one B200).
class Context {
public:
    Context(const ura::GfContext& gf, const ura::DenoiserParams& p, const ura::ParityCheckMatrix& h, int device = 0,
            int precision = CIDER_FP32)
        : checks_(h.checks()), slots_(h.slots()), q_(p.q), dim_(p.dim) {
        cider_model_desc md{};
        md.m = gf.m();
        md.prim_poly = gf.prim_poly();
        md.dim = p.dim;
        md.hidden = p.gate_a.hidden;
        md.layers = 1;
        md.heads = 0;
        md.tau_demix = p.tau_demix;
        md.evidence_scale = p.evidence_scale;
        md.precision = precision;
        const auto w = flatten(p);
        edges_ = edges_of(h);
        cider_code_desc cd{h.checks(), h.slots(), int(edges_.size() / 3), edges_.data()};
        cider_ctx* c = nullptr;
        check(cider_create(&md, w.data(), &cd, device, &c));
        ctx_.reset(c);
    }
    // config mode (BASELINE configs: N stacked blocks, MLP width H, attention heads): cider.h's flat
    // weight layout (cider_weights_init) and model descriptor
    Context(const cider_model_desc& md, const std::vector<float>& weights, const ura::ParityCheckMatrix& h, int device = 0)
        : checks_(h.checks()), slots_(h.slots()), q_(1 << md.m), dim_(md.dim) {
        if (weights.size() != cider_weights_count(&md)) throw std::domain_error("cider: weight count does not match the model");
        edges_ = edges_of(h);
        cider_code_desc cd{h.checks(), h.slots(), int(edges_.size() / 3), edges_.data()};
        cider_ctx* c = nullptr;
        check(cider_create(&md, weights.data(), &cd, device, &c));
        ctx_.reset(c);
    }
    cider_ctx* get() const { return ctx_.get(); }
    int q() const { return q_; }
    int slots() const { return slots_; }
    // the context is built for one parity-check matrix; calls must pass the same one
    void require_same(const ura::ParityCheckMatrix& h) const {
        if (h.checks() != checks_ || h.slots() != slots_ || edges_of(h) != edges_)
            throw std::domain_error("cider: parity-check matrix differs from the one the context was built with");
    }

private:
    struct Del {
        void operator()(cider_ctx* c) const { cider_destroy(c); }
    };
    std::unique_ptr<cider_ctx, Del> ctx_;
    int checks_, slots_, q_, dim_;
    std::vector<int32_t> edges_;
};

// Per-step drop-in for ura::StructuredDenoiser (denoiser.cpp:253-259). Thread-safe like the
// reference's const logits(): the context serialises calls internally.
class GpuStructuredDenoiser : public ura::Denoiser {
public:
    explicit GpuStructuredDenoiser(std::shared_ptr<Context> ctx) : ctx_(std::move(ctx)) {}
    ura::LogitGrid logits(const ura::MaskedGrid& x, const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h,
                          double /*mask_ratio: time-homogeneous*/) const override {
        ctx_->require_same(h);
        if (s.slots != ctx_->slots() || s.q != ctx_->q() || x.cols != ctx_->slots())
            throw std::domain_error("module_b: slot count mismatch");
        std::vector<int32_t> X(x.v.begin(), x.v.end());
        std::vector<float> S(s.v.begin(), s.v.end());
        std::vector<float> lg(size_t(x.rows) * x.cols * s.q);
        check(cider_denoise(ctx_->get(), 1, x.rows, X.data(), S.data(), lg.data(), nullptr));
        ura::LogitGrid out(x.rows, x.cols, s.q);
        for (size_t i = 0; i < lg.size(); ++i) out.v[i] = lg[i];
        return out;
    }

private:
    std::shared_ptr<Context> ctx_;
};

// Whole-pass drop-in (the device runs the T-step loop, reveal, gamma=0 pass and remasking).
class GpuRefiner {
public:
    explicit GpuRefiner(std::shared_ptr<Context> ctx) : ctx_(std::move(ctx)) {}

    // = ura::run_refinement(den, s, h, sched, k, l) for one bin
    ura::SymbolGrid run_refinement(const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h,
                                   const ura::RevealSchedule& sched, int k) const {
        return run(s, h, sched, nullptr, k);
    }
    // = ura::run_refinement(den, s, h, sched, k, l, trace, final_pass_logits) (refine.hpp:60-62)
    ura::SymbolGrid run_refinement(const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h,
                                   const ura::RevealSchedule& sched, int k, ura::RefineTrace* trace,
                                   ura::LogitGrid* final_pass_logits) const {
        ctx_->require_same(h);
        const int L = ctx_->slots(), Q = ctx_->q();
        std::vector<float> S(s.v.begin(), s.v.end());
        std::vector<int32_t> g(size_t(k) * L);
        std::vector<float> fl(final_pass_logits ? size_t(k) * L * Q : 0);
        TraceBuf tb(k, L, sched.steps);
        const cider_schedule sc = schedule(sched);
        check(cider_refine(ctx_->get(), 1, k, S.data(), &sc, nullptr, g.data(), final_pass_logits ? fl.data() : nullptr,
                           trace ? &tb.t : nullptr));
        if (trace) tb.fold(*trace, k, L, false);
        if (final_pass_logits) *final_pass_logits = logits_of(fl, k, L, Q);
        ura::SymbolGrid out(k, L);
        std::copy(g.begin(), g.end(), out.v.begin());
        return out;
    }
    // = ura::remask_pass (refine.hpp:97-100, refine.cpp:238-275): rows with confidences[k] < threshold
    // re-decoded on the device, the others bit-identical; final_pass_logits / trace as the reference
    ura::SymbolGrid remask_pass(const ura::SymbolGrid& grid, const std::vector<double>& confidences, double threshold,
                                const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h,
                                const ura::RevealSchedule& sched, ura::RefineTrace* trace = nullptr,
                                ura::LogitGrid* final_pass_logits = nullptr) const {
        ctx_->require_same(h);
        if (static_cast<int>(confidences.size()) != grid.rows)
            throw std::domain_error("remask_pass: one confidence per row required");
        const int k = grid.rows, L = ctx_->slots(), Q = ctx_->q();
        int n_low = 0;
        for (double c : confidences) n_low += c < threshold;
        if (n_low == 0) return grid;
        std::vector<float> S(s.v.begin(), s.v.end());
        std::vector<int32_t> gin(grid.v.begin(), grid.v.end()), gout(gin.size());
        std::vector<float> fl(final_pass_logits ? size_t(k) * L * Q : 0);
        TraceBuf tb(k, L, sched.steps);
        const cider_schedule sc = schedule(sched);
        check(cider_remask_pass(ctx_->get(), 1, k, S.data(), &sc, gin.data(), confidences.data(), threshold, gout.data(),
                                final_pass_logits ? fl.data() : nullptr, trace ? &tb.t : nullptr));
        if (trace) tb.fold(*trace, k, L, true);
        if (final_pass_logits) *final_pass_logits = logits_of(fl, k, L, Q);
        ura::SymbolGrid out(k, L);
        std::copy(gout.begin(), gout.end(), out.v.begin());
        return out;
    }
    // = ura::run_with_remasking(den, scorer, s, h, sched, remask, k, l, trace) (refine.cpp:277-292) with
    // any ConfidenceScorer: the passes run on the device, the scorer on the host between them
    ura::SymbolGrid run_with_remasking(const ura::ConfidenceScorer& scorer, const ura::EvidenceMatrix& s,
                                       const ura::ParityCheckMatrix& h, const ura::RevealSchedule& sched,
                                       const ura::RemaskConfig& remask, int k, ura::RefineTrace* trace = nullptr) const {
        ura::validate_remask_config(remask);
        ura::LogitGrid fl;
        ura::SymbolGrid grid = run_refinement(s, h, sched, k, trace, &fl);
        for (double threshold : remask.thresholds) {
            auto conf = scorer.score_rows(grid, fl);
            bool any_low = false;
            for (double c : conf) any_low = any_low || c < threshold;
            if (!any_low) break;
            grid = remask_pass(grid, conf, threshold, s, h, sched, trace, &fl);
        }
        return grid;
    }
    // = ura::run_with_remasking(den, MaxProbScorer, s, h, sched, remask, k, l)
    ura::SymbolGrid run_with_remasking(const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h,
                                       const ura::RevealSchedule& sched, const ura::RemaskConfig& remask, int k) const {
        cider_remask rm{};
        rm.mode = remask.thresholds.empty() ? CIDER_REMASK_NONE : CIDER_REMASK_THRESHOLD;
        if (remask.thresholds.size() > CIDER_MAX_THRESHOLDS) throw std::domain_error("remask: too many thresholds");
        rm.n_thresholds = int(remask.thresholds.size());
        for (size_t i = 0; i < remask.thresholds.size(); ++i) rm.thresholds[i] = remask.thresholds[i];
        return run(s, h, sched, &rm, k);
    }
    // batched: B evidence matrices -> B grids in one device call
    std::vector<ura::SymbolGrid> run_batch(const std::vector<const ura::EvidenceMatrix*>& ss, const ura::ParityCheckMatrix& h,
                                           const ura::RevealSchedule& sched, const cider_remask* rm, int k) const {
        ctx_->require_same(h);
        const int B = int(ss.size()), L = ctx_->slots(), Q = ctx_->q();
        std::vector<float> S(size_t(B) * L * Q);
        for (int b = 0; b < B; ++b)
            for (size_t i = 0; i < size_t(L) * Q; ++i) S[size_t(b) * L * Q + i] = float(ss[b]->v[i]);
        std::vector<int32_t> g(size_t(B) * k * L);
        cider_schedule sc{sched.steps, sched.tau_max, sched.tau_min, sched.first_reveal ? 1 : 0};
        check(cider_refine(ctx_->get(), B, k, S.data(), &sc, rm, g.data(), nullptr, nullptr));
        std::vector<ura::SymbolGrid> out(B, ura::SymbolGrid(k, L));
        for (int b = 0; b < B; ++b) std::copy(g.begin() + size_t(b) * k * L, g.begin() + size_t(b + 1) * k * L, out[b].v.begin());
        return out;
    }

    // ragged loads in one call (cider_refine_ragged): bin b has loads[b] users, decoded with the
    // reference's per-load schedule and remask thresholds (default_steps_for_load /
    // default_remask_thresholds, refine.cpp:28-46) — what a DecoderBank of make_bin_decoder applies
    // bin by bin inside run_protocol_frame (protocol.cpp:41-88), as one batch per load
    std::vector<ura::SymbolGrid> run_ragged(const std::vector<const ura::EvidenceMatrix*>& ss, const std::vector<int>& loads,
                                            const ura::ParityCheckMatrix& h, int k_max, bool per_load_remask = true) const {
        ctx_->require_same(h);
        const int B = int(ss.size()), L = ctx_->slots(), Q = ctx_->q();
        if (int(loads.size()) != B) throw std::domain_error("run_ragged: one load per bin");
        std::vector<float> S(size_t(B) * L * Q);
        for (int b = 0; b < B; ++b)
            for (size_t i = 0; i < size_t(L) * Q; ++i) S[size_t(b) * L * Q + i] = float(ss[b]->v[i]);
        std::vector<cider_schedule> sc(k_max);
        std::vector<cider_remask> rm(k_max);
        for (int k = 1; k <= k_max; ++k) {
            sc[k - 1] = cider_schedule{ura::default_steps_for_load(k), 1.0, 1.0, 1};
            rm[k - 1] = cider_remask{};
            rm[k - 1].mode = CIDER_REMASK_NONE;
            if (per_load_remask) {
                const auto th = ura::default_remask_thresholds(k);
                if (th.size() > CIDER_MAX_THRESHOLDS) throw std::domain_error("remask: too many thresholds");
                rm[k - 1].mode = th.empty() ? CIDER_REMASK_NONE : CIDER_REMASK_THRESHOLD;
                rm[k - 1].n_thresholds = int(th.size());
                for (size_t i = 0; i < th.size(); ++i) rm[k - 1].thresholds[i] = th[i];
            }
        }
        std::vector<int32_t> ld(loads.begin(), loads.end());
        size_t rows = 0;
        for (int k : loads) rows += size_t(k);
        std::vector<int32_t> g(rows * L);
        check(cider_refine_ragged(ctx_->get(), B, ld.data(), S.data(), k_max, sc.data(), rm.data(), g.data()));
        std::vector<ura::SymbolGrid> out;
        size_t o = 0;
        for (int b = 0; b < B; ++b) {
            out.emplace_back(loads[b], L);
            std::copy(g.begin() + o * L, g.begin() + (o + loads[b]) * L, out.back().v.begin());
            o += size_t(loads[b]);
        }
        return out;
    }

private:
    // cider_trace buffers of one bin, folded into a ura::RefineTrace like run_masked_loop / remask_pass
    // record it (refine.cpp:160-170, 261-264): reveal_counts / first_step_sites replaced by the last
    // pass's, pass_first_reveals / remask stages appended
    struct TraceBuf {
        std::vector<int32_t> first, rows, steps, mask, pass_first, n_passes, counts, n_counts;
        std::vector<uint8_t> sites;
        cider_trace t{};
        TraceBuf(int k, int L, int max_steps)
            : first(1), rows(CIDER_MAX_THRESHOLDS), steps(CIDER_MAX_THRESHOLDS), mask(k), pass_first(1 + CIDER_MAX_THRESHOLDS),
              n_passes(1), counts(std::max(1, max_steps)), n_counts(1), sites(size_t(k) * L) {
            t = cider_trace{first.data(), rows.data(), steps.data(), mask.data(), pass_first.data(), n_passes.data(),
                            std::max(1, max_steps), counts.data(), n_counts.data(), sites.data()};
        }
        void fold(ura::RefineTrace& tr, int k, int L, bool stage) const {
            if (n_passes[0] == 0) return;
            for (int p = 0; p < n_passes[0] && p < 1 + CIDER_MAX_THRESHOLDS; ++p) tr.pass_first_reveals.push_back(pass_first[p]);
            if (stage) {
                tr.remask_rows_per_stage.push_back(rows[0]);
                tr.remask_steps_per_stage.push_back(steps[0]);
            }
            tr.reveal_counts.assign(counts.begin(), counts.begin() + std::min<size_t>(counts.size(), size_t(n_counts[0])));
            tr.first_step_sites.clear();
            for (int r = 0; r < k; ++r)
                for (int l = 0; l < L; ++l)
                    if (sites[size_t(r) * L + l]) tr.first_step_sites.emplace_back(r, l);
        }
    };
    static cider_schedule schedule(const ura::RevealSchedule& sched) {
        return cider_schedule{sched.steps, sched.tau_max, sched.tau_min, sched.first_reveal ? 1 : 0};
    }
    static ura::LogitGrid logits_of(const std::vector<float>& fl, int k, int L, int Q) {
        ura::LogitGrid out(k, L, Q);
        for (size_t i = 0; i < fl.size(); ++i) out.v[i] = fl[i];
        return out;
    }
    ura::SymbolGrid run(const ura::EvidenceMatrix& s, const ura::ParityCheckMatrix& h, const ura::RevealSchedule& sched,
                        const cider_remask* rm, int k) const {
        return run_batch({&s}, h, sched, rm, k)[0];
    }
    std::shared_ptr<Context> ctx_;
};

// ura::BinDecoder (protocol.hpp:40) for run_protocol_frame (protocol.cpp:73); bins of load K
// with the default per-load schedule (refine.cpp:28-46) unless `sched_override.steps > 0`.
inline ura::BinDecoder make_bin_decoder(std::shared_ptr<Context> ctx, ura::RevealSchedule sched_override = {0, 1.0, 1.0, true},
                                        bool per_load_remask = true) {
    auto refiner = std::make_shared<GpuRefiner>(ctx);
    return [refiner, sched_override, per_load_remask](const ura::BinTask& t) {
        ura::RevealSchedule sched = sched_override;
        if (sched.steps <= 0) sched.steps = ura::default_steps_for_load(t.load);
        ura::RemaskConfig rm;
        if (per_load_remask) rm.thresholds = ura::default_remask_thresholds(t.load);
        return refiner->run_with_remasking(t.evidence, t.h, sched, rm, t.load);
    };
}

// Request-coalescing BinDecoder: run_protocol (protocol.cpp:97-110) calls the decoder bank from
// parallel_for worker threads, one bin at a time per frame. Each call here enqueues its bin and
// blocks; a dispatcher thread drains everything pending (after the first request waited `window`, or
// as soon as `max_batch` bins are queued) into ONE ragged device batch (GpuRefiner::run_ragged: the
// reference's per-load schedule and remask thresholds) and hands every caller its grid. Results are
// those of the per-bin make_bin_decoder (run_ragged == per-load calls, tests). Evidence is read
// during the call only (the caller's BinTask outlives it).
class BinCoalescer {
public:
    BinCoalescer(std::shared_ptr<Context> ctx, int k_max, size_t max_batch = 4096,
                 std::chrono::microseconds window = std::chrono::microseconds(200), bool per_load_remask = true)
        : refiner_(std::make_shared<GpuRefiner>(std::move(ctx))), k_max_(k_max), max_batch_(max_batch), window_(window),
          per_load_remask_(per_load_remask), worker_([this] { loop(); }) {}
    ~BinCoalescer() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        worker_.join();
    }
    BinCoalescer(const BinCoalescer&) = delete;
    BinCoalescer& operator=(const BinCoalescer&) = delete;

    ura::SymbolGrid decode(const ura::BinTask& t) {
        if (t.load < 1 || t.load > k_max_) throw std::domain_error("BinCoalescer: load outside 1..k_max");
        Req r{&t.evidence, &t.h, t.load, {}};
        auto fut = r.done.get_future();
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (q_.empty()) first_ = std::chrono::steady_clock::now();
            q_.push_back(&r);
        }
        cv_.notify_all();
        return fut.get(); // rethrows the batch's exception
    }
    int64_t batches() const { return batches_; }

private:
    struct Req {
        const ura::EvidenceMatrix* s;
        const ura::ParityCheckMatrix* h;
        int load;
        std::promise<ura::SymbolGrid> done;
    };
    void loop() {
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
            if (q_.empty() && stop_) return;
            // gather: until the window since the first pending request has passed, or the batch is full
            cv_.wait_until(lk, first_ + window_, [this] { return stop_ || q_.size() >= max_batch_; });
            std::vector<Req*> batch;
            while (!q_.empty() && batch.size() < max_batch_) {
                batch.push_back(q_.front());
                q_.pop_front();
            }
            if (!q_.empty()) first_ = std::chrono::steady_clock::now();
            lk.unlock();
            run(batch);
            lk.lock();
        }
    }
    void run(const std::vector<Req*>& batch) {
        // one code per context: bins whose H differs from the first are decoded (and rejected) alone
        std::vector<const ura::EvidenceMatrix*> ss;
        std::vector<int> loads;
        std::vector<Req*> in;
        for (Req* r : batch) {
            if (r->h != batch.front()->h) {
                try {
                    r->done.set_value(refiner_->run_ragged({r->s}, {r->load}, *r->h, k_max_, per_load_remask_)[0]);
                } catch (...) {
                    r->done.set_exception(std::current_exception());
                }
                continue;
            }
            ss.push_back(r->s);
            loads.push_back(r->load);
            in.push_back(r);
        }
        if (in.empty()) return;
        try {
            auto out = refiner_->run_ragged(ss, loads, *in.front()->h, k_max_, per_load_remask_);
            ++batches_;
            for (size_t i = 0; i < in.size(); ++i) in[i]->done.set_value(std::move(out[i]));
        } catch (...) {
            for (Req* r : in) r->done.set_exception(std::current_exception());
        }
    }
    std::shared_ptr<GpuRefiner> refiner_;
    int k_max_;
    size_t max_batch_;
    std::chrono::microseconds window_;
    bool per_load_remask_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Req*> q_;
    std::chrono::steady_clock::time_point first_{};
    bool stop_ = false;
    int64_t batches_ = 0;
    std::thread worker_; // last: started after every member above is initialised
};

inline ura::BinDecoder make_coalescing_bin_decoder(std::shared_ptr<BinCoalescer> c) {
    return [c](const ura::BinTask& t) { return c->decode(t); };
}

// The device FFT-BP decoder for one code (cider_bp_* in cider.h). Implements the WHT backend
// (bp.cpp:222-269); a direct-backend config is refused rather than silently substituted.
class GpuBp {
public:
    GpuBp(const ura::GfContext& gf, const ura::ParityCheckMatrix& h, int device = 0)
        : slots_(h.slots()), q_(gf.q()) {
        const auto e = edges_of(h);
        cider_code_desc cd{h.checks(), h.slots(), int(e.size() / 3), e.data()};
        cider_bp_ctx* c = nullptr;
        check(cider_bp_create(gf.m(), gf.prim_poly(), &cd, device, &c));
        ctx_.reset(c, cider_bp_destroy);
    }

    // = ura::bp_decode (bp.cpp:271-347); final_state is not exported by the device decoder
    ura::BpResult bp_decode(const std::vector<std::vector<double>>& lambda, const ura::BpConfig& cfg) const {
        if (static_cast<int>(lambda.size()) != slots_) throw std::domain_error("bp_decode: belief count must equal slot count");
        std::vector<double> lam(size_t(slots_) * q_);
        for (int l = 0; l < slots_; ++l) std::copy(lambda[l].begin(), lambda[l].end(), lam.begin() + size_t(l) * q_);
        std::vector<int32_t> hard(slots_);
        std::vector<double> marg(lam.size());
        int32_t conv = 0, its = 0;
        const cider_bp_config c = config(cfg);
        check(cider_bp_decode(ctx_.get(), 1, lam.data(), &c, hard.data(), marg.data(), &conv, &its));
        ura::BpResult r;
        r.hard.assign(hard.begin(), hard.end());
        r.marginals.assign(slots_, std::vector<double>(q_));
        for (int l = 0; l < slots_; ++l) std::copy(marg.begin() + size_t(l) * q_, marg.begin() + size_t(l + 1) * q_, r.marginals[l].begin());
        r.converged = conv != 0;
        r.iters_used = its;
        return r;
    }

    // = ura::sic_decode (bp.cpp:349-368) for many bins in one device batch
    std::vector<ura::SicResult> sic_decode_batch(const std::vector<const ura::EvidenceMatrix*>& bins, int k,
                                                 const ura::BpConfig& cfg,
                                                 double cancel_value = std::numeric_limits<double>::quiet_NaN()) const {
        const int B = static_cast<int>(bins.size());
        std::vector<double> S(size_t(B) * slots_ * q_);
        for (int b = 0; b < B; ++b) {
            if (bins[b]->slots != slots_ || bins[b]->q != q_) throw std::domain_error("sic_decode: evidence shape mismatch");
            std::copy(bins[b]->v.begin(), bins[b]->v.end(), S.begin() + size_t(b) * slots_ * q_);
        }
        std::vector<int32_t> grid(size_t(B) * k * slots_), sc(size_t(B) * k), si(size_t(B) * k);
        const cider_bp_config c = config(cfg);
        check(cider_sic_decode(ctx_.get(), B, k, S.data(), &c, cancel_value, grid.data(), sc.data(), si.data()));
        std::vector<ura::SicResult> out(B);
        for (int b = 0; b < B; ++b) {
            out[b].grid = ura::SymbolGrid(k, slots_);
            for (int r = 0; r < k; ++r) {
                for (int l = 0; l < slots_; ++l) out[b].grid.at(r, l) = grid[(size_t(b) * k + r) * slots_ + l];
                out[b].stages.push_back({sc[size_t(b) * k + r] != 0, si[size_t(b) * k + r]});
            }
        }
        return out;
    }
    ura::SicResult sic_decode(const ura::EvidenceMatrix& s, int k, const ura::BpConfig& cfg,
                              double cancel_value = std::numeric_limits<double>::quiet_NaN()) const {
        return sic_decode_batch({&s}, k, cfg, cancel_value)[0];
    }

private:
    static cider_bp_config config(const ura::BpConfig& cfg) {
        if (cfg.backend != ura::CheckBackend::wht) throw std::domain_error("cider: the device BP decoder implements the WHT backend");
        return cider_bp_config{cfg.max_iters, cfg.message_floor, cfg.early_exit ? 1 : 0};
    }
    int slots_, q_;
    std::shared_ptr<cider_bp_ctx> ctx_;
};

// ura::BinDecoder running SIC-BP on the device for bins of load K (the paper's FFT-BP baseline).
inline ura::BinDecoder make_sic_bin_decoder(std::shared_ptr<GpuBp> bp, ura::BpConfig cfg = {}) {
    return [bp, cfg](const ura::BinTask& t) { return bp->sic_decode(t.evidence, t.load, cfg).grid; };
}

} // namespace cider
