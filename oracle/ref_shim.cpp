// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// C-ABI shim around the reference implementation itself. oracle/Makefile compiles the
// reference's own sources straight from /root/reference/proj/src (gf, ldpc, denoiser, refine,
// metrics, parallel, bp) together with this file into oracle/_ref/libura_ref.so. Nothing from
// the reference is copied into this repository; this file only *calls* the reference API.
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs may load it.
//
// Ref-exact mode (layers=1, hidden=dim, heads=0) is ura::StructuredDenoiser verbatim
// (denoiser.cpp:253-259). Config mode composes the reference's own
// module_a / module_b / final_logits per layer with shared E, W, V; heads>0 swaps Module B's
// sum-pool Psi for the extrinsic pooling attention defined in DESIGN.md §2, built from the
// reference's coeff_action (denoiser.cpp:162-179) and TwoLayerMap::apply_gelu (denoiser.cpp:29-34).
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <random>
#include <thread>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ura/amp.hpp"
#include "ura/bp.hpp"
#include "ura/denoiser.hpp"
#include "ura/gf.hpp"
#include "ura/ldpc.hpp"
#include "ura/metrics.hpp"
#include "ura/parallel.hpp"
#include "ura/refine.hpp"
#include "ura/seeding.hpp"
#include "ura/sim.hpp"

#include "cider.h"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::domain_error& e) {
        return fail(e, CIDER_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, CIDER_ERUNTIME);
    }
}

ura::GfContext make_gf(const cider_model_desc* m) {
    uint32_t poly = m->prim_poly ? m->prim_poly : ura::GfContext::default_prim_poly(m->m);
    return ura::GfContext(m->m, poly);
}

ura::ParityCheckMatrix make_h(int q, const cider_code_desc* c) {
    std::vector<ura::ParityEdge> e(c->n_edges);
    for (int i = 0; i < c->n_edges; ++i)
        e[i] = ura::ParityEdge{c->edges[3 * i], c->edges[3 * i + 1], c->edges[3 * i + 2]};
    return ura::ParityCheckMatrix(c->checks, c->slots, q, std::move(e));
}

struct AttnParams {
    std::vector<double> query; // D
    std::vector<double> key;   // D x D, row-major [out][in]
};

// Unpacks the flat weight layout of cider.h into per-layer reference DenoiserParams.
struct Model {
    int q = 0, dim = 0, hidden = 0, layers = 0, heads = 0;
    std::vector<ura::DenoiserParams> p; // one per layer; tables replicated (shared values)
    std::vector<AttnParams> attn;

    Model(const cider_model_desc* m, const double* w) {
        q = 1 << m->m;
        dim = m->dim;
        hidden = m->hidden;
        layers = m->layers;
        heads = m->heads;
        if (layers < 1 || dim < 1 || hidden < 1 || heads < 0 || (heads > 0 && dim % heads))
            throw std::domain_error("ref_shim: bad model dimensions");
        size_t off = 0;
        auto take = [&](std::vector<double>& v, size_t n) {
            v.assign(w + off, w + off + n);
            off += n;
        };
        ura::DenoiserParams base;
        base.q = q;
        base.dim = dim;
        base.tau_demix = m->tau_demix;
        base.evidence_scale = m->evidence_scale;
        take(base.embed, size_t(q + 1) * dim);
        take(base.out_proj, size_t(q) * dim);
        take(base.sym_embed, size_t(q) * dim);
        auto map = [&](ura::TwoLayerMap& t, int in) {
            t.in = in;
            t.hidden = hidden;
            t.out = dim;
            take(t.w1, size_t(hidden) * in);
            take(t.b1, hidden);
            take(t.w2, size_t(dim) * hidden);
            take(t.b2, dim);
        };
        for (int l = 0; l < layers; ++l) {
            ura::DenoiserParams pl = base;
            map(pl.gate_a, 2 * dim);
            map(pl.check_agg, dim);
            map(pl.fuse_b, 2 * dim);
            p.push_back(std::move(pl));
        }
        if (heads > 0) {
            for (int l = 0; l < layers; ++l) {
                AttnParams a;
                take(a.query, dim);
                take(a.key, size_t(dim) * dim);
                attn.push_back(std::move(a));
            }
        }
    }
};

// Module B with attention Psi, composed of reference primitives ("attention Psi").
ura::LatentGrid module_b_attn(const ura::GfContext& gf, const ura::LatentGrid& zt,
                              const ura::ParityCheckMatrix& h, const ura::DenoiserParams& p,
                              const AttnParams& a, int heads, ura::LatentGrid* incoming_out) {
    const int dim = p.dim, dh = dim / heads;
    const double scale = 1.0 / std::sqrt(double(dh));
    ura::LatentGrid acc(zt.rows, zt.cols, dim);
    std::vector<double> pooled(dim), mapped(dim);
    for (int k = 0; k < zt.rows; ++k) {
        for (int j = 0; j < h.checks(); ++j) {
            const auto& edges = h.check_edges(j);
            const int d = int(edges.size());
            std::vector<std::vector<double>> nrm(d);
            std::vector<std::vector<double>> score(d, std::vector<double>(heads, 0.0));
            for (int i = 0; i < d; ++i) {
                const ura::ParityEdge& e = h.edge(edges[i]);
                nrm[i] = ura::coeff_action(gf, p, zt.at(k, e.slot), e.coeff);
                for (int hh = 0; hh < heads; ++hh) {
                    double s = 0.0;
                    for (int t = hh * dh; t < (hh + 1) * dh; ++t) {
                        double key = 0.0;
                        for (int c = 0; c < dim; ++c) key += a.key[size_t(t) * dim + c] * nrm[i][c];
                        s += a.query[t] * key;
                    }
                    score[i][hh] = s * scale;
                }
            }
            for (int i = 0; i < d; ++i) {
                std::fill(pooled.begin(), pooled.end(), 0.0);
                for (int hh = 0; hh < heads; ++hh) {
                    double mx = -INFINITY;
                    for (int i2 = 0; i2 < d; ++i2)
                        if (i2 != i) mx = std::max(mx, score[i2][hh]);
                    double den = 0.0;
                    for (int i2 = 0; i2 < d; ++i2)
                        if (i2 != i) den += std::exp(score[i2][hh] - mx);
                    for (int i2 = 0; i2 < d; ++i2) {
                        if (i2 == i) continue;
                        double wgt = double(d - 1) * std::exp(score[i2][hh] - mx) / den;
                        for (int t = hh * dh; t < (hh + 1) * dh; ++t) pooled[t] += wgt * nrm[i2][t];
                    }
                }
                p.check_agg.apply_gelu(pooled.data(), mapped.data());
                const ura::ParityEdge& e = h.edge(edges[i]);
                auto msg = ura::coeff_action(gf, p, mapped.data(), gf.inv(e.coeff));
                double* dst = acc.at(k, e.slot);
                for (int t = 0; t < dim; ++t) dst[t] += msg[t];
            }
        }
    }
    if (incoming_out) *incoming_out = acc;
    ura::LatentGrid out(zt.rows, zt.cols, dim);
    std::vector<double> cat(2 * dim), res(dim);
    for (int k = 0; k < zt.rows; ++k)
        for (int l = 0; l < zt.cols; ++l) {
            std::copy(zt.at(k, l), zt.at(k, l) + dim, cat.data());
            std::copy(acc.at(k, l), acc.at(k, l) + dim, cat.data() + dim);
            p.fuse_b.apply_gelu(cat.data(), res.data());
            for (int t = 0; t < dim; ++t) out.at(k, l)[t] = zt.at(k, l)[t] + res[t];
        }
    return out;
}

// Stacked denoiser: the reference's layer functions, N times.
class StackedDenoiser : public ura::Denoiser {
public:
    StackedDenoiser(ura::GfContext gf, const Model& m) : gf_(std::move(gf)), m_(m) {}

    ura::LogitGrid forward(const ura::MaskedGrid& x, const ura::EvidenceMatrix& s,
                           const ura::ParityCheckMatrix& h,
                           std::vector<ura::LatentGrid>* incoming) const {
        if (m_.layers == 1 && m_.heads == 0 && !incoming) {
            // ref-exact: the reference's own StructuredDenoiser end to end
            ura::StructuredDenoiser den(gf_, m_.p[0]);
            return den.logits(x, s, h, 0.0);
        }
        ura::LatentGrid z = ura::embed_grid(x, m_.p[0]);
        for (int l = 0; l < m_.layers; ++l) {
            ura::LatentGrid zt = ura::module_a(z, s, m_.p[l]);
            ura::LatentGrid in;
            if (m_.heads == 0)
                z = ura::module_b(gf_, zt, h, m_.p[l], &in);
            else
                z = module_b_attn(gf_, zt, h, m_.p[l], m_.attn[l], m_.heads, &in);
            if (incoming) incoming->push_back(std::move(in));
        }
        return ura::final_logits(z, m_.p[0]);
    }

    ura::LogitGrid logits(const ura::MaskedGrid& x, const ura::EvidenceMatrix& s,
                          const ura::ParityCheckMatrix& h, double) const override {
        return forward(x, s, h, nullptr);
    }

private:
    ura::GfContext gf_;
    const Model& m_;
};

// §7.1(3) rank adapter: confidences 0 for the k_low lowest rows (ties -> lower row), 1 otherwise.
std::vector<double> rank_confidences(const std::vector<double>& conf, int k_low) {
    const int k = int(conf.size());
    std::vector<int> order(k);
    for (int i = 0; i < k; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return conf[a] < conf[b]; });
    std::vector<double> out(k, 1.0);
    for (int i = 0; i < k_low; ++i) out[order[i]] = 0.0;
    return out;
}

void refine_one(const Model& model, const ura::GfContext& gf, const ura::ParityCheckMatrix& h,
                int K, const double* S, const cider_schedule* sc, const cider_remask* rm,
                int32_t* grid, double* final_logits, int32_t* first, int32_t* rows,
                int32_t* steps, int32_t* mask, const ura::Denoiser* den_override = nullptr) {
    const int q = model.q, L = h.slots();
    StackedDenoiser stacked(gf, model);
    const ura::Denoiser& den = den_override ? *den_override : stacked;
    ura::EvidenceMatrix s(L, q);
    std::copy(S, S + size_t(L) * q, s.v.begin());
    ura::RevealSchedule sched;
    sched.steps = sc->steps;
    sched.tau_max = sc->tau_max;
    sched.tau_min = sc->tau_min;
    sched.first_reveal = sc->first_reveal != 0;
    ura::RefineTrace trace;
    ura::LogitGrid fl;
    ura::SymbolGrid out;
    std::vector<int> last_mask(K, 0);
    const int mode = rm ? rm->mode : CIDER_REMASK_NONE;
    if (mode == CIDER_REMASK_THRESHOLD) {
        ura::RemaskConfig cfg;
        cfg.thresholds.assign(rm->thresholds, rm->thresholds + rm->n_thresholds);
        ura::validate_remask_config(cfg);
        // run_with_remasking, unrolled so final-pass logits and the selected rows are observable;
        // every call below is the reference's own (refine.cpp:277-292).
        ura::MaxProbScorer scorer;
        out = ura::run_refinement(den, s, h, sched, K, L, &trace, &fl);
        for (double thr : cfg.thresholds) {
            auto conf = scorer.score_rows(out, fl);
            bool any = false;
            for (double c : conf) any = any || c < thr;
            if (!any) break;
            for (int k = 0; k < K; ++k) last_mask[k] = conf[k] < thr;
            out = ura::remask_pass(out, conf, thr, den, s, h, sched, &trace, &fl);
        }
    } else {
        out = ura::run_refinement(den, s, h, sched, K, L, &trace, &fl);
        if (mode == CIDER_REMASK_RANK) {
            ura::MaxProbScorer scorer;
            auto conf = scorer.score_rows(out, fl);
            int k_low = int(std::floor(rm->rank_fraction * K));
            if (k_low > 0) {
                auto adj = rank_confidences(conf, k_low);
                for (int k = 0; k < K; ++k) last_mask[k] = adj[k] < 0.5;
                out = ura::remask_pass(out, adj, 0.5, den, s, h, sched, &trace, &fl);
            }
        }
    }
    std::copy(out.v.begin(), out.v.end(), grid);
    if (final_logits) std::copy(fl.v.begin(), fl.v.end(), final_logits);
    if (first) *first = trace.pass_first_reveals.empty() ? 0 : trace.pass_first_reveals.front();
    for (int i = 0; i < CIDER_MAX_THRESHOLDS; ++i) {
        if (rows) rows[i] = i < int(trace.remask_rows_per_stage.size()) ? trace.remask_rows_per_stage[i] : 0;
        if (steps) steps[i] = i < int(trace.remask_steps_per_stage.size()) ? trace.remask_steps_per_stage[i] : 0;
    }
    if (mask) std::copy(last_mask.begin(), last_mask.end(), mask);
}

// ---- the reference arm of bench.py: decodes paused between forwards ------------------------------
// A decode of a config-3/5 bin is 22 fp64 forwards of ~9 s each; bench.py must time bounded steps.
// Each worker thread decodes its bins with the reference's own engine (refine_one above:
// ura::run_refinement + MaxProbScorer + ura::remask_pass), through a Denoiser whose logits() waits for
// a token: ref_session_advance grants every worker n forwards and returns once all of them are
// parked again, so K bench steps time exactly the reference's decode work of those forwards.
struct Session;
class GatedDenoiser : public ura::Denoiser {
public:
    GatedDenoiser(Session& s, int w, const ura::Denoiser& inner) : s_(s), w_(w), inner_(inner) {}
    ura::LogitGrid logits(const ura::MaskedGrid& x, const ura::EvidenceMatrix& ev, const ura::ParityCheckMatrix& h,
                          double r) const override;

private:
    Session& s_;
    int w_;
    const ura::Denoiser& inner_;
};

struct Stopped : std::exception {};

struct Session {
    enum State { RUNNING, PARKED, EXITED };
    Model model;
    ura::GfContext gf;
    ura::ParityCheckMatrix h;
    int K, L, q, n_bins, threads;
    cider_schedule sched;
    cider_remask remask;
    std::vector<double> S;
    std::vector<int32_t> grids;
    std::vector<char> done;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<int> tokens;
    std::vector<State> state;
    bool stop = false;
    int64_t forwards = 0, bins_done = 0;
    std::string error;
    std::vector<std::thread> workers;

    Session(const cider_model_desc* md, const double* w, const cider_code_desc* code, int K_, int n, const double* S_,
            const cider_schedule* sc, const cider_remask* rm, int threads_)
        : model(md, w), gf(make_gf(md)), h(make_h(1 << md->m, code)), K(K_), L(code->slots), q(1 << md->m), n_bins(n),
          threads(threads_), sched(*sc), remask(rm ? *rm : cider_remask{}), S(S_, S_ + size_t(n) * code->slots * (1 << md->m)),
          grids(size_t(n) * K_ * code->slots, -1), done(n, 0), tokens(threads_, 0), state(threads_, RUNNING) {
        for (int t = 0; t < threads; ++t) workers.emplace_back([this, t] { run(t); });
    }
    ~Session() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : workers) t.join();
    }
    void run(int t) {
        StackedDenoiser inner(gf, model);
        GatedDenoiser den(*this, t, inner);
        try {
            for (int b = t; b < n_bins; b += threads) {
                refine_one(model, gf, h, K, S.data() + size_t(b) * L * q, &sched, &remask, grids.data() + size_t(b) * K * L,
                           nullptr, nullptr, nullptr, nullptr, nullptr, &den);
                std::lock_guard<std::mutex> lk(mu);
                done[b] = 1;
                ++bins_done;
            }
        } catch (const Stopped&) {
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lk(mu);
            if (error.empty()) error = e.what();
        }
        std::lock_guard<std::mutex> lk(mu);
        state[t] = EXITED;
        tokens[t] = 0;
        cv.notify_all();
    }
    bool all_parked() const {
        for (int t = 0; t < threads; ++t)
            if (!(state[t] == EXITED || (state[t] == PARKED && tokens[t] == 0))) return false;
        return true;
    }
    void advance(int n) {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return all_parked(); });
        for (int t = 0; t < threads; ++t)
            if (state[t] != EXITED) tokens[t] += n;
        cv.notify_all();
        cv.wait(lk, [&] { return all_parked(); });
        if (!error.empty()) throw std::runtime_error(error);
    }
};

ura::LogitGrid GatedDenoiser::logits(const ura::MaskedGrid& x, const ura::EvidenceMatrix& ev,
                                     const ura::ParityCheckMatrix& h, double r) const {
    {
        std::unique_lock<std::mutex> lk(s_.mu);
        s_.state[w_] = Session::PARKED;
        s_.cv.notify_all();
        s_.cv.wait(lk, [&] { return s_.stop || s_.tokens[w_] > 0; });
        if (s_.stop) throw Stopped();
        --s_.tokens[w_];
        s_.state[w_] = Session::RUNNING;
    }
    ura::LogitGrid out = inner_.logits(x, ev, h, r);
    std::lock_guard<std::mutex> lk(s_.mu);
    ++s_.forwards;
    return out;
}

} // namespace

extern "C" {

// cider_weights_init's layout and draw order with the reference's own seeding: one
// make_rng(seed) stream of uniform(-1/sqrt(D), 1/sqrt(D)) draws in random_init's order (tables, then per
// layer gate_a, check_agg, fuse_b), attention parameters from make_rng(derive_seed(seed, 1000 + layer)).
// N = 1, H = D, heads = 0 is DenoiserParams::random_init (denoiser.cpp:41-69) value for value.
int ref_weights_init(const cider_model_desc* md, uint64_t seed, double* out) {
    return guarded([&] {
        const size_t q = size_t(1) << md->m, D = md->dim, H = md->hidden;
        const double bound = 1.0 / std::sqrt(double(D));
        std::uniform_real_distribution<double> u(-bound, bound);
        auto rng = ura::make_rng(seed);
        size_t off = 0;
        auto fill = [&](std::mt19937_64& g, size_t n) {
            for (size_t i = 0; i < n; ++i) out[off++] = u(g);
        };
        fill(rng, (q + 1) * D);
        fill(rng, q * D);
        fill(rng, q * D);
        for (int l = 0; l < md->layers; ++l)
            for (size_t in : {2 * D, D, 2 * D}) {
                fill(rng, H * in);
                fill(rng, H);
                fill(rng, D * H);
                fill(rng, D);
            }
        if (md->heads > 0)
            for (int l = 0; l < md->layers; ++l) {
                auto ra = ura::make_rng(ura::derive_seed(seed, 1000 + uint64_t(l)));
                fill(ra, D);
                fill(ra, D * D);
            }
    });
}

// The BASELINE evidence model over the reference's own code construction: bin b's
// stream is make_rng(derive_seed(master, 16 + b)); truth = sample_codewords(gf, derive_generator(gf, H),
// K, rng) (ldpc.cpp:153-195); then per slot K erasure draws, one false-candidate draw (+ its symbol),
// Q normals; S = log_softmax, rounded to fp32 (what both arms decode). Bins fan out over threads.
int ref_workload_bins(int m, const cider_code_desc* code, int K, double snr_db, double p_erase, double p_false,
                      uint64_t master, int64_t first, int n, int32_t* truth, double* S, int threads) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        auto h = make_h(gf.q(), code);
        auto gen = ura::derive_generator(gf, h);
        const int L = code->slots, Q = gf.q();
        const double sigma = std::pow(10.0, -snr_db / 20.0);
        ura::parallel_for(
            n,
            [&](int i) {
                auto rng = ura::make_rng(ura::derive_seed(master, uint64_t(16 + first + i)));
                auto g = ura::sample_codewords(gf, gen, K, rng);
                if (truth) std::copy(g.v.begin(), g.v.end(), truth + size_t(i) * K * L);
                std::uniform_real_distribution<double> uni(0.0, 1.0);
                std::normal_distribution<double> nrm(0.0, 1.0);
                std::uniform_int_distribution<int> sym(0, Q - 1);
                std::vector<double> y(Q);
                for (int l = 0; l < L; ++l) {
                    std::fill(y.begin(), y.end(), 0.0);
                    for (int k = 0; k < K; ++k) {
                        bool erased = uni(rng) < p_erase;
                        if (!erased) y[g.v[size_t(k) * L + l]] += 1.0;
                    }
                    if (uni(rng) < p_false) y[sym(rng)] += 1.0;
                    for (int a = 0; a < Q; ++a) y[a] += sigma * nrm(rng);
                    double mx = y[0];
                    for (int a = 1; a < Q; ++a) mx = std::max(mx, y[a]);
                    double se = 0.0;
                    for (int a = 0; a < Q; ++a) se += std::exp(y[a] - mx);
                    const double lse = mx + std::log(se);
                    for (int a = 0; a < Q; ++a) S[(size_t(i) * L + l) * Q + a] = double(float(y[a] - lse));
                }
            },
            threads);
    });
}

int ref_session_create(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int K, int n_bins,
                       const double* S, const cider_schedule* sched, const cider_remask* remask, int threads, void** out) {
    return guarded([&] {
        if (threads < 1 || n_bins < 1) throw std::domain_error("ref_session: need threads >= 1 and bins >= 1");
        *out = new Session(md, weights, code, K, n_bins, S, sched, remask, threads);
    });
}
// every live worker runs n more forwards (with the decode logic between them); returns when all are parked
int ref_session_advance(void* s, int n) {
    return guarded([&] { static_cast<Session*>(s)->advance(n); });
}
int ref_session_status(void* s, int64_t* forwards, int64_t* bins_done, int32_t* grids, int32_t* done) {
    return guarded([&] {
        auto* ss = static_cast<Session*>(s);
        std::lock_guard<std::mutex> lk(ss->mu);
        *forwards = ss->forwards;
        *bins_done = ss->bins_done;
        if (grids) std::copy(ss->grids.begin(), ss->grids.end(), grids);
        if (done) for (int b = 0; b < ss->n_bins; ++b) done[b] = ss->done[b];
    });
}
void ref_session_destroy(void* s) { delete static_cast<Session*>(s); }


const char* ref_last_error(void) { return g_err.c_str(); }

// ura::DenoiserParams::random_init flattened in draw order (denoiser.cpp:41-69).
int ref_random_init(int q, int dim, uint64_t seed, double* out) {
    return guarded([&] {
        auto p = ura::DenoiserParams::random_init(q, dim, seed);
        size_t off = 0;
        auto put = [&](const std::vector<double>& v) {
            std::copy(v.begin(), v.end(), out + off);
            off += v.size();
        };
        put(p.embed);
        put(p.out_proj);
        put(p.sym_embed);
        for (const ura::TwoLayerMap* t : {&p.gate_a, &p.check_agg, &p.fuse_b}) {
            put(t->w1);
            put(t->b1);
            put(t->w2);
            put(t->b2);
        }
    });
}

// build_random_ldpc(gf, L, P, w, make_rng(seed)) (ldpc.cpp:80-120); edges sorted (check, slot).
int ref_build_ldpc(int m, int slots, int checks, int col_weight, uint64_t seed, int32_t* edges) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        auto rng = ura::make_rng(seed);
        auto h = ura::build_random_ldpc(gf, slots, checks, col_weight, rng);
        for (int e = 0; e < h.edge_count(); ++e) {
            edges[3 * e] = h.edge(e).check;
            edges[3 * e + 1] = h.edge(e).slot;
            edges[3 * e + 2] = h.edge(e).coeff;
        }
    });
}

// sample_codewords(gf, derive_generator(gf, H), K, make_rng(seed)) (ldpc.cpp:153-195).
int ref_sample_codewords(int m, const cider_code_desc* code, int k, uint64_t seed, int32_t* out) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        auto h = make_h(gf.q(), code);
        auto gen = ura::derive_generator(gf, h);
        auto rng = ura::make_rng(seed);
        auto g = ura::sample_codewords(gf, gen, k, rng);
        std::copy(g.v.begin(), g.v.end(), out);
        auto syn_ok = true;
        for (int r = 0; r < k; ++r) {
            std::vector<int> cw(g.v.begin() + size_t(r) * g.cols, g.v.begin() + size_t(r + 1) * g.cols);
            for (int x : h.syndrome(gf, cw)) syn_ok = syn_ok && x == 0;
        }
        if (!syn_ok) throw std::runtime_error("ref_sample_codewords: nonzero syndrome");
    });
}

int ref_gf_mul(int m, int a, int b) { return ura::GfContext::with_default_poly(m).mul(a, b); }
int ref_gf_inv(int m, int a) { return ura::GfContext::with_default_poly(m).inv(a); }

int ref_ser_cer(int K, int L, const int32_t* truth, const int32_t* pred, double* ser, double* cer) {
    return guarded([&] {
        ura::SymbolGrid t(K, L), p(K, L);
        std::copy(truth, truth + K * L, t.v.begin());
        std::copy(pred, pred + K * L, p.v.begin());
        auto r = ura::ser_cer(t, p);
        *ser = r.ser;
        *cer = r.cer;
    });
}

// One denoiser forward (Denoiser::logits) for one bin; incoming: layers x K x L x D (nullable).
int ref_denoise(const cider_model_desc* md, const double* weights, const cider_code_desc* code,
                int K, const int32_t* X, const double* S, double* logits, double* incoming) {
    return guarded([&] {
        Model model(md, weights);
        auto gf = make_gf(md);
        auto h = make_h(gf.q(), code);
        const int L = h.slots(), q = gf.q();
        ura::MaskedGrid x(K, L);
        std::copy(X, X + K * L, x.v.begin());
        ura::EvidenceMatrix s(L, q);
        std::copy(S, S + size_t(L) * q, s.v.begin());
        StackedDenoiser den(gf, model);
        std::vector<ura::LatentGrid> in;
        auto lam = den.forward(x, s, h, incoming ? &in : nullptr);
        if (logits) std::copy(lam.v.begin(), lam.v.end(), logits);
        if (incoming)
            for (size_t l = 0; l < in.size(); ++l)
                std::copy(in[l].v.begin(), in[l].v.end(), incoming + l * in[l].v.size());
    });
}

// ura::reveal_step on caller-provided logits (refine.cpp:83-127).
int ref_reveal_step(int K, int L, int q, const int32_t* X, const double* logits, int target,
                    double tau, int first, int32_t* out) {
    return guarded([&] {
        ura::MaskedGrid x(K, L);
        std::copy(X, X + K * L, x.v.begin());
        ura::LogitGrid lam(K, L, q);
        std::copy(logits, logits + size_t(K) * L * q, lam.v.begin());
        auto y = ura::reveal_step(x, lam, target, tau, first != 0);
        std::copy(y.v.begin(), y.v.end(), out);
    });
}

// Full decode of B bins through the reference engine; bins fan out over ura::parallel_for
// (parallel.cpp:20-51) with `workers` threads (0 = URADEC_WORKERS / hardware_concurrency).
int ref_refine(const cider_model_desc* md, const double* weights, const cider_code_desc* code,
               int B, int K, const double* S, const cider_schedule* sched,
               const cider_remask* remask, int32_t* grid, double* final_logits,
               int32_t* first_reveals, int32_t* remask_rows, int32_t* remask_steps,
               int32_t* remask_mask, int workers) {
    return guarded([&] {
        Model model(md, weights);
        auto gf = make_gf(md);
        auto h = make_h(gf.q(), code);
        const int L = h.slots(), q = gf.q();
        ura::parallel_for(
            B,
            [&](int b) {
                refine_one(model, gf, h, K, S + size_t(b) * L * q, sched, remask,
                           grid + size_t(b) * K * L,
                           final_logits ? final_logits + size_t(b) * K * L * q : nullptr,
                           first_reveals ? first_reveals + b : nullptr,
                           remask_rows ? remask_rows + size_t(b) * CIDER_MAX_THRESHOLDS : nullptr,
                           remask_steps ? remask_steps + size_t(b) * CIDER_MAX_THRESHOLDS : nullptr,
                           remask_mask ? remask_mask + size_t(b) * K : nullptr);
            },
            workers);
    });
}

// ura::remask_pass (refine.cpp:238-275) on caller confidences, per bin, through the stacked denoiser.
int ref_remask_pass(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int B, int K,
                    const double* S, const cider_schedule* sc, const int32_t* grid_in, const double* conf, double threshold,
                    int32_t* grid_out, double* final_logits, int workers) {
    return guarded([&] {
        Model model(md, weights);
        auto gf = make_gf(md);
        auto h = make_h(gf.q(), code);
        const int L = h.slots(), q = gf.q();
        ura::parallel_for(
            B,
            [&](int b) {
                StackedDenoiser den(gf, model);
                ura::EvidenceMatrix s(L, q);
                std::copy(S + size_t(b) * L * q, S + size_t(b + 1) * L * q, s.v.begin());
                ura::SymbolGrid g(K, L);
                std::copy(grid_in + size_t(b) * K * L, grid_in + size_t(b + 1) * K * L, g.v.begin());
                ura::RevealSchedule sched;
                sched.steps = sc->steps;
                sched.tau_max = sc->tau_max;
                sched.tau_min = sc->tau_min;
                sched.first_reveal = sc->first_reveal != 0;
                std::vector<double> cf(conf + size_t(b) * K, conf + size_t(b + 1) * K);
                ura::LogitGrid fl;
                auto out = ura::remask_pass(g, cf, threshold, den, s, h, sched, nullptr, &fl);
                std::copy(out.v.begin(), out.v.end(), grid_out + size_t(b) * K * L);
                if (final_logits && !fl.v.empty()) std::copy(fl.v.begin(), fl.v.end(), final_logits + size_t(b) * K * L * q);
            },
            workers);
    });
}

// Reference GF(Q) FFT-BP check update (bp.cpp:128-149) — the north_star-named WHT kernel's oracle.
int ref_check_update_wht(int m, int n_in, const double* incoming, const int32_t* coeffs,
                         int target_coeff, double* out) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        const int q = gf.q();
        std::vector<std::vector<double>> in(n_in, std::vector<double>(q));
        std::vector<int> c(n_in);
        for (int i = 0; i < n_in; ++i) {
            std::copy(incoming + size_t(i) * q, incoming + size_t(i + 1) * q, in[i].begin());
            c[i] = coeffs[i];
        }
        auto r = ura::check_update_wht(gf, in, c, target_coeff);
        std::copy(r.begin(), r.end(), out);
    });
}

int ref_check_update_direct(int m, int n_in, const double* incoming, const int32_t* coeffs,
                            int target_coeff, double* out) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        const int q = gf.q();
        std::vector<std::vector<double>> in(n_in, std::vector<double>(q));
        std::vector<int> c(n_in);
        for (int i = 0; i < n_in; ++i) {
            std::copy(incoming + size_t(i) * q, incoming + size_t(i + 1) * q, in[i].begin());
            c[i] = coeffs[i];
        }
        auto r = ura::check_update_direct(gf, in, c, target_coeff);
        std::copy(r.begin(), r.end(), out);
    });
}

// Reference FFT-BP decoders (bp.cpp:271-368), WHT backend, for B independent inputs: the oracle of
// the GPU decoder behind cider_bp_decode / cider_sic_decode.
int ref_bp_decode(int m, const cider_code_desc* code, int B, const double* lambda, int max_iters,
                  double message_floor, int early_exit, int32_t* hard, double* marginals, int32_t* converged,
                  int32_t* iters) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        const int q = gf.q();
        auto h = make_h(q, code);
        const int L = h.slots();
        ura::BpConfig cfg;
        cfg.max_iters = max_iters;
        cfg.message_floor = message_floor;
        cfg.early_exit = early_exit != 0;
        cfg.backend = ura::CheckBackend::wht;
        for (int b = 0; b < B; ++b) {
            std::vector<std::vector<double>> lam(L, std::vector<double>(q));
            for (int l = 0; l < L; ++l)
                std::copy(lambda + (size_t(b) * L + l) * q, lambda + (size_t(b) * L + l + 1) * q, lam[l].begin());
            auto r = ura::bp_decode(lam, gf, h, cfg);
            for (int l = 0; l < L; ++l) {
                hard[size_t(b) * L + l] = r.hard[l];
                if (marginals) std::copy(r.marginals[l].begin(), r.marginals[l].end(), marginals + (size_t(b) * L + l) * q);
            }
            if (converged) converged[b] = r.converged ? 1 : 0;
            if (iters) iters[b] = r.iters_used;
        }
    });
}

int ref_sic_decode(int m, const cider_code_desc* code, int B, int K, const double* S, int max_iters,
                   double message_floor, int early_exit, double cancel_value, int32_t* grid, int32_t* stage_converged,
                   int32_t* stage_iters) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        const int q = gf.q();
        auto h = make_h(q, code);
        const int L = h.slots();
        ura::BpConfig cfg;
        cfg.max_iters = max_iters;
        cfg.message_floor = message_floor;
        cfg.early_exit = early_exit != 0;
        cfg.backend = ura::CheckBackend::wht;
        for (int b = 0; b < B; ++b) {
            ura::EvidenceMatrix ev(L, q);
            std::copy(S + size_t(b) * L * q, S + size_t(b + 1) * L * q, ev.v.begin());
            auto r = ura::sic_decode(ev, gf, h, K, cfg, cancel_value);
            for (int k = 0; k < K; ++k) {
                for (int l = 0; l < L; ++l) grid[(size_t(b) * K + k) * L + l] = r.grid.at(k, l);
                if (stage_converged) stage_converged[size_t(b) * K + k] = r.stages[k].converged ? 1 : 0;
                if (stage_iters) stage_iters[size_t(b) * K + k] = r.stages[k].iters_used;
            }
        }
    });
}

// ura::save_parity_file / load_parity_file (ldpc.cpp:197-226): the F4 file-format oracle
int ref_save_parity_file(const char* path, int m, const cider_code_desc* code, int col_weight, uint32_t prim_poly,
                         uint64_t seed) {
    return guarded([&] {
        auto gf = ura::GfContext::with_default_poly(m);
        auto h = make_h(gf.q(), code);
        ura::save_parity_file(path, h, ura::LdpcFileMeta{col_weight, prim_poly, seed});
    });
}
int ref_load_parity_file(const char* path, int max_edges, int32_t* edges, int* n_edges, int* checks, int* slots, int* q,
                         int* col_weight, uint32_t* prim_poly, uint64_t* seed) {
    return guarded([&] {
        ura::LdpcFileMeta meta;
        auto h = ura::load_parity_file(path, &meta);
        if (h.edge_count() > max_edges) throw std::runtime_error("ref_load_parity_file: buffer too small");
        for (int e = 0; e < h.edge_count(); ++e) {
            edges[3 * e] = h.edge(e).check;
            edges[3 * e + 1] = h.edge(e).slot;
            edges[3 * e + 2] = h.edge(e).coeff;
        }
        *n_edges = h.edge_count();
        *checks = h.checks();
        *slots = h.slots();
        *q = h.q();
        *col_weight = meta.col_weight;
        *prim_poly = meta.prim_poly;
        *seed = meta.seed;
    });
}

int ref_cosine_target(int t, int steps, int initially_masked, int base) {
    return base + int(std::lround(ura::cosine_fraction(t, steps) * initially_masked));
}
double ref_infer_temperature(int t, int steps, double tmax, double tmin) {
    return ura::infer_temperature(t, steps, tmax, tmin);
}
int ref_remask_steps(int steps, int k_low, int k) { return ura::remask_steps(steps, k_low, k); }

// ---- AMP slot detector -----------------------------------------------------
// make_dictionaries(q, n_s, slots, seed) (sim.cpp:74-80): slots x q x n_s complex, interleaved.
int ref_amp_make_dicts(int q, int n_s, int slots, uint64_t seed, double* dicts) {
    return guarded([&] {
        auto d = ura::make_dictionaries(q, n_s, slots, seed);
        for (int l = 0; l < slots; ++l)
            for (size_t i = 0; i < d[l].cols.size(); ++i) {
                dicts[(size_t(l) * q * n_s + i) * 2] = d[l].cols[i].real();
                dicts[(size_t(l) * q * n_s + i) * 2 + 1] = d[l].cols[i].imag();
            }
    });
}

static std::vector<ura::SensingMatrix> dicts_from(int q, int n_s, int slots, const double* dicts) {
    std::vector<ura::SensingMatrix> d(slots);
    for (int l = 0; l < slots; ++l) {
        d[l].slot = l;
        d[l].n_s = n_s;
        d[l].q = q;
        d[l].cols.resize(size_t(q) * n_s);
        for (size_t i = 0; i < d[l].cols.size(); ++i)
            d[l].cols[i] = ura::cplx(dicts[(size_t(l) * q * n_s + i) * 2], dicts[(size_t(l) * q * n_s + i) * 2 + 1]);
    }
    return d;
}

// Observations of K users' symbols per slot: activity_vector + transmit on make_rng(seed), slot by
// slot (as generate_frame does after sampling the codewords, sim.cpp:82-103). y: slots x n_s complex.
int ref_amp_observe(int q, int n_s, int slots, const double* dicts, int k, const int32_t* symbols, double p_sym,
                    double noise_var, uint64_t seed, double* y) {
    return guarded([&] {
        auto d = dicts_from(q, n_s, slots, dicts);
        auto rng = ura::make_rng(seed);
        std::vector<int> col(k);
        for (int l = 0; l < slots; ++l) {
            for (int j = 0; j < k; ++j) col[j] = symbols[l * k + j];
            auto yl = ura::transmit(d[l], ura::activity_vector(col, q), p_sym, noise_var, rng);
            for (int r = 0; r < n_s; ++r) {
                y[(size_t(l) * n_s + r) * 2] = yl[r].real();
                y[(size_t(l) * n_s + r) * 2 + 1] = yl[r].imag();
            }
        }
    });
}

// detect_frame (amp.cpp:133-148): S slots x q.
int ref_amp_detect_frame(int q, int n_s, int slots, const double* dicts, const double* y, int iters, double rho_bg,
                         double sigma_u2, double evidence_floor, double* S) {
    return guarded([&] {
        auto d = dicts_from(q, n_s, slots, dicts);
        std::vector<std::vector<ura::cplx>> obs(slots, std::vector<ura::cplx>(n_s));
        for (int l = 0; l < slots; ++l)
            for (int r = 0; r < n_s; ++r) obs[l][r] = ura::cplx(y[(size_t(l) * n_s + r) * 2], y[(size_t(l) * n_s + r) * 2 + 1]);
        ura::AmpConfig cfg;
        cfg.iters = iters;
        cfg.rho_bg = rho_bg;
        cfg.sigma_u2 = sigma_u2;
        cfg.evidence_floor = evidence_floor;
        auto ev = ura::detect_frame(obs, d, cfg);
        for (int l = 0; l < slots; ++l)
            for (int a = 0; a < q; ++a) S[size_t(l) * q + a] = ev.at(l, a);
    });
}

double ref_symbol_power(double eb_db, int payload_bits, int slots) { return ura::symbol_power(eb_db, payload_bits, slots); }

} // extern "C"
