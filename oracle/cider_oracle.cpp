// cider_oracle.cpp — TEST INFRASTRUCTURE ONLY: the CPU oracle for the CIDER refinement path.
//
// A from-scratch fp64 restatement of the reference algorithm (no reference source is compiled
// in here), used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
// checker. It is pinned against the reference itself: tests/test_oracle.py compares it with
// oracle/_ref/libura_ref.so (the reference's own code, built by oracle/Makefile) and with the
// committed golden vectors under tests/golden/ (made by tests/golden/make_golden.py from the
// reference). In ref-exact mode it reproduces the reference bit for bit (same fp64 operation
// order, same libm).
//
// Each routine cites the reference file:line it restates (paths under /root/reference/proj).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>
#include <atomic>

#include "cider.h"

namespace {

thread_local std::string g_err;

// ---- GF(2^m) (gf.cpp:8-46) ---------------------------------------------------------------
struct Field {
    int q = 0;
    std::vector<int> lg, ex;
    explicit Field(int m, uint32_t poly) {
        static const uint32_t dflt[9] = {0, 0x3, 0x7, 0xB, 0x13, 0x25, 0x43, 0x89, 0x11D};
        if (m < 1 || m > 8) throw std::domain_error("oracle: field degree must be in 1..8");
        if (!poly) poly = dflt[m];
        q = 1 << m;
        lg.assign(q, -1);
        ex.assign(q - 1, 0);
        uint32_t v = 1;
        for (int i = 0; i < q - 1; ++i) {
            if (lg[v] != -1) throw std::domain_error("oracle: polynomial not primitive");
            ex[i] = int(v);
            lg[v] = i;
            v <<= 1;
            if (v & (1u << m)) v ^= poly;
        }
    }
    int mul(int a, int b) const {
        if (!a || !b) return 0;
        int s = lg[a] + lg[b];
        if (s >= q - 1) s -= q - 1;
        return ex[s];
    }
    int inv(int a) const {
        if (!a) throw std::domain_error("oracle: zero has no inverse");
        return ex[(q - 1 - lg[a]) % (q - 1)];
    }
};

// ---- Tanner graph (ldpc.cpp:11-30): edges sorted by (check, slot) ------------------------
struct Tanner {
    int P = 0, L = 0;
    std::vector<int> chk, slot, coef;       // per edge
    std::vector<int> cbeg;                   // check j owns edges [cbeg[j], cbeg[j+1])
    Tanner(const cider_code_desc* c, int q) {
        P = c->checks;
        L = c->slots;
        if (P <= 0 || L <= 0) throw std::domain_error("oracle: empty parity-check matrix");
        std::vector<int> idx(c->n_edges);
        for (int i = 0; i < c->n_edges; ++i) idx[i] = i;
        auto E = c->edges;
        std::sort(idx.begin(), idx.end(), [&](int a, int b) {
            return E[3 * a] != E[3 * b] ? E[3 * a] < E[3 * b] : E[3 * a + 1] < E[3 * b + 1];
        });
        cbeg.assign(P + 1, 0);
        for (int n = 0; n < c->n_edges; ++n) {
            int i = idx[n];
            int j = E[3 * i], l = E[3 * i + 1], a = E[3 * i + 2];
            if (j < 0 || j >= P || l < 0 || l >= L) throw std::domain_error("oracle: edge out of range");
            if (a <= 0 || a >= q) throw std::domain_error("oracle: coefficient must be nonzero");
            if (n && chk.back() == j && slot.back() == l) throw std::domain_error("oracle: duplicate edge");
            chk.push_back(j);
            slot.push_back(l);
            coef.push_back(a);
            cbeg[j + 1]++;
        }
        for (int j = 0; j < P; ++j) cbeg[j + 1] += cbeg[j];
    }
};

// Speed without changing a single bit: the reference sums every dot product in index order, seeded
// with its bias; dot4 runs four such chains side by side (instruction-level parallelism only, each
// chain's operation order unchanged), and par_for spreads independent rows / sites over threads.
inline void dot4(const double* a0, const double* a1, const double* a2, const double* a3, const double* x, int n,
                 double* s) {
    double s0 = s[0], s1 = s[1], s2 = s[2], s3 = s[3];
    for (int i = 0; i < n; ++i) {
        const double xi = x[i];
        s0 += a0[i] * xi;
        s1 += a1[i] * xi;
        s2 += a2[i] * xi;
        s3 += a3[i] * xi;
    }
    s[0] = s0; s[1] = s1; s[2] = s2; s[3] = s3;
}
inline double dot1(const double* a, const double* x, int n, double s) {
    for (int i = 0; i < n; ++i) s += a[i] * x[i];
    return s;
}
// rows r of a row-major matrix m (ld) against x, s[r] seeded by init[r] (or 0)
void matvec(const double* m, size_t ld, int rows, const double* x, int n, const double* init, double* out) {
    int r = 0;
    for (; r + 4 <= rows; r += 4) {
        double s[4] = {init ? init[r] : 0.0, init ? init[r + 1] : 0.0, init ? init[r + 2] : 0.0, init ? init[r + 3] : 0.0};
        dot4(m + size_t(r) * ld, m + size_t(r + 1) * ld, m + size_t(r + 2) * ld, m + size_t(r + 3) * ld, x, n, s);
        out[r] = s[0]; out[r + 1] = s[1]; out[r + 2] = s[2]; out[r + 3] = s[3];
    }
    for (; r < rows; ++r) out[r] = dot1(m + size_t(r) * ld, x, n, init ? init[r] : 0.0);
}

thread_local int g_intra = 1; // threads one forward may use (set per call by the C entry points)
void par_for(int n, const std::function<void(int)>& fn) {
    const int T = std::min(g_intra, n);
    if (T <= 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<int> next{0};
    std::exception_ptr err;
    std::atomic<bool> bad{false};
    auto work = [&] {
        for (;;) {
            int i = next.fetch_add(1);
            if (i >= n || bad) return;
            try { fn(i); } catch (...) { if (!bad.exchange(true)) err = std::current_exception(); return; }
        }
    };
    std::vector<std::thread> ts;
    for (int w = 1; w < T; ++w) ts.emplace_back(work);
    work();
    for (auto& t : ts) t.join();
    if (err) std::rethrow_exception(err);
}

double gelu(double x) { return 0.5 * x * (1.0 + std::erf(x / std::sqrt(2.0))); } // denoiser.cpp:13
double sigm(double x) { return 1.0 / (1.0 + std::exp(-x)); }                       // denoiser.cpp:15

struct Mlp {
    int in = 0, hid = 0, out = 0;
    const double *w1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;
    // y = W2 gelu(W1 x + b1) + b2, each affine row seeded with its bias (denoiser.cpp:17-34)
    void run(const double* x, double* y) const {
        std::vector<double> h(hid);
        matvec(w1, size_t(in), hid, x, in, b1, h.data());
        for (int r = 0; r < hid; ++r) h[r] = gelu(h[r]);
        matvec(w2, size_t(hid), out, h.data(), hid, b2, y);
    }
};

struct Layer {
    Mlp gate, agg, fuse;
    const double* aq = nullptr; // attention query (D)
    const double* ak = nullptr; // attention key map (D x D)
};

struct Net {
    int q, D, H, N, heads;
    double tau, beta;
    const double *E, *W, *V;
    std::vector<Layer> layer;
    Net(const cider_model_desc* m, const double* w) {
        q = 1 << m->m;
        D = m->dim;
        H = m->hidden;
        N = m->layers;
        heads = m->heads;
        tau = m->tau_demix;
        beta = m->evidence_scale;
        if (N < 1 || D < 1 || H < 1 || heads < 0 || (heads && D % heads))
            throw std::domain_error("oracle: bad model dimensions");
        if (!(tau > 0.0)) throw std::domain_error("demix_responsibilities: tau must be positive");
        size_t o = 0;
        auto take = [&](size_t n) { const double* p = w + o; o += n; return p; };
        E = take(size_t(q + 1) * D);
        W = take(size_t(q) * D);
        V = take(size_t(q) * D);
        layer.resize(N);
        auto mk = [&](Mlp& f, int in) {
            f.in = in; f.hid = H; f.out = D;
            f.w1 = take(size_t(H) * in); f.b1 = take(H);
            f.w2 = take(size_t(D) * H); f.b2 = take(D);
        };
        for (auto& L : layer) { mk(L.gate, 2 * D); mk(L.agg, D); mk(L.fuse, 2 * D); }
        if (heads)
            for (auto& L : layer) { L.aq = take(D); L.ak = take(size_t(D) * D); }
    }
    const double* w(int a) const { return W + size_t(a) * D; }
};

// T_alpha(x) = W^T Pi_alpha W x (denoiser.cpp:162-179): exact zeros of the permuted symbol
// vector are skipped, as the reference does.
void coeff_act(const Net& n, const Field& f, const double* x, int alpha, double* out) {
    if (!alpha) throw std::domain_error("coeff_action: alpha must be nonzero");
    std::vector<double> sym(n.q), perm(n.q, 0.0);
    matvec(n.W, size_t(n.D), n.q, x, n.D, nullptr, sym.data());
    for (int a = 0; a < n.q; ++a) perm[f.mul(alpha, a)] = sym[a];
    std::fill(out, out + n.D, 0.0);
    for (int a = 0; a < n.q; ++a) {
        if (perm[a] == 0.0) continue;
        for (int i = 0; i < n.D; ++i) out[i] += perm[a] * n.w(a)[i];
    }
}

// One denoiser forward, Z is K x L x D row-major (denoiser.cpp:71-259 restated). Sites, slots
// and (row, check) pairs are independent, so they run under par_for; Module B's messages are
// produced per (row, check) into per-edge buffers and then summed into each slot sequentially in
// the reference's (row, check, edge) order, so the result is bit-identical at any thread count.
void forward(const Net& n, const Field& f, const Tanner& t, int K, const int* X, const double* S,
             double* logits, double* incoming) {
    const int L = t.L, Q = n.q, D = n.D;
    const size_t KL = size_t(K) * L;
    const int NE = int(t.slot.size());
    std::vector<double> Z(KL * D), Zt(KL * D), e(KL * D), acc(KL * D), msgs(size_t(K) * NE * D);
    // embed_grid (denoiser.cpp:71-84)
    for (size_t s = 0; s < KL; ++s) {
        int tok = X[s];
        if (tok != -1 && (tok < 0 || tok >= Q)) throw std::domain_error("embed_grid: token out of range");
        int row = tok == -1 ? Q : tok;
        std::copy(n.E + size_t(row) * D, n.E + size_t(row + 1) * D, Z.begin() + s * D);
    }
    std::vector<double> lbar(KL * Q), r(KL * Q);
    for (int li = 0; li < n.N; ++li) {
        const Layer& Ly = n.layer[li];
        // intermediate logits (denoiser.cpp:86-101)
        par_for(int(KL), [&](int si) {
            const size_t s = size_t(si);
            const int l = int(s % L);
            matvec(n.W, size_t(D), Q, &Z[s * D], D, nullptr, &lbar[s * Q]);
            for (int a = 0; a < Q; ++a) lbar[s * Q + a] = lbar[s * Q + a] + n.beta * S[size_t(l) * Q + a];
        });
        // demixing softmax over rows, normaliser summed in descending order (denoiser.cpp:103-122)
        par_for(L, [&](int l) {
            std::vector<double> ex(K), srt(K);
            for (int a = 0; a < Q; ++a) {
                double mx = lbar[size_t(l) * Q + a];
                for (int k = 1; k < K; ++k) mx = std::max(mx, lbar[(size_t(k) * L + l) * Q + a]);
                for (int k = 0; k < K; ++k) ex[k] = std::exp((lbar[(size_t(k) * L + l) * Q + a] - mx) / n.tau);
                srt = ex;
                std::sort(srt.begin(), srt.end(), std::greater<double>());
                double den = 0.0;
                for (double v : srt) den += v;
                for (int k = 0; k < K; ++k) r[(size_t(k) * L + l) * Q + a] = ex[k] / den;
            }
        });
        // evidence embedding (denoiser.cpp:124-139) and gated fusion (denoiser.cpp:141-160), per site
        par_for(int(KL), [&](int si) {
            const size_t s = size_t(si);
            const int l = int(s % L);
            double* es = &e[s * D];
            std::fill(es, es + D, 0.0);
            for (int a = 0; a < Q; ++a) {
                double wgt = r[s * Q + a] * S[size_t(l) * Q + a];
                if (wgt == 0.0) continue;
                for (int i = 0; i < D; ++i) es[i] += wgt * n.V[size_t(a) * D + i];
            }
            std::vector<double> cat(2 * D), g(D);
            std::copy(&Z[s * D], &Z[s * D] + D, cat.begin());
            std::copy(es, es + D, cat.begin() + D);
            Ly.gate.run(cat.data(), g.data());
            for (int i = 0; i < D; ++i) g[i] = sigm(g[i]);
            for (int i = 0; i < D; ++i) Zt[s * D + i] = g[i] * Z[s * D + i] + (1.0 - g[i]) * es[i];
        });
        // parity-aware propagation (denoiser.cpp:181-228); heads>0: extrinsic pooling attention
        const int dh = n.heads ? D / n.heads : D;
        par_for(K * t.P, [&](int kj) {
            const int k = kj / t.P, j = kj % t.P;
            const int b0 = t.cbeg[j], d = t.cbeg[j + 1] - t.cbeg[j];
            std::vector<double> nv(size_t(d) * D), sc(size_t(d) * std::max(1, n.heads));
            std::vector<double> pooled(D), mapped(D), kv(dh);
            for (int i = 0; i < d; ++i)
                coeff_act(n, f, &Zt[(size_t(k) * L + t.slot[b0 + i]) * D], t.coef[b0 + i], &nv[size_t(i) * D]);
            if (n.heads) {
                const double scale = 1.0 / std::sqrt(double(dh));
                for (int i = 0; i < d; ++i)
                    for (int h = 0; h < n.heads; ++h) {
                        matvec(Ly.ak + size_t(h) * dh * D, size_t(D), dh, &nv[size_t(i) * D], D, nullptr, kv.data());
                        double s = 0.0;
                        for (int o = 0; o < dh; ++o) s += Ly.aq[h * dh + o] * kv[o];
                        sc[size_t(i) * n.heads + h] = s * scale;
                    }
            }
            for (int i = 0; i < d; ++i) {
                std::fill(pooled.begin(), pooled.end(), 0.0);
                if (!n.heads) {
                    for (int i2 = 0; i2 < d; ++i2) {
                        if (i2 == i) continue;
                        for (int o = 0; o < D; ++o) pooled[o] += nv[size_t(i2) * D + o];
                    }
                } else {
                    for (int h = 0; h < n.heads; ++h) {
                        double mx = -INFINITY, den = 0.0;
                        for (int i2 = 0; i2 < d; ++i2)
                            if (i2 != i) mx = std::max(mx, sc[size_t(i2) * n.heads + h]);
                        for (int i2 = 0; i2 < d; ++i2)
                            if (i2 != i) den += std::exp(sc[size_t(i2) * n.heads + h] - mx);
                        for (int i2 = 0; i2 < d; ++i2) {
                            if (i2 == i) continue;
                            double wgt = double(d - 1) * std::exp(sc[size_t(i2) * n.heads + h] - mx) / den;
                            for (int o = h * dh; o < (h + 1) * dh; ++o) pooled[o] += wgt * nv[size_t(i2) * D + o];
                        }
                    }
                }
                Ly.agg.run(pooled.data(), mapped.data());
                coeff_act(n, f, mapped.data(), f.inv(t.coef[b0 + i]), &msgs[(size_t(k) * NE + b0 + i) * D]);
            }
        });
        std::fill(acc.begin(), acc.end(), 0.0);
        for (int k = 0; k < K; ++k)
            for (int ed = 0; ed < NE; ++ed) { // edges are sorted by (check, slot): the reference's order
                const double* msg = &msgs[(size_t(k) * NE + ed) * D];
                double* dst = &acc[(size_t(k) * L + t.slot[ed]) * D];
                for (int o = 0; o < D; ++o) dst[o] += msg[o];
            }
        if (incoming) std::copy(acc.begin(), acc.end(), incoming + size_t(li) * KL * D);
        par_for(int(KL), [&](int si) {
            const size_t s = size_t(si);
            std::vector<double> cat(2 * D), g(D);
            std::copy(&Zt[s * D], &Zt[s * D] + D, cat.begin());
            std::copy(&acc[s * D], &acc[s * D] + D, cat.begin() + D);
            Ly.fuse.run(cat.data(), g.data());
            for (int i = 0; i < D; ++i) Z[s * D + i] = Zt[s * D + i] + g[i];
        });
    }
    // final logits (denoiser.cpp:230-245)
    par_for(int(KL), [&](int si) {
        matvec(n.W, size_t(D), Q, &Z[size_t(si) * D], D, nullptr, &logits[size_t(si) * Q]);
    });
}

// ---- the engine (refine.cpp:11-292 restated) ---------------------------------------------
const double kPi = 3.14159265358979323846;
double cosfrac(int t, int T) {
    if (T < 1) throw std::domain_error("cosine_fraction: need T >= 1");
    return 0.5 * (1.0 - std::cos(kPi * t / T));
}
double temperature(int t, int T, double tmax, double tmin) {
    if (T <= 1) return tmin;
    double w = 0.5 * (1.0 + std::cos(kPi * (t - 1) / (T - 1)));
    return tmax * w + tmin * (1.0 - w);
}
int rm_steps(int T, int low, int K) {
    int s = int((static_cast<long long>(T) * low) / K);
    return s < 1 ? 1 : s;
}
int amax(const double* v, int q) {
    int b = 0;
    for (int a = 1; a < q; ++a)
        if (v[a] > v[b]) b = a;
    return b;
}
double kappa(const double* v, int q, double tau) {
    double m = v[0];
    for (int a = 1; a < q; ++a) m = std::max(m, v[a]);
    double s = 0.0;
    for (int a = 0; a < q; ++a) s += std::exp((v[a] - m) / tau);
    return 1.0 / s;
}

void reveal(int K, int L, int Q, std::vector<int>& x, const double* lam, int target, double tau, bool first) {
    if (!(tau > 0.0)) throw std::domain_error("reveal_step: tau must be positive");
    std::vector<int> y = x;
    if (first) { // refine.cpp:88-103: one site per slot, strict > keeps the lowest row
        for (int l = 0; l < L; ++l) {
            int br = -1;
            double bk = 0.0;
            for (int k = 0; k < K; ++k) {
                if (x[size_t(k) * L + l] != -1) continue;
                double c = kappa(lam + (size_t(k) * L + l) * Q, Q, tau);
                if (br < 0 || c > bk) { br = k; bk = c; }
            }
            if (br >= 0) y[size_t(br) * L + l] = amax(lam + (size_t(br) * L + l) * Q, Q);
        }
        x.swap(y);
        return;
    }
    int revealed = 0;
    for (int v : x) revealed += v != -1;
    if (revealed >= target) return;
    struct Site { double c; int k, l; };
    std::vector<Site> st;
    for (int k = 0; k < K; ++k)
        for (int l = 0; l < L; ++l)
            if (x[size_t(k) * L + l] == -1) st.push_back({kappa(lam + (size_t(k) * L + l) * Q, Q, tau), k, l});
    std::sort(st.begin(), st.end(), [](const Site& a, const Site& b) {
        if (a.c != b.c) return a.c > b.c;
        if (a.k != b.k) return a.k < b.k;
        return a.l < b.l;
    });
    for (const Site& s : st) {
        if (revealed >= target) break;
        y[size_t(s.k) * L + s.l] = amax(lam + (size_t(s.k) * L + s.l) * Q, Q);
        ++revealed;
    }
    x.swap(y);
}

// run_masked_loop (refine.cpp:134-195)
std::vector<int> masked_loop(const Net& n, const Field& f, const Tanner& t, int K, const double* S,
                             const cider_schedule& sc, std::vector<int> x, const std::vector<char>& upd,
                             std::vector<double>& fl, int* first_count) {
    if (sc.steps < 1) throw std::domain_error("run_refinement: need T >= 1");
    if (!(sc.tau_min > 0.0) || sc.tau_max < sc.tau_min)
        throw std::domain_error("run_refinement: need tau_max >= tau_min > 0");
    const int L = t.L, Q = n.q, total = K * L;
    int init_masked = 0;
    for (int v : x) init_masked += v == -1;
    const int base = total - init_masked;
    std::vector<double> lam(size_t(total) * Q);
    for (int step = 1; step <= sc.steps; ++step) {
        try {
            forward(n, f, t, K, x.data(), S, lam.data(), nullptr);
        } catch (const std::exception& e) {
            throw std::runtime_error("denoiser failed at step " + std::to_string(step) + ": " + e.what());
        }
        double tau = temperature(step, sc.steps, sc.tau_max, sc.tau_min);
        int target = base + int(std::lround(cosfrac(step, sc.steps) * init_masked));
        int before = 0;
        for (int v : x) before += v == -1;
        reveal(K, L, Q, x, lam.data(), target, tau, step == 1 && sc.first_reveal);
        if (step == 1 && first_count) {
            int after = 0;
            for (int v : x) after += v == -1;
            *first_count = before - after;
        }
    }
    for (int s = 0; s < total; ++s)
        if (x[s] == -1) x[s] = amax(&lam[size_t(s) * Q], Q);
    fl.assign(size_t(total) * Q, 0.0);
    try {
        forward(n, f, t, K, x.data(), S, fl.data(), nullptr);
    } catch (const std::exception& e) {
        throw std::runtime_error(std::string("denoiser failed at the final pass: ") + e.what());
    }
    std::vector<int> out = x;
    for (int k = 0; k < K; ++k)
        if (upd[k])
            for (int l = 0; l < L; ++l) out[size_t(k) * L + l] = amax(&fl[(size_t(k) * L + l) * Q], Q);
    return out;
}

// MaxProbScorer + row_confidence (refine.cpp:207-225)
std::vector<double> row_conf(int K, int L, int Q, const std::vector<double>& fl) {
    std::vector<double> c(K);
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int l = 0; l < L; ++l) s += kappa(&fl[(size_t(k) * L + l) * Q], Q, 1.0);
        c[k] = s / L;
    }
    return c;
}

// remask_pass (refine.cpp:238-275) with an explicit low-row set.
std::vector<int> remask(const Net& n, const Field& f, const Tanner& t, int K, const double* S,
                        const cider_schedule& sc, const std::vector<int>& grid, const std::vector<char>& low,
                        std::vector<double>& fl, int* rows, int* steps) {
    const int L = t.L;
    int nlow = 0;
    for (char c : low) nlow += c != 0;
    if (!nlow) return grid;
    std::vector<int> x0 = grid;
    for (int k = 0; k < K; ++k)
        if (low[k])
            for (int l = 0; l < L; ++l) x0[size_t(k) * L + l] = -1;
    cider_schedule rm = sc;
    rm.steps = rm_steps(sc.steps, nlow, K);
    *rows = nlow;
    *steps = rm.steps;
    auto redone = masked_loop(n, f, t, K, S, rm, x0, low, fl, nullptr);
    std::vector<int> merged = grid;
    for (int k = 0; k < K; ++k)
        if (low[k])
            for (int l = 0; l < L; ++l) merged[size_t(k) * L + l] = redone[size_t(k) * L + l];
    return merged;
}

void decode(const Net& n, const Field& f, const Tanner& t, int K, const double* S,
            const cider_schedule& sc, const cider_remask* rmc, int* grid, double* flo, int* first,
            int* rows, int* steps, int* mask) {
    const int L = t.L, Q = n.q;
    std::vector<double> fl;
    std::vector<char> all(K, 1);
    int fr = 0;
    std::vector<int> g = masked_loop(n, f, t, K, S, sc, std::vector<int>(size_t(K) * L, -1), all, fl, &fr);
    std::vector<int> r(CIDER_MAX_THRESHOLDS, 0), s(CIDER_MAX_THRESHOLDS, 0), lastmask(K, 0);
    const int mode = rmc ? rmc->mode : CIDER_REMASK_NONE;
    if (mode == CIDER_REMASK_THRESHOLD) {
        double prev = 1.0; // validate_remask_config (refine.cpp:48-57)
        for (int i = 0; i < rmc->n_thresholds; ++i) {
            double th = rmc->thresholds[i];
            if (th <= 0.0 || th >= 1.0) throw std::domain_error("remask thresholds must lie in (0,1)");
            if (th >= prev) throw std::domain_error("remask thresholds must be strictly descending");
            prev = th;
        }
        int stage = 0;
        for (int i = 0; i < rmc->n_thresholds; ++i) {
            auto c = row_conf(K, L, Q, fl);
            std::vector<char> low(K, 0);
            bool any = false;
            for (int k = 0; k < K; ++k) { low[k] = c[k] < rmc->thresholds[i]; any = any || low[k]; }
            if (!any) break;
            for (int k = 0; k < K; ++k) lastmask[k] = low[k];
            g = remask(n, f, t, K, S, sc, g, low, fl, &r[stage], &s[stage]);
            ++stage;
        }
    } else if (mode == CIDER_REMASK_RANK) {
        int klow = int(std::floor(rmc->rank_fraction * K));
        if (klow > 0) {
            auto c = row_conf(K, L, Q, fl);
            std::vector<int> ord(K);
            for (int k = 0; k < K; ++k) ord[k] = k;
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return c[a] < c[b]; });
            std::vector<char> low(K, 0);
            for (int i = 0; i < klow; ++i) low[ord[i]] = 1;
            for (int k = 0; k < K; ++k) lastmask[k] = low[k];
            g = remask(n, f, t, K, S, sc, g, low, fl, &r[0], &s[0]);
        }
    }
    std::copy(g.begin(), g.end(), grid);
    if (flo) std::copy(fl.begin(), fl.end(), flo);
    if (first) *first = fr;
    if (rows) std::copy(r.begin(), r.end(), rows);
    if (steps) std::copy(s.begin(), s.end(), steps);
    if (mask) std::copy(lastmask.begin(), lastmask.end(), mask);
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return CIDER_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CIDER_ERUNTIME;
    }
}

// n independent jobs over `threads` workers (0 = all cores); when there are fewer jobs than
// threads, each job's forwards get the spare threads (g_intra)
void pool_for(int n, int threads, const std::function<void(int)>& fn) {
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    const int workers = std::min(threads, std::max(n, 1));
    const int intra = std::max(1, threads / std::max(workers, 1));
    std::atomic<int> next{0};
    std::exception_ptr err;
    std::atomic<bool> bad{false};
    std::vector<std::thread> ts;
    for (int w = 0; w < workers; ++w)
        ts.emplace_back([&] {
            g_intra = intra;
            for (;;) {
                int i = next.fetch_add(1);
                if (i >= n || bad) return;
                try { fn(i); } catch (...) { if (!bad.exchange(true)) err = std::current_exception(); return; }
            }
        });
    for (auto& t : ts) t.join();
    if (err) std::rethrow_exception(err);
}

// ---- GF(Q) FFT-BP check update, WHT domain (bp.cpp:128-149, 195-206) ----------------------
void wht(long double* v, int q) {
    for (int len = 1; len < q; len <<= 1)
        for (int i = 0; i < q; i += 2 * len)
            for (int j = i; j < i + len; ++j) {
                long double a = v[j], b = v[j + len];
                v[j] = a + b;
                v[j + len] = a - b;
            }
}

} // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_denoise(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int K,
                   const int32_t* X, const double* S, double* logits, double* incoming) {
    return guarded([&] {
        Net n(md, weights);
        Field f(md->m, md->prim_poly);
        Tanner t(code, f.q);
        std::vector<double> lam(size_t(K) * t.L * f.q);
        forward(n, f, t, K, X, S, logits ? logits : lam.data(), incoming);
    });
}

// B independent forwards (X: B x K x L, S: B x L x Q, logits: B x K x L x Q) on `threads` threads
int oracle_denoise_batch(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int B,
                         int K, const int32_t* X, const double* S, double* logits, int threads) {
    return guarded([&] {
        Net n(md, weights);
        Field f(md->m, md->prim_poly);
        Tanner t(code, f.q);
        const size_t nx = size_t(K) * t.L, nq = nx * f.q;
        pool_for(B, threads, [&](int b) {
            forward(n, f, t, K, X + size_t(b) * nx, S + size_t(b) * t.L * f.q, logits + size_t(b) * nq, nullptr);
        });
    });
}

int oracle_reveal_step(int K, int L, int Q, const int32_t* X, const double* logits, int target, double tau,
                       int first, int32_t* out) {
    return guarded([&] {
        std::vector<int> x(X, X + K * L);
        reveal(K, L, Q, x, logits, target, tau, first != 0);
        std::copy(x.begin(), x.end(), out);
    });
}

int oracle_refine(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int B,
                  int K, const double* S, const cider_schedule* sched, const cider_remask* remask_cfg,
                  int32_t* grid, double* final_logits, int32_t* first, int32_t* rows, int32_t* steps,
                  int32_t* mask, int threads) {
    return guarded([&] {
        Net n(md, weights);
        Field f(md->m, md->prim_poly);
        Tanner t(code, f.q);
        const int L = t.L, Q = f.q;
        pool_for(B, threads, [&](int b) {
            decode(n, f, t, K, S + size_t(b) * L * Q, *sched, remask_cfg, grid + size_t(b) * K * L,
                   final_logits ? final_logits + size_t(b) * K * L * Q : nullptr, first ? first + b : nullptr,
                   rows ? rows + size_t(b) * CIDER_MAX_THRESHOLDS : nullptr,
                   steps ? steps + size_t(b) * CIDER_MAX_THRESHOLDS : nullptr, mask ? mask + size_t(b) * K : nullptr);
        });
    });
}

// remask_pass with caller row confidences (refine.cpp:238-275): rows with conf < threshold re-decoded.
int oracle_remask_pass(const cider_model_desc* md, const double* weights, const cider_code_desc* code, int B, int K,
                       const double* S, const cider_schedule* sched, const int32_t* grid_in, const double* conf,
                       double threshold, int32_t* grid_out, double* final_logits, int threads) {
    return guarded([&] {
        Net n(md, weights);
        Field f(md->m, md->prim_poly);
        Tanner t(code, f.q);
        const int L = t.L, Q = f.q;
        pool_for(B, threads, [&](int b) {
            std::vector<int> g(grid_in + size_t(b) * K * L, grid_in + size_t(b + 1) * K * L);
            std::vector<char> low(K, 0);
            for (int k = 0; k < K; ++k) low[k] = conf[size_t(b) * K + k] < threshold;
            std::vector<double> fl;
            int rows = 0, steps = 0;
            auto out = remask(n, f, t, K, S + size_t(b) * L * Q, *sched, g, low, fl, &rows, &steps);
            std::copy(out.begin(), out.end(), grid_out + size_t(b) * K * L);
            if (final_logits && rows) std::copy(fl.begin(), fl.end(), final_logits + size_t(b) * K * L * Q);
        });
    });
}

// Check->variable message of one GF(Q) parity check in the WHT domain (bp.cpp:128-149):
// permute each input by its coefficient, transform, multiply, transform back, gather by the
// target coefficient, clamp at 0, normalise (uniform if all mass vanished, bp.cpp:11-19).
int oracle_check_update_wht(int m, int n_in, const double* incoming, const int32_t* coeffs, int target,
                            double* out) {
    return guarded([&] {
        Field f(m, 0);
        const int q = f.q;
        std::vector<long double> acc(q, 1.0L), y(q);
        for (int i = 0; i < n_in; ++i) {
            std::fill(y.begin(), y.end(), 0.0L);
            for (int a = 0; a < q; ++a) y[f.mul(coeffs[i], a)] = incoming[size_t(i) * q + a];
            wht(y.data(), q);
            for (int a = 0; a < q; ++a) acc[a] *= y[a];
        }
        wht(acc.data(), q);
        const long double sc = 1.0L / q;
        double sum = 0.0;
        for (int a = 0; a < q; ++a) {
            out[a] = std::max(double(acc[f.mul(target, a)] * sc), 0.0);
        }
        for (int a = 0; a < q; ++a) sum += out[a];
        if (sum > 0.0) {
            double inv = 1.0 / sum;
            for (int a = 0; a < q; ++a) out[a] *= inv;
        } else {
            for (int a = 0; a < q; ++a) out[a] = 1.0 / q;
        }
    });
}

} // extern "C"
