// host.cpp — GF tables, Tanner graph validation, weight initialisation, the BASELINE workload
// generator and the permutation-invariant SER/CER of libcider. Host C++ only.
//
// Bit-compatibility with the reference matters here: the weights and the code/codewords must
// be the ones the reference would draw from the same seeds, so the draws below follow the
// reference's draw ORDER with the same libstdc++ distribution types (implementation-defined,
// hence generated on the host with the same toolchain — SURVEY §7.1(2)). They are pinned by
// tests/test_workload.py against oracle/_ref (the reference's own code).
#include <algorithm>
#include <atomic>
#include <fstream>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <set>
#include <thread>

#include "host.hpp"

namespace cider {

uint32_t Gf::default_poly(int m) {
    // conventional primitive polynomials (gf.cpp:8-20)
    static const uint32_t p[9] = {0, 0x3, 0x7, 0xB, 0x13, 0x25, 0x43, 0x89, 0x11D};
    if (m < 1 || m > 8) throw InvalidInput("GfContext: extension degree must be in 1..8");
    return p[m];
}

Gf::Gf(int m_, uint32_t poly_) : m(m_) {
    if (m < 1 || m > 8) throw InvalidInput("GfContext: extension degree must be in 1..8");
    poly = poly_ ? poly_ : default_poly(m);
    if ((poly >> m) != 1u) throw InvalidInput("GfContext: prim_poly must have degree exactly m");
    q = 1 << m;
    lg.assign(q, -1);
    ex.assign(q - 1, 0);
    uint32_t e = 1;
    for (int i = 0; i < q - 1; ++i) {
        if (lg[e] != -1) throw InvalidInput("GfContext: polynomial is not primitive");
        ex[i] = int(e);
        lg[e] = i;
        e <<= 1;
        if (e & (1u << m)) e ^= poly;
    }
    if (e != 1) throw InvalidInput("GfContext: polynomial is not primitive");
}

int Gf::inv(int a) const {
    if (!a) throw InvalidInput("gf_inv: zero has no inverse");
    return ex[(q - 1 - lg[a]) % (q - 1)];
}

Tanner::Tanner(const cider_code_desc* c, int q_) : q(q_) {
    if (!c || c->checks <= 0 || c->slots <= 0) throw InvalidInput("ParityCheckMatrix: empty dimensions");
    checks = c->checks;
    slots = c->slots;
    if (c->n_edges < 0 || (c->n_edges && !c->edges)) throw InvalidInput("ParityCheckMatrix: bad edge list");
    std::vector<int> idx(c->n_edges);
    for (int i = 0; i < c->n_edges; ++i) idx[i] = i;
    const int32_t* E = c->edges;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) {
        return E[3 * a] != E[3 * b] ? E[3 * a] < E[3 * b] : E[3 * a + 1] < E[3 * b + 1];
    });
    check_ptr.assign(checks + 1, 0);
    slot_ptr.assign(slots + 1, 0);
    for (int n = 0; n < c->n_edges; ++n) {
        int i = idx[n];
        int j = E[3 * i], l = E[3 * i + 1], a = E[3 * i + 2];
        if (j < 0 || j >= checks || l < 0 || l >= slots)
            throw InvalidInput("ParityCheckMatrix: edge index out of range");
        if (a <= 0 || a >= q) throw InvalidInput("ParityCheckMatrix: coefficient must be a nonzero field element");
        if (n && chk.back() == j && slot.back() == l)
            throw InvalidInput("ParityCheckMatrix: duplicate (check, slot) entry");
        chk.push_back(j);
        slot.push_back(l);
        coef.push_back(a);
        check_ptr[j + 1]++;
        slot_ptr[l + 1]++;
    }
    for (int j = 0; j < checks; ++j) check_ptr[j + 1] += check_ptr[j];
    for (int l = 0; l < slots; ++l) slot_ptr[l + 1] += slot_ptr[l];
    slot_edge.assign(chk.size(), 0);
    std::vector<int> fill(slot_ptr.begin(), slot_ptr.end() - 1);
    for (int e = 0; e < n_edges(); ++e) slot_edge[fill[slot[e]]++] = e; // ascending edge = ascending check
}

void validate_model(const cider_model_desc* m) {
    if (!m) throw InvalidInput("cider: null model");
    if (m->m < 1 || m->m > 8) throw InvalidInput("GfContext: extension degree must be in 1..8");
    if (m->dim < 1 || m->hidden < 1 || m->layers < 1)
        throw InvalidInput("DenoiserParams: bad dimensions");
    if (m->heads < 0 || (m->heads > 0 && m->dim % m->heads))
        throw InvalidInput("cider: heads must divide dim");
    if (!(m->tau_demix > 0.0)) throw InvalidInput("demix_responsibilities: tau must be positive");
    if (m->precision != CIDER_FP32 && m->precision != CIDER_BF16)
        throw InvalidInput("cider: unknown precision");
}

size_t weights_count(const cider_model_desc* m) {
    const size_t q = size_t(1) << m->m, D = m->dim, H = m->hidden, N = m->layers;
    size_t n = (q + 1) * D + 2 * q * D;
    size_t per_layer = (H * 2 * D + H + D * H + D) + (H * D + H + D * H + D) + (H * 2 * D + H + D * H + D);
    n += N * per_layer;
    if (m->heads > 0) n += N * (D + D * D);
    return n;
}

namespace {

// Draw order = DenoiserParams::random_init (denoiser.cpp:41-69) generalised to N layers and
// hidden width H; attention parameters from their own streams
// derive_seed(seed, 1000 + layer) so heads = 0 leaves the base stream untouched.
void init_weights(const cider_model_desc* m, uint64_t seed, double* out) {
    validate_model(m);
    const double bound = 1.0 / std::sqrt(double(m->dim));
    std::uniform_real_distribution<double> u(-bound, bound);
    std::mt19937_64 rng(seed);
    const size_t q = size_t(1) << m->m, D = m->dim, H = m->hidden;
    size_t off = 0;
    auto fill = [&](std::mt19937_64& g, size_t n) {
        for (size_t i = 0; i < n; ++i) out[off++] = u(g);
    };
    fill(rng, (q + 1) * D); // embed
    fill(rng, q * D);       // out_proj
    fill(rng, q * D);       // sym_embed
    for (int l = 0; l < m->layers; ++l) {
        for (size_t in : {2 * D, D, 2 * D}) { // gate_a, check_agg, fuse_b
            fill(rng, H * in);
            fill(rng, H);
            fill(rng, D * H);
            fill(rng, D);
        }
    }
    if (m->heads > 0)
        for (int l = 0; l < m->layers; ++l) {
            std::mt19937_64 ra(derive_seed(seed, 1000 + uint64_t(l)));
            fill(ra, D);
            fill(ra, D * D);
        }
}

// ---- code construction (the reference's ldpc.cpp:80-195 algorithms, host-side) -----------

int gf_rank(const Gf& gf, std::vector<std::vector<int>> a, std::vector<int>* pivots) {
    const int rows = int(a.size()), cols = rows ? int(a[0].size()) : 0;
    int r = 0;
    for (int c = 0; c < cols && r < rows; ++c) {
        int p = -1;
        for (int i = r; i < rows; ++i)
            if (a[i][c]) { p = i; break; }
        if (p < 0) continue;
        std::swap(a[r], a[p]);
        int s = gf.inv(a[r][c]);
        for (int j = 0; j < cols; ++j) a[r][j] = gf.mul(s, a[r][j]);
        for (int i = 0; i < rows; ++i) {
            if (i == r || !a[i][c]) continue;
            int f = a[i][c];
            for (int j = 0; j < cols; ++j) a[i][j] ^= gf.mul(f, a[r][j]);
        }
        if (pivots) pivots->push_back(c);
        ++r;
    }
    return r;
}

struct Systematic {
    std::vector<int> pivot, info;
    std::vector<std::vector<int>> red; // red[i][j]: info symbol j's coefficient in pivot row i
};

Systematic systematic_form(const Gf& gf, const Tanner& t) {
    std::vector<std::vector<int>> a(t.checks, std::vector<int>(t.slots, 0));
    for (int e = 0; e < t.n_edges(); ++e) a[t.chk[e]][t.slot[e]] = t.coef[e];
    // reduce in place (same elimination as gf_rank, keeping the reduced rows)
    Systematic s;
    const int rows = t.checks, cols = t.slots;
    int r = 0;
    for (int c = 0; c < cols && r < rows; ++c) {
        int p = -1;
        for (int i = r; i < rows; ++i)
            if (a[i][c]) { p = i; break; }
        if (p < 0) continue;
        std::swap(a[r], a[p]);
        int sc = gf.inv(a[r][c]);
        for (int j = 0; j < cols; ++j) a[r][j] = gf.mul(sc, a[r][j]);
        for (int i = 0; i < rows; ++i) {
            if (i == r || !a[i][c]) continue;
            int f = a[i][c];
            for (int j = 0; j < cols; ++j) a[i][j] ^= gf.mul(f, a[r][j]);
        }
        s.pivot.push_back(c);
        ++r;
    }
    if (r != rows) throw std::runtime_error("derive_generator: H is rank deficient");
    std::vector<char> isp(cols, 0);
    for (int c : s.pivot) isp[c] = 1;
    for (int c = 0; c < cols; ++c)
        if (!isp[c]) s.info.push_back(c);
    s.red.assign(rows, std::vector<int>(s.info.size()));
    for (int i = 0; i < rows; ++i)
        for (size_t j = 0; j < s.info.size(); ++j) s.red[i][j] = a[i][s.info[j]];
    return s;
}

std::vector<int> encode(const Gf& gf, const Systematic& s, int slots, const std::vector<int>& info) {
    std::vector<int> c(slots, 0);
    for (size_t j = 0; j < s.info.size(); ++j) c[s.info[j]] = info[j];
    for (size_t i = 0; i < s.pivot.size(); ++i) {
        int acc = 0;
        for (size_t j = 0; j < s.info.size(); ++j) acc ^= gf.mul(s.red[i][j], info[j]);
        c[s.pivot[i]] = acc;
    }
    return c;
}

// regular-column construction with greedy balanced rows (ldpc.cpp:80-120)
std::vector<int> random_ldpc(const Gf& gf, int slots, int checks, int w, std::mt19937_64& rng) {
    if (checks >= slots) throw InvalidInput("build_random_ldpc: need P < L");
    if (w < 2) throw InvalidInput("build_random_ldpc: col_weight must be >= 2");
    if (w > checks) throw InvalidInput("build_random_ldpc: col_weight exceeds check count");
    std::uniform_int_distribution<int> coeff(1, gf.q - 1);
    std::vector<int> cand;
    for (int attempt = 0; attempt < 64; ++attempt) {
        std::vector<int> deg(checks, 0), edges;
        for (int l = 0; l < slots; ++l) {
            std::vector<char> used(checks, 0);
            for (int k = 0; k < w; ++k) {
                // (the reference starts the scan at checks + 1, ldpc.cpp:103: once every free check has a
                // larger degree — dense codes, 3 L / P > P + 1 — its candidate list is empty and the draw is
                // undefined behaviour; an unbounded start gives the same codes wherever the reference is defined)
                int lo = std::numeric_limits<int>::max();
                for (int j = 0; j < checks; ++j)
                    if (!used[j] && deg[j] < lo) lo = deg[j];
                cand.clear();
                for (int j = 0; j < checks; ++j)
                    if (!used[j] && deg[j] == lo) cand.push_back(j);
                std::uniform_int_distribution<size_t> pick(0, cand.size() - 1);
                int j = cand[pick(rng)];
                used[j] = 1;
                ++deg[j];
                int a = coeff(rng);
                edges.insert(edges.end(), {j, l, a});
            }
        }
        cider_code_desc cd{checks, slots, int(edges.size() / 3), edges.data()};
        Tanner t(&cd, gf.q);
        std::vector<std::vector<int>> a(checks, std::vector<int>(slots, 0));
        for (int e = 0; e < t.n_edges(); ++e) a[t.chk[e]][t.slot[e]] = t.coef[e];
        if (gf_rank(gf, a, nullptr) == checks) {
            std::vector<int> out;
            for (int e = 0; e < t.n_edges(); ++e) out.insert(out.end(), {t.chk[e], t.slot[e], t.coef[e]});
            return out;
        }
    }
    throw std::runtime_error("build_random_ldpc: no full-rank matrix within the retry budget");
}

// K codewords from K distinct uniform info vectors (ldpc.cpp:174-195)
void codewords(const Gf& gf, const Systematic& s, int slots, int k, std::mt19937_64& rng, int32_t* out) {
    std::uniform_int_distribution<int> sym(0, gf.q - 1);
    std::set<std::vector<int>> seen;
    int n = 0;
    while (n < k) {
        std::vector<int> info(s.info.size());
        for (int& x : info) x = sym(rng);
        if (!seen.insert(info).second) continue;
        auto c = encode(gf, s, slots, info);
        std::copy(c.begin(), c.end(), out + size_t(n) * slots);
        ++n;
    }
}

template <class F>
void parallel(int n, int threads, F&& fn) {
    if (threads <= 0) threads = int(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::max(1, std::min(threads, n));
    if (threads == 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&] {
            for (int i; (i = next.fetch_add(1)) < n;) fn(i);
        });
    for (auto& t : pool) t.join();
}

// Lexicographically smallest minimum-cost assignment for K <= 16 via DP over column subsets
// (same optimum and tie rule as metrics.cpp:79-122).
void assignment(int K, const std::vector<int>& cost, std::vector<int>& perm, int& total) {
    const int full = 1 << K;
    std::vector<int> best(full, 0); // best[mask] = optimal cost of rows popcount(mask).. over cols ~mask
    for (int mask = full - 2; mask >= 0; --mask) {
        int row = __builtin_popcount(mask);
        int b = 1 << 30;
        for (int c = 0; c < K; ++c)
            if (!(mask & (1 << c))) b = std::min(b, cost[row * K + c] + best[mask | (1 << c)]);
        best[mask] = b;
    }
    best[full - 1] = 0;
    total = best[0];
    perm.assign(K, -1);
    int mask = 0;
    for (int row = 0; row < K; ++row)
        for (int c = 0; c < K; ++c)
            if (!(mask & (1 << c)) && cost[row * K + c] + best[mask | (1 << c)] == best[mask]) {
                perm[row] = c;
                mask |= 1 << c;
                break;
            }
}

thread_local std::string g_host_err;
thread_local uint64_t g_host_err_tick = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return CIDER_OK;
    } catch (const std::domain_error& e) {
        g_host_err = e.what();
        g_host_err_tick = error_tick();
        return CIDER_EINVAL;
    } catch (const std::exception& e) {
        g_host_err = e.what();
        g_host_err_tick = error_tick();
        return CIDER_ERUNTIME;
    }
}

} // namespace

void systematic_tables(const Gf& gf, const Tanner& t, std::vector<int>& info, std::vector<int>& pivot,
                       std::vector<uint8_t>& red) {
    Systematic s = systematic_form(gf, t);
    info = s.info;
    pivot = s.pivot;
    red.assign(s.pivot.size() * s.info.size(), 0);
    for (size_t i = 0; i < s.pivot.size(); ++i)
        for (size_t j = 0; j < s.info.size(); ++j) red[i * s.info.size() + j] = uint8_t(s.red[i][j]);
}


const char* host_last_error() { return g_host_err.c_str(); }
uint64_t host_error_tick() { return g_host_err_tick; }
void set_host_error(const std::string& msg) {
    g_host_err = msg;
    g_host_err_tick = error_tick();
}
uint64_t error_tick() { // per-thread order of failures across the host and engine halves of the ABI
    static thread_local uint64_t t = 0;
    return ++t;
}

} // namespace cider

using namespace cider;

extern "C" {

size_t cider_weights_count(const cider_model_desc* m) {
    try {
        validate_model(m);
        return weights_count(m);
    } catch (...) {
        return 0;
    }
}

int cider_weights_init_f64(const cider_model_desc* m, uint64_t seed, double* out) {
    return guard([&] { init_weights(m, seed, out); });
}

int cider_weights_init(const cider_model_desc* m, uint64_t seed, float* out) {
    return guard([&] {
        validate_model(m);
        std::vector<double> w(weights_count(m));
        init_weights(m, seed, w.data());
        for (size_t i = 0; i < w.size(); ++i) out[i] = float(w[i]);
    });
}

int cider_workload_code(const cider_workload_desc* w, int32_t* edges) {
    return guard([&] {
        Gf gf(w->m, 0);
        std::mt19937_64 rng(derive_seed(w->master_seed, 1));
        auto e = random_ldpc(gf, w->slots, w->checks, w->col_weight, rng);
        std::copy(e.begin(), e.end(), edges);
    });
}

// Evidence model of BASELINE.json configs: per slot l,
//   y = sum_k onehot(c_kl)*[not erased] + onehot(false candidate)*[p_false] + sigma*N(0,1),
//   S_l = log_softmax(y),  sigma = 10^(-snr/20).
// Draw order per bin (after sample_codewords on the same stream): for l: for k: one U(0,1)
// for the erasure; then one U(0,1) for the false candidate and, if it fires, one symbol;
// then Q normals.
int cider_workload_bins(const cider_workload_desc* w, const int32_t* edges, int64_t first, int n,
                        int32_t* truth, float* S, int threads) {
    return guard([&] {
        Gf gf(w->m, 0);
        const int L = w->slots, P = w->checks, K = w->k, Q = gf.q;
        cider_code_desc cd{P, L, L * w->col_weight, edges};
        Tanner t(&cd, Q);
        Systematic sys = systematic_form(gf, t);
        if (K < 1) throw InvalidInput("sample_codewords: need K >= 1");
        const double sigma = std::pow(10.0, -w->snr_db / 20.0);
        parallel(n, threads, [&](int i) {
            std::mt19937_64 rng(derive_seed(w->master_seed, uint64_t(16 + first + i)));
            std::vector<int32_t> cw(size_t(K) * L);
            codewords(gf, sys, L, K, rng, cw.data());
            if (truth) std::copy(cw.begin(), cw.end(), truth + size_t(i) * K * L);
            std::uniform_real_distribution<double> uni(0.0, 1.0);
            std::normal_distribution<double> nrm(0.0, 1.0);
            std::uniform_int_distribution<int> sym(0, Q - 1);
            std::vector<double> y(Q);
            for (int l = 0; l < L; ++l) {
                std::fill(y.begin(), y.end(), 0.0);
                for (int k = 0; k < K; ++k) {
                    bool erased = uni(rng) < w->p_erase;
                    if (!erased) y[cw[size_t(k) * L + l]] += 1.0;
                }
                if (uni(rng) < w->p_false) y[sym(rng)] += 1.0;
                for (int a = 0; a < Q; ++a) y[a] += sigma * nrm(rng);
                double mx = y[0];
                for (int a = 1; a < Q; ++a) mx = std::max(mx, y[a]);
                double se = 0.0;
                for (int a = 0; a < Q; ++a) se += std::exp(y[a] - mx);
                double lse = mx + std::log(se);
                if (S)
                    for (int a = 0; a < Q; ++a) S[(size_t(i) * L + l) * Q + a] = float(y[a] - lse);
            }
        });
    });
}

// Parity-check file (ldpc.cpp:197-226): header "P L Q col_weight prim_poly seed",
// then one "check slot coeff" line per edge; load validates like ParityCheckMatrix (ldpc.cpp:11-30).
int cider_save_parity_file(const char* path, const cider_code_desc* code, int q, int col_weight, uint32_t prim_poly,
                           uint64_t seed) {
    return guard([&] {
        Tanner t(code, q); // validates and sorts (check, slot) like the reference's constructor
        std::ofstream out(path);
        if (!out) throw std::runtime_error(std::string("save_parity_file: cannot open ") + path);
        out << t.checks << ' ' << t.slots << ' ' << q << ' ' << col_weight << ' ' << prim_poly << ' ' << seed << '\n';
        for (int e = 0; e < t.n_edges(); ++e) out << t.chk[e] << ' ' << t.slot[e] << ' ' << t.coef[e] << '\n';
        if (!out) throw std::runtime_error(std::string("save_parity_file: write failed for ") + path);
    });
}

int cider_load_parity_file(const char* path, int max_edges, int32_t* edges, int* n_edges, int* checks, int* slots, int* q,
                           int* col_weight, uint32_t* prim_poly, uint64_t* seed) {
    return guard([&] {
        std::ifstream in(path);
        if (!in) throw std::runtime_error(std::string("load_parity_file: cannot open ") + path);
        int p = 0, l = 0, qq = 0, w = 0;
        uint32_t poly = 0;
        uint64_t sd = 0;
        if (!(in >> p >> l >> qq >> w >> poly >> sd))
            throw std::runtime_error(std::string("load_parity_file: malformed header in ") + path);
        std::vector<int32_t> e;
        int a, b, c;
        while (in >> a >> b >> c) e.insert(e.end(), {a, b, c});
        if (!in.eof()) throw std::runtime_error(std::string("load_parity_file: malformed entry line in ") + path);
        cider_code_desc cd{p, l, int(e.size() / 3), e.data()};
        try {
            Tanner t(&cd, qq);
            if (t.n_edges() > max_edges) throw std::runtime_error("load_parity_file: edge buffer too small");
            for (int i = 0; i < t.n_edges(); ++i) {
                edges[3 * i] = t.chk[i];
                edges[3 * i + 1] = t.slot[i];
                edges[3 * i + 2] = t.coef[i];
            }
            *n_edges = t.n_edges();
        } catch (const InvalidInput& err) {
            throw std::runtime_error(std::string("load_parity_file: invalid matrix in ") + path + ": " + err.what());
        }
        *checks = p;
        *slots = l;
        *q = qq;
        *col_weight = w;
        *prim_poly = poly;
        *seed = sd;
    });
}

int cider_ser_cer(int n, int K, int L, const int32_t* truth, const int32_t* pred, double* ser_sum,
                  double* cer_sum) {
    return guard([&] {
        if (K < 1 || K > 16 || L < 1) throw InvalidInput("ser_cer: unsupported shape");
        double ser = 0.0, cer = 0.0;
        std::vector<int> cost(K * K), perm;
        for (int b = 0; b < n; ++b) {
            const int32_t* t = truth + size_t(b) * K * L;
            const int32_t* p = pred + size_t(b) * K * L;
            for (int i = 0; i < K; ++i)
                for (int j = 0; j < K; ++j) {
                    int d = 0;
                    for (int c = 0; c < L; ++c) d += p[i * L + c] != t[j * L + c];
                    cost[i * K + j] = d;
                }
            int total = 0;
            assignment(K, cost, perm, total);
            int bad = 0;
            for (int i = 0; i < K; ++i) bad += cost[i * K + perm[i]] > 0;
            ser += double(total) / (double(K) * L);
            cer += double(bad) / K;
        }
        *ser_sum = ser;
        *cer_sum = cer;
    });
}

} // extern "C"
