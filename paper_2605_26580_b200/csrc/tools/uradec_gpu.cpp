// uradec_gpu.cpp — `uradec decode` on the B200: the reference CLI's decode
// subcommand (uradec.cpp:519-547) for its refine-structured and sic-bp decoders, over the C ABI of
// libcider only. Reads the reference's JSON Lines dataset (cider_dataset_load) and parity file
// (cider_load_parity_file), decodes every frame on the device in one batch, and writes the same CSV:
// the "# uradec 0.1.0" / "# config: ..." preamble, the decode header and one row with identical
// columns (ms_per_sample is this tool's own per-frame device time).
//
//   uradec-gpu decode --dataset D.jsonl --hfile H.txt --decoder refine-structured|sic-bp
//       [--steps N --tau-max X --tau-min X --no-first-reveal --remask-thresholds a,b,...
//        --scorer maxprob|oracle --param-seed S --latent-dim D --backend wht --bp-iters N
//        --no-early-exit --precision fp32|bf16 --device I --out F --per-frame F]
//
// refine-structured = RefineDecoder (uradec.cpp:170-224): DenoiserParams::random_init(q, latent_dim,
// param_seed) (cider_weights_init, ref-exact model), per-load steps unless --steps, MaxProb or oracle
// (truth-row) scorer driving the remask stages. sic-bp = SicBpDecoder (uradec.cpp:122-145).
// Exit codes as uradec (uradec.cpp:817-829): 2 usage, 3 bad input (CIDER_EINVAL), 4 runtime failure.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cider.h"

namespace {

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(int rc) {
    if (rc != CIDER_OK) throw Fail(rc == CIDER_EINVAL ? 3 : 4, cider_last_error());
}
// load_and_check wraps every dataset / parity-file failure as a DataError (exit 3, uradec.cpp:466-485)
void ck_data(int rc) {
    if (rc != CIDER_OK) throw Fail(3, cider_last_error());
}

std::string fmt(double x) { // format_double (dataset.cpp:57-61)
    char b[64];
    ck(cider_format_double(x, b, sizeof(b)));
    return b;
}

int default_steps_for_load(int k) { // refine.cpp:28-40
    switch (k) {
        case 2: return 12;
        case 3: return 24;
        case 4: return 42;
        case 5: return 60;
        case 6: return 50;
        case 7: return 62;
        case 8: return 74;
        default: return k <= 1 ? 12 : 74;
    }
}

struct Opts {
    std::string dataset, hfile, decoder = "sic-bp", backend = "wht", scorer = "maxprob", out, per_frame, precision = "fp32";
    int bp_iters = 50, steps = 0, latent_dim = 128, device = 0;
    bool early_exit = true, first_reveal = true;
    double tau_max = 1.0, tau_min = 1.0;
    std::vector<double> thresholds;
    uint64_t param_seed = 1;
};

Opts parse(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "decode") throw Fail(2, "usage: uradec-gpu decode --dataset D --hfile H [options]");
    Opts o;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw Fail(2, a + " needs a value");
            return argv[++i];
        };
        if (a == "--dataset") o.dataset = val();
        else if (a == "--hfile") o.hfile = val();
        else if (a == "--decoder") o.decoder = val();
        else if (a == "--backend") o.backend = val();
        else if (a == "--bp-iters") o.bp_iters = std::stoi(val());
        else if (a == "--no-early-exit") o.early_exit = false;
        else if (a == "--steps") o.steps = std::stoi(val());
        else if (a == "--tau-max") o.tau_max = std::stod(val());
        else if (a == "--tau-min") o.tau_min = std::stod(val());
        else if (a == "--no-first-reveal") o.first_reveal = false;
        else if (a == "--remask-thresholds") {
            std::stringstream ss(val());
            std::string t;
            while (std::getline(ss, t, ',')) o.thresholds.push_back(std::stod(t));
        } else if (a == "--scorer") o.scorer = val();
        else if (a == "--param-seed") o.param_seed = std::stoull(val());
        else if (a == "--latent-dim") o.latent_dim = std::stoi(val());
        else if (a == "--precision") o.precision = val();
        else if (a == "--device") o.device = std::stoi(val());
        else if (a == "--out") o.out = val();
        else if (a == "--per-frame") o.per_frame = val();
        else throw Fail(2, "unknown option " + a);
    }
    if (o.dataset.empty() || o.hfile.empty()) throw Fail(2, "--dataset and --hfile are required");
    return o;
}

double snr_db(double eb_db, int slots, int n_s, int payload_bits) { // sim.cpp:70-72
    return eb_db - 10.0 * std::log10(static_cast<double>(slots) * n_s / payload_bits);
}

int field_degree(int q) {
    for (int m = 1; m <= 8; ++m)
        if ((1 << m) == q) return m;
    throw Fail(3, "RunConfig: Q must be a power of two in 2..256");
}

struct FrameOut {
    std::vector<int32_t> grid;
    bool converged = true;
    int iters = 0, first_reveal = 0, stages = 0, rows = 0, trm = 0;
};

int run(const Opts& o) {
    // ---- load_and_check (uradec.cpp:465-494) ----
    cider_run_config cfg{};
    char fp[17] = {0}, hfp[17] = {0};
    int n = 0;
    ck_data(cider_dataset_load(o.dataset.c_str(), &cfg, fp, hfp, &n, 0, nullptr, nullptr, nullptr, nullptr));
    const int K = cfg.k, L = cfg.l, Q = cfg.q;
    std::vector<uint64_t> seeds(n);
    std::vector<int32_t> truth(size_t(n) * K * L);
    std::vector<double> ev(size_t(n) * L * Q), snr(n);
    ck_data(cider_dataset_load(o.dataset.c_str(), &cfg, fp, hfp, &n, n, seeds.data(), truth.data(), ev.data(), snr.data()));
    std::vector<int32_t> edges(size_t(1) << 20);
    int ne = 0, hp = 0, hl = 0, hq = 0, cw = 0;
    uint32_t poly = 0;
    uint64_t hseed = 0;
    ck_data(cider_load_parity_file(o.hfile.c_str(), int(edges.size() / 3), edges.data(), &ne, &hp, &hl, &hq, &cw, &poly, &hseed));
    if (hl != cfg.l || hp != cfg.p || hq != cfg.q) throw Fail(3, "parity file dimensions disagree with the dataset config");
    if (hfp[0]) {
        char f2[17];
        ck_data(cider_file_fingerprint(o.hfile.c_str(), f2));
        if (std::string(f2) != hfp) throw Fail(3, "parity file fingerprint disagrees with the dataset header");
    }
    const int m = field_degree(Q);
    cider_code_desc code{hp, hl, ne, edges.data()};

    // ---- decode every frame (one device batch) ----
    std::vector<FrameOut> res(n);
    double ms_total = 0.0;
    if (o.decoder == "sic-bp") {
        if (o.backend != "wht") throw Fail(3, "the device BP decoder implements the wht backend");
        cider_bp_ctx* bp = nullptr;
        ck(cider_bp_create(m, poly, &code, o.device, &bp));
        cider_bp_config bc{o.bp_iters, 1e-30, o.early_exit ? 1 : 0};
        std::vector<int32_t> grid(size_t(n) * K * L), sc(size_t(n) * K), si(size_t(n) * K);
        auto t0 = std::chrono::steady_clock::now();
        const int rc = cider_sic_decode(bp, n, K, ev.data(), &bc, std::nan(""), grid.data(), sc.data(), si.data());
        ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        cider_bp_destroy(bp);
        ck(rc);
        for (int i = 0; i < n; ++i) {
            res[i].grid.assign(grid.begin() + size_t(i) * K * L, grid.begin() + size_t(i + 1) * K * L);
            for (int s = 0; s < K; ++s) {
                res[i].converged = res[i].converged && sc[size_t(i) * K + s];
                res[i].iters += si[size_t(i) * K + s];
            }
        }
    } else if (o.decoder == "refine-structured") {
        if (o.scorer != "maxprob" && o.scorer != "oracle") throw Fail(3, "unknown scorer: " + o.scorer);
        cider_model_desc md{};
        md.m = m;
        md.prim_poly = poly;
        md.dim = o.latent_dim;
        md.hidden = o.latent_dim;
        md.layers = 1;
        md.heads = 0;
        md.tau_demix = 1.0;
        md.evidence_scale = 1.0;
        md.precision = o.precision == "bf16" ? CIDER_BF16 : CIDER_FP32;
        std::vector<float> w(cider_weights_count(&md));
        ck(cider_weights_init(&md, o.param_seed, w.data()));
        cider_ctx* ctx = nullptr;
        ck(cider_create(&md, w.data(), &code, o.device, &ctx));
        cider_schedule sc{o.steps > 0 ? o.steps : default_steps_for_load(K), o.tau_max, o.tau_min, o.first_reveal ? 1 : 0};
        std::vector<float> S(ev.begin(), ev.end());
        std::vector<int32_t> grid(size_t(n) * K * L), first(n), rows(size_t(n) * CIDER_MAX_THRESHOLDS),
            stp(size_t(n) * CIDER_MAX_THRESHOLDS);
        cider_trace tr{};
        tr.first_reveals = first.data();
        tr.remask_rows = rows.data();
        tr.remask_steps = stp.data();
        auto t0 = std::chrono::steady_clock::now();
        try {
            if (o.scorer == "maxprob" || o.thresholds.empty()) {
                // MaxProbScorer stages on the device (run_with_remasking, refine.cpp:277-292)
                cider_remask rm{};
                rm.mode = o.thresholds.empty() ? CIDER_REMASK_NONE : CIDER_REMASK_THRESHOLD;
                if (o.thresholds.size() > CIDER_MAX_THRESHOLDS) throw Fail(3, "remask: too many thresholds");
                rm.n_thresholds = int(o.thresholds.size());
                for (size_t i = 0; i < o.thresholds.size(); ++i) rm.thresholds[i] = o.thresholds[i];
                ck(cider_refine(ctx, n, K, S.data(), &sc, &rm, grid.data(), nullptr, &tr));
                for (int i = 0; i < n; ++i)
                    for (int s = 0; s < CIDER_MAX_THRESHOLDS; ++s)
                        if (rows[size_t(i) * CIDER_MAX_THRESHOLDS + s]) {
                            ++res[i].stages;
                            res[i].rows += rows[size_t(i) * CIDER_MAX_THRESHOLDS + s];
                            res[i].trm += stp[size_t(i) * CIDER_MAX_THRESHOLDS + s];
                        }
            } else {
                // OracleRowScorer (refine.cpp:227-236): 1 for a row equal to the truth row, else 0; the
                // stage loop of run_with_remasking on the host, each pass on the device (cider_remask_pass)
                cider_remask none{};
                ck(cider_refine(ctx, n, K, S.data(), &sc, &none, grid.data(), nullptr, &tr));
                double prev = 1.0;
                for (double t : o.thresholds) {
                    if (t <= 0.0 || t >= 1.0) throw Fail(3, "remask thresholds must lie in (0,1)");
                    if (t >= prev) throw Fail(3, "remask thresholds must be strictly descending");
                    prev = t;
                }
                std::vector<char> live(n, 1);
                for (double t : o.thresholds) {
                    std::vector<int> idx;
                    std::vector<double> conf;
                    for (int i = 0; i < n; ++i) {
                        if (!live[i]) continue;
                        std::vector<double> c(K);
                        bool any = false;
                        for (int k = 0; k < K; ++k) {
                            bool ok = true;
                            for (int l = 0; l < L; ++l)
                                ok = ok && grid[(size_t(i) * K + k) * L + l] == truth[(size_t(i) * K + k) * L + l];
                            c[k] = ok ? 1.0 : 0.0;
                            any = any || c[k] < t;
                        }
                        if (!any) { live[i] = 0; continue; } // the reference's break for this frame
                        idx.push_back(i);
                        conf.insert(conf.end(), c.begin(), c.end());
                    }
                    if (idx.empty()) break;
                    const int B = int(idx.size());
                    std::vector<float> Sb(size_t(B) * L * Q);
                    std::vector<int32_t> gin(size_t(B) * K * L), gout(gin.size()), f1(B), r1(size_t(B) * CIDER_MAX_THRESHOLDS),
                        s1(size_t(B) * CIDER_MAX_THRESHOLDS);
                    for (int j = 0; j < B; ++j) {
                        std::copy(S.begin() + size_t(idx[j]) * L * Q, S.begin() + size_t(idx[j] + 1) * L * Q, Sb.begin() + size_t(j) * L * Q);
                        std::copy(grid.begin() + size_t(idx[j]) * K * L, grid.begin() + size_t(idx[j] + 1) * K * L, gin.begin() + size_t(j) * K * L);
                    }
                    cider_trace t1{};
                    t1.first_reveals = f1.data();
                    t1.remask_rows = r1.data();
                    t1.remask_steps = s1.data();
                    ck(cider_remask_pass(ctx, B, K, Sb.data(), &sc, gin.data(), conf.data(), t, gout.data(), nullptr, &t1));
                    for (int j = 0; j < B; ++j) {
                        std::copy(gout.begin() + size_t(j) * K * L, gout.begin() + size_t(j + 1) * K * L, grid.begin() + size_t(idx[j]) * K * L);
                        ++res[idx[j]].stages;
                        res[idx[j]].rows += r1[size_t(j) * CIDER_MAX_THRESHOLDS];
                        res[idx[j]].trm += s1[size_t(j) * CIDER_MAX_THRESHOLDS];
                    }
                }
            }
        } catch (...) {
            cider_destroy(ctx);
            throw;
        }
        ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        cider_destroy(ctx);
        for (int i = 0; i < n; ++i) {
            res[i].grid.assign(grid.begin() + size_t(i) * K * L, grid.begin() + size_t(i + 1) * K * L);
            res[i].first_reveal = first[i];
        }
    } else {
        throw Fail(3, "unknown decoder: " + o.decoder);
    }

    // ---- run_decoder_over_frames + write_decode_row (uradec.cpp:255-341) ----
    char cj[1024];
    ck(cider_config_to_json(&cfg, cj, sizeof(cj)));
    std::ofstream fout;
    if (!o.out.empty()) {
        fout.open(o.out);
        if (!fout) throw Fail(4, "cannot open output file " + o.out);
    }
    std::ostream& os = o.out.empty() ? std::cout : fout;
    auto preamble = [&](std::ostream& s) { s << "# uradec 0.1.0\n# config: " << cj << "\n"; };
    preamble(os);
    os << "decoder,backend,scale,q,l,p,k,eb_db,snr_db,seed,samples,ser,cer,ms_per_sample,converged_frac,mean_iters,"
          "telemetry,status,config_fp\n";
    const double per_ms = n ? ms_total / n : 0.0;
    if (!o.per_frame.empty()) {
        std::ofstream pf(o.per_frame);
        if (!pf) throw Fail(4, "cannot open per-frame output " + o.per_frame);
        preamble(pf);
        pf << "frame,seed,ser,cer,ms,converged,iters\n";
        for (int i = 0; i < n; ++i) {
            double s = 0, c = 0;
            ck(cider_ser_cer(1, K, L, truth.data() + size_t(i) * K * L, res[i].grid.data(), &s, &c));
            pf << i << ',' << seeds[i] << ',' << fmt(s) << ',' << fmt(c) << ',' << fmt(per_ms) << ','
               << (res[i].converged ? 1 : 0) << ',' << res[i].iters << "\n";
        }
    }
    double ser = 0, cer = 0, conv = 0, iters = 0, fr = 0, stg = 0, rws = 0, trm = 0;
    for (int i = 0; i < n; ++i) {
        double s = 0, c = 0;
        ck(cider_ser_cer(1, K, L, truth.data() + size_t(i) * K * L, res[i].grid.data(), &s, &c));
        ser += s;
        cer += c;
        conv += res[i].converged;
        iters += res[i].iters;
        fr += res[i].first_reveal;
        stg += res[i].stages;
        rws += res[i].rows;
        trm += res[i].trm;
    }
    if (n > 0) {
        ser /= n;
        cer /= n;
        conv /= n;
        iters /= n;
    }
    const bool bp = o.decoder == "sic-bp";
    std::string tel;
    if (!bp && n > 0)
        tel = "first_reveal=" + fmt(fr / n) + ";remask_stages=" + fmt(stg / n) + ";remask_rows=" + fmt(rws / n) + ";t_rm=" +
              fmt(trm / n);
    const int payload = field_degree(Q) * (cfg.l - cfg.p);
    os << o.decoder << ',' << o.backend << ',' << cfg.scale << ',' << cfg.q << ',' << cfg.l << ',' << cfg.p << ',' << cfg.k
       << ',' << fmt(cfg.eb_db) << ',' << fmt(snr_db(cfg.eb_db, cfg.l, cfg.n_s, payload)) << ',' << cfg.seed << ',' << n
       << ',' << fmt(ser) << ',' << fmt(cer) << ',' << fmt(per_ms) << ',';
    if (bp) os << fmt(conv) << ',' << fmt(iters);
    else os << ',';
    os << ',' << tel << ",ok," << fp << "\n";
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    try {
        return run(parse(argc, argv));
    } catch (const Fail& f) {
        std::cerr << (f.code == 2 ? "usage error: " : f.code == 3 ? "validation error: " : "runtime failure: ") << f.what() << "\n";
        return f.code;
    } catch (const std::invalid_argument& e) {
        std::cerr << "usage error: bad option value (" << e.what() << ")\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "runtime failure: " << e.what() << "\n";
        return 4;
    }
}
