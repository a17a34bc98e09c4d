// ref_cli_shim.cpp — TEST INFRASTRUCTURE ONLY: the reference's dataset format and `uradec`'s
// simulate / decode steps, composed from the reference's own library (dataset.cpp compiled against
// nlohmann/json 3.11.3 — the header the reference vendors but does not ship; oracle/Makefile takes
// the copy in the image's cudnn_frontend include tree). The CLI itself (tools/uradec.cpp) needs
// CLI11, which is absent, so its cmd_simulate (uradec.cpp:496-517) and cmd_decode / RefineDecoder /
// SicBpDecoder / run_decoder_over_frames / write_decode_row (uradec.cpp:122-341, 519-547) are
// restated here as calls into the reference library, to produce the reference's dataset files and
// CSV rows for tests/test_dataset.py. Nothing here is on the product path.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ura/amp.hpp"
#include "ura/bp.hpp"
#include "ura/dataset.hpp"
#include "ura/denoiser.hpp"
#include "ura/ldpc.hpp"
#include "ura/metrics.hpp"
#include "ura/parallel.hpp"
#include "ura/refine.hpp"
#include "ura/seeding.hpp"
#include "ura/sim.hpp"

#include "cider.h"

namespace {
thread_local std::string g_cli_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::domain_error& e) {
        g_cli_err = e.what();
        return CIDER_EINVAL;
    } catch (const std::exception& e) {
        g_cli_err = e.what();
        return CIDER_ERUNTIME;
    }
}

ura::RunConfig to_cfg(const cider_run_config& c) {
    ura::RunConfig r;
    r.scale = c.scale;
    r.q = c.q; r.l = c.l; r.p = c.p; r.col_weight = c.col_weight; r.k = c.k; r.n_s = c.n_s;
    r.eb_db = c.eb_db; r.noise_var = c.noise_var; r.amp_iters = c.amp_iters; r.rho_bg = c.rho_bg;
    r.sigma_u2 = c.sigma_u2; r.evidence_floor = c.evidence_floor; r.seed = c.seed; r.frames = c.frames;
    return r;
}

void put_str(const std::string& s, char* out, int cap) {
    if (int(s.size()) >= cap) throw std::runtime_error("ref_cli: output buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
}
} // namespace

extern "C" {

const char* refcli_last_error(void) { return g_cli_err.c_str(); }

int refcli_config_to_json(const cider_run_config* c, char* out, int cap) {
    return guarded([&] { put_str(ura::config_to_json(to_cfg(*c)), out, cap); });
}
int refcli_config_fingerprint(const cider_run_config* c, char* out, int cap) {
    return guarded([&] { put_str(ura::config_fingerprint(to_cfg(*c)), out, cap); });
}
int refcli_format_double(double x, char* out, int cap) {
    return guarded([&] { put_str(ura::format_double(x), out, cap); });
}
// nlohmann's dump of one double (the number layout config_to_json uses)
int refcli_json_double(double x, char* out, int cap) {
    return guarded([&] {
        cider_run_config c{};
        std::strcpy(c.scale, "x");
        c.eb_db = x;
        const std::string j = ura::config_to_json(to_cfg(c));
        const size_t a = j.find("\"eb_db\":") + 8, b = j.find(',', a);
        put_str(j.substr(a, b - a), out, cap);
    });
}

// cmd_simulate (uradec.cpp:496-517): build_code, save_parity_file, frames through generate_frame +
// detect_frame, write_dataset
int refcli_simulate(const cider_run_config* c, const char* dataset_path, const char* hfile) {
    return guarded([&] {
        ura::RunConfig cfg = to_cfg(*c);
        ura::GfContext gf = ura::GfContext::with_default_poly(cfg.field_degree());
        auto rng = ura::make_rng(ura::derive_seed(cfg.seed, 1));
        ura::ParityCheckMatrix h = ura::build_random_ldpc(gf, cfg.l, cfg.p, cfg.col_weight, rng);
        ura::GeneratorForm gen = ura::derive_generator(gf, h);
        auto dicts = ura::make_dictionaries(cfg.q, cfg.n_s, cfg.l, ura::derive_seed(cfg.seed, 2));
        ura::save_parity_file(hfile, h, ura::LdpcFileMeta{cfg.col_weight, gf.prim_poly(), cfg.seed});
        ura::FrameConfig fc = cfg.frame_config();
        ura::AmpConfig amp = cfg.amp_config();
        const double snr = ura::snr_db(cfg.eb_db, cfg.l, cfg.n_s, cfg.payload_bits());
        std::vector<ura::DatasetFrame> frames(cfg.frames);
        ura::parallel_for(cfg.frames, [&](int i) {
            auto frame = ura::generate_frame(fc, gf, gen, dicts, ura::derive_seed(cfg.seed, 16 + i));
            ura::DatasetFrame df;
            df.seed = frame.seed;
            df.truth = std::move(frame.truth);
            df.evidence = ura::detect_frame(frame.observations, dicts, amp);
            df.snr_db = snr;
            frames[i] = std::move(df);
        });
        ura::write_dataset(dataset_path, cfg, ura::file_fingerprint(hfile), frames);
    });
}

// load_dataset's view of a file: header fields + frames (for the reader's round-trip test)
int refcli_load(const char* path, cider_run_config* c, char* fp, char* hfp, int* n, int cap, uint64_t* seeds, int32_t* truth,
                double* evidence, double* snr) {
    return guarded([&] {
        ura::Dataset ds = ura::load_dataset(path);
        const ura::RunConfig& r = ds.config;
        std::memset(c, 0, sizeof(*c));
        std::snprintf(c->scale, sizeof(c->scale), "%s", r.scale.c_str());
        c->q = r.q; c->l = r.l; c->p = r.p; c->col_weight = r.col_weight; c->k = r.k; c->n_s = r.n_s;
        c->eb_db = r.eb_db; c->noise_var = r.noise_var; c->amp_iters = r.amp_iters; c->rho_bg = r.rho_bg;
        c->sigma_u2 = r.sigma_u2; c->evidence_floor = r.evidence_floor; c->seed = r.seed; c->frames = r.frames;
        put_str(ds.fingerprint, fp, 17);
        put_str(ds.h_fingerprint, hfp, 17);
        *n = int(ds.frames.size());
        for (int i = 0; i < std::min(cap, *n); ++i) {
            const auto& f = ds.frames[i];
            seeds[i] = f.seed;
            snr[i] = f.snr_db;
            std::copy(f.truth.v.begin(), f.truth.v.end(), truth + size_t(i) * r.k * r.l);
            std::copy(f.evidence.v.begin(), f.evidence.v.end(), evidence + size_t(i) * r.l * r.q);
        }
    });
}

// cmd_decode's CSV row (uradec.cpp:519-547) for refine-structured (scorer maxprob | oracle) or sic-bp,
// decoded by the reference library; f32 != 0 rounds the evidence and the denoiser parameters to fp32
// first (the inputs the device's FP32 mode computes with). ms_per_sample is written as 0.
int refcli_decode_row(const char* dataset_path, const char* hfile, const char* decoder, const char* scorer, int steps,
                      const double* thresholds, int n_thr, int latent_dim, uint64_t param_seed, int f32, char* out, int cap) {
    return guarded([&] {
        ura::Dataset ds = ura::load_dataset(dataset_path);
        ura::LdpcFileMeta meta;
        ura::ParityCheckMatrix h = ura::load_parity_file(hfile, &meta);
        const ura::RunConfig& cfg = ds.config;
        if (h.slots() != cfg.l || h.checks() != cfg.p || h.q() != cfg.q)
            throw std::runtime_error("parity file dimensions disagree with the dataset config");
        if (!ds.h_fingerprint.empty() && ura::file_fingerprint(hfile) != ds.h_fingerprint)
            throw std::runtime_error("parity file fingerprint disagrees with the dataset header");
        ura::GfContext gf(cfg.field_degree(), meta.prim_poly);
        const int n = int(ds.frames.size()), K = cfg.k, L = cfg.l;
        if (f32)
            for (auto& f : ds.frames)
                for (double& x : f.evidence.v) x = double(float(x));
        const std::string dec(decoder);
        std::vector<ura::SymbolGrid> grids(n);
        std::vector<int> conv(n, 1), iters(n, 0), first(n, 0), stages(n, 0), rows(n, 0), trm(n, 0);
        if (dec == "sic-bp") {
            ura::BpConfig bc;
            ura::parallel_for(n, [&](int i) {
                auto r = ura::sic_decode(ds.frames[i].evidence, gf, h, K, bc);
                grids[i] = r.grid;
                for (const auto& st : r.stages) {
                    conv[i] = conv[i] && st.converged;
                    iters[i] += st.iters_used;
                }
            });
        } else {
            auto params = ura::DenoiserParams::random_init(gf.q(), latent_dim, param_seed);
            if (f32) {
                auto rd = [](std::vector<double>& v) { for (double& x : v) x = double(float(x)); };
                rd(params.embed); rd(params.out_proj); rd(params.sym_embed);
                for (auto* t : {&params.gate_a, &params.check_agg, &params.fuse_b}) { rd(t->w1); rd(t->b1); rd(t->w2); rd(t->b2); }
            }
            ura::StructuredDenoiser den(gf, params);
            ura::RevealSchedule sched;
            sched.steps = steps > 0 ? steps : ura::default_steps_for_load(K);
            ura::RemaskConfig rm;
            rm.thresholds.assign(thresholds, thresholds + n_thr);
            ura::validate_remask_config(rm);
            const std::string sc(scorer);
            ura::parallel_for(n, [&](int i) {
                std::unique_ptr<ura::ConfidenceScorer> s;
                if (sc == "oracle") s = std::make_unique<ura::OracleRowScorer>(ds.frames[i].truth);
                else s = std::make_unique<ura::MaxProbScorer>();
                ura::RefineTrace tr;
                grids[i] = rm.thresholds.empty()
                               ? ura::run_refinement(den, ds.frames[i].evidence, h, sched, K, L, &tr)
                               : ura::run_with_remasking(den, *s, ds.frames[i].evidence, h, sched, rm, K, L, &tr);
                first[i] = tr.pass_first_reveals.empty() ? 0 : tr.pass_first_reveals.front();
                stages[i] = int(tr.remask_rows_per_stage.size());
                for (int r : tr.remask_rows_per_stage) rows[i] += r;
                for (int t : tr.remask_steps_per_stage) trm[i] += t;
            });
        }
        double ser = 0, cer = 0, cv = 0, it = 0, fr = 0, stg = 0, rw = 0, tm = 0;
        for (int i = 0; i < n; ++i) {
            auto m = ura::ser_cer(ds.frames[i].truth, grids[i]);
            ser += m.ser; cer += m.cer; cv += conv[i]; it += iters[i];
            fr += first[i]; stg += stages[i]; rw += rows[i]; tm += trm[i];
        }
        if (n > 0) { ser /= n; cer /= n; cv /= n; it /= n; }
        const bool bp = dec == "sic-bp";
        std::ostringstream os;
        const double snr = ura::snr_db(cfg.eb_db, cfg.l, cfg.n_s, cfg.payload_bits());
        os << dec << ",wht," << cfg.scale << ',' << cfg.q << ',' << cfg.l << ',' << cfg.p << ',' << cfg.k << ','
           << ura::format_double(cfg.eb_db) << ',' << ura::format_double(snr) << ',' << cfg.seed << ',' << n << ','
           << ura::format_double(ser) << ',' << ura::format_double(cer) << ",0,";
        if (bp) os << ura::format_double(cv) << ',' << ura::format_double(it);
        else os << ',';
        os << ',';
        if (!bp && n > 0)
            os << "first_reveal=" << ura::format_double(fr / n) << ";remask_stages=" << ura::format_double(stg / n)
               << ";remask_rows=" << ura::format_double(rw / n) << ";t_rm=" << ura::format_double(tm / n);
        os << ",ok," << ura::config_fingerprint(cfg);
        put_str(os.str(), out, cap);
    });
}

} // extern "C"
