// adapter_test.cpp — TEST PROGRAM: the reference's own engine driving the B200 denoiser.
//
// Built by oracle/Makefile (only where /root/reference exists) against the reference objects in
// oracle/_ref/obj and libcider.so; the binary travels to the GPU box in oracle/_ref/ and is run by
// tests/test_gpu.py::test_reference_engine_with_gpu_denoiser. It checks the drop-in boundary:
//   (1) ura::run_refinement + ura::StructuredDenoiser        (the reference, CPU, fp64)
//   (2) ura::run_refinement + cider::GpuStructuredDenoiser   (reference loop, B200 forward)
//   (3) cider::GpuRefiner::run_refinement                    (whole loop on the B200)
//   (4) ura::run_with_remasking vs GpuRefiner::run_with_remasking, and a BinDecoder call
//   (5) ura::sic_decode vs cider::GpuBp::sic_decode (FFT-BP, WHT backend), and a SIC BinDecoder
//   (6) RefineTrace (reveal_counts, first_step_sites, pass_first_reveals, remask stages) and
//       run_with_remasking with a pluggable ConfidenceScorer (ura::OracleRowScorer) vs the reference
//   (7) ura::run_protocol / run_protocol_frame (protocol.cpp:41-113) with a CPU decoder bank vs the
//       request-coalescing GPU bank: identical per-bin grids and identical frame SER / CER
// on fp32-rounded parameters and evidence (FP32 mode), and requires identical grids.
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>

#include <map>
#include <mutex>

#include "cider_ura.hpp"
#include "ura/ldpc.hpp"
#include "ura/metrics.hpp"
#include "ura/protocol.hpp"
#include "ura/seeding.hpp"

static void round_f32(std::vector<double>& v) {
    for (double& x : v) x = double(float(x));
}

int main() {
    int fails = 0;
    try {
        auto gf = ura::GfContext::with_default_poly(6);
        auto rng = ura::make_rng(ura::derive_seed(0, 1));
        auto h = ura::build_random_ldpc(gf, 16, 8, 3, rng);
        auto p = ura::DenoiserParams::random_init(64, 32, 1);
        for (auto* v : {&p.embed, &p.out_proj, &p.sym_embed}) round_f32(*v);
        for (auto* t : {&p.gate_a, &p.check_agg, &p.fuse_b}) {
            round_f32(t->w1);
            round_f32(t->b1);
            round_f32(t->w2);
            round_f32(t->b2);
        }
        auto ctx = std::make_shared<cider::Context>(gf, p, h, 0, CIDER_FP32);
        ura::StructuredDenoiser cpu(gf, p);
        cider::GpuStructuredDenoiser gpu(ctx);
        cider::GpuRefiner refiner(ctx);
        ura::RevealSchedule sched;
        sched.steps = 5;
        int identical = 0, identical_loop = 0, identical_rm = 0;
        const int bins = 6;
        for (int b = 0; b < bins; ++b) {
            ura::EvidenceMatrix s(16, 64);
            auto er = ura::make_rng(ura::derive_seed(7, b));
            std::uniform_real_distribution<double> u(-8.0, 0.0);
            for (double& x : s.v) x = double(float(u(er)));
            const int k = 3;
            auto a = ura::run_refinement(cpu, s, h, sched, k, 16);
            auto g = ura::run_refinement(gpu, s, h, sched, k, 16);
            auto d = refiner.run_refinement(s, h, sched, k);
            identical += (a == g);
            identical_loop += (a == d);
            ura::RemaskConfig rm{{0.9, 0.5}};
            ura::MaxProbScorer scorer;
            auto ar = ura::run_with_remasking(cpu, scorer, s, h, sched, rm, k, 16);
            auto dr = refiner.run_with_remasking(s, h, sched, rm, k);
            identical_rm += (ar == dr);
        }
        std::printf("reference loop + GPU denoiser: %d/%d identical grids\n", identical, bins);
        std::printf("GPU loop vs reference:         %d/%d identical grids\n", identical_loop, bins);
        std::printf("GPU remasking vs reference:    %d/%d identical grids\n", identical_rm, bins);
        fails += identical != bins;
        fails += identical_loop != bins;
        fails += identical_rm != bins;
        // BinDecoder plug-in (protocol.hpp:40)
        auto dec = cider::make_bin_decoder(ctx, sched, false);
        ura::EvidenceMatrix s(16, 64, -1.0);
        ura::SymbolGrid truth(2, 16);
        ura::BinTask task{gf, h, s, truth, 2};
        auto out = dec(task);
        const bool shape_ok = out.rows == 2 && out.cols == 16;
        std::printf("BinDecoder call: %s\n", shape_ok ? "ok" : "FAILED");
        fails += !shape_ok;
        // (4b) ragged loads: one GpuRefiner::run_ragged call == per-bin BinDecoder calls (per-load defaults)
        {
            auto bank_dec = cider::make_bin_decoder(ctx);
            std::mt19937_64 r4(11);
            std::normal_distribution<double> nd(0.0, 1.0);
            std::vector<ura::EvidenceMatrix> ev(6, ura::EvidenceMatrix(16, 64));
            std::vector<const ura::EvidenceMatrix*> ptrs;
            const std::vector<int> loads{1, 2, 3, 3, 1, 2};
            for (auto& m : ev) {
                for (double& x : m.v) x = double(float(1.2 * nd(r4)));
                ptrs.push_back(&m);
            }
            auto rag = refiner.run_ragged(ptrs, loads, h, 3);
            int same = 0;
            for (size_t b = 0; b < ev.size(); ++b) {
                ura::SymbolGrid tk(loads[b], 16);
                auto one = bank_dec(ura::BinTask{gf, h, ev[b], tk, loads[b]});
                same += one.v == rag[b].v && one.rows == rag[b].rows;
            }
            std::printf("ragged batch vs per-bin decoder: %d/%d identical grids\n", same, int(ev.size()));
            fails += same != int(ev.size());
        }
        // (4c) request coalescing: 8 threads x 6 bins through one BinCoalescer == per-bin decoder
        {
            auto co = std::make_shared<cider::BinCoalescer>(ctx, 3);
            auto cdec = cider::make_coalescing_bin_decoder(co);
            auto pdec = cider::make_bin_decoder(ctx);
            const int T = 8, NB = 6;
            std::vector<ura::EvidenceMatrix> ev(T * NB, ura::EvidenceMatrix(16, 64));
            std::mt19937_64 r5(5);
            std::normal_distribution<double> nd(0.0, 1.0);
            for (auto& m : ev)
                for (double& x : m.v) x = double(float(1.2 * nd(r5)));
            std::vector<ura::SymbolGrid> got(T * NB, ura::SymbolGrid(1, 16));
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    for (int i = 0; i < NB; ++i) {
                        const int b = t * NB + i, load = 1 + b % 3;
                        ura::SymbolGrid tk(load, 16);
                        got[b] = cdec(ura::BinTask{gf, h, ev[b], tk, load});
                    }
                });
            for (auto& x : th) x.join();
            int same = 0;
            for (int b = 0; b < T * NB; ++b) {
                const int load = 1 + b % 3;
                ura::SymbolGrid tk(load, 16);
                auto one = pdec(ura::BinTask{gf, h, ev[b], tk, load});
                same += one.v == got[b].v && one.rows == got[b].rows;
            }
            std::printf("coalesced (8 threads, %lld device batches) vs per-bin decoder: %d/%d identical grids\n",
                        (long long)co->batches(), same, T * NB);
            fails += same != T * NB;
        }
        // (5) SIC-BP: ura::sic_decode vs cider::GpuBp (bp.hpp:72-93), same evidence, identical grids
        {
            cider::GpuBp gbp(gf, h);
            std::mt19937_64 r3(7);
            std::normal_distribution<double> nd(0.0, 1.0);
            ura::BpConfig bcfg;
            bcfg.max_iters = 20;
            std::vector<ura::EvidenceMatrix> ev(6, ura::EvidenceMatrix(16, 64));
            std::vector<const ura::EvidenceMatrix*> ptrs;
            for (auto& m : ev) {
                for (double& x : m.v) x = 1.5 * nd(r3);
                ptrs.push_back(&m);
            }
            auto gpu_res = gbp.sic_decode_batch(ptrs, 2, bcfg);
            int same = 0;
            for (size_t b = 0; b < ev.size(); ++b) {
                auto ref_res = ura::sic_decode(ev[b], gf, h, 2, bcfg);
                bool ok = ref_res.grid.v == gpu_res[b].grid.v;
                for (int st = 0; st < 2; ++st)
                    ok = ok && ref_res.stages[st].converged == gpu_res[b].stages[st].converged &&
                         ref_res.stages[st].iters_used == gpu_res[b].stages[st].iters_used;
                same += ok;
            }
            std::printf("GPU SIC-BP vs reference:       %d/%d identical grids + stage stats\n", same, int(ev.size()));
            fails += same != int(ev.size());
            auto sdec = cider::make_sic_bin_decoder(std::make_shared<cider::GpuBp>(gf, h), bcfg);
            ura::BinTask t2{gf, h, ev[0], truth, 2};
            const bool sic_ok = sdec(t2).v == gpu_res[0].grid.v;
            std::printf("SIC BinDecoder call: %s\n", sic_ok ? "ok" : "FAILED");
            fails += !sic_ok;
        }
        // (6) RefineTrace + pluggable ConfidenceScorer (refine.hpp:48-92)
        {
            int same = 0, same_tr = 0;
            const int n6 = 4, k = 3;
            for (int b = 0; b < n6; ++b) {
                ura::EvidenceMatrix s6(16, 64);
                auto er = ura::make_rng(ura::derive_seed(21, b));
                std::uniform_real_distribution<double> u(-8.0, 0.0);
                for (double& x : s6.v) x = double(float(u(er)));
                ura::SymbolGrid truth6(k, 16);
                auto tr6 = ura::make_rng(ura::derive_seed(22, b));
                std::uniform_int_distribution<int> sym(0, 63);
                for (int& v : truth6.v) v = sym(tr6);
                ura::OracleRowScorer scorer(truth6); // every row "wrong" -> all rows re-decoded per stage
                ura::RemaskConfig rm{{0.9, 0.5}};
                ura::RefineTrace ta, tg;
                auto a = ura::run_with_remasking(cpu, scorer, s6, h, sched, rm, k, 16, &ta);
                auto g = refiner.run_with_remasking(scorer, s6, h, sched, rm, k, &tg);
                same += a == g;
                same_tr += ta.reveal_counts == tg.reveal_counts && ta.first_step_sites == tg.first_step_sites &&
                           ta.pass_first_reveals == tg.pass_first_reveals && ta.remask_rows_per_stage == tg.remask_rows_per_stage &&
                           ta.remask_steps_per_stage == tg.remask_steps_per_stage;
            }
            std::printf("scored remasking (OracleRowScorer) vs reference: %d/%d identical grids, %d/%d identical traces\n", same,
                        n6, same_tr, n6);
            fails += same != n6;
            fails += same_tr != n6;
        }
        // (7) the stochastic-binning protocol: reference CPU bank vs the coalescing GPU bank
        {
            ura::FrameConfig base;
            base.q = 64;
            base.slots = 16;
            base.n_s = 24;
            base.eb_db = 8.0;
            base.payload_bits = 6 * 8;
            auto gen = ura::derive_generator(gf, h);
            auto dicts = ura::make_dictionaries(base.q, base.n_s, base.slots, 5);
            ura::ProtocolConfig pc;
            pc.k_tot = 6;
            pc.zeta = 2;
            pc.k_max = 4;
            std::mutex mu;
            using Key = std::vector<double>;
            std::map<Key, ura::SymbolGrid> cpu_out, gpu_out;
            auto f32 = [](const ura::EvidenceMatrix& e) {
                ura::EvidenceMatrix r = e;
                for (double& x : r.v) x = double(float(x)); // both banks decode the fp32-rounded evidence
                return r;
            };
            ura::BinDecoder cpu_dec = [&](const ura::BinTask& t) {
                ura::RevealSchedule sc;
                sc.steps = ura::default_steps_for_load(t.load);
                ura::RemaskConfig rm;
                rm.thresholds = ura::default_remask_thresholds(t.load);
                ura::MaxProbScorer mp;
                auto ev = f32(t.evidence);
                auto g = ura::run_with_remasking(cpu, mp, ev, t.h, sc, rm, t.load, t.evidence.slots);
                std::lock_guard<std::mutex> lk(mu);
                cpu_out[ev.v] = g;
                return g;
            };
            auto co = std::make_shared<cider::BinCoalescer>(ctx, pc.k_max);
            auto gdec = cider::make_coalescing_bin_decoder(co);
            ura::BinDecoder gpu_dec = [&](const ura::BinTask& t) {
                auto ev = f32(t.evidence);
                auto g = gdec(ura::BinTask{t.gf, t.h, ev, t.truth, t.load});
                std::lock_guard<std::mutex> lk(mu);
                gpu_out[ev.v] = g;
                return g;
            };
            const int frames = 12;
            auto ra = ura::run_protocol(pc, base, gf, h, gen, dicts, ura::DecoderBank::uniform(cpu_dec, pc.k_max), frames, 3);
            auto rg = ura::run_protocol(pc, base, gf, h, gen, dicts, ura::DecoderBank::uniform(gpu_dec, pc.k_max), frames, 3);
            int same = 0;
            for (auto& [k, g] : cpu_out) {
                auto it = gpu_out.find(k);
                same += it != gpu_out.end() && it->second == g;
            }
            const bool agg = ra.ser == rg.ser && ra.cer == rg.cer && ra.overflow_rate == rg.overflow_rate;
            std::printf("run_protocol (%d frames, %d decoded bins, %lld device batches): %d/%d identical bin grids, "
                        "SER %.6f / %.6f, CER %.6f / %.6f: %s\n",
                        frames, int(cpu_out.size()), (long long)co->batches(), same, int(cpu_out.size()), ra.ser, rg.ser, ra.cer,
                        rg.cer, agg ? "ok" : "FAILED");
            fails += same != int(cpu_out.size()) || cpu_out.size() != gpu_out.size() || cpu_out.empty();
            fails += !agg;
        }
        // (8) config-mode context (N = 2 layers, hidden 48, 2 attention heads) through the adapter: the
        // reference's own loop driving GpuStructuredDenoiser equals the device loop (GpuRefiner), FP32
        {
            cider_model_desc md{};
            md.m = 6;
            md.dim = 32;
            md.hidden = 48;
            md.layers = 2;
            md.heads = 2;
            md.tau_demix = 1.0;
            md.evidence_scale = 1.0;
            md.precision = CIDER_FP32;
            std::vector<float> w(cider_weights_count(&md));
            cider::check(cider_weights_init(&md, 4, w.data()));
            auto cctx = std::make_shared<cider::Context>(md, w, h, 0);
            cider::GpuStructuredDenoiser cden(cctx);
            cider::GpuRefiner cref(cctx);
            int same = 0;
            for (int b = 0; b < 4; ++b) {
                ura::EvidenceMatrix s8(16, 64);
                auto er = ura::make_rng(ura::derive_seed(31, b));
                std::uniform_real_distribution<double> u(-8.0, 0.0);
                for (double& x : s8.v) x = double(float(u(er)));
                auto a = ura::run_refinement(cden, s8, h, sched, 3, 16);
                auto d = cref.run_refinement(s8, h, sched, 3);
                same += a == d;
            }
            std::printf("config-mode context (2 layers, attention): reference loop vs device loop %d/4 identical grids\n", same);
            fails += same != 4;
        }
        // error contract: a different H must be rejected like a bad input
        auto rng2 = ura::make_rng(99);
        auto h2 = ura::build_random_ldpc(gf, 16, 8, 3, rng2);
        try {
            gpu.logits(ura::all_masked_grid(2, 16), s, h2, 0.0);
            std::printf("foreign H accepted: FAILED\n");
            ++fails;
        } catch (const std::domain_error&) {
            std::printf("foreign H rejected with std::domain_error: ok\n");
        }
    } catch (const std::exception& e) {
        std::printf("exception: %s\n", e.what());
        ++fails;
    }
    return fails;
}
