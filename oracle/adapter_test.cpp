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
// on fp32-rounded parameters and evidence (FP32 mode), and requires identical grids.
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>

#include "cider_ura.hpp"
#include "ura/ldpc.hpp"
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
