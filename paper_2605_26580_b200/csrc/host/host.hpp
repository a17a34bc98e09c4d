// host.hpp — host-side helpers of libcider (no CUDA): seeding, GF(2^m) tables, Tanner graph.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "cider.h"

namespace cider {

struct InvalidInput : std::domain_error {
    using std::domain_error::domain_error;
};

// splitmix64 finaliser and the counter-based seed split of seeding.hpp:10-22.
inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t derive_seed(uint64_t master, uint64_t index) {
    return mix64(master ^ mix64(index + 0x517cc1b727220a95ULL));
}

// GF(2^m) with symbols labelled by their polynomial bitmask (gf.hpp:14-37).
struct Gf {
    int m = 0, q = 0;
    uint32_t poly = 0;
    std::vector<int> lg, ex;
    Gf(int m_, uint32_t poly_);
    static uint32_t default_poly(int m);
    int mul(int a, int b) const {
        if (!a || !b) return 0;
        int s = lg[a] + lg[b];
        if (s >= q - 1) s -= q - 1;
        return ex[s];
    }
    int inv(int a) const;
};

// Validated, (check, slot)-sorted edge list with CSR views (ldpc.cpp:11-30).
struct Tanner {
    int checks = 0, slots = 0, q = 0;
    std::vector<int> chk, slot, coef;     // per edge, sorted by (check, slot)
    std::vector<int> check_ptr;           // check j: edges [check_ptr[j], check_ptr[j+1])
    std::vector<int> slot_ptr, slot_edge; // slot l: slot_edge[slot_ptr[l] .. slot_ptr[l+1]), ascending check
    Tanner(const cider_code_desc* c, int q);
    int n_edges() const { return int(chk.size()); }
};

// failure ordering for cider_last_error (the most recent message of either half of the ABI)
uint64_t error_tick();
uint64_t host_error_tick();
void set_host_error(const std::string& msg); // a host-half failure for cider_last_error

// systematic encoder of H (info slots, pivot slots, pivot-row coefficients [pivot][info]) for the
// device workload generator (kernels/workload.cuh)
void systematic_tables(const Gf& gf, const Tanner& t, std::vector<int>& info, std::vector<int>& pivot,
                       std::vector<uint8_t>& red);

size_t weights_count(const cider_model_desc* m);
void validate_model(const cider_model_desc* m);

} // namespace cider
