// dataset.cpp — the reference's on-disk dataset format: JSON Lines datasets
// (dataset.hpp:19-99, dataset.cpp:139-220), their config fingerprint, and the number formatting of
// uradec's CSV rows — host C++ of libcider, so `uradec-gpu decode` reads the reference's datasets.
//
// The reference serialises with nlohmann::json (a vendored third-party header the reference tree
// does not ship; the copy pinned by this repo's tests is nlohmann/json 3.11.3, found in the image's
// cudnn_frontend include tree). Two of its behaviours are part of the format and are restated here:
//   * object keys are emitted in sorted order (json::object_t is a std::map), so the config
//     fingerprint FNV-1a(config_to_json(cfg)) hashes {"amp_iters":..,"col_weight":..,...} in that order;
//   * doubles are dumped with Grisu2 digits (Loitsch 2010; not always the shortest form), laid out
//     by its format_buffer rule (fixed for decimal exponents in (-4, 15], with ".0" on integral
//     values; else d.ddde+XX with at least two exponent digits).
// tests/test_dataset.py pins both against the reference's own write_dataset / config_fingerprint
// (oracle/_ref, dataset.cpp compiled against that json.hpp) and round-trips reference-written files.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "host.hpp"

namespace cider {
namespace {

// ---- a minimal JSON value / parser (objects, arrays, strings, numbers, literals) --------------
struct JVal;
using JObj = std::map<std::string, JVal>;
using JArr = std::vector<JVal>;
struct JVal {
    enum Kind { NUL, BOOL, INT, UINT, DBL, STR, ARR, OBJ } kind = NUL;
    bool b = false;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0.0;
    std::string s;
    std::shared_ptr<JArr> a;
    std::shared_ptr<JObj> o;

    bool is_num() const { return kind == INT || kind == UINT || kind == DBL; }
    double as_double() const {
        if (kind == DBL) return d;
        if (kind == INT) return double(i);
        if (kind == UINT) return double(u);
        throw std::runtime_error("type must be number");
    }
    int64_t as_int() const {
        if (kind == INT) return i;
        if (kind == UINT) return int64_t(u);
        if (kind == DBL) return int64_t(d); // nlohmann get<int> truncates a float
        throw std::runtime_error("type must be number");
    }
    uint64_t as_uint() const {
        if (kind == UINT) return u;
        if (kind == INT) return uint64_t(i);
        if (kind == DBL) return uint64_t(d);
        throw std::runtime_error("type must be number");
    }
    const std::string& as_str() const {
        if (kind != STR) throw std::runtime_error("type must be string");
        return s;
    }
    const JArr& arr() const {
        if (kind != ARR) throw std::runtime_error("type must be array");
        return *a;
    }
    const JObj& obj() const {
        if (kind != OBJ) throw std::runtime_error("type must be object");
        return *o;
    }
    bool contains(const std::string& k) const { return kind == OBJ && o->count(k); }
    const JVal& at(const std::string& k) const {
        auto it = obj().find(k);
        if (it == o->end()) throw std::runtime_error("key '" + k + "' not found");
        return it->second;
    }
};

struct Parser {
    const std::string& t;
    size_t p = 0;
    explicit Parser(const std::string& text) : t(text) {}
    [[noreturn]] void fail(const char* what) const {
        throw std::runtime_error(std::string("parse error at byte ") + std::to_string(p + 1) + ": " + what);
    }
    void ws() {
        while (p < t.size() && (t[p] == ' ' || t[p] == '\t' || t[p] == '\n' || t[p] == '\r')) ++p;
    }
    JVal value() {
        ws();
        if (p >= t.size()) fail("unexpected end of input");
        const char c = t[p];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            JVal v;
            v.kind = JVal::STR;
            v.s = str();
            return v;
        }
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        return literal();
    }
    JVal object() {
        JVal v;
        v.kind = JVal::OBJ;
        v.o = std::make_shared<JObj>();
        ++p;
        ws();
        if (p < t.size() && t[p] == '}') { ++p; return v; }
        for (;;) {
            ws();
            if (p >= t.size() || t[p] != '"') fail("expected object key");
            std::string k = str();
            ws();
            if (p >= t.size() || t[p] != ':') fail("expected ':'");
            ++p;
            (*v.o)[k] = value();
            ws();
            if (p < t.size() && t[p] == ',') { ++p; continue; }
            if (p < t.size() && t[p] == '}') { ++p; return v; }
            fail("expected ',' or '}'");
        }
    }
    JVal array() {
        JVal v;
        v.kind = JVal::ARR;
        v.a = std::make_shared<JArr>();
        ++p;
        ws();
        if (p < t.size() && t[p] == ']') { ++p; return v; }
        for (;;) {
            v.a->push_back(value());
            ws();
            if (p < t.size() && t[p] == ',') { ++p; continue; }
            if (p < t.size() && t[p] == ']') { ++p; return v; }
            fail("expected ',' or ']'");
        }
    }
    std::string str() {
        ++p; // opening quote
        std::string out;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c != '\\') { out.push_back(c); continue; }
            if (p >= t.size()) fail("bad escape");
            char e = t[p++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    if (p + 4 > t.size()) fail("bad \\u escape");
                    unsigned cp = std::stoul(t.substr(p, 4), nullptr, 16);
                    p += 4;
                    if (cp < 0x80) out.push_back(char(cp));
                    else if (cp < 0x800) { out.push_back(char(0xC0 | (cp >> 6))); out.push_back(char(0x80 | (cp & 0x3F))); }
                    else { out.push_back(char(0xE0 | (cp >> 12))); out.push_back(char(0x80 | ((cp >> 6) & 0x3F))); out.push_back(char(0x80 | (cp & 0x3F))); }
                    break;
                }
                default: fail("bad escape");
            }
        }
        if (p >= t.size()) fail("unterminated string");
        ++p;
        return out;
    }
    JVal number() {
        const size_t b = p;
        if (t[p] == '-') ++p;
        bool flt = false;
        while (p < t.size()) {
            const char c = t[p];
            if (c >= '0' && c <= '9') { ++p; continue; }
            if (c == '.' || c == 'e' || c == 'E' || c == '+' || (c == '-' && p > b)) { flt = true; ++p; continue; }
            break;
        }
        const std::string num = t.substr(b, p - b);
        JVal v;
        const char* s0 = num.c_str();
        char* end = nullptr;
        if (!flt) { // integers as nlohmann stores them: unsigned when non-negative, else signed
            errno = 0;
            if (num[0] == '-') {
                v.kind = JVal::INT;
                v.i = std::strtoll(s0, &end, 10);
            } else {
                v.kind = JVal::UINT;
                v.u = std::strtoull(s0, &end, 10);
            }
            if (errno == 0 && end && *end == '\0') return v;
        }
        v.kind = JVal::DBL;
        v.d = std::strtod(s0, &end); // correctly rounded, as nlohmann's parser
        if (!end || *end != '\0') fail("bad number");
        return v;
    }
    JVal literal() {
        JVal v;
        auto take = [&](const char* w) {
            const size_t n = std::strlen(w);
            if (t.compare(p, n, w) != 0) fail("unexpected token");
            p += n;
        };
        if (t[p] == 't') { take("true"); v.kind = JVal::BOOL; v.b = true; }
        else if (t[p] == 'f') { take("false"); v.kind = JVal::BOOL; v.b = false; }
        else { take("null"); v.kind = JVal::NUL; }
        return v;
    }
    JVal parse_all() {
        JVal v = value();
        ws();
        if (p != t.size()) fail("trailing characters");
        return v;
    }
};

// ---- number formatting -------------------------------------------------------------------------
// nlohmann::json dumps a double with Grisu2 (F. Loitsch, "Printing floating-point numbers quickly and
// accurately with integers", PLDI 2010) — usually, not always, the shortest round-trip digits — then
// lays them out with its format_buffer rule. Both are restated here from the published algorithm:
// boundaries m-/m+ of v, a cached power 10^-k bringing the scaled exponent into [alpha, gamma] =
// [-60, -32], digit generation from the conservative upper bound M+ - 1 ulp until the remainder is
// within the interval, then the closest-digit adjustment ("round / weed") toward v.
struct DiyFp {
    uint64_t f;
    int e;
};
DiyFp diy_sub(DiyFp a, DiyFp b) { return {a.f - b.f, a.e}; }
DiyFp diy_mul(DiyFp a, DiyFp b) { // upper 64 bits of the 128-bit product, rounded half up
    const unsigned __int128 p = (unsigned __int128)a.f * b.f;
    uint64_t hi = uint64_t(p >> 64);
    hi += uint64_t(p >> 63) & 1u;
    return {hi, a.e + b.e + 64};
}
DiyFp diy_normalize(DiyFp x) {
    while ((x.f >> 63) == 0) { x.f <<= 1; --x.e; }
    return x;
}
DiyFp diy_normalize_to(DiyFp x, int e) { return {x.f << (x.e - e), e}; }

// 10^k = f x 2^e (f normalised, rounded to nearest) for k = -300, -292, ..., 324 (generated offline
// with exact rational arithmetic)
struct CachedPow {
    uint64_t f;
    int e, k;
};
const CachedPow kPow10[] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300},
    {0xFF77B1FCBEBCDC4FULL, -1034, -292},
    {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276},
    {0xD3515C2831559A83ULL, -954, -268},
    {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252},
    {0xAECC49914078536DULL, -874, -244},
    {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228},
    {0x9096EA6F3848984FULL, -794, -220},
    {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204},
    {0xEF340A98172AACE5ULL, -715, -196},
    {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180},
    {0xC5DD44271AD3CDBAULL, -635, -172},
    {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156},
    {0xA3AB66580D5FDAF6ULL, -555, -148},
    {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132},
    {0x87625F056C7C4A8BULL, -475, -124},
    {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108},
    {0xDFF9772470297EBDULL, -396, -100},
    {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84},
    {0xB94470938FA89BCFULL, -316, -76},
    {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60},
    {0x993FE2C6D07B7FACULL, -236, -52},
    {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36},
    {0xFD87B5F28300CA0EULL, -157, -28},
    {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12},
    {0xD1B71758E219652CULL, -77, -4},
    {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12},
    {0xAD78EBC5AC620000ULL, 3, 20},
    {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36},
    {0x8F7E32CE7BEA5C70ULL, 83, 44},
    {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60},
    {0xED63A231D4C4FB27ULL, 162, 68},
    {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84},
    {0xC45D1DF942711D9AULL, 242, 92},
    {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108},
    {0xA26DA3999AEF774AULL, 322, 116},
    {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132},
    {0x865B86925B9BC5C2ULL, 402, 140},
    {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156},
    {0xDE469FBD99A05FE3ULL, 481, 164},
    {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180},
    {0xB7DCBF5354E9BECEULL, 561, 188},
    {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204},
    {0x98165AF37B2153DFULL, 641, 212},
    {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228},
    {0xFB9B7CD9A4A7443CULL, 720, 236},
    {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252},
    {0xD01FEF10A657842CULL, 800, 260},
    {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276},
    {0xAC2820D9623BF429ULL, 880, 284},
    {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300},
    {0x8E679C2F5E44FF8FULL, 960, 308},
    {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324}
};

void grisu2(double v, char* buf, int& len, int& dec_exp) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const uint64_t F = bits & ((uint64_t(1) << 52) - 1);
    const int E = int((bits >> 52) & 0x7FF);
    constexpr int kBias = 1075; // 1023 + 52
    const uint64_t f = E == 0 ? F : F + (uint64_t(1) << 52);
    const int e = E == 0 ? 1 - kBias : E - kBias;
    const bool lower_closer = F == 0 && E > 1;
    const DiyFp mp = diy_normalize({2 * f + 1, e - 1});
    const DiyFp mm = diy_normalize_to(lower_closer ? DiyFp{4 * f - 1, e - 2} : DiyFp{2 * f - 1, e - 1}, mp.e);
    const DiyFp w = diy_normalize({f, e});
    // cached power for the exponent of m+
    constexpr int kAlpha = -60;
    const int fk = kAlpha - mp.e - 1;
    const int k = (fk * 78913) / (1 << 18) + (fk > 0 ? 1 : 0);
    const int idx = (300 + k + 7) / 8;
    const CachedPow& c = kPow10[idx];
    const DiyFp cm{c.f, c.e};
    const DiyFp W = diy_mul(w, cm), Wm = diy_mul(mm, cm), Wp = diy_mul(mp, cm);
    const DiyFp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
    dec_exp = -c.k;
    // digit generation
    uint64_t delta = diy_sub(Mp, Mm).f;
    uint64_t dist = diy_sub(Mp, W).f;
    const int sh = -Mp.e;
    const uint64_t one = uint64_t(1) << sh;
    uint32_t p1 = uint32_t(Mp.f >> sh);
    uint64_t p2 = Mp.f & (one - 1);
    uint32_t pow10 = 1;
    int n = 1;
    while (n < 10 && p1 >= pow10 * 10ull) { pow10 *= 10; ++n; }
    len = 0;
    auto round_weed = [&](uint64_t rest, uint64_t ten_k) {
        while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
            --buf[len - 1];
            rest += ten_k;
        }
    };
    while (n > 0) {
        const uint32_t d = p1 / pow10;
        p1 %= pow10;
        buf[len++] = char('0' + d);
        --n;
        const uint64_t rest = (uint64_t(p1) << sh) + p2;
        if (rest <= delta) {
            dec_exp += n;
            round_weed(rest, uint64_t(pow10) << sh);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const uint64_t d = p2 >> sh;
        p2 &= one - 1;
        buf[len++] = char('0' + d);
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dec_exp -= m;
    round_weed(p2, one);
}

std::string json_double(double x) {
    if (!std::isfinite(x)) return "null";
    std::string out;
    if (std::signbit(x)) { out.push_back('-'); x = -x; }
    if (x == 0.0) return out + "0.0";
    char buf[32];
    int k = 0, de = 0;
    grisu2(x, buf, k, de);
    const std::string digits(buf, size_t(k));
    const int n = k + de; // decimal point position relative to the digit string
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {
        out += digits;
        out.append(size_t(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= kMaxExp) {
        out += digits.substr(0, size_t(n));
        out.push_back('.');
        out += digits.substr(size_t(n));
    } else if (kMinExp < n && n <= 0) {
        out += "0.";
        out.append(size_t(-n), '0');
        out += digits;
    } else {
        out.push_back(digits[0]);
        if (k > 1) {
            out.push_back('.');
            out += digits.substr(1);
        }
        out.push_back('e');
        const int ex = n - 1;
        out.push_back(ex < 0 ? '-' : '+');
        const int ax = ex < 0 ? -ex : ex;
        char eb[8];
        std::snprintf(eb, sizeof(eb), ax < 10 ? "0%d" : "%d", ax);
        out += eb;
    }
    return out;
}

std::string json_string(const std::string& s) {
    std::string out = "\"";
    for (unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (c < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    out += b;
                } else {
                    out.push_back(char(c));
                }
        }
    }
    return out + "\"";
}

// config_to_json (dataset.cpp:63-81, 114): the object's keys in sorted order, as nlohmann dumps them
std::string config_json(const cider_run_config& c) {
    std::ostringstream o;
    o << "{\"amp_iters\":" << c.amp_iters << ",\"col_weight\":" << c.col_weight << ",\"eb_db\":" << json_double(c.eb_db)
      << ",\"evidence_floor\":" << json_double(c.evidence_floor) << ",\"frames\":" << c.frames << ",\"k\":" << c.k
      << ",\"l\":" << c.l << ",\"n_s\":" << c.n_s << ",\"noise_var\":" << json_double(c.noise_var) << ",\"p\":" << c.p
      << ",\"q\":" << c.q << ",\"rho_bg\":" << json_double(c.rho_bg) << ",\"scale\":" << json_string(c.scale)
      << ",\"seed\":" << c.seed << ",\"sigma_u2\":" << json_double(c.sigma_u2) << "}";
    return o.str();
}

std::string fnv1a(const std::string& data) { // dataset.cpp:118-128
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : data) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    char buf[17];
    std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(h));
    return buf;
}

// RunConfig defaults (dataset.hpp:19-36) overridden by the keys present (config_from_json_obj)
cider_run_config config_from(const JVal& j) {
    cider_run_config c{};
    std::snprintf(c.scale, sizeof(c.scale), "%s", "tiny");
    c.q = 64; c.l = 12; c.p = 8; c.col_weight = 3; c.k = 2; c.n_s = 24;
    c.eb_db = 10.0; c.noise_var = 1.0; c.amp_iters = 20; c.rho_bg = -1.0; c.sigma_u2 = -1.0;
    c.evidence_floor = -40.0; c.seed = 1; c.frames = 100;
    if (j.contains("scale")) {
        const std::string& s = j.at("scale").as_str();
        if (s.size() >= sizeof(c.scale)) throw std::runtime_error("load_dataset: scale name too long");
        std::snprintf(c.scale, sizeof(c.scale), "%s", s.c_str());
    }
    auto gi = [&](const char* k, int& f) { if (j.contains(k)) f = int(j.at(k).as_int()); };
    auto gd = [&](const char* k, double& f) { if (j.contains(k)) f = j.at(k).as_double(); };
    gi("q", c.q); gi("l", c.l); gi("p", c.p); gi("col_weight", c.col_weight); gi("k", c.k); gi("n_s", c.n_s);
    gd("eb_db", c.eb_db); gd("noise_var", c.noise_var); gi("amp_iters", c.amp_iters); gd("rho_bg", c.rho_bg);
    gd("sigma_u2", c.sigma_u2); gd("evidence_floor", c.evidence_floor);
    if (j.contains("seed")) c.seed = j.at("seed").as_uint();
    gi("frames", c.frames);
    return c;
}

struct LoadedFrame {
    uint64_t seed;
    double snr;
    int rows;
    std::vector<int32_t> truth;
    std::vector<double> ev;
};

template <class F>
int guard2(F&& f) {
    try {
        f();
        return CIDER_OK;
    } catch (const std::domain_error& e) {
        set_host_error(e.what());
        return CIDER_EINVAL;
    } catch (const std::exception& e) {
        set_host_error(e.what());
        return CIDER_ERUNTIME;
    }
}

} // namespace
} // namespace cider

using namespace cider;

extern "C" {

int cider_format_double(double x, char* out, int cap) {
    // format_double (dataset.cpp:57-61): std::to_chars shortest round-trip form
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), x);
    const int n = int(r.ptr - buf);
    if (!out || cap <= n) return CIDER_EINVAL;
    std::memcpy(out, buf, size_t(n));
    out[n] = '\0';
    return CIDER_OK;
}

int cider_config_to_json(const cider_run_config* cfg, char* out, int cap) {
    if (!cfg || !out) return CIDER_EINVAL;
    const std::string s = config_json(*cfg);
    if (cap <= int(s.size())) return CIDER_EINVAL;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return CIDER_OK;
}

int cider_config_fingerprint(const cider_run_config* cfg, char out[17]) {
    if (!cfg || !out) return CIDER_EINVAL;
    const std::string h = fnv1a(config_json(*cfg));
    std::memcpy(out, h.c_str(), 17);
    return CIDER_OK;
}

int cider_file_fingerprint(const char* path, char out[17]) {
    return guard2([&] { // dataset.cpp:132-137
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("file_fingerprint: cannot open ") + path);
        std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        std::memcpy(out, fnv1a(data).c_str(), 17);
    });
}

int cider_dataset_load(const char* path, cider_run_config* cfg, char fingerprint[17], char h_fingerprint[17],
                       int* n_frames, int frames_cap, uint64_t* seeds, int32_t* truth, double* evidence, double* snr_db) {
    return guard2([&] { // load_dataset (dataset.cpp:176-220)
        const std::string ps(path ? path : "");
        std::ifstream in(ps);
        if (!in) throw std::runtime_error("load_dataset: cannot open " + ps);
        std::string line;
        if (!std::getline(in, line)) throw std::runtime_error("load_dataset: empty file " + ps);
        JVal header = Parser(line).parse_all();
        if (!header.contains("type") || header.at("type").kind != JVal::STR || header.at("type").s != "header")
            throw std::runtime_error("load_dataset: missing header record in " + ps);
        const cider_run_config c = config_from(header.at("config"));
        const std::string fp = header.at("fingerprint").as_str();
        const std::string hfp = header.contains("h_fingerprint") && header.at("h_fingerprint").kind == JVal::STR
                                    ? header.at("h_fingerprint").s : std::string();
        if (fp != fnv1a(config_json(c))) throw std::runtime_error("load_dataset: config fingerprint mismatch in " + ps);
        std::vector<LoadedFrame> frames;
        while (std::getline(in, line)) {
            if (line.empty()) continue;
            JVal rec = Parser(line).parse_all();
            LoadedFrame f;
            f.seed = rec.at("seed").as_uint();
            f.snr = rec.at("snr_db").as_double();
            if (rec.at("config_fp").as_str() != fp)
                throw std::runtime_error("load_dataset: frame/config fingerprint mismatch in " + ps);
            const JArr& tr = rec.at("truth").arr();
            const int rows = int(tr.size()), cols = int(tr.at(0).arr().size());
            f.rows = rows;
            for (int k = 0; k < rows; ++k)
                for (int l = 0; l < cols; ++l) f.truth.push_back(int32_t(tr[k].arr().at(l).as_int()));
            const JArr& ev = rec.at("evidence").arr();
            const int slots = int(ev.size()), q = int(ev.at(0).arr().size());
            for (int l = 0; l < slots; ++l)
                for (int a = 0; a < q; ++a) f.ev.push_back(ev[l].arr().at(a).as_double());
            if (cols != c.l || slots != c.l || q != c.q)
                throw std::runtime_error("load_dataset: frame dimensions disagree with config");
            if (rows != c.k) // every frame of a dataset carries the configured K users (cmd_simulate)
                throw std::runtime_error("load_dataset: frame user count disagrees with config k");
            frames.push_back(std::move(f));
        }
        if (cfg) *cfg = c;
        if (fingerprint) std::memcpy(fingerprint, fp.c_str(), std::min<size_t>(fp.size(), 16) + 1);
        if (h_fingerprint) {
            std::memset(h_fingerprint, 0, 17);
            std::memcpy(h_fingerprint, hfp.c_str(), std::min<size_t>(hfp.size(), 16));
        }
        if (n_frames) *n_frames = int(frames.size());
        const int n = std::min(frames_cap, int(frames.size()));
        const size_t tk = size_t(c.k) * c.l, eq = size_t(c.l) * c.q;
        for (int i = 0; i < n; ++i) {
            if (seeds) seeds[i] = frames[i].seed;
            if (snr_db) snr_db[i] = frames[i].snr;
            if (truth) std::copy(frames[i].truth.begin(), frames[i].truth.end(), truth + size_t(i) * tk);
            if (evidence) std::copy(frames[i].ev.begin(), frames[i].ev.end(), evidence + size_t(i) * eq);
        }
    });
}

} // extern "C"
