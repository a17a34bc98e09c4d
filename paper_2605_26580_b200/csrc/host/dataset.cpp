// dataset.cpp — the reference's on-disk dataset format: JSON Lines datasets
// (dataset.hpp:19-99, dataset.cpp:139-220), their config fingerprint, and the number formatting of
// uradec's CSV rows — host C++ of libcider, so `uradec-gpu decode` reads the reference's datasets.
//
// The reference serialises with nlohmann::json (a vendored third-party header the reference tree
// does not ship; the copy pinned by this repo's tests is nlohmann/json 3.11.3, found in the image's
// cudnn_frontend include tree). Two of its behaviours are part of the format and are restated here:
//   * object keys are emitted in sorted order (json::object_t is a std::map), so the config
//     fingerprint FNV-1a(config_to_json(cfg)) hashes {"amp_iters":..,"col_weight":..,...} in that order;
//   * doubles are dumped as the shortest round-trip decimal digits, laid out by its
//     format_buffer rule (fixed for decimal exponents in (-4, 15], with ".0" on integral values;
//     else d.ddde+XX with at least two exponent digits).
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
// nlohmann::json's dump of a double: shortest round-trip digits, then its format_buffer layout
// (min_exp = -4, max_exp = 15 for doubles).
std::string json_double(double x) {
    if (!std::isfinite(x)) return "null";
    if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific); // shortest, d.ddde±XX
    std::string sci(buf, r.ptr);
    std::string out;
    size_t i = 0;
    if (sci[0] == '-') { out.push_back('-'); i = 1; }
    const size_t epos = sci.find('e');
    std::string digits;
    for (size_t j = i; j < epos; ++j)
        if (sci[j] != '.') digits.push_back(sci[j]);
    const int e10 = std::stoi(sci.substr(epos + 1)); // value = d.ddd x 10^e10
    const int k = int(digits.size());
    const int n = e10 + 1; // decimal point position relative to the digit string
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
