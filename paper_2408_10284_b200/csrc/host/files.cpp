// Artifact files of the reference (see files.hpp).  The writer reproduces the reference's
// nlohmann::json output byte for byte (sorted object keys, shortest round-trip doubles formatted
// like nlohmann's dtoa, dump(2) pretty printing), so files written here are interchangeable with
// the reference's `moesim` tools and profile_hash matches.
#include "files.hpp"

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <map>
#include <sstream>
#include <string_view>
#include <thread>

namespace adapmoe {

namespace {

// ---- minimal JSON DOM -----------------------------------------------------------------------
struct JVal {
    enum Type { Null, Bool, Num, Str, Arr, Obj } t = Null;
    bool b = false;
    double n = 0.0;
    bool integral = false;           // the number had no fraction / exponent
    long long i = 0;                 // exact value when integral
    std::string s;
    std::vector<JVal> a;
    bool num_array = false;          // fast path: array of numbers only (kept in nums)
    std::vector<double> nums;
    std::vector<char> nums_int;      // per number: was integral
    std::map<std::string, JVal> o;   // sorted keys, like nlohmann::json's default object

    const JVal* get(const std::string& k) const {
        if (t != Obj) return nullptr;
        auto it = o.find(k);
        return it == o.end() ? nullptr : &it->second;
    }
    size_t size() const { return t == Arr ? (num_array ? nums.size() : a.size()) : 0; }
};

[[noreturn]] void parse_fail(const std::string& where, const std::string& what) {
    fail(Status::Format, where + ": parse error: " + what);
}
[[noreturn]] void schema_fail(const std::string& where, const std::string& what) { fail(Status::Format, where + ": " + what); }

class Parser {
public:
    Parser(const char* b, const char* e, std::string where) : p_(b), end_(e), where_(std::move(where)) {}
    JVal parse_document() {
        JVal v = value();
        ws();
        if (p_ != end_) parse_fail(where_, "trailing characters");
        return v;
    }

private:
    void ws() {
        while (p_ < end_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
    }
    bool number_start(char c) const { return c == '-' || (c >= '0' && c <= '9'); }
    void number(double& out, bool& integral, long long& iv) {
        const char* b = p_;
        integral = true;
        while (p_ < end_ && (number_start(*p_) || *p_ == '+' || *p_ == '.' || *p_ == 'e' || *p_ == 'E')) {
            if (*p_ == '.' || *p_ == 'e' || *p_ == 'E') integral = false;
            ++p_;
        }
        auto r = std::from_chars(b, p_, out);
        if (r.ec != std::errc() || r.ptr != p_) parse_fail(where_, "bad number");
        if (integral) {
            auto ri = std::from_chars(b, p_, iv);
            if (ri.ec != std::errc() || ri.ptr != p_) integral = false;
        }
    }
    std::string string() {
        if (*p_ != '"') parse_fail(where_, "expected string");
        ++p_;
        std::string s;
        while (p_ < end_ && *p_ != '"') {
            if (*p_ == '\\') {
                ++p_;
                if (p_ >= end_) break;
                const char c = *p_++;
                switch (c) {
                    case 'n': s += '\n'; break;
                    case 't': s += '\t'; break;
                    case 'r': s += '\r'; break;
                    case 'b': s += '\b'; break;
                    case 'f': s += '\f'; break;
                    case 'u': {
                        if (end_ - p_ < 4) parse_fail(where_, "bad \\u escape");
                        unsigned cp = 0;
                        std::from_chars(p_, p_ + 4, cp, 16);
                        p_ += 4;
                        if (cp < 0x80) s += static_cast<char>(cp);
                        else if (cp < 0x800) {
                            s += static_cast<char>(0xC0 | (cp >> 6));
                            s += static_cast<char>(0x80 | (cp & 0x3F));
                        } else {
                            s += static_cast<char>(0xE0 | (cp >> 12));
                            s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                            s += static_cast<char>(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: s += c;
                }
            } else {
                s += *p_++;
            }
        }
        if (p_ >= end_) parse_fail(where_, "unterminated string");
        ++p_;
        return s;
    }
    JVal value() {
        ws();
        if (p_ >= end_) parse_fail(where_, "unexpected end of input");
        JVal v;
        const char c = *p_;
        if (c == '{') {
            v.t = JVal::Obj;
            ++p_;
            ws();
            if (p_ < end_ && *p_ == '}') {
                ++p_;
                return v;
            }
            for (;;) {
                ws();
                std::string k = string();
                ws();
                if (p_ >= end_ || *p_ != ':') parse_fail(where_, "expected ':'");
                ++p_;
                v.o[k] = value();
                ws();
                if (p_ < end_ && *p_ == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < end_ && *p_ == '}') {
                    ++p_;
                    return v;
                }
                parse_fail(where_, "expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.t = JVal::Arr;
            ++p_;
            ws();
            if (p_ < end_ && *p_ == ']') {
                ++p_;
                v.num_array = true;
                return v;
            }
            v.num_array = true;
            for (;;) {
                ws();
                if (p_ < end_ && v.num_array && number_start(*p_)) {
                    double d;
                    bool integral;
                    long long iv;
                    number(d, integral, iv);
                    v.nums.push_back(d);
                    v.nums_int.push_back(integral ? 1 : 0);
                } else {
                    if (v.num_array) {  // leave the fast path
                        for (size_t q = 0; q < v.nums.size(); ++q) {
                            JVal e;
                            e.t = JVal::Num;
                            e.n = v.nums[q];
                            e.integral = v.nums_int[q] != 0;
                            e.i = static_cast<long long>(e.n);
                            v.a.push_back(e);
                        }
                        v.nums.clear();
                        v.num_array = false;
                    }
                    v.a.push_back(value());
                }
                ws();
                if (p_ < end_ && *p_ == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < end_ && *p_ == ']') {
                    ++p_;
                    return v;
                }
                parse_fail(where_, "expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.t = JVal::Str;
            v.s = string();
            return v;
        }
        if (number_start(c)) {
            v.t = JVal::Num;
            number(v.n, v.integral, v.i);
            return v;
        }
        auto lit = [&](const char* w, size_t len) { return static_cast<size_t>(end_ - p_) >= len && !std::memcmp(p_, w, len); };
        if (lit("true", 4)) {
            p_ += 4;
            v.t = JVal::Bool;
            v.b = true;
            return v;
        }
        if (lit("false", 5)) {
            p_ += 5;
            v.t = JVal::Bool;
            return v;
        }
        if (lit("null", 4)) {
            p_ += 4;
            return v;
        }
        parse_fail(where_, "unexpected character");
    }
    const char* p_;
    const char* end_;
    std::string where_;
};

JVal parse_text(std::string_view text, const std::string& where) {
    return Parser(text.data(), text.data() + text.size(), where).parse_document();
}

std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(Status::Io, "cannot open " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return buf.str();
}

void write_file(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(Status::Io, "cannot open " + path + " for writing");
    out << text;
    if (!out) fail(Status::Io, "write failed: " + path);
}

// ---- schema helpers (inc/io.hpp:73-83 detail::require) ----------------------------------------
const JVal& field(const JVal& j, const char* k, const std::string& where) {
    const JVal* v = j.get(k);
    if (!v) schema_fail(where, std::string("missing field \"") + k + "\"");
    return *v;
}
[[noreturn]] void wrong_type(const char* k, const std::string& where) {
    schema_fail(where, std::string("field \"") + k + "\" has the wrong type");
}
double req_double(const JVal& j, const char* k, const std::string& where) {
    const JVal& v = field(j, k, where);
    if (v.t != JVal::Num) wrong_type(k, where);
    return v.n;
}
long long req_int(const JVal& j, const char* k, const std::string& where) {
    const JVal& v = field(j, k, where);
    if (v.t != JVal::Num) wrong_type(k, where);
    return v.integral ? v.i : static_cast<long long>(v.n);  // nlohmann get<int> truncates a float
}
std::string req_string(const JVal& j, const char* k, const std::string& where) {
    const JVal& v = field(j, k, where);
    if (v.t != JVal::Str) wrong_type(k, where);
    return v.s;
}
std::vector<double> req_doubles(const JVal& j, const char* k, const std::string& where) {
    const JVal& v = field(j, k, where);
    if (v.t != JVal::Arr || !v.num_array) wrong_type(k, where);
    return v.nums;
}
std::vector<int> req_ints(const JVal& j, const char* k, const std::string& where) {
    const JVal& v = field(j, k, where);
    if (v.t != JVal::Arr || !v.num_array) wrong_type(k, where);
    std::vector<int> out(v.nums.size());
    for (size_t q = 0; q < out.size(); ++q) out[q] = static_cast<int>(v.nums[q]);
    return out;
}

// inc/io.hpp:41-50
void check_header(const JVal& j, const char* kind, const std::string& path) {
    if (j.t != JVal::Obj) schema_fail(path, "expected a JSON object");
    const JVal* fv = j.get("format_version");
    if (!fv || fv->t != JVal::Num || !fv->integral) schema_fail(path, "missing format_version");
    if (fv->i != kFormatVersion) fail(Status::Format, path + ": unsupported format_version " + std::to_string(fv->i));
    const JVal* k = j.get("kind");
    if (!k || k->t != JVal::Str || k->s != kind) schema_fail(path, std::string("expected kind \"") + kind + "\"");
}

ModelSpec spec_from(const JVal& j, const std::string& path) {
    const JVal* m = j.get("model");
    if (!m) schema_fail(path, "missing model");
    ModelSpec s;
    s.num_layers = static_cast<int>(req_int(*m, "num_layers", path));
    s.experts_per_layer = static_cast<int>(req_int(*m, "experts_per_layer", path));
    s.top_k = static_cast<int>(req_int(*m, "top_k", path));
    s.hidden_dim = static_cast<int>(req_int(*m, "hidden_dim", path));
    return s;
}


// ---- shortest round-trip doubles exactly as nlohmann::json prints them -------------------------
// Grisu2 (F. Loitsch, "Printing floating-point numbers quickly and accurately with integers",
// PLDI 2010) with the boundaries / cached-power / digit-generation / round-weed steps nlohmann's
// to_chars uses, so the digits (which are not always the shortest) match the reference's files.
struct DiyFp {
    std::uint64_t f;
    int e;
};
DiyFp diy_mul(DiyFp x, DiyFp y) {
    const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f + (static_cast<unsigned __int128>(1) << 63);
    return DiyFp{static_cast<std::uint64_t>(p >> 64), x.e + y.e + 64};
}
DiyFp diy_normalize(DiyFp x) {
    while ((x.f >> 63) == 0) {
        x.f <<= 1;
        x.e -= 1;
    }
    return x;
}
struct CachedPower {
    std::uint64_t f;
    int e, k;
};
// 10^k, k = -300, -292, ..., 324, as normalised 64-bit significands (round to nearest)
constexpr CachedPower kCachedPowers[] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};

void grisu2_digits(double value, char* buf, int& len, int& decimal_exponent) {
    constexpr int kAlpha = -60;
    std::uint64_t bits;
    std::memcpy(&bits, &value, 8);
    const std::uint64_t E = bits >> 52, F = bits & ((std::uint64_t{1} << 52) - 1);
    const DiyFp v = E == 0 ? DiyFp{F, -1074} : DiyFp{F + (std::uint64_t{1} << 52), static_cast<int>(E) - 1075};
    const bool lower_closer = F == 0 && E > 1;
    const DiyFp m_plus{2 * v.f + 1, v.e - 1};
    const DiyFp m_minus = lower_closer ? DiyFp{4 * v.f - 1, v.e - 2} : DiyFp{2 * v.f - 1, v.e - 1};
    const DiyFp w_plus = diy_normalize(m_plus);
    const DiyFp w_minus{m_minus.f << (m_minus.e - w_plus.e), w_plus.e};
    const DiyFp w_v = diy_normalize(v);
    // cached power c ~ 10^-k with kAlpha <= e_c + e + 64 <= kGamma
    const int fexp = kAlpha - w_plus.e - 1;
    const int kk = (fexp * 78913) / (1 << 18) + static_cast<int>(fexp > 0);
    const int index = (300 + kk + 7) / 8;
    const CachedPower cached = kCachedPowers[index];
    const DiyFp c{cached.f, cached.e};
    const DiyFp w = diy_mul(w_v, c), wm = diy_mul(w_minus, c), wp = diy_mul(w_plus, c);
    const DiyFp M_minus{wm.f + 1, wm.e}, M_plus{wp.f - 1, wp.e};
    decimal_exponent = -cached.k;
    // digit generation
    std::uint64_t delta = M_plus.f - M_minus.f;
    std::uint64_t dist = M_plus.f - w.f;
    const int sh = -M_plus.e;
    const std::uint64_t one = std::uint64_t{1} << sh;
    std::uint32_t p1 = static_cast<std::uint32_t>(M_plus.f >> sh);
    std::uint64_t p2 = M_plus.f & (one - 1);
    std::uint32_t pow10 = 1;
    int n = 1;
    {
        const std::uint32_t tens[] = {1000000000u, 100000000u, 10000000u, 1000000u, 100000u, 10000u, 1000u, 100u, 10u};
        n = 1;
        pow10 = 1;
        for (int q = 0; q < 9; ++q)
            if (p1 >= tens[q]) {
                n = 10 - q;
                pow10 = tens[q];
                break;
            }
    }
    len = 0;
    auto round_weed = [&](std::uint64_t rest, std::uint64_t ten_k) {
        while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
            buf[len - 1]--;
            rest += ten_k;
        }
    };
    while (n > 0) {
        const std::uint32_t d = p1 / pow10, r = p1 % pow10;
        buf[len++] = static_cast<char>('0' + d);
        p1 = r;
        n--;
        const std::uint64_t rest = (static_cast<std::uint64_t>(p1) << sh) + p2;
        if (rest <= delta) {
            decimal_exponent += n;
            round_weed(rest, static_cast<std::uint64_t>(pow10) << sh);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const std::uint64_t d = p2 >> sh, r = p2 & (one - 1);
        buf[len++] = static_cast<char>('0' + d);
        p2 = r;
        m++;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    decimal_exponent -= m;
    round_weed(p2, one);
}

// ---- writer: nlohmann::json dump() format ------------------------------------------------------
// Digits from grisu2_digits, laid out like nlohmann's dtoa format_buffer (min_exp -4, max_exp 15).
std::string fmt_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    std::string out;
    if (v < 0) {
        out = "-";
        v = -v;
    }
    char buf[32];
    int k = 0, dexp = 0;
    grisu2_digits(v, buf, k, dexp);
    const std::string digits(buf, buf + k);
    const int n = k + dexp;  // position of the decimal point
    if (k <= n && n <= 15) {
        out += digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(-n, '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

// value builders
JVal num(double d) {
    JVal v;
    v.t = JVal::Num;
    v.n = d;
    return v;
}
JVal inum(long long i) {
    JVal v;
    v.t = JVal::Num;
    v.integral = true;
    v.i = i;
    v.n = static_cast<double>(i);
    return v;
}
JVal str(const std::string& s) {
    JVal v;
    v.t = JVal::Str;
    v.s = s;
    return v;
}
JVal darr(const std::vector<double>& d) {
    JVal v;
    v.t = JVal::Arr;
    v.num_array = true;
    v.nums = d;
    v.nums_int.assign(d.size(), 0);
    return v;
}
JVal iarr(const std::vector<int>& d) {
    JVal v;
    v.t = JVal::Arr;
    v.num_array = true;
    v.nums.assign(d.begin(), d.end());
    v.nums_int.assign(d.size(), 1);
    return v;
}
JVal obj() {
    JVal v;
    v.t = JVal::Obj;
    return v;
}
JVal arr() {
    JVal v;
    v.t = JVal::Arr;
    return v;
}

void dump(const JVal& v, std::string& out, int indent, int level) {
    const bool pretty = indent >= 0;
    auto nl = [&](int lvl) {
        if (pretty) {
            out += '\n';
            out.append(static_cast<size_t>(lvl) * indent, ' ');
        }
    };
    switch (v.t) {
        case JVal::Null: out += "null"; return;
        case JVal::Bool: out += v.b ? "true" : "false"; return;
        case JVal::Num: out += v.integral ? std::to_string(v.i) : fmt_double(v.n); return;
        case JVal::Str: out += quote(v.s); return;
        case JVal::Arr: {
            const size_t n = v.size();
            if (n == 0) {
                out += "[]";
                return;
            }
            out += '[';
            for (size_t q = 0; q < n; ++q) {
                if (q) out += ',';
                nl(level + 1);
                if (v.num_array) {
                    out += v.nums_int[q] ? std::to_string(static_cast<long long>(v.nums[q])) : fmt_double(v.nums[q]);
                } else {
                    dump(v.a[q], out, indent, level + 1);
                }
            }
            nl(level);
            out += ']';
            return;
        }
        case JVal::Obj: {
            if (v.o.empty()) {
                out += "{}";
                return;
            }
            out += '{';
            bool first = true;
            for (const auto& [k, e] : v.o) {
                if (!first) out += ',';
                first = false;
                nl(level + 1);
                out += quote(k);
                out += pretty ? ": " : ":";
                dump(e, out, indent, level + 1);
            }
            nl(level);
            out += '}';
            return;
        }
    }
}

std::string dumps(const JVal& v, int indent = -1) {
    std::string s;
    dump(v, s, indent, 0);
    return s;
}

JVal spec_json(const ModelSpec& s) {
    JVal m = obj();
    m.o["num_layers"] = inum(s.num_layers);
    m.o["experts_per_layer"] = inum(s.experts_per_layer);
    m.o["top_k"] = inum(s.top_k);
    m.o["hidden_dim"] = inum(s.hidden_dim);
    return m;
}

JVal header(const char* kind) {
    JVal j = obj();
    j.o["format_version"] = inum(kFormatVersion);
    j.o["kind"] = str(kind);
    return j;
}

std::uint64_t fnv1a(const std::string& bytes) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : bytes) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

// binary trace container ----------------------------------------------------------------------
constexpr char kTraceMagic[8] = {'M', 'O', 'E', 'T', 'R', 'B', '1', '\0'};

}  // namespace

// ---- traces ----------------------------------------------------------------------------------
TraceData load_trace_file(const std::string& path) {
    const std::string text = read_file(path);
    TraceData t;
    if (text.size() >= 8 && !std::memcmp(text.data(), kTraceMagic, 8)) {
        const char* p = text.data() + 8;
        auto take = [&](void* dst, size_t n) {
            if (static_cast<size_t>(p - text.data()) + n > text.size()) fail(Status::Format, path + ": truncated binary trace");
            std::memcpy(dst, p, n);
            p += n;
        };
        int32_t hdr[6];
        take(hdr, sizeof hdr);
        t.spec = ModelSpec{hdr[0], hdr[1], hdr[2], hdr[3]};
        t.tokens = hdr[4];
        if (hdr[5] != kFormatVersion) fail(Status::Format, path + ": unsupported format_version " + std::to_string(hdr[5]));
        const size_t T = t.tokens, L = t.spec.num_layers, N = t.spec.experts_per_layer, K = t.spec.top_k,
                     D = t.spec.hidden_dim;
        t.token_index.resize(T);
        t.activations.resize(T * L * D);
        t.scores.resize(T * L * N);
        t.selected_count.resize(T * L);
        t.selected.resize(T * L * K);
        take(t.token_index.data(), T * 4);
        take(t.activations.data(), T * L * D * 8);
        take(t.scores.data(), T * L * N * 8);
        take(t.selected_count.data(), T * L * 4);
        take(t.selected.data(), T * L * K * 4);
        return t;
    }
    // JSON Lines: header, then one token per line (inc/io.hpp:146-186)
    size_t pos = 0;
    int line_no = 0;
    auto next_line = [&](std::string& line) {
        if (pos >= text.size()) return false;
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        line.assign(text, pos, e - pos);
        pos = e + 1;
        ++line_no;
        return true;
    };
    std::string line;
    if (!next_line(line)) fail(Status::Format, path + ":1: empty file");
    const JVal head = parse_text(line, path + ":1");
    check_header(head, "trace", path);
    t.spec = spec_from(head, path);
    const int L = t.spec.num_layers, N = t.spec.experts_per_layer, K = t.spec.top_k, D = t.spec.hidden_dim;
    // token lines parse independently on host threads; results (and the first error, in line
    // order) are assembled sequentially, as a one-pass reader would report them
    struct Span {
        size_t pos, len;
        int line_no;
    };
    std::vector<Span> spans;
    while (pos < text.size()) {
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        ++line_no;
        if (e > pos) spans.push_back(Span{pos, e - pos, line_no});
        pos = e + 1;
    }
    struct Parsed {
        int tok = 0;
        std::vector<double> act, sc;
        std::vector<int> cnt, sel;
        std::vector<std::string> violations;
        std::exception_ptr error;
    };
    std::vector<Parsed> parsed(spans.size());
    auto parse_line = [&](size_t q) {
        Parsed& r = parsed[q];
        try {
            const std::string where = path + ":" + std::to_string(spans[q].line_no);
            const JVal j = parse_text(std::string_view(text.data() + spans[q].pos, spans[q].len), where);
            const int tok = static_cast<int>(req_int(j, "token", where));
            const JVal* layers = j.get("layers");
            if (!layers || layers->t != JVal::Arr) schema_fail(where, "missing layers array");
            r.tok = tok;
            const int nl = static_cast<int>(layers->size());
            if (nl != L)
                r.violations.push_back("token " + std::to_string(tok) + ": expected " + std::to_string(L) +
                                       " layers, got " + std::to_string(nl));
            r.act.reserve(static_cast<size_t>(L) * D);
            r.sc.reserve(static_cast<size_t>(L) * N);
            for (int l = 0; l < L; ++l) {
                std::vector<double> act, sc;
                std::vector<int> sel;
                if (l < nl) {
                    const JVal& jl = layers->a[l];
                    act = req_doubles(jl, "activation", where);
                    sc = req_doubles(jl, "scores", where);
                    sel = req_ints(jl, "selected", where);
                    if (static_cast<int>(act.size()) != D)
                        r.violations.push_back("token " + std::to_string(tok) + " layer " + std::to_string(l) +
                                               ": activation dim " + std::to_string(act.size()) + " != " +
                                               std::to_string(D));
                    if (static_cast<int>(sc.size()) != N)
                        r.violations.push_back("token " + std::to_string(tok) + " layer " + std::to_string(l) +
                                               ": score vector length mismatch");
                }
                act.resize(D, 0.0);
                sc.resize(N, 0.0);
                r.act.insert(r.act.end(), act.begin(), act.end());
                r.sc.insert(r.sc.end(), sc.begin(), sc.end());
                r.cnt.push_back(static_cast<int>(sel.size()));
                for (int k = 0; k < K; ++k) r.sel.push_back(k < static_cast<int>(sel.size()) ? sel[k] : -1);
                if (static_cast<int>(sel.size()) > K)
                    r.violations.push_back("token " + std::to_string(tok) + " layer " + std::to_string(l) +
                                           ": selected count " + std::to_string(sel.size()));
            }
        } catch (...) {
            r.error = std::current_exception();
        }
    };
    const int n_threads = std::max(1, std::min({static_cast<int>(std::thread::hardware_concurrency()), 16,
                                                static_cast<int>(spans.size())}));
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (size_t q; (q = next.fetch_add(1)) < spans.size();) parse_line(q);
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < n_threads; ++w) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    for (const Parsed& r : parsed) {
        if (r.error) std::rethrow_exception(r.error);
        t.token_index.push_back(r.tok);
        t.shape_violations.insert(t.shape_violations.end(), r.violations.begin(), r.violations.end());
        t.activations.insert(t.activations.end(), r.act.begin(), r.act.end());
        t.scores.insert(t.scores.end(), r.sc.begin(), r.sc.end());
        t.selected_count.insert(t.selected_count.end(), r.cnt.begin(), r.cnt.end());
        t.selected.insert(t.selected.end(), r.sel.begin(), r.sel.end());
    }
    t.tokens = static_cast<int>(t.token_index.size());
    return t;
}

void save_trace_jsonl(const std::string& path, const TraceData& t) {
    const int L = t.spec.num_layers, N = t.spec.experts_per_layer, K = t.spec.top_k, D = t.spec.hidden_dim;
    JVal h = header("trace");
    h.o["model"] = spec_json(t.spec);
    // one line per token: lines are formatted independently on host threads, written in order
    std::vector<std::string> lines(t.tokens);
    auto format = [&](int tok) {
        JVal j = obj();
        j.o["token"] = inum(t.token_index.empty() ? tok : t.token_index[tok]);
        JVal layers = arr();
        for (int l = 0; l < L; ++l) {
            const size_t tl = static_cast<size_t>(tok) * L + l;
            JVal jl = obj();
            jl.o["activation"] = darr(std::vector<double>(t.activations.begin() + tl * D, t.activations.begin() + (tl + 1) * D));
            jl.o["scores"] = darr(std::vector<double>(t.scores.begin() + tl * N, t.scores.begin() + (tl + 1) * N));
            std::vector<int> sel;
            const int cnt = t.selected_count.empty() ? K : t.selected_count[tl];
            for (int k = 0; k < cnt && k < K; ++k) sel.push_back(t.selected[tl * K + k]);
            jl.o["selected"] = iarr(sel);
            layers.a.push_back(std::move(jl));
        }
        j.o["layers"] = std::move(layers);
        lines[tok] = dumps(j) + "\n";
    };
    const int n_threads = std::max(1, std::min({static_cast<int>(std::thread::hardware_concurrency()), 16, t.tokens}));
    std::atomic<int> next{0};
    std::vector<std::exception_ptr> errors(n_threads);
    auto worker = [&](int w) {
        try {
            for (int tok; (tok = next.fetch_add(1)) < t.tokens;) format(tok);
        } catch (...) {
            errors[w] = std::current_exception();
        }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < n_threads; ++w) pool.emplace_back(worker, w);
    worker(0);
    for (auto& th : pool) th.join();
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
    size_t total = 0;
    for (const auto& l : lines) total += l.size();
    std::string out = dumps(h) + "\n";
    out.reserve(out.size() + total);
    for (const auto& l : lines) out += l;
    write_file(path, out);
}

void save_trace_binary(const std::string& path, const TraceData& t) {
    const size_t T = t.tokens, L = t.spec.num_layers, N = t.spec.experts_per_layer, K = t.spec.top_k,
                 D = t.spec.hidden_dim;
    if (t.activations.size() != T * L * D || t.scores.size() != T * L * N || t.selected.size() != T * L * K)
        fail(Status::Usage, "save_trace_binary: array sizes do not match the spec");
    std::string out(kTraceMagic, 8);
    const int32_t hdr[6] = {t.spec.num_layers, t.spec.experts_per_layer, t.spec.top_k, t.spec.hidden_dim, t.tokens,
                            kFormatVersion};
    auto put = [&](const void* p, size_t n) { out.append(static_cast<const char*>(p), n); };
    put(hdr, sizeof hdr);
    std::vector<int32_t> idx(T), cnt(T * L, static_cast<int32_t>(K));
    for (size_t q = 0; q < T; ++q) idx[q] = t.token_index.empty() ? static_cast<int32_t>(q) : t.token_index[q];
    if (!t.selected_count.empty()) cnt.assign(t.selected_count.begin(), t.selected_count.end());
    put(idx.data(), T * 4);
    put(t.activations.data(), T * L * D * 8);
    put(t.scores.data(), T * L * N * 8);
    put(cnt.data(), T * L * 4);
    put(t.selected.data(), T * L * K * 4);
    write_file(path, out);
}

// inc/core.hpp:249-297 (kScoreTolerance, inc/core.hpp)
std::vector<std::string> validate_trace(const TraceData& t) {
    constexpr double kScoreTolerance = 1e-6;
    std::vector<std::string> v = t.shape_violations;
    const int L = t.spec.num_layers, N = t.spec.experts_per_layer, K = t.spec.top_k;
    for (int tok = 0; tok < t.tokens; ++tok)
        for (int l = 0; l < L; ++l) {
            const size_t tl = static_cast<size_t>(tok) * L + l;
            const std::string at = "token " + std::to_string(t.token_index[tok]) + " layer " + std::to_string(l) + ": ";
            double sum = 0.0;
            bool negative = false;
            for (int j = 0; j < N; ++j) {
                sum += t.scores[tl * N + j];
                negative |= t.scores[tl * N + j] < 0.0;
            }
            if (negative) v.push_back(at + "negative score");
            if (std::abs(sum - 1.0) > kScoreTolerance) v.push_back(at + "score normalization: sum " + std::to_string(sum));
            const int cnt = t.selected_count[tl];
            if (cnt != 1 && cnt != K) v.push_back(at + "selected count " + std::to_string(cnt));
            std::vector<int> seen;
            for (int k = 0; k < std::min(cnt, K); ++k) {
                const int e = t.selected[tl * K + k];
                if (e < 0 || e >= N)
                    v.push_back(at + "expert index out of range: " + std::to_string(e));
                else if (std::find(seen.begin(), seen.end(), e) != seen.end())
                    v.push_back(at + "duplicate selected expert: " + std::to_string(e));
                seen.push_back(e);
            }
        }
    return v;
}

// ---- gates -----------------------------------------------------------------------------------
namespace {
JVal gate_json(const std::vector<double>& w, int d, int n) {
    JVal g = obj();
    g.o["hidden_dim"] = inum(d);
    g.o["num_experts"] = inum(n);
    g.o["weights"] = darr(w);
    return g;
}
std::vector<double> gate_from(const JVal& jg, const std::string& path, int d, int n) {
    const int gd = static_cast<int>(req_int(jg, "hidden_dim", path));
    const int gn = static_cast<int>(req_int(jg, "num_experts", path));
    std::vector<double> w = req_doubles(jg, "weights", path);
    if (w.size() != static_cast<size_t>(gd) * gn) schema_fail(path, "gate weight count does not match shape");
    if (gd != d || gn != n) fail(Status::Validation, path + ": gate shape does not match the model");
    return w;
}
}  // namespace

GatesData load_gates_file(const std::string& path) {
    const JVal j = parse_text(read_file(path), path);
    check_header(j, "gates", path);
    GatesData g;
    g.spec = spec_from(j, path);
    const JVal* arr_g = j.get("gates");
    if (!arr_g || arr_g->t != JVal::Arr) schema_fail(path, "missing gates array");
    const int D = g.spec.hidden_dim, N = g.spec.experts_per_layer;
    if (static_cast<int>(arr_g->size()) != g.spec.num_layers)
        fail(Status::Validation, path + ": gate count does not match num_layers");
    for (const JVal& jg : arr_g->a) {
        std::vector<double> w = gate_from(jg, path, D, N);
        g.gates.insert(g.gates.end(), w.begin(), w.end());
    }
    const JVal* jp = j.get("predictive_gate");
    if (jp && jp->t != JVal::Null) {
        const JVal* pg = jp->get("gate");
        if (!pg) schema_fail(path, "predictive_gate missing gate");
        g.first_gate = gate_from(*pg, path, D, N);
        g.learning_rate = req_double(*jp, "learning_rate", path);
        g.steps = static_cast<int>(req_int(*jp, "steps", path));
        g.seed = static_cast<std::uint64_t>(req_int(*jp, "seed", path));
    }
    return g;
}

void save_gates_file(const std::string& path, const GatesData& g) {
    const int L = g.spec.num_layers, D = g.spec.hidden_dim, N = g.spec.experts_per_layer;
    JVal j = header("gates");
    j.o["model"] = spec_json(g.spec);
    JVal gates = arr();
    const size_t one = static_cast<size_t>(D) * N;
    for (int l = 0; l < L; ++l)
        gates.a.push_back(gate_json(std::vector<double>(g.gates.begin() + l * one, g.gates.begin() + (l + 1) * one), D, N));
    j.o["gates"] = std::move(gates);
    if (g.first_gate) {
        JVal p = obj();
        p.o["gate"] = gate_json(*g.first_gate, D, N);
        p.o["learning_rate"] = num(g.learning_rate);
        p.o["steps"] = inum(g.steps);
        p.o["seed"] = inum(static_cast<long long>(g.seed));
        j.o["predictive_gate"] = std::move(p);
    }
    write_file(path, dumps(j, 2) + "\n");
}

// ---- profiles / threshold / allocation / cost table -------------------------------------------
namespace {
JVal profiles_json(const ProfilesData& p) {
    JVal j = header("profiles");
    j.o["model"] = spec_json(p.spec);
    JVal layers = arr();
    for (size_t l = 0; l < p.alpha.size(); ++l) {
        JVal e = obj();
        e.o["single_expert_prob"] = num(p.alpha[l]);
        e.o["prefetch_accuracy"] = num(p.beta[l]);
        e.o["fisher_diag_sum"] = num(p.fisher[l]);
        layers.a.push_back(std::move(e));
    }
    j.o["layers"] = std::move(layers);
    return j;
}
}  // namespace

ProfilesData load_profiles_file(const std::string& path) {
    const JVal j = parse_text(read_file(path), path);
    check_header(j, "profiles", path);
    ProfilesData p;
    p.spec = spec_from(j, path);
    const JVal* layers = j.get("layers");
    if (!layers || layers->t != JVal::Arr) schema_fail(path, "missing layers array");
    for (const JVal& jl : layers->a) {
        p.alpha.push_back(req_double(jl, "single_expert_prob", path));
        p.beta.push_back(req_double(jl, "prefetch_accuracy", path));
        p.fisher.push_back(req_double(jl, "fisher_diag_sum", path));
    }
    return p;
}

void save_profiles_file(const std::string& path, const ProfilesData& p) { write_file(path, dumps(profiles_json(p), 2) + "\n"); }

std::string profile_hash(const ProfilesData& p) {
    std::uint64_t v = fnv1a(dumps(profiles_json(p)));
    static const char* digits = "0123456789abcdef";
    std::string out(16, '0');
    for (int i = 15; i >= 0; --i) {
        out[i] = digits[v & 0xf];
        v >>= 4;
    }
    return out;
}

ThresholdData load_threshold_file(const std::string& path) {
    const JVal j = parse_text(read_file(path), path);
    check_header(j, "threshold", path);
    return ThresholdData{req_double(j, "tau", path), req_double(j, "target_single_ratio", path),
                         req_double(j, "realized_single_ratio", path)};
}

void save_threshold_file(const std::string& path, const ThresholdData& t) {
    JVal j = header("threshold");
    j.o["tau"] = num(t.tau);
    j.o["target_single_ratio"] = num(t.target_single_ratio);
    j.o["realized_single_ratio"] = num(t.realized_single_ratio);
    write_file(path, dumps(j, 2) + "\n");
}

AllocationData load_allocation_file(const std::string& path) {
    const JVal j = parse_text(read_file(path), path);
    check_header(j, "allocation", path);
    AllocationData a;
    a.budget = static_cast<int>(req_int(j, "budget", path));
    a.capacities = req_ints(j, "capacities", path);
    a.total_cost = req_double(j, "total_cost", path);
    a.profile_hash = req_string(j, "profile_hash", path);
    return a;
}

void save_allocation_file(const std::string& path, const AllocationData& a) {
    JVal j = header("allocation");
    j.o["budget"] = inum(a.budget);
    j.o["capacities"] = iarr(a.capacities);
    j.o["total_cost"] = num(a.total_cost);
    j.o["profile_hash"] = str(a.profile_hash);
    write_file(path, dumps(j, 2) + "\n");
}

CostTableData load_cost_table_file(const std::string& path) {
    const JVal j = parse_text(read_file(path), path);
    check_header(j, "cost_table", path);
    CostTableData c;
    c.experts_per_layer = static_cast<int>(req_int(j, "experts_per_layer", path));
    const JVal& loads = field(j, "loads", path);
    if (loads.t != JVal::Arr) wrong_type("loads", path);
    for (const JVal& row : loads.a) {
        if (row.t != JVal::Arr || !row.num_array) wrong_type("loads", path);
        c.loads.push_back(row.nums);
    }
    return c;
}

void save_cost_table_file(const std::string& path, const CostTableData& c) {
    JVal j = header("cost_table");
    j.o["experts_per_layer"] = inum(c.experts_per_layer);
    JVal loads = arr();
    for (const auto& row : c.loads) loads.a.push_back(darr(row));
    j.o["loads"] = std::move(loads);
    write_file(path, dumps(j, 2) + "\n");
}

}  // namespace adapmoe
