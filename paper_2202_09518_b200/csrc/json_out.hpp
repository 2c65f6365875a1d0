// Minimal JSON value + writer whose dump() reproduces the byte layout of the reference's
// nlohmann::json::dump() as the reference is compiled in this image (nlohmann 3.11.3 from
// cudnn_frontend's thirdparty tree, oracle/Makefile): object keys in sorted order (std::map),
// `"key": value` with an `indent`-space step, arrays of integers on one line (`[0,45]`, that
// tree's patch) and every other non-empty array one element per line, floats as nlohmann's
// to_chars writes them (Grisu2 digits, below; integral values get ".0"; non-finite -> null),
// strings escaped like
// dump_escaped(ensure_ascii = false). Used by SelectionReport::to_json and the oocnmf CLI's
// counters / stats / manifest files (tools/oocnmf_cli.cpp:74-104,166-195). Pinned against the
// compiled nlohmann by tests/test_cli_cpu.py (parse + dump is a fixed point of this output).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace oocnmf::jsonout {

class Json {
public:
    enum class Type { null, boolean, integer, unsigned_integer, floating, string, array, object };

    Json() = default;
    Json(std::nullptr_t) {}
    Json(bool b) : t_(Type::boolean), b_(b) {}
    Json(int v) : t_(Type::integer), i_(v) {}
    Json(long v) : t_(Type::integer), i_(v) {}
    Json(long long v) : t_(Type::integer), i_(v) {}
    Json(unsigned v) : t_(Type::unsigned_integer), u_(v) {}
    Json(unsigned long v) : t_(Type::unsigned_integer), u_(v) {}
    Json(unsigned long long v) : t_(Type::unsigned_integer), u_(v) {}
    Json(double v) : t_(Type::floating), d_(v) {}
    Json(const char* s) : t_(Type::string), s_(s) {}
    Json(std::string s) : t_(Type::string), s_(std::move(s)) {}

    static Json array() {
        Json j;
        j.t_ = Type::array;
        return j;
    }
    static Json object() {
        Json j;
        j.t_ = Type::object;
        return j;
    }

    Type type() const { return t_; }
    Json& operator[](const std::string& key) {
        if (t_ == Type::null) t_ = Type::object;
        return o_[key];
    }
    void push_back(Json v) {
        if (t_ == Type::null) t_ = Type::array;
        a_.push_back(std::move(v));
    }

    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

private:
    Type t_ = Type::null;
    bool b_ = false;
    std::int64_t i_ = 0;
    std::uint64_t u_ = 0;
    double d_ = 0;
    std::string s_;
    std::vector<Json> a_;
    std::map<std::string, Json> o_;

    static void escaped(std::string& out, const std::string& s) {
        for (unsigned char ch : s) {
            switch (ch) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                case '\n': out += "\\n"; break;
                case '\r': out += "\\r"; break;
                case '\t': out += "\\t"; break;
                default:
                    if (ch < 0x20) {
                        char b[8];
                        std::snprintf(b, sizeof b, "\\u%04x", unsigned(ch));
                        out += b;
                    } else {
                        out += char(ch);
                    }
            }
        }
    }

public:
    // Float text as nlohmann::detail::to_chars writes it: Grisu2 (Loitsch, "Printing
    // Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010) with the rounding
    // interval narrowed by one unit on each side, cached powers 10^k for k = -300, -292, ..., 324
    // and target binary exponents in [-60, -32]; then fixed notation for decimal point positions
    // in (-4, 15], else d.ddde±XX. Grisu2 is not always the shortest round-trip string (e.g.
    // 1.1607702651454979e+17), which is why the digits are generated here rather than by
    // std::to_chars.
    static std::string number(double x) {
        if (!std::isfinite(x)) return "null";
        std::string out;
        if (std::signbit(x)) out += '-', x = -x;
        if (x == 0) return out + "0.0";
        char digits[24];
        int len = 0, dexp = 0;
        grisu2(x, digits, len, dexp);
        const int k = len, n = len + dexp;  // value = digits * 10^dexp, point after n digits
        const std::string d(digits, std::size_t(len));
        if (k <= n && n <= 15) {
            out += d + std::string(std::size_t(n - k), '0') + ".0";
        } else if (0 < n && n <= 15) {
            out += d.substr(0, std::size_t(n)) + "." + d.substr(std::size_t(n));
        } else if (-4 < n && n <= 0) {
            out += "0." + std::string(std::size_t(-n), '0') + d;
        } else {
            out += d.substr(0, 1);
            if (k > 1) out += "." + d.substr(1);
            const int ex = n - 1;
            char b[16];
            std::snprintf(b, sizeof b, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
            out += b;
        }
        return out;
    }

private:
    struct Fp {  // f * 2^e
        std::uint64_t f;
        int e;
    };
    static Fp mul(Fp a, Fp b) {  // upper 64 bits of the 128-bit product, rounded half up
        const unsigned __int128 p = (unsigned __int128)a.f * b.f + ((unsigned __int128)1 << 63);
        return {std::uint64_t(p >> 64), a.e + b.e + 64};
    }
    static Fp normalize(Fp x) {
        while (!(x.f >> 63)) x.f <<= 1, --x.e;
        return x;
    }
    struct Cached {
        std::uint64_t f;
        int e, k;
    };
    // round-to-nearest 64-bit significands of 10^k (tools-independent constants)
    static constexpr Cached kPowers[79] = {
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
        {0x9E19DB92B4E31BA9ULL, 1013, 324}};

    static void grisu2(double value, char* buf, int& len, int& dexp) {
        std::uint64_t bits;
        std::memcpy(&bits, &value, 8);
        const std::uint64_t F = bits & ((std::uint64_t(1) << 52) - 1);
        const int E = int(bits >> 52);
        const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (std::uint64_t(1) << 52), E - 1075};
        const bool lower_closer = F == 0 && E > 1;
        const Fp mp = normalize({2 * v.f + 1, v.e - 1});
        Fp mm = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
        mm = {mm.f << (mm.e - mp.e), mp.e};
        const Fp w = normalize(v);
        // cached power 10^-k bringing the exponent into [-60, -32]
        const int f = -60 - mp.e - 1;
        const int kk = (f * 78913) / (1 << 18) + (f > 0);
        const Cached& c = kPowers[(300 + kk + 7) / 8];
        const Fp cm{c.f, c.e};
        const Fp W = mul(w, cm), Wm = mul(mm, cm), Wp = mul(mp, cm);
        const Fp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
        dexp = -c.k;
        len = 0;
        digit_gen(buf, len, dexp, Mm, W, Mp);
    }

    static void round_weed(char* buf, int len, std::uint64_t dist, std::uint64_t delta, std::uint64_t rest,
                           std::uint64_t ten_k) {
        while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
            buf[len - 1]--;
            rest += ten_k;
        }
    }

    static void digit_gen(char* buf, int& len, int& dexp, Fp Mm, Fp w, Fp Mp) {
        std::uint64_t delta = Mp.f - Mm.f, dist = Mp.f - w.f;
        const int sh = -Mp.e;
        const std::uint64_t one = std::uint64_t(1) << sh;
        std::uint32_t p1 = std::uint32_t(Mp.f >> sh);
        std::uint64_t p2 = Mp.f & (one - 1);
        std::uint32_t pow10 = 1;
        int n = 1;
        while (n < 10 && p1 >= pow10 * 10u) pow10 *= 10u, ++n;
        while (n > 0) {
            const std::uint32_t d = p1 / pow10;
            p1 %= pow10;
            buf[len++] = char('0' + d);
            --n;
            const std::uint64_t rest = (std::uint64_t(p1) << sh) + p2;
            if (rest <= delta) {
                dexp += n;
                round_weed(buf, len, dist, delta, rest, std::uint64_t(pow10) << sh);
                return;
            }
            pow10 /= 10u;
        }
        int m = 0;
        for (;;) {
            p2 *= 10, delta *= 10, dist *= 10;
            buf[len++] = char('0' + (p2 >> sh));
            p2 &= one - 1;
            ++m;
            if (p2 <= delta) break;
        }
        dexp -= m;
        round_weed(buf, len, dist, delta, p2, one);
    }

private:
    void write(std::string& out, int indent, int cur) const {
        const bool pretty = indent >= 0;
        switch (t_) {
            case Type::null: out += "null"; return;
            case Type::boolean: out += b_ ? "true" : "false"; return;
            case Type::integer: out += std::to_string(i_); return;
            case Type::unsigned_integer: out += std::to_string(u_); return;
            case Type::floating: out += number(d_); return;
            case Type::string:
                out += '"';
                escaped(out, s_);
                out += '"';
                return;
            case Type::array: {
                if (a_.empty()) {
                    out += "[]";
                    return;
                }
                const bool ints = a_[0].t_ == Type::integer || a_[0].t_ == Type::unsigned_integer;
                if (pretty && !ints) {
                    out += "[\n";
                    for (std::size_t i = 0; i < a_.size(); ++i) {
                        out += std::string(std::size_t(cur + indent), ' ');
                        a_[i].write(out, indent, cur + indent);
                        out += i + 1 < a_.size() ? ",\n" : "\n";
                    }
                    out += std::string(std::size_t(cur), ' ') + "]";
                } else {
                    out += '[';
                    for (std::size_t i = 0; i < a_.size(); ++i) {
                        a_[i].write(out, -1, cur);
                        if (i + 1 < a_.size()) out += ',';
                    }
                    out += ']';
                }
                return;
            }
            case Type::object: {
                if (o_.empty()) {
                    out += "{}";
                    return;
                }
                out += pretty ? "{\n" : "{";
                std::size_t i = 0;
                for (const auto& [key, val] : o_) {
                    if (pretty) out += std::string(std::size_t(cur + indent), ' ');
                    out += '"';
                    escaped(out, key);
                    out += pretty ? "\": " : "\":";
                    val.write(out, indent, cur + indent);
                    if (++i < o_.size()) out += pretty ? ",\n" : ",";
                }
                if (pretty) out += "\n" + std::string(std::size_t(cur), ' ');
                out += '}';
                return;
            }
        }
    }
};

}  // namespace oocnmf::jsonout
