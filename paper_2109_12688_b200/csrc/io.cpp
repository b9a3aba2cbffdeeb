// DREG volume container and JSON run report (reference io.hpp:15-67, io.cpp).
//
// Host-side file formats around the registration path: the
// GPU library reads and writes the reference's on-disk volumes and deformation fields
// byte-for-byte, so files move between the two implementations unchanged.
//
// Container (little-endian, io.hpp:15-22, README.md:99-114):
//   0 "DREG" | 4 u32 version 1 | 8 u8 kind (0 scalar, 1 vector, 2 label)
//   9 3 x u32 dims (M, N, H) | 21 3 x f64 spacing | 45 payload
// Payload: f32 (scalar M*N*H, vector 3*M*N*H interleaved) or u16 (label), x fastest.
// Readers reject, in this order (io.cpp:88-158): short header, bad magic, version,
// kind > 2, an extent outside [1, 65536], more than 2^31 voxels, non-finite or
// non-positive spacing, a short payload, trailing bytes, a non-finite f32 value.
//
// Report (io.cpp:263-298): an insertion-ordered JSON object dumped with a 2-space
// indent; every double rounded to 6 significant digits ("%.6g" then strtod) and
// printed with the digits and number layout of the reference's
// JSON serialiser (integral doubles keep ".0", exponents carry a sign and >= 2 digits).
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "dreg_cuda.h"

namespace {

constexpr size_t kHeader = 45;
constexpr uint32_t kVersion = 1;
constexpr uint32_t kMaxExtent = 65536;

struct IoFail {
    std::string msg;
};

void set_err(char* err, size_t len, const std::string& m) {
    if (!err || len == 0) return;
    const size_t n = m.size() < len - 1 ? m.size() : len - 1;
    std::memcpy(err, m.data(), n);
    err[n] = '\0';
}

template <class F>
int io_guard(char* err, size_t len, F&& f) {
    try {
        f();
        set_err(err, len, "");
        return DREG_OK;
    } catch (const IoFail& e) {
        set_err(err, len, e.msg);
        return DREG_IO_ERROR;
    } catch (const std::bad_alloc&) {
        set_err(err, len, "host allocation failed");
        return DREG_RUNTIME;
    }
}

uint32_t rd32(const unsigned char* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
uint64_t rd64(const unsigned char* p) {
    return (uint64_t)rd32(p) | ((uint64_t)rd32(p + 4) << 32);
}
void wr32(unsigned char* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (unsigned char)(v >> (8 * i));
}
void wr64(unsigned char* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (unsigned char)(v >> (8 * i));
}
double as_f64(uint64_t b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}
uint64_t f64_bits(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// Whole-file read; the reference also loads the file in one piece (io.cpp:150-163).
std::vector<unsigned char> slurp(const std::string& path, size_t limit) {
    File h;
    h.f = std::fopen(path.c_str(), "rb");
    if (!h.f) throw IoFail{"cannot open: " + path};
    if (std::fseek(h.f, 0, SEEK_END) != 0) throw IoFail{"read failed: " + path};
    const long size = std::ftell(h.f);
    if (size < 0) throw IoFail{"read failed: " + path};
    std::fseek(h.f, 0, SEEK_SET);
    const size_t want = limit < (size_t)size ? limit : (size_t)size;
    std::vector<unsigned char> bytes(want);
    if (want && std::fread(bytes.data(), 1, want, h.f) != want) throw IoFail{"read failed: " + path};
    return bytes;
}

dreg_volume_info decode_header(const unsigned char* b, size_t size, const std::string& path) {
    if (size < kHeader) throw IoFail{"truncated header: " + path};
    if (std::memcmp(b, "DREG", 4) != 0) throw IoFail{"bad magic: " + path};
    if (rd32(b + 4) != kVersion) throw IoFail{"unsupported version: " + path};
    if (b[8] > 2) throw IoFail{"unknown volume kind: " + path};
    dreg_volume_info h{};
    h.kind = b[8];
    uint64_t voxels = 1;
    uint32_t ext[3];
    for (int a = 0; a < 3; ++a) {
        ext[a] = rd32(b + 9 + 4 * a);
        if (ext[a] < 1 || ext[a] > kMaxExtent) throw IoFail{"dims out of range: " + path};
        voxels *= ext[a];
    }
    if (voxels > (uint64_t{1} << 31)) throw IoFail{"volume too large: " + path};
    h.dims = {(int)ext[0], (int)ext[1], (int)ext[2]};
    h.spacing = {as_f64(rd64(b + 21)), as_f64(rd64(b + 29)), as_f64(rd64(b + 37))};
    const double s[3] = {h.spacing.x, h.spacing.y, h.spacing.z};
    for (double v : s)
        if (!std::isfinite(v) || v <= 0.0) throw IoFail{"invalid spacing: " + path};
    return h;
}

size_t payload_bytes(const dreg_volume_info& h) {
    const size_t n = (size_t)h.dims.x * h.dims.y * h.dims.z;
    return h.kind == DREG_KIND_LABEL ? 2 * n : (h.kind == DREG_KIND_VECTOR ? 12 * n : 4 * n);
}

const char* kind_name(int kind) {
    return kind == DREG_KIND_SCALAR ? "a scalar volume" : kind == DREG_KIND_VECTOR ? "a vector field" : "a label volume";
}

// ---- JSON numbers ------------------------------------------------------------------
double sig6(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6g", v);
    return std::strtod(buf, nullptr);
}

// Decimal digits of a positive finite double by Grisu2 (Loitsch, "Printing
// Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010), the
// algorithm of the reference's JSON serialiser (nlohmann::json 3.x, the library
// io.cpp:11 includes; not vendored in the reference tree).  Grisu2 is not always
// shortest (e.g. 6.600579999999999e+20 for sig6(6.60058e20)), so matching its exact
// digit choice -- boundary shrink by one unit, alpha/gamma = -60/-32 cached powers of
// ten, round-to-nearest 64x64 products, the weed-out rounding loop -- is what makes the
// report text byte-identical.  value = digits * 10^exp10.
struct Fp {
    uint64_t f;
    int e;
};

Fp fp_mul(Fp x, Fp y) {  // 64x64 -> upper 64 bits, rounded half up
    const uint64_t a = x.f >> 32, b = x.f & 0xffffffffu, c = y.f >> 32, d = y.f & 0xffffffffu;
    const uint64_t ac = a * c, bc = b * c, ad = a * d, bd = b * d;
    uint64_t mid = (bd >> 32) + (ad & 0xffffffffu) + (bc & 0xffffffffu);
    mid += uint64_t{1} << 31;
    return {ac + (ad >> 32) + (bc >> 32) + (mid >> 32), x.e + y.e + 64};
}

Fp fp_norm(Fp x) {
    while (!(x.f >> 63)) {
        x.f <<= 1;
        x.e -= 1;
    }
    return x;
}

struct Pow10 {
    uint64_t f;
    int e;
    int k;
};

// 10^k for k = -300, -292, ..., 324: 64-bit significand rounded to nearest.
const Pow10 kPow10[] = {
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

void grisu2(double v, std::string& digits, int& exp10) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
    const int E = (int)(bits >> 52);
    const Fp w0 = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (uint64_t{1} << 52), E - 1075};
    const bool closer_below = F == 0 && E > 1;
    const Fp hi = fp_norm({2 * w0.f + 1, w0.e - 1});
    Fp lo = closer_below ? Fp{4 * w0.f - 1, w0.e - 2} : Fp{2 * w0.f - 1, w0.e - 1};
    lo = {lo.f << (lo.e - hi.e), hi.e};
    const Fp w = fp_norm(w0);

    // cached power c = 10^-k with -60 <= e_c + hi.e + 64 <= -32
    const int t = -60 - hi.e - 1;
    const int k = (t * 78913) / (1 << 18) + (t > 0 ? 1 : 0);
    const Pow10& c = kPow10[(300 + k + 7) / 8];
    const Fp cf{c.f, c.e};
    const Fp W = fp_mul(w, cf);
    Fp Mlo = fp_mul(lo, cf), Mhi = fp_mul(hi, cf);
    Mlo.f += 1;  // shrink the rounding interval by one unit on both sides
    Mhi.f -= 1;
    exp10 = -c.k;

    uint64_t delta = Mhi.f - Mlo.f;
    uint64_t dist = Mhi.f - W.f;
    const int sh = -Mhi.e;
    const uint64_t one = uint64_t{1} << sh;
    uint32_t p1 = (uint32_t)(Mhi.f >> sh);
    uint64_t p2 = Mhi.f & (one - 1);
    digits.clear();

    auto weed = [&](uint64_t rest, uint64_t ten_k) {
        while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
            digits.back() = (char)(digits.back() - 1);
            rest += ten_k;
        }
    };

    int n = 1;
    uint32_t pow10 = 1;
    while (n < 10 && p1 >= pow10 * 10ull) {
        pow10 *= 10;
        ++n;
    }
    while (n > 0) {
        digits.push_back((char)('0' + p1 / pow10));
        p1 %= pow10;
        --n;
        const uint64_t rest = ((uint64_t)p1 << sh) + p2;
        if (rest <= delta) {
            exp10 += n;
            weed(rest, (uint64_t)pow10 << sh);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        digits.push_back((char)('0' + (p2 >> sh)));
        p2 &= one - 1;
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    exp10 -= m;
    weed(p2, one);
}

// Number layout of the reference's serialiser (min_exp -4, max_exp 15).
std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    std::string out = v < 0 ? "-" : "";
    std::string d;
    int e10;
    grisu2(std::fabs(v), d, e10);
    const int k = (int)d.size();
    const int n = k + e10;  // decimal point position
    if (k <= n && n <= 15) {
        out += d + std::string((size_t)(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += d.substr(0, (size_t)n) + "." + d.substr((size_t)n);
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string((size_t)(-n), '0') + d;
    } else {
        out += d.substr(0, 1);
        if (k > 1) out += "." + d.substr(1);
        const int e = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

std::string json_string(const char* s) {
    std::string out = "\"";
    for (const char* c = s ? s : ""; *c; ++c) {
        const unsigned char u = (unsigned char)*c;
        switch (u) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (u < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", u);
                    out += b;
                } else {
                    out += (char)u;
                }
        }
    }
    return out + "\"";
}

std::string label_map(int n, const int* labels, const double* values, const std::string& indent) {
    std::map<int, double> m;  // RunReport keeps std::map<int, double> (io.hpp:60-61)
    for (int i = 0; i < n; ++i) m[labels[i]] = values[i];
    if (m.empty()) return "{}";
    std::string out = "{\n";
    bool first = true;
    for (const auto& [label, value] : m) {
        if (!first) out += ",\n";
        first = false;
        out += indent + "  " + json_string(std::to_string(label).c_str()) + ": " + json_double(sig6(value));
    }
    return out + "\n" + indent + "}";
}

}  // namespace

extern "C" {

int dreg_volume_info_read(const char* path, dreg_volume_info* out, char* err, size_t err_len) {
    return io_guard(err, err_len, [&] {
        if (!path || !out) throw IoFail{"null argument"};
        const auto b = slurp(path, kHeader);
        *out = decode_header(b.data(), b.size(), path);
    });
}

int dreg_volume_read(const char* path, int expected_kind, dreg_volume_info* info, void* payload,
                     size_t capacity, char* err, size_t err_len) {
    return io_guard(err, err_len, [&] {
        if (!path) throw IoFail{"null argument"};
        const std::string p = path;
        const auto b = slurp(p, (size_t)-1);
        const dreg_volume_info h = decode_header(b.data(), b.size(), p);
        const size_t need = kHeader + payload_bytes(h);
        if (b.size() < need) throw IoFail{"truncated payload: " + p};
        if (b.size() > need) throw IoFail{"trailing bytes: " + p};
        if (h.kind != DREG_KIND_LABEL) {
            const unsigned char* q = b.data() + kHeader;
            for (size_t i = 0; i < payload_bytes(h); i += 4) {
                const uint32_t bits = rd32(q + i);
                float f;
                std::memcpy(&f, &bits, 4);
                if (!std::isfinite(f)) throw IoFail{"non-finite payload value: " + p};
            }
        }
        if (expected_kind >= 0 && h.kind != expected_kind)
            throw IoFail{std::string("expected ") + kind_name(expected_kind) + ": " + p};
        if (info) *info = h;
        if (payload) {
            if (capacity < payload_bytes(h)) throw IoFail{"payload buffer too small: " + p};
            // the container is little-endian like the host; copy the words as stored
            std::memcpy(payload, b.data() + kHeader, payload_bytes(h));
        }
    });
}

int dreg_volume_write(const char* path, int kind, dreg_dims3 dims, dreg_spacing3 spacing, const void* payload,
                      char* err, size_t err_len) {
    return io_guard(err, err_len, [&] {
        if (!path || !payload) throw IoFail{"null argument"};
        if (kind < 0 || kind > 2) throw IoFail{"unknown volume kind"};
        if (dims.x < 1 || dims.y < 1 || dims.z < 1) throw IoFail{"volume dims must be positive"};
        dreg_volume_info h{kind, dims, spacing};
        const size_t nb = payload_bytes(h);
        std::vector<unsigned char> bytes(kHeader + nb);
        unsigned char* b = bytes.data();
        std::memcpy(b, "DREG", 4);
        wr32(b + 4, kVersion);
        b[8] = (unsigned char)kind;
        wr32(b + 9, (uint32_t)dims.x);
        wr32(b + 13, (uint32_t)dims.y);
        wr32(b + 17, (uint32_t)dims.z);
        wr64(b + 21, f64_bits(spacing.x));
        wr64(b + 29, f64_bits(spacing.y));
        wr64(b + 37, f64_bits(spacing.z));
        std::memcpy(b + kHeader, payload, nb);
        File h2;
        h2.f = std::fopen(path, "wb");
        if (!h2.f) throw IoFail{std::string("cannot open for writing: ") + path};
        if (std::fwrite(b, 1, bytes.size(), h2.f) != bytes.size() || std::fflush(h2.f) != 0)
            throw IoFail{std::string("write failed: ") + path};
    });
}

int dreg_report_write(const char* path, const dreg_run_report* r, char* err, size_t err_len) {
    return io_guard(err, err_len, [&] {
        if (!path || !r) throw IoFail{"null argument"};
        const dreg_report_config& c = r->config;
        std::string j = "{\n";
        j += "  \"dice\": " + label_map(r->n_dice, r->dice_labels, r->dice, "  ") + ",\n";
        j += "  \"hausdorff_mm\": " + label_map(r->n_hausdorff, r->hausdorff_labels, r->hausdorff_mm, "  ") + ",\n";
        j += "  \"jacobian_pct_nonpositive\": " + json_double(sig6(r->jacobian_pct_nonpositive)) + ",\n";
        j += "  \"runtime_seconds\": " + json_double(sig6(r->runtime_seconds)) + ",\n";
        j += "  \"velocity_count\": " + std::to_string(r->velocity_count) + ",\n";
        j += "  \"config\": {\n";
        j += "    \"data_term\": " + json_string(c.data_term) + ",\n";
        j += "    \"order\": " + std::to_string(c.order) + ",\n";
        j += "    \"lambda\": " + json_double(sig6(c.lambda)) + ",\n";
        j += "    \"theta\": " + json_double(sig6(c.theta)) + ",\n";
        j += "    \"levels\": " + std::to_string(c.levels) + ",\n";
        j += "    \"profile\": " + json_string(c.profile) + ",\n";
        j += "    \"tol\": " + json_double(sig6(c.tol)) + ",\n";
        j += "    \"warp_improvement_threshold\": " + json_double(sig6(c.warp_improvement_threshold)) + ",\n";
        j += "    \"epsilon\": " + json_double(sig6(c.epsilon)) + ",\n";
        j += "    \"threads\": " + std::to_string(c.threads) + "\n";
        j += "  }\n}\n";
        File h;
        h.f = std::fopen(path, "w");
        if (!h.f) throw IoFail{std::string("cannot open for writing: ") + path};
        if (std::fwrite(j.data(), 1, j.size(), h.f) != j.size() || std::fflush(h.f) != 0)
            throw IoFail{std::string("write failed: ") + path};
    });
}

}  // extern "C"
