// Host orchestration of the B200 FlashIPA layer.  See layer.hpp.
#include "layer.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <tuple>
#include <mutex>
#include <numbers>
#include <sstream>
#include <thread>

namespace fipa_b200 {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

namespace {

template <class... P>
std::string cat(P&&... parts) {
    std::ostringstream os;
    (os << ... << parts);
    return os.str();
}

#define REQUIRE(cond, ...)                                      \
    do {                                                        \
        if (!(cond)) throw ::fipa_b200::ValueError(cat(__VA_ARGS__)); \
    } while (0)

std::size_t round_up(std::size_t x, std::size_t m) { return (x + m - 1) / m * m; }

// Inference attention kernel: the CTA-pair kernel where its budget allows, the two-pass pair
// kernel for wider lifted rows (rank 3-4), else the single-CTA kernel.  Tuning::attn forces an
// alternative (A/B checks); the single-CTA kernel does not read sharded keys, so a sharded
// forward never takes it.
enum class AttnImpl { pair, pass, one_sm };
// bf16 dK / dV hand-off to the unpack (AttnBwdArgs::dk16); FIPA_BF16_ACC=0 keeps them fp32 (A/B)
bool bf16_acc_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FIPA_BF16_ACC");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}
AttnImpl attention_impl(const LayerDims& d, Tuning::Attn forced, bool sharded) {
    if (forced == Tuning::Attn::one_sm && !sharded) return AttnImpl::one_sm;
    if (forced == Tuning::Attn::pass && attn_fwd_pass_supported(d)) return AttnImpl::pass;
    if (attn_fwd_2sm_supported(d)) return AttnImpl::pair;
    if (attn_fwd_pass_supported(d)) return AttnImpl::pass;
    return AttnImpl::one_sm;
}
bool bf16_attention_supported(const LayerDims& d) {
    return attn_fwd_2sm_supported(d) || attn_fwd_pass_supported(d);
}

// ------------------------------------------------------------------ Rng
// Counter-based splitmix64 + Box-Muller, bit-identical to the reference generator
// (proj/src/rng.cpp:11-41): draw n = mix64(seed + n*golden), uniform in (0,1].
class Rng {
public:
    explicit Rng(std::uint64_t seed) : seed_(seed) {}
    std::uint64_t next_u64() {
        counter_ += 1;
        std::uint64_t z = seed_ + counter_ * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
    double gaussian() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        const double u1 = uniform();
        const double u2 = uniform();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * std::numbers::pi * u2;
        spare_ = radius * std::sin(angle);
        have_spare_ = true;
        return radius * std::cos(angle);
    }

private:
    std::uint64_t seed_;
    std::uint64_t counter_ = 0;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

std::size_t numel(const std::vector<std::size_t>& s) {
    std::size_t n = 1;
    for (auto d : s) n *= d;
    return n;
}

constexpr double kGammaRawUnit = 0.5413248546129181;  // ln(e - 1), proj/src/ipa.cpp:30

double softplus(double x) {  // proj/src/ipa.cpp:25-27
    return x > 0.0 ? x + std::log1p(std::exp(-x)) : std::log1p(std::exp(x));
}

}  // namespace

// ------------------------------------------------------------------ Tuning
Tuning Tuning::from_env() {
    Tuning t;
    if (const char* e = std::getenv("FIPA_ATTN_IMPL")) {
        const std::string v(e);
        t.attn = v == "1sm" ? Attn::one_sm : v == "pass" ? Attn::pass : v == "pair" ? Attn::pair : Attn::automatic;
    }
    if (const char* e = std::getenv("FIPA_FUSED_PACK")) t.fused_pack = std::string(e) != "0";
    if (const char* e = std::getenv("FIPA_BWD_DS")) t.bwd_ds = std::atoi(e) != 0 ? 1 : 0;
    if (const char* e = std::getenv("FIPA_F32_TC")) t.f32_tc = std::string(e) != "0";
    if (const char* e = std::getenv("FIPA_GRAPHS")) t.graphs = std::string(e) != "0";
    if (const char* e = std::getenv("FIPA_HOST_CHUNK")) t.host_chunk = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("FIPA_MICRO")) t.micro = std::min(4, std::max(1, std::atoi(e)));
    if (const char* e = std::getenv("FIPA_DS_CAP_MB")) t.ds_cap_mb = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FIPA_SHARD_CHUNKS")) t.shard_chunks = std::min(8, std::max(0, std::atoi(e)));
    if (const char* e = std::getenv("FIPA_BWD_RING"))
        std::sscanf(e, "%d,%d,%d,%d,%d", &t.bwd_ring[0], &t.bwd_ring[1], &t.bwd_ring[2], &t.bwd_ring[3],
                    &t.bwd_ring[4]);
    if (const char* e = std::getenv("FIPA_PASS_RING"))
        std::sscanf(e, "%d,%d,%d,%d", &t.pass_ring[0], &t.pass_ring[1], &t.pass_ring[2], &t.pass_ring[3]);
    return t;
}

// ------------------------------------------------------------------ Config
void Config::validate() const {
    REQUIRE(d_in > 0 && d_z > 0 && heads > 0 && c > 0 && n_query > 0 && n_value > 0 && rank > 0,
            "all IpaConfig dimensions must be positive");
    if (enforce_head_cap) {
        const std::size_t widest = std::max(qk_width(), v_width());
        REQUIRE(widest <= head_cap, "lifted head width ", widest, " exceeds the cap of ", head_cap,
                "; shrink c/N/r*d_z or set enforce_head_cap=false");
    }
}

LayerDims Config::dims() const {
    LayerDims d{};
    d.d_in = int(d_in);
    d.d_z = int(d_z);
    d.heads = int(heads);
    d.c = int(c);
    d.n_query = int(n_query);
    d.n_value = int(n_value);
    d.rank = int(rank);
    d.n_proj = int(heads * (3 * c + 6 * n_query + 3 * n_value));
    // 21 translation/bias columns, padded so the pair-factor block starts 16-byte aligned
    d.zq = int(round_up(c + 3 * n_query + 21, 8));
    d.dqk_used = d.zq + int(rank * d_z);
    d.dqk_mma = int(round_up(d.dqk_used, 16));
    d.dqk_pad = int(round_up(d.dqk_used, 64));
    d.dv_used = int(c + rank * d_z + 3 * n_value + 6);
    d.dv_mma = int(round_up(d.dv_used, 16));
    d.dv_pad = int(round_up(d.dv_used, 64));
    // TMEM budget of the tcgen05 attention: O (dv_tc) + S (64) + P (32) <= 512 columns.
    d.dv_tc = std::min(d.dv_mma, 416);
    d.dv_simt = std::max(0, d.dv_used - d.dv_tc);
    d.seg = int(d_z + c + 4 * n_value);
    d.feat = int(heads) * d.seg;
    d.din_ld = int(round_up(d_in, 8));
    d.feat_ld = int(round_up(d.feat, 8));
    return d;
}

HostWeights& HostWeights::operator=(const HostWeights& o) {
    for (int i = 0; i < 10; ++i) *slots[i] = *o.slots[i];
    w_l = o.w_l;
    w_c = o.w_c;
    stored_f32 = o.stored_f32;
    return *this;
}

std::vector<std::vector<std::size_t>> weight_shapes(const Config& c) {
    const std::size_t seg = c.d_z + c.c + 4 * c.n_value;
    return {{c.d_in, c.heads * c.c},           {c.d_in, c.heads * c.c},
            {c.d_in, c.heads * c.c},           {c.d_in, c.heads * c.n_query * 3},
            {c.d_in, c.heads * c.n_query * 3}, {c.d_in, c.heads * c.n_value * 3},
            {c.heads, c.d_z},                  {c.heads},
            {c.heads * seg, c.d_in},           {c.d_in}};
}

const char* const* weight_names() {
    static const char* names[10] = {"w_q",    "w_k",       "w_v",   "w_qp",  "w_kp",
                                    "w_vp",   "w_bias",    "gamma_raw", "w_out", "b_out"};
    return names;
}

// IpaWeights::init (proj/src/ipa.cpp:172-193): draw order w_q w_k w_v w_qp w_kp w_vp
// (sigma 1/sqrt(d_in)), w_bias (1/sqrt(d_z)), w_out (1/sqrt(H*seg)); gamma_raw = ln(e-1),
// b_out = 0, w_l = sqrt(1/3), w_c = sqrt(2/(9 Nq)).  round_f32 mirrors f32 storage.
HostWeights init_weights(const Config& cfg, std::uint64_t seed, bool round_f32) {
    cfg.validate();
    const auto shapes = weight_shapes(cfg);
    Rng rng(seed);
    HostWeights w;
    auto draw = [&](std::vector<double>& dst, const std::vector<std::size_t>& shape, double sd) {
        dst.resize(numel(shape));
        for (auto& v : dst) {
            v = sd * rng.gaussian();
            if (round_f32) v = static_cast<double>(static_cast<float>(v));
        }
    };
    const double s_in = 1.0 / std::sqrt(static_cast<double>(cfg.d_in));
    for (int i = 0; i < 6; ++i) draw(*w.slots[i], shapes[i], s_in);
    draw(w.w_bias, shapes[6], 1.0 / std::sqrt(static_cast<double>(cfg.d_z)));
    w.gamma_raw.assign(cfg.heads, round_f32 ? double(float(kGammaRawUnit)) : kGammaRawUnit);
    draw(w.w_out, shapes[8], 1.0 / std::sqrt(static_cast<double>(shapes[8][0])));
    w.b_out.assign(cfg.d_in, 0.0);
    w.w_l = std::sqrt(1.0 / 3.0);
    w.w_c = std::sqrt(2.0 / (9.0 * static_cast<double>(cfg.n_query)));
    w.stored_f32 = round_f32;
    return w;
}

// ------------------------------------------------------------ weights file
// Layout (proj/include/fipa/model_io.hpp:15-21, README "Weights file format"):
//   "FIPA" | u16 version=1 | u16 count | entries
//   entry: u16 name_len | name | u8 precision (0 f32, 1 f64) | u8 rank | u64 dims[rank] | payload
// w_l / w_c travel as 1-element f64 tensors.  Bit-exact round trips.
namespace {

void put_u16(std::string& o, std::uint16_t v) {
    o.push_back(char(v & 0xff));
    o.push_back(char(v >> 8));
}
void put_u64(std::string& o, std::uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(char((v >> (8 * i)) & 0xff));
}
void put_entry(std::string& o, const std::string& name, const std::vector<double>& vals,
               const std::vector<std::size_t>& shape, bool f32) {
    put_u16(o, static_cast<std::uint16_t>(name.size()));
    o.append(name);
    o.push_back(char(f32 ? 0 : 1));
    o.push_back(char(shape.size()));
    for (auto d : shape) put_u64(o, d);
    for (double v : vals) {
        if (f32) {
            const auto bits = std::bit_cast<std::uint32_t>(static_cast<float>(v));
            for (int b = 0; b < 4; ++b) o.push_back(char((bits >> (8 * b)) & 0xff));
        } else {
            put_u64(o, std::bit_cast<std::uint64_t>(v));
        }
    }
}

struct Cursor {
    const std::string& buf;
    std::size_t pos = 0;
    void need(std::size_t n) const {
        if (pos + n > buf.size()) throw IoError("weights file: truncated payload");
    }
    std::uint8_t u8() {
        need(1);
        return static_cast<std::uint8_t>(buf[pos++]);
    }
    std::uint16_t u16() {
        need(2);
        const std::uint16_t v = std::uint16_t(std::uint8_t(buf[pos])) |
                                std::uint16_t(std::uint16_t(std::uint8_t(buf[pos + 1])) << 8);
        pos += 2;
        return v;
    }
    std::uint64_t u64() {
        need(8);
        std::uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= std::uint64_t(std::uint8_t(buf[pos + i])) << (8 * i);
        pos += 8;
        return v;
    }
    std::string bytes(std::size_t n) {
        need(n);
        std::string s = buf.substr(pos, n);
        pos += n;
        return s;
    }
};

struct Entry {
    bool f32 = false;
    std::vector<std::size_t> shape;
    std::vector<double> vals;
};

}  // namespace

void save_weights_file(const HostWeights& w, const std::vector<std::vector<std::size_t>>& shapes,
                       const std::string& path) {
    std::string buf("FIPA");
    put_u16(buf, 1);
    put_u16(buf, 12);
    for (int i = 0; i < 10; ++i) put_entry(buf, weight_names()[i], *w.slots[i], shapes[i], w.stored_f32);
    put_entry(buf, "w_l", {w.w_l}, {1}, false);
    put_entry(buf, "w_c", {w.w_c}, {1}, false);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open '" + path + "' for writing");
    out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
    if (!out) throw IoError("short write to '" + path + "'");
}

HostWeights load_weights_file(const std::string& path,
                              const std::vector<std::vector<std::size_t>>& shapes) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open '" + path + "' for reading");
    std::ostringstream ss;
    ss << in.rdbuf();
    const std::string buf = ss.str();
    Cursor cur{buf};
    if (cur.bytes(4) != "FIPA") throw IoError("weights file: bad magic");
    const std::uint16_t version = cur.u16();
    if (version != 1) throw IoError(cat("weights file: version ", version, ", expected 1"));
    const std::uint16_t count = cur.u16();
    std::map<std::string, Entry> table;
    for (std::uint16_t e = 0; e < count; ++e) {
        const std::uint16_t nl = cur.u16();
        std::string name = cur.bytes(nl);
        Entry ent;
        const std::uint8_t tag = cur.u8();
        if (tag > 1) throw IoError("weights file: unknown precision tag");
        ent.f32 = tag == 0;
        const std::uint8_t rank = cur.u8();
        if (rank == 0) throw IoError("weights file: rank-0 tensor entry");
        std::size_t n = 1;
        for (int r = 0; r < rank; ++r) {
            const std::uint64_t d = cur.u64();
            if (d == 0) throw IoError("weights file: zero dimension");
            ent.shape.push_back(d);
            n *= d;
        }
        cur.need(n * (ent.f32 ? 4 : 8));
        ent.vals.resize(n);
        for (std::size_t i = 0; i < n; ++i) {
            if (ent.f32) {
                std::uint32_t bits = 0;
                for (int b = 0; b < 4; ++b)
                    bits |= std::uint32_t(std::uint8_t(buf[cur.pos + b])) << (8 * b);
                cur.pos += 4;
                ent.vals[i] = static_cast<double>(std::bit_cast<float>(bits));
            } else {
                ent.vals[i] = std::bit_cast<double>(cur.u64());
            }
        }
        if (!table.emplace(std::move(name), std::move(ent)).second)
            throw IoError("weights file: duplicate tensor entry");
    }
    if (cur.pos != buf.size()) throw IoError("weights file: trailing bytes");
    auto take = [&](const char* name) {
        auto it = table.find(name);
        if (it == table.end()) throw IoError(std::string("weights file: missing tensor '") + name + "'");
        Entry e = std::move(it->second);
        table.erase(it);
        return e;
    };
    HostWeights w;
    for (int i = 0; i < 10; ++i) {
        Entry e = take(weight_names()[i]);
        if (e.shape != shapes[i])
            throw ValueError(cat("weights file: tensor '", weight_names()[i],
                                 "' has a shape that disagrees with the layer configuration"));
        if (i == 0) w.stored_f32 = e.f32;
        *w.slots[i] = std::move(e.vals);
    }
    w.w_l = take("w_l").vals.at(0);
    w.w_c = take("w_c").vals.at(0);
    if (!table.empty()) throw IoError("weights file: unexpected tensor '" + table.begin()->first + "'");
    return w;
}

// ------------------------------------------------------------------ layer
FlashIpaLayer::FlashIpaLayer(const Config& cfg) : cfg_(cfg) {
    cfg_.validate();
    dims_ = cfg_.dims();
    if (cudaGetDevice(&device_) != cudaSuccess) {
        device_ = 0;
        cudaGetLastError();
    }
    w_ = fipa_b200::init_weights(cfg_, 0, cfg_.weights_f32);
    dirty_ = true;  // device copies are made lazily by the first forward
}

FlashIpaLayer::~FlashIpaLayer() {
    release_device();
    release_host_pipe();
    clear_graphs();
    if (capture_stream_) cudaStreamDestroy(capture_stream_);
    for (auto& st : side_streams_)
        if (st) cudaStreamDestroy(st);
    if (fork_ev_) cudaEventDestroy(fork_ev_);
    for (auto& e : join_ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    for (auto& e : evb_)
        if (e) cudaEventDestroy(e);
}

void FlashIpaLayer::release_device() {
    for (void* p : {static_cast<void*>(d_wproj_t_), static_cast<void*>(d_wout_t_), static_cast<void*>(d_wheads_),
                    static_cast<void*>(d_wproj_), static_cast<void*>(d_wout_),
                    static_cast<void*>(d_bout_), static_cast<void*>(d_head_g_),
                    static_cast<void*>(d_wl_bias_), static_cast<void*>(d_bwd_scale_),
                    static_cast<void*>(d_wproj_cat_), static_cast<void*>(d_wout_cat_)}) {
        if (p) cudaFree(p);
    }
    d_wproj_t_ = d_wout_t_ = d_wheads_ = nullptr;
    d_wproj_ = d_wout_ = d_bout_ = d_head_g_ = d_wl_bias_ = d_bwd_scale_ = nullptr;
    d_wproj_cat_ = d_wout_cat_ = nullptr;
}

void FlashIpaLayer::init_weights(std::uint64_t seed) {
    w_ = fipa_b200::init_weights(cfg_, seed, cfg_.weights_f32);
    dirty_ = true;
}

void FlashIpaLayer::set_weights(const HostWeights& w) {
    const auto shapes = weight_shapes(cfg_);
    for (int i = 0; i < 10; ++i)
        REQUIRE(w.slots[i]->size() == numel(shapes[i]), "weights tensor '", weight_names()[i],
                "' has ", w.slots[i]->size(), " elements, expected ", numel(shapes[i]));
    w_ = w;
    dirty_ = true;
}

void FlashIpaLayer::save(const std::string& path) const { save_weights_file(w_, weight_shapes(cfg_), path); }

void FlashIpaLayer::load(const std::string& path) {
    w_ = load_weights_file(path, weight_shapes(cfg_));
    dirty_ = true;
}

// Device copies: fused projection matrix in the reference column order
// (w_q | w_k | w_v | w_qp | w_kp | w_vp), output projection, per-head scalars.
void FlashIpaLayer::upload_weights() {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    clear_graphs();  // captured graphs hold the old device weight pointers
    release_device();
    const LayerDims& d = dims_;
    const std::size_t din = cfg_.d_in, np = d.n_proj, feat = d.feat, H = cfg_.heads;
    std::vector<double> wproj(din * np);  // [d_in, n_proj]
    std::size_t col0 = 0;
    for (int i = 0; i < 6; ++i) {
        const std::vector<double>& src = *w_.slots[i];
        const std::size_t w = src.size() / din;
        for (std::size_t r = 0; r < din; ++r)
            for (std::size_t c = 0; c < w; ++c) wproj[r * np + col0 + c] = src[r * w + c];
        col0 += w;
    }
    auto up = [&](auto** dst, const auto& host) {
        using T = std::remove_reference_t<decltype(host[0])>;
        cuda_check(cudaMalloc(reinterpret_cast<void**>(dst), host.size() * sizeof(T)), "cudaMalloc");
        cuda_check(cudaMemcpy(*dst, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice),
                   "cudaMemcpy H2D");
    };
    if (cfg_.precision == Precision::bf16) {
        const std::size_t dld = d.din_ld, fld = d.feat_ld;
        std::vector<__nv_bfloat16> t(np * dld, __float2bfloat16_rn(0.f));
        for (std::size_t r = 0; r < din; ++r)
            for (std::size_t c = 0; c < np; ++c)
                t[c * dld + r] = __float2bfloat16_rn(static_cast<float>(wproj[r * np + c]));
        up(&d_wproj_t_, t);
        if (proj_pack_supported(d)) {
            // head-major copy for the fused projection+pack kernel: per head the rows
            // q (c) | k (c) | v (c) | q_p (3Nq) | k_p (3Nq) | v_p (3Nv), zero-padded to NH rows
            const std::size_t NH = std::size_t(proj_pack_head_width(d)), c = cfg_.c, Nq = cfg_.n_query,
                              Nv = cfg_.n_value;
            std::vector<__nv_bfloat16> wh(H * NH * dld, __float2bfloat16_rn(0.f));
            for (std::size_t h = 0; h < H; ++h) {
                std::size_t n = 0;
                auto put = [&](std::size_t col0, std::size_t width) {  // fused column block -> head rows
                    for (std::size_t e = 0; e < width; ++e, ++n)
                        for (std::size_t r = 0; r < din; ++r)
                            wh[(h * NH + n) * dld + r] = __float2bfloat16_rn(static_cast<float>(wproj[r * np + col0 + e]));
                };
                put(0 * H * c + h * c, c);
                put(1 * H * c + h * c, c);
                put(2 * H * c + h * c, c);
                put(3 * H * c + h * 3 * Nq, 3 * Nq);
                put(3 * H * c + 3 * H * Nq + h * 3 * Nq, 3 * Nq);
                put(3 * H * c + 6 * H * Nq + h * 3 * Nv, 3 * Nv);
            }
            up(&d_wheads_, wh);
        }
        std::vector<__nv_bfloat16> o(din * fld, __float2bfloat16_rn(0.f));
        for (std::size_t r = 0; r < feat; ++r)
            for (std::size_t c = 0; c < din; ++c)
                o[c * fld + r] = __float2bfloat16_rn(static_cast<float>(w_.w_out[r * din + c]));
        up(&d_wout_t_, o);
    }
    {  // fp32 copies: the f32 path, and the quadratic-memory arm (reference_forward) at any precision
        std::vector<float> t(wproj.begin(), wproj.end());
        up(&d_wproj_, t);
        std::vector<float> o(w_.w_out.begin(), w_.w_out.end());
        up(&d_wout_, o);
    }
    if (f32_tensor_cores()) {
        // 3xTF32 B operands (K-major): row n = [w_lo | w_hi | w_hi] over the K extent, zero padded,
        // against A' = [a_hi | a_lo | a_hi]: the two small cross terms accumulate first, then the
        // large hi.hi term.  hi = tf32(w) (round to nearest, ties away, like cvt.rna), lo = w - hi.
        auto tf32 = [](double w) {
            const float f = static_cast<float>(w);
            std::uint32_t u = std::bit_cast<std::uint32_t>(f);
            if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
            return std::bit_cast<float>(u);
        };
        auto cat = [&](std::size_t rows, std::size_t K, std::size_t Kp, auto&& val) {
            std::vector<float> v(rows * 3 * Kp, 0.f);
            for (std::size_t r = 0; r < rows; ++r)
                for (std::size_t k = 0; k < K; ++k) {
                    const double w = val(r, k);
                    const float hi = tf32(w), lo = static_cast<float>(w - static_cast<double>(hi));
                    float* row = v.data() + r * 3 * Kp;
                    row[k] = lo;
                    row[Kp + k] = hi;
                    row[2 * Kp + k] = hi;
                }
            return v;
        };
        up(&d_wproj_cat_, cat(np, din, std::size_t(din_p()), [&](std::size_t n, std::size_t k) { return wproj[k * np + n]; }));
        up(&d_wout_cat_, cat(din, feat, std::size_t(feat_p()), [&](std::size_t n, std::size_t k) { return w_.w_out[k * din + n]; }));
    }
    std::vector<float> bout(w_.b_out.begin(), w_.b_out.end());
    up(&d_bout_, bout);
    std::vector<float> g(H), wlb(H * cfg_.d_z);
    for (std::size_t h = 0; h < H; ++h) g[h] = static_cast<float>(softplus(w_.gamma_raw[h]) * w_.w_l * w_.w_c);
    for (std::size_t e = 0; e < wlb.size(); ++e) wlb[e] = static_cast<float>(w_.w_l * w_.w_bias[e]);
    up(&d_head_g_, g);
    up(&d_wl_bias_, wlb);
    std::vector<float> bs(H + 1);
    for (std::size_t h = 0; h < H; ++h)
        bs[h] = static_cast<float>(w_.w_l * w_.w_c / (1.0 + std::exp(-w_.gamma_raw[h])));
    bs[H] = static_cast<float>(w_.w_l);
    up(&d_bwd_scale_, bs);
    k_scale_ = static_cast<float>(w_.w_l / std::sqrt(static_cast<double>(cfg_.c)));
    dirty_ = false;
}

FlashIpaLayer::Workspace FlashIpaLayer::carve(void* base, std::int64_t B, std::int64_t L, bool train) const {
    const LayerDims& d = dims_;
    const std::size_t BL = std::size_t(B) * L, BHL = BL * d.heads;
    const std::size_t el = cfg_.precision == Precision::bf16 ? 2 : 4;
    Workspace w;
    std::size_t off = 0;
    auto take = [&](std::size_t bytes) {
        char* p = reinterpret_cast<char*>(reinterpret_cast<std::uintptr_t>(base) + off);
        off += round_up(bytes, 256);
        return p;
    };
    w.trans_c = reinterpret_cast<float*>(take(BL * 3 * 4));
    if (cfg_.precision == Precision::bf16) {
        w.s_bf16 = reinterpret_cast<__nv_bfloat16*>(take(BL * d.din_ld * 2));
        w.z1q = reinterpret_cast<__nv_bfloat16*>(take(BL * std::size_t(d.rank) * d.d_z * 2));
        w.z2b = reinterpret_cast<__nv_bfloat16*>(take(BL * std::size_t(d.rank) * d.d_z * 2));
    }
    w.proj = reinterpret_cast<float*>(take(BL * d.n_proj * 4));
    w.qhat = take(BHL * d.dqk_pad * el);
    w.khat = take(BHL * d.dqk_pad * el);
    w.vhat = take(BHL * d.dv_pad * el);
    w.colbias = reinterpret_cast<float*>(take(BHL * 4));
    w.lse = reinterpret_cast<float*>(take(BHL * 4));
    w.feat = take(BL * d.feat_ld * el);
    if (f32_tensor_cores()) {
        w.s_cat = reinterpret_cast<float*>(take(BL * 3 * std::size_t(din_p()) * 4));
        w.qs = reinterpret_cast<float*>(take(2 * BHL * d.dqk_pad * 4));
        w.ks = reinterpret_cast<float*>(take(2 * BHL * d.dqk_pad * 4));
        w.vs = reinterpret_cast<float*>(take(2 * std::size_t(B) * d.heads * d.dv_pad * round_up(std::size_t(L), 4) * 4));
        w.feat_cat = reinterpret_cast<float*>(take(BL * 3 * std::size_t(feat_p()) * 4));
    }
    if (train) {
        const std::size_t rdz = std::size_t(d.rank) * d.d_z;
        w.o_hat = reinterpret_cast<float*>(take(BHL * d.dv_pad * 4));
        w.dout_bf16 = reinterpret_cast<__nv_bfloat16*>(take(BL * d.din_ld * 2));
        w.dfeat = reinterpret_cast<__nv_bfloat16*>(take(BL * d.feat_ld * 2));
        w.do_hat = reinterpret_cast<__nv_bfloat16*>(take(BHL * d.dv_pad * 2));
        w.Dvec = reinterpret_cast<float*>(take(BHL * 4));
        w.dq_acc = reinterpret_cast<float*>(take(BHL * acc_ld() * 4));
        w.dk_acc = reinterpret_cast<float*>(take(BHL * acc_ld() * 4));
        w.dv_acc = reinterpret_cast<float*>(take(BHL * acc_ld() * 4));
        if (!dense_backward()) {
            w.dk16 = reinterpret_cast<__nv_bfloat16*>(take(BHL * acc_ld() * 2));
            w.dv16 = reinterpret_cast<__nv_bfloat16*>(take(BHL * acc_ld() * 2));
            w.dq16 = reinterpret_cast<__nv_bfloat16*>(take(BHL * acc_ld() * 2));
        }
        w.dproj = reinterpret_cast<__nv_bfloat16*>(take(BL * nproj_ld() * 2));
        w.dz1_epi = reinterpret_cast<float*>(take(BL * rdz * 4));
        w.geo_epi = reinterpret_cast<float*>(take(BL * 12 * 4));
        w.dt_c = reinterpret_cast<float*>(take(BL * 3 * 4));
        w.red = reinterpret_cast<float*>(take((d.heads + d.heads * std::size_t(d.d_z)) * 4));
        w.dwproj = reinterpret_cast<float*>(take(std::size_t(d.d_in) * d.n_proj * 4));
        if (dense_backward()) {
            // materialised S / dP (fp32) and P / dS (bf16) for as many whole samples as fit the
            // dS budget (Tuning::ds_cap_mb), at least one
            w.att_ld = static_cast<int>(round_up(std::size_t(L), 64));
            const double per_sample = double(d.heads) * double(L) * double(w.att_ld) * 12.0;
            const double cap = double(tuning_.ds_cap_mb) * double(1 << 20);
            w.att_samples = static_cast<int>(std::max<std::int64_t>(
                1, std::min<std::int64_t>(B, static_cast<std::int64_t>(cap / per_sample))));
            const std::size_t n = std::size_t(w.att_samples) * d.heads * L * w.att_ld;
            w.att_s = reinterpret_cast<float*>(take(n * 4));
            w.att_dp = reinterpret_cast<float*>(take(n * 4));
            w.att_p = reinterpret_cast<__nv_bfloat16*>(take(n * 2));
            w.att_ds = reinterpret_cast<__nv_bfloat16*>(take(n * 2));
        } else if (const std::int64_t qc = ds_chunk(B, L)) {
            w.ds_ld = static_cast<int>(qc);  // whole 64-column blocks: all queries, or a query chunk
            w.ds = reinterpret_cast<__nv_bfloat16*>(take(BHL * w.ds_ld * 2));
        }
    }
    w.bytes = off;
    return w;
}

FlashIpaLayer::Workspace FlashIpaLayer::slice(const Workspace& w, std::int64_t b0, std::int64_t L) const {
    const LayerDims& d = dims_;
    const std::size_t n = std::size_t(b0) * L, H = d.heads, rdz = std::size_t(d.rank) * d.d_z;
    const std::size_t el = cfg_.precision == Precision::bf16 ? 2 : 4;
    auto adv = [](auto* p, std::size_t bytes) {
        using T = std::remove_pointer_t<decltype(p)>;
        return p == nullptr ? p : reinterpret_cast<T*>(reinterpret_cast<char*>(p) + bytes);
    };
    Workspace v = w;
    v.trans_c = adv(w.trans_c, n * 3 * 4);
    v.s_bf16 = adv(w.s_bf16, n * d.din_ld * 2);
    v.z1q = adv(w.z1q, n * rdz * 2);
    v.z2b = adv(w.z2b, n * rdz * 2);
    v.proj = adv(w.proj, n * d.n_proj * 4);
    v.qhat = adv(static_cast<char*>(w.qhat), n * H * d.dqk_pad * el);
    v.khat = adv(static_cast<char*>(w.khat), n * H * d.dqk_pad * el);
    v.vhat = adv(static_cast<char*>(w.vhat), n * H * d.dv_pad * el);
    v.colbias = adv(w.colbias, n * H * 4);
    v.lse = adv(w.lse, n * H * 4);
    v.feat = adv(static_cast<char*>(w.feat), n * d.feat_ld * el);
    v.o_hat = adv(w.o_hat, n * H * d.dv_pad * 4);
    v.dout_bf16 = adv(w.dout_bf16, n * d.din_ld * 2);
    v.dfeat = adv(w.dfeat, n * d.feat_ld * 2);
    v.do_hat = adv(w.do_hat, n * H * d.dv_pad * 2);
    v.Dvec = adv(w.Dvec, n * H * 4);
    v.dq_acc = adv(w.dq_acc, n * H * acc_ld() * 4);
    v.dk_acc = adv(w.dk_acc, n * H * acc_ld() * 4);
    v.dv_acc = adv(w.dv_acc, n * H * acc_ld() * 4);
    v.dk16 = adv(w.dk16, n * H * acc_ld() * 2);
    v.dv16 = adv(w.dv16, n * H * acc_ld() * 2);
    v.dq16 = adv(w.dq16, n * H * acc_ld() * 2);
    v.dproj = adv(w.dproj, n * nproj_ld() * 2);
    v.dz1_epi = adv(w.dz1_epi, n * rdz * 4);
    v.geo_epi = adv(w.geo_epi, n * 12 * 4);
    v.dt_c = adv(w.dt_c, n * 3 * 4);
    v.ds = adv(w.ds, n * H * std::size_t(w.ds_ld) * 2);
    return v;  // red / dwproj: shared accumulators; the fp32-path planes are not sliced (bf16 only)
}

bool FlashIpaLayer::f32_tensor_cores() const {
    return cfg_.precision == Precision::f32 && tuning_.f32_tc && attn_fwd_f32tc_supported(dims_);
}

bool FlashIpaLayer::materialize_ds(std::int64_t B, std::int64_t L) const { return ds_chunk(B, L) > 0; }

// Query columns of dS held at once by the materialised-dS backward (0: streaming dQ kernel).  dS is
// B*H*L*cols*2 bytes: the whole [L keys x L queries] matrix up to L = 8192 and 2 GiB, where the dQ GEMM
// over it is ~3x faster than the streaming kernel's recompute of S, P and dP (B=2 L=4096: 0.29 vs
// 0.98 ms); beyond, query chunks of a multiple of 256 columns within the same 2 GiB (the dK/dV kernel
// runs once per chunk, later chunks adding their partial dK / dV by TMA reduction), so the workspace
// stays linear in L.
std::int64_t FlashIpaLayer::ds_chunk(std::int64_t B, std::int64_t L) const {
    if (tuning_.bwd_ds == 0) return 0;
    const double cap = double(tuning_.ds_cap_mb) * double(1 << 20), per_col = double(B) * dims_.heads * double(L) * 2.0;
    const std::int64_t full = (L + 63) / 64 * 64;
    if (L <= 8192 && per_col * double(full) <= cap) return full;
    const std::int64_t qc = std::int64_t(cap / per_col) / 256 * 256;
    return qc >= 256 ? std::min(qc, full) : 0;
}

std::size_t FlashIpaLayer::workspace_size(std::int64_t B, std::int64_t L) const {
    return carve(nullptr, B, L).bytes;
}

std::size_t FlashIpaLayer::train_workspace_size(std::int64_t B, std::int64_t L) const {
    return carve(nullptr, B, L, true).bytes;
}

std::size_t FlashIpaLayer::num_weights() const {
    std::size_t n = 0;
    for (const auto& sh : weight_shapes(cfg_)) n += numel(sh);
    return n;
}

bool FlashIpaLayer::fused_backward_supported() const {
    return cfg_.precision == Precision::bf16 && attn_fwd_2sm_supported(dims_) && attn_bwd_supported(dims_) &&
           dims_.n_value <= 32 && dims_.n_query <= 32;
}

bool FlashIpaLayer::dense_backward() const {
    return cfg_.precision == Precision::bf16 && !fused_backward_supported() && bf16_attention_supported(dims_) &&
           dims_.n_value <= 32 && dims_.n_query <= 32 && dims_.heads <= 16;
}

bool FlashIpaLayer::backward_supported() const { return fused_backward_supported() || dense_backward(); }

int FlashIpaLayer::launches_per_backward() const {
    // dout cast, dfeat GEMM, dW_out GEMM, prep, attn KV, dQ (GEMM or attention kernel), unpack
    // (geometry + streaming), recenter, ds GEMM, dW_proj GEMM, finish (scatter + scalings); memsets
    // are not kernels of ours; a query-chunked dS adds two launches per further chunk
    return 12;
}

int FlashIpaLayer::step_launches(std::int64_t B, std::int64_t L, bool train) const {
    // the captured graphs run micro_chunks(...) sample chains (forward_micro / backward_micro): every
    // chain launches the per-call kernels; the backward's finish kernel runs once after the join
    const bool graphs = tuning_.graphs && !timing_;
    const int nf = graphs && !(train && dense_backward()) ? micro_chunks(B, L, true) : 1;
    int n = nf * launches_per_forward();
    if (train) {
        const int nb = graphs && !dense_backward() ? micro_chunks(B, L) : 1;
        n += nb > 1 ? nb * (launches_per_backward() - 1) + 1 : launches_per_backward();
    }
    return n;
}

int FlashIpaLayer::launches_per_forward() const {
    // fp32 tensor-core path: recenter, split s, projection GEMM, pack, split q/k/v, attention,
    // split feat, output GEMM
    if (f32_tensor_cores()) return 10;
    if (cfg_.precision != Precision::bf16) return 5;
    // fused: cast (+ recentre), projection+pack, attention, output GEMM; else recenter, cast,
    // projection GEMM, pack, attention, output GEMM
    return (proj_pack_supported(dims_) && tuning_.fused_pack) ? 4 : 6;
}

void FlashIpaLayer::set_timing(bool on) {
    timing_ = on;
    if (on && !ev_[0]) {
        for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        for (auto& e : evb_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    }
}

std::vector<float> FlashIpaLayer::bwd_stage_times() const {
    std::vector<float> out;
    if (!bwd_timed_once_) return out;
    for (int i = 0; i < kBwdStages; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, evb_[i], evb_[i + 1]) != cudaSuccess) ms = -1.f;
        out.push_back(ms);
    }
    return out;
}

std::vector<float> FlashIpaLayer::stage_times() const {
    std::vector<float> out;
    if (!timed_once_) return out;
    for (int i = 0; i < kStages; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev_[i], ev_[i + 1]) != cudaSuccess) ms = -1.f;
        out.push_back(ms);
    }
    return out;
}

bool FlashIpaLayer::GraphKey::operator<(const GraphKey& o) const {
    return std::tie(kind, B, L, ptrs, ws_bytes) < std::tie(o.kind, o.B, o.L, o.ptrs, o.ws_bytes);
}

void FlashIpaLayer::clear_graphs() {
    std::lock_guard<std::mutex> lk(graph_mu_);
    for (auto& [k, g] : graphs_) cudaGraphExecDestroy(g);
    graphs_.clear();
    graph_order_.clear();
}

// Replays the graph captured for `key` on `stream` (capturing it first); false when graphs do not
// apply (then the caller launches kernel by kernel).
template <class F>
bool FlashIpaLayer::run_graph(const GraphKey& key, cudaStream_t stream, F&& launch) {
    if (!tuning_.graphs || timing_) return false;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return false;  // the caller is capturing its own graph: launch into it directly
    }
    std::lock_guard<std::mutex> lk(graph_mu_);
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        if (!capture_stream_)
            cuda_check(cudaStreamCreateWithFlags(&capture_stream_, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamBeginCapture(capture_stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            launch(capture_stream_);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(capture_stream_, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            throw;
        }
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamEndCapture(capture_stream_, &graph), "end capture");
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(e, "graph instantiate");
        if (graph_order_.size() >= 32) {  // bounded cache: drop the oldest
            auto old = graphs_.find(graph_order_.front());
            if (old != graphs_.end()) {
                cudaGraphExecDestroy(old->second);
                graphs_.erase(old);
            }
            graph_order_.erase(graph_order_.begin());
        }
        it = graphs_.emplace(key, exec).first;
        graph_order_.push_back(key);
    }
    cuda_check(cudaGraphLaunch(it->second, stream), "graph launch");
    return true;
}

void FlashIpaLayer::forward(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                            const float* z2, const float* rot, const float* trans,
                            const std::uint8_t* mask, float* out, void* workspace,
                            std::size_t workspace_bytes, cudaStream_t stream, bool train,
                            const ShardStage* shard) {
    if (shard == nullptr && B >= 1 && L >= 1 && s && z1 && z2 && rot && trans && out && workspace) {
        cuda_check(cudaSetDevice(device_), "cudaSetDevice");
        if (dirty_) {
            std::lock_guard<std::mutex> lk(upload_mu_);
            if (dirty_) upload_weights();
        }
        GraphKey key{train ? 1 : 0, B, L, {s, z1, z2, rot, trans, mask, out, workspace}, workspace_bytes};
        if (run_graph(key, stream, [&](cudaStream_t cs) {
                if (micro_chunks(B, L, true) > 1 && !(train && dense_backward()))
                    forward_micro(B, L, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes, cs, train);
                else
                    forward_impl(B, L, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes, cs, train,
                                 nullptr);
            }))
            return;
    }
    forward_impl(B, L, s, z1, z2, rot, trans, mask, out, workspace, workspace_bytes, stream, train, shard);
}

void FlashIpaLayer::forward_impl(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                 const float* z2, const float* rot, const float* trans,
                                 const std::uint8_t* mask, float* out, void* workspace,
                                 std::size_t workspace_bytes, cudaStream_t stream, bool train,
                                 const ShardStage* shard, const Workspace* view) {
    REQUIRE(B >= 1, "batch must be >= 1");
    REQUIRE(L >= 1, "empty frame set");
    REQUIRE(s && z1 && z2 && rot && trans && out, "null input/output pointer");
    REQUIRE(!train || backward_supported(),
            "training (forward_train/backward) needs precision='bf16'");
    REQUIRE(shard == nullptr || (cfg_.precision == Precision::bf16 && bf16_attention_supported(dims_)),
            "query-row sharding needs precision='bf16'");
    const bool do_pack = shard == nullptr || shard->stage == 1;
    const bool do_attend = shard == nullptr || shard->stage == 2 || shard->stage == 3;
    // stage 2 with a head range (hc > 0): that chunk's attention only; stage 3: the output GEMM
    const bool attn_part = shard == nullptr || shard->stage == 2;
    const bool out_part = shard == nullptr || shard->stage == 3 || (shard->stage == 2 && shard->hc == 0);
    const Workspace ws = view ? *view : carve(workspace, B, L, train);
    REQUIRE(view != nullptr || (workspace != nullptr && workspace_bytes >= ws.bytes), "workspace too small: need ",
            ws.bytes, " bytes, got ", workspace_bytes);
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    if (dirty_) {
        std::lock_guard<std::mutex> lk(upload_mu_);
        if (dirty_) upload_weights();
    }
    const LayerDims& d = dims_;
    const int BL = static_cast<int>(B * L);
    auto mark = [&](int i) {
        if (timing_) cuda_check(cudaEventRecord(ev_[i], stream), "cudaEventRecord");
    };
    mark(0);
    const bool fused = do_pack && d_wheads_ != nullptr && tuning_.fused_pack;
    if (shard == nullptr && !fused) {
        launch_recenter(trans, mask, ws.trans_c, int(B), int(L), stream);
    } else if (shard != nullptr && do_pack) {
        launch_recenter_with_sums(trans, shard->sums, ws.trans_c, int(B), int(L), stream);
    }
    mark(1);
    if (fused) {
        // fused projection GEMM + frame application + packing (proj_pack.cu); the input cast
        // also recentres the translations (unsharded)
        launch_cast_inputs(s, ws.s_bf16, d.d_in, d.din_ld, z1, z2, ws.z1q, ws.z2b, d.rank * d.d_z, BL, stream,
                           shard == nullptr ? trans : nullptr, mask, ws.trans_c, int(B), int(L));
        mark(2);
        ProjPackArgs pp{};
        pp.s_bf16 = ws.s_bf16;
        pp.w_heads = d_wheads_;
        pp.z1 = z1;
        pp.z2 = z2;
        pp.z1q = ws.z1q;
        pp.z2b = ws.z2b;
        pp.rot = rot;
        pp.trans = ws.trans_c;
        pp.mask = mask;
        pp.head_g = d_head_g_;
        pp.wl_bias = d_wl_bias_;
        pp.k_scale = k_scale_;
        pp.proj = ws.proj;
        pp.colbias = ws.colbias;
        pp.qhat = static_cast<__nv_bfloat16*>(ws.qhat);
        pp.khat = static_cast<__nv_bfloat16*>(ws.khat);
        pp.vhat = static_cast<__nv_bfloat16*>(ws.vhat);
        pp.B = int(B);
        pp.L = int(L);
        launch_proj_pack(d, pp, stream);
        mark(3);
    } else if (do_pack) {
    if (cfg_.precision == Precision::bf16) {
        launch_f32_to_bf16_2d(s, ws.s_bf16, BL, d.d_in, d.din_ld, stream);
        mark(2);
        GemmArgs g;
        g.A = ws.s_bf16;
        g.lda = d.din_ld;
        g.B = d_wproj_t_;
        g.ldb = d.din_ld;
        g.C = ws.proj;
        g.ldc = d.n_proj;
        g.M = BL;
        g.N = d.n_proj;
        g.K = d.d_in;
        launch_gemm_bf16(g, stream);
    } else if (f32_tensor_cores()) {
        // 3xTF32: proj = [s_hi | s_lo | s_hi] . [W_lo | W_hi | W_hi]^T on the tensor cores
        launch_split3(s, BL, d.d_in, d.d_in, ws.s_cat, din_p(), 3 * int64_t(din_p()), 0b010, 3, stream);
        mark(2);
        GemmF32Args g;
        g.A = ws.s_cat;
        g.lda = 3 * din_p();
        g.B = d_wproj_cat_;
        g.ldb = 3 * din_p();
        g.C = ws.proj;
        g.ldc = d.n_proj;
        g.M = BL;
        g.N = d.n_proj;
        g.K = 3 * din_p();
        launch_gemm_tf32(g, stream);
    } else {
        mark(2);
        launch_gemm_f32(s, d.d_in, d_wproj_, ws.proj, BL, d.n_proj, d.d_in, nullptr, nullptr, stream);
    }
    mark(3);
    PackArgs pa{};
    pa.proj = ws.proj;
    pa.z1 = z1;
    pa.z2 = z2;
    pa.rot = rot;
    pa.trans = ws.trans_c;
    pa.mask = mask;
    pa.head_g = d_head_g_;
    pa.wl_bias = d_wl_bias_;
    pa.k_scale = k_scale_;
    pa.qhat = ws.qhat;
    pa.khat = ws.khat;
    pa.vhat = ws.vhat;
    pa.colbias = ws.colbias;
    pa.B = int(B);
    pa.L = int(L);
    pa.out_f32 = cfg_.precision == Precision::f32;
    launch_pack(d, pa, stream);
    }
    mark(4);
    if (!do_attend) {
        cuda_check(cudaGetLastError(), "kernel launch");
        return;
    }
    if (cfg_.precision == Precision::bf16) {
        if (attn_part) {
        AttnArgs aa{};
        aa.qhat = static_cast<const __nv_bfloat16*>(ws.qhat);
        aa.khat = static_cast<const __nv_bfloat16*>(ws.khat);
        aa.vhat = static_cast<const __nv_bfloat16*>(ws.vhat);
        aa.colbias = ws.colbias;
        aa.z1 = z1;
        aa.rot = rot;
        aa.trans = ws.trans_c;
        aa.feat = static_cast<__nv_bfloat16*>(ws.feat);
        aa.lse = ws.lse;
        // (the materialised backward recomputes O_hat from P and V_hat)
        aa.o_save = train && !dense_backward() ? ws.o_hat : nullptr;
        aa.B = int(B);
        aa.L = int(L);
        if (shard != nullptr) {  // keys = all shards' rows, gathered [G][B*H][L][pad]
            aa.khat = static_cast<const __nv_bfloat16*>(shard->k_all);
            aa.vhat = static_cast<const __nv_bfloat16*>(shard->v_all);
            aa.Lk = int(L) * shard->groups;
            aa.kchunk = int(L);
        }
        for (int i = 0; i < 4; ++i) aa.pass_ring[i] = tuning_.pass_ring[i];
        const AttnImpl impl = train && !dense_backward() ? AttnImpl::pair
                                                         : attention_impl(d, tuning_.attn, shard != nullptr);
        if (shard != nullptr && shard->hc > 0) {
            REQUIRE(impl == AttnImpl::pair, "head-chunked sharded attention needs the CTA-pair kernel");
            aa.h0 = shard->h0;
            aa.hc = shard->hc;
        }
        if (impl == AttnImpl::pair) {
            launch_attn_fwd_2sm(d, aa, stream);
        } else if (impl == AttnImpl::pass) {
            launch_attn_fwd_pass(d, aa, stream);
        } else {
            launch_attn_fwd_tc(d, aa, stream);
        }
        mark(5);
        }
        if (out_part) {
        GemmArgs g;
        g.A = static_cast<const __nv_bfloat16*>(ws.feat);
        g.lda = d.feat_ld;
        g.B = d_wout_t_;
        g.ldb = d.feat_ld;
        g.C = out;
        g.ldc = d.d_in;
        g.M = BL;
        g.N = d.d_in;
        g.K = d.feat;
        g.bias = d_bout_;
        g.row_mask = mask;
        launch_gemm_bf16(g, stream);
        }
    } else if (f32_tensor_cores()) {
        const int64_t BHL = int64_t(B) * d.heads * L;
        const int64_t pq = BHL * d.dqk_pad;
        launch_split3(static_cast<const float*>(ws.qhat), BHL, d.dqk_pad, d.dqk_pad, ws.qs, d.dqk_pad, d.dqk_pad, 0b10, 2,
                      stream, pq);
        launch_split3(static_cast<const float*>(ws.khat), BHL, d.dqk_pad, d.dqk_pad, ws.ks, d.dqk_pad, d.dqk_pad, 0b10, 2,
                      stream, pq);
        const int Lp = int((L + 3) / 4 * 4);
        const int64_t pv = int64_t(B) * d.heads * d.dv_pad * Lp;
        launch_split_t(static_cast<const float*>(ws.vhat), int(B) * d.heads, int(L), d.dv_pad, ws.vs, Lp, pv, stream);
        mark(4);  // the operand splits count with the pack stage; the attention stage is the kernel alone
        AttnF32TcArgs aa{};
        aa.q_hi = ws.qs;
        aa.q_lo = ws.qs + pq;
        aa.k_hi = ws.ks;
        aa.k_lo = ws.ks + pq;
        aa.v_hi = ws.vs;
        aa.v_lo = ws.vs + pv;
        aa.z1 = z1;
        aa.rot = rot;
        aa.trans = ws.trans_c;
        aa.feat = static_cast<float*>(ws.feat);
        aa.lse = ws.lse;
        aa.B = int(B);
        aa.L = int(L);
        launch_attn_fwd_f32tc(d, aa, stream);
        mark(5);
        launch_split3(static_cast<const float*>(ws.feat), BL, d.feat, d.feat_ld, ws.feat_cat, feat_p(),
                      3 * int64_t(feat_p()), 0b010, 3, stream);
        GemmF32Args g;
        g.A = ws.feat_cat;
        g.lda = 3 * feat_p();
        g.B = d_wout_cat_;
        g.ldb = 3 * feat_p();
        g.C = out;
        g.ldc = d.d_in;
        g.M = BL;
        g.N = d.d_in;
        g.K = 3 * feat_p();
        g.bias = d_bout_;
        g.row_mask = mask;
        launch_gemm_tf32(g, stream);
    } else {
        AttnF32Args aa{};
        aa.qhat = static_cast<const float*>(ws.qhat);
        aa.khat = static_cast<const float*>(ws.khat);
        aa.vhat = static_cast<const float*>(ws.vhat);
        aa.colbias = ws.colbias;
        aa.z1 = z1;
        aa.rot = rot;
        aa.trans = ws.trans_c;
        aa.feat = static_cast<float*>(ws.feat);
        aa.lse = ws.lse;
        aa.B = int(B);
        aa.L = int(L);
        launch_attn_fwd_f32(d, aa, stream);
        mark(5);
        launch_gemm_f32(static_cast<const float*>(ws.feat), d.feat_ld, d_wout_, out, BL, d.d_in, d.feat, d_bout_,
                        mask, stream);
    }
    mark(6);
    if (timing_) timed_once_ = true;
    cuda_check(cudaGetLastError(), "kernel launch");
}

// ------------------------------------------------------------ quadratic-memory arm
namespace {
struct DenseLayout {
    std::size_t proj, gq, gk, vcat, z, logits, ov, oz, feat, bytes;
};
DenseLayout dense_layout(const LayerDims& d, std::int64_t B, std::int64_t L) {
    DenseLayout l{};
    std::size_t off = 0;
    auto take = [&](std::size_t floats) {
        const std::size_t o = off;
        off += round_up(floats * 4, 256);
        return o;
    };
    const std::size_t BL = std::size_t(B) * L, H = d.heads, vw = d.c + 3 * d.n_value;
    l.proj = take(BL * d.n_proj);
    l.gq = take(BL * H * d.n_query * 3);
    l.gk = take(BL * H * d.n_query * 3);
    l.vcat = take(BL * H * vw);
    l.z = take(BL * std::size_t(L) * d.d_z);
    l.logits = take(BL * H * std::size_t(L));
    l.ov = take(BL * H * vw);
    l.oz = take(BL * H * d.d_z);
    l.feat = take(BL * d.feat);
    l.bytes = off;
    return l;
}
}  // namespace

std::size_t FlashIpaLayer::reference_workspace_size(std::int64_t B, std::int64_t L) const {
    return dense_layout(dims_, B, L).bytes;
}

void FlashIpaLayer::reference_forward(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                      const float* z2, const float* rot, const float* trans,
                                      const std::uint8_t* mask, float* out, void* workspace,
                                      std::size_t workspace_bytes, cudaStream_t stream) {
    REQUIRE(B >= 1, "batch must be >= 1");
    REQUIRE(L >= 1, "empty frame set");
    REQUIRE(s && z1 && z2 && rot && trans && out, "null input/output pointer");
    REQUIRE(B * L <= std::int64_t(1) << 31 && L <= 65535, "dense arm: B*L or L too large");
    const DenseLayout lay = dense_layout(dims_, B, L);
    REQUIRE(workspace != nullptr && workspace_bytes >= lay.bytes, "reference workspace too small: need ",
            lay.bytes, " bytes");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    if (dirty_) {
        std::lock_guard<std::mutex> lk(upload_mu_);
        if (dirty_) upload_weights();
    }
    char* base = static_cast<char*>(workspace);
    auto at = [&](std::size_t o) { return reinterpret_cast<float*>(base + o); };
    DenseArgs a{};
    a.B = int(B);
    a.L = int(L);
    a.s = s;
    a.z1 = z1;
    a.z2 = z2;
    a.rot = rot;
    a.trans = trans;
    a.mask = mask;
    a.wproj = d_wproj_;
    a.wout = d_wout_;
    a.bout = d_bout_;
    a.head_g = d_head_g_;
    a.wl_bias = d_wl_bias_;
    a.k_scale = k_scale_;
    a.proj = at(lay.proj);
    a.gq = at(lay.gq);
    a.gk = at(lay.gk);
    a.vcat = at(lay.vcat);
    a.z = at(lay.z);
    a.logits = at(lay.logits);
    a.ov = at(lay.ov);
    a.oz = at(lay.oz);
    a.feat = at(lay.feat);
    a.out = out;
    launch_dense_ipa(dims_, a, stream);
    cuda_check(cudaGetLastError(), "kernel launch");
}

// Backward of the layer (no reference counterpart: proj/SPEC.md:8).  Order of work:
//   dOut (masked rows zeroed, proj/src/flash_ipa.cpp:213-216) -> db_out, dfeat = dOut.w_out^T,
//   dw_out = feat^T.dOut -> bwd_prep (epilogue^T) -> attention backward (attn_bwd.cu)
//   -> bwd_unpack (lifts^T) -> ds = dproj.W^T, dW = s^T.dproj, d(w_bias), d(gamma_raw).
void FlashIpaLayer::backward(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                             const float* z2, const float* rot, const float* trans,
                             const std::uint8_t* mask, const float* dout, float* ds, float* dz1,
                             float* dz2, float* drot, float* dtrans, float* dweights, void* workspace,
                             std::size_t workspace_bytes, cudaStream_t stream, const BwdShard* shard) {
    if (shard == nullptr && !dirty_ && B >= 1 && L >= 1 && s && z1 && z2 && rot && trans && dout && ds && dz1 &&
        dz2 && dweights && workspace && backward_supported()) {
        cuda_check(cudaSetDevice(device_), "cudaSetDevice");
        GraphKey key{2, B, L, {s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace},
                     workspace_bytes};
        if (run_graph(key, stream, [&](cudaStream_t cs) {
                if (micro_chunks(B, L) > 1 && !dense_backward())
                    backward_micro(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights,
                                   workspace, workspace_bytes, cs);
                else
                    backward_impl(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights,
                                  workspace, workspace_bytes, cs, nullptr);
            }))
            return;
    }
    backward_impl(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
                  workspace_bytes, stream, shard);
}

void FlashIpaLayer::backward_impl(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                  const float* z2, const float* rot, const float* trans,
                                  const std::uint8_t* mask, const float* dout, float* ds, float* dz1,
                                  float* dz2, float* drot, float* dtrans, float* dweights, void* workspace,
                                  std::size_t workspace_bytes, cudaStream_t stream, const BwdShard* shard,
                                  const Workspace* view, int parts) {
    REQUIRE(B >= 1, "batch must be >= 1");
    REQUIRE(L >= 1, "empty frame set");
    REQUIRE(s && z1 && z2 && rot && trans && dout && ds && dz1 && dz2 && dweights,
            "null input/output pointer");
    REQUIRE(backward_supported(), "backward needs precision='bf16'");
    const Workspace ws = view ? *view : carve(workspace, B, L, true);
    // chunks of a micro-batched call accumulate the weight gradients concurrently: atomic GEMM
    // epilogues (split-K >= 2), accumulators zeroed once (part 1) and scattered once (part 4)
    const bool chunked = parts != 7;
    REQUIRE(workspace != nullptr && workspace_bytes >= ws.bytes, "train workspace too small: need ",
            ws.bytes, " bytes, got ", workspace_bytes);
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    REQUIRE(!dirty_, "backward: weights changed since the training forward");
    const LayerDims& d = dims_;
    const int BL = static_cast<int>(B * L);
    const int H = d.heads;
    // dweights regions (reference order)
    const auto shapes = weight_shapes(cfg_);
    std::size_t woff[11] = {0};
    for (int i = 0; i < 10; ++i) woff[i + 1] = woff[i] + numel(shapes[i]);
    float* dw_bias = dweights + woff[6];
    float* dgamma = dweights + woff[7];
    float* dw_out = dweights + woff[8];
    float* db_out = dweights + woff[9];

    auto mark = [&](int i) {
        if (timing_ && shard == nullptr) cuda_check(cudaEventRecord(evb_[i], stream), "cudaEventRecord");
    };
    const int G = shard ? shard->groups : 1;
    if (shard != nullptr) {
        REQUIRE(shard->stage >= 1 && shard->stage <= 3, "backward shard stage must be 1, 2 or 3");
        REQUIRE(G == 1 || L % 256 == 0, "sharded backward needs L_local % 256 == 0");
        REQUIRE(shard->stage != 1 || (shard->k_all && shard->v_all && shard->dk_part && shard->dv_part),
                "backward shard stage 1 needs the gathered keys and the partial-gradient buffers");
        REQUIRE(shard->stage != 2 || (shard->dk_own && shard->dv_own && shard->dt_sums),
                "backward shard stage 2 needs the reduced key gradients and a dt_sums buffer");
        REQUIRE(shard->stage != 3 || shard->dt_sums, "backward shard stage 3 needs the global dt_sums");
    }
    const bool st1 = shard == nullptr || shard->stage == 1;
    const bool st2 = shard == nullptr || shard->stage == 2;
    const bool st3 = shard == nullptr || shard->stage == 3;
    mark(0);
    if (st1 && (parts & 1)) {
    cuda_check(cudaMemsetAsync(dw_out, 0, (woff[10] - woff[8]) * 4, stream), "memset");
    cuda_check(cudaMemsetAsync(ws.red, 0, (H + std::size_t(H) * d.d_z) * 4, stream), "memset");
    cuda_check(cudaMemsetAsync(ws.dwproj, 0, std::size_t(d.d_in) * d.n_proj * 4, stream), "memset");
    }
    if (st1 && (parts & 2)) {

    launch_bwd_dout(dout, mask, ws.dout_bf16, d.din_ld, db_out, BL, d.d_in, stream);
    mark(1);
    {  // dfeat = dOut . w_out^T
        GemmArgs g;
        g.A = ws.dout_bf16;
        g.lda = d.din_ld;
        g.B = d_wout_t_;
        g.ldb = d.feat_ld;
        g.b_mn_major = true;
        g.C = ws.dfeat;
        g.ldc = d.feat_ld;
        g.out_bf16 = true;
        g.M = BL;
        g.N = d.feat;
        g.K = d.d_in;
        launch_gemm_bf16(g, stream);
    }
    mark(2);
    {  // dw_out = feat^T . dOut
        GemmArgs g;
        g.A = static_cast<const __nv_bfloat16*>(ws.feat);
        g.lda = d.feat_ld;
        g.a_mn_major = true;
        g.B = ws.dout_bf16;
        g.ldb = d.din_ld;
        g.b_mn_major = true;
        g.C = dw_out;
        g.ldc = d.d_in;
        g.M = d.feat;
        g.N = d.d_in;
        g.K = BL;
        const int tiles = ((d.feat + 127) / 128) * ((d.d_in + 127) / 128);
        g.split_k = std::max(chunked ? 2 : 1, std::min(148 / std::max(tiles, 1), std::max(1, BL / 512)));
        launch_gemm_bf16(g, stream);
    }
    mark(3);
    if (dense_backward()) {
        REQUIRE(shard == nullptr, "query-row sharded training needs the fused attention backward (lifted widths <= 448)");
        dense_attention_backward(B, L, z1, rot, ws, stream);
        mark(4);
        mark(5);
    } else {
    {
        BwdPrepArgs a{};
        a.dfeat = ws.dfeat;
        a.ohat = ws.o_hat;
        a.z1 = z1;
        a.rot = rot;
        a.trans_c = ws.trans_c;
        a.dohat = ws.do_hat;
        a.Dvec = ws.Dvec;
        a.dz1_epi = ws.dz1_epi;
        a.geo_epi = ws.geo_epi;
        a.B = int(B);
        a.L = int(L);
        launch_bwd_prep(d, a, stream);
    }
    mark(4);
    {
        AttnBwdArgs a{};
        a.qhat = static_cast<const __nv_bfloat16*>(ws.qhat);
        a.khat = static_cast<const __nv_bfloat16*>(ws.khat);
        a.vhat = static_cast<const __nv_bfloat16*>(ws.vhat);
        a.dohat = ws.do_hat;
        a.lse = ws.lse;
        a.Dvec = ws.Dvec;
        a.dq_acc = ws.dq_acc;
        a.dk_acc = ws.dk_acc;
        a.dv_acc = ws.dv_acc;
        a.acc_ld = acc_ld();
        a.B = int(B);
        a.L = int(L);
        for (int i = 0; i < 5; ++i) a.ring[i] = tuning_.bwd_ring[i];
        if (shard != nullptr) {  // local queries against all G shards' keys; partial dK / dV
            a.khat = static_cast<const __nv_bfloat16*>(shard->k_all);
            a.vhat = static_cast<const __nv_bfloat16*>(shard->v_all);
            a.Lk = int(L) * G;
            a.kchunk = int(L);
            a.dk_acc = shard->dk_part;
            a.dv_acc = shard->dv_part;
        } else if (ws.ds != nullptr) {
            a.ds = ws.ds;
            a.ds_ld = ws.ds_ld;
        }
        // bf16 dK / dV copies for the unpack (unsharded whole-query launches; the query-chunked
        // dS accumulates by TMA reduction, the sharded one reduce-scatters fp32 partials)
        const bool acc16 = bf16_acc_enabled() && shard == nullptr && ws.dk16 != nullptr && !(ws.ds != nullptr && ws.ds_ld < L);
        if (acc16) {
            a.dk16 = ws.dk16;
            a.dv16 = ws.dv16;
            if (ws.ds != nullptr) a.dq16 = ws.dq16;  // dQ by the GEMM over the stored dS
        }
        if (shard == nullptr && ws.ds != nullptr && ws.ds_ld < L) {
            // query-chunked materialised dS: dK/dV kernel + dQ GEMM per chunk of ds_ld queries
            for (int q0 = 0; q0 < int(L); q0 += ws.ds_ld) {
                a.q0 = q0;
                a.qn = std::min<int>(ws.ds_ld, int(L) - q0);
                a.acc_add = q0 > 0 ? 1 : 0;
                launch_attn_bwd(d, a, stream, 1);
                launch_attn_bwd(d, a, stream, 2);
            }
            mark(5);
        } else {
        launch_attn_bwd(d, a, stream, 1);
        if (shard != nullptr && shard->kv_done != nullptr) cuda_check(cudaEventRecord(shard->kv_done, stream), "event");
        mark(5);
        launch_attn_bwd(d, a, stream, 2);
        }
    }
    }  // fused
    mark(6);
    }  // stage 1
    if (st2 && (parts & 2)) {
    {
        BwdUnpackArgs a{};
        a.dq_acc = ws.dq_acc;
        a.dk_acc = shard ? shard->dk_own : ws.dk_acc;
        a.dv_acc = shard ? shard->dv_own : ws.dv_acc;
        a.acc_ld = acc_ld();
        if (bf16_acc_enabled() && shard == nullptr && ws.dk16 != nullptr && !(ws.ds != nullptr && ws.ds_ld < L) &&
            !dense_backward()) {
            a.dk16 = ws.dk16;  // written by the dK/dV kernel above (same condition)
            a.dv16 = ws.dv16;
            if (ws.ds != nullptr) a.dq16 = ws.dq16;
        }
        a.proj = ws.proj;
        a.rot = rot;
        a.trans_c = ws.trans_c;
        a.z2 = z2;
        a.head_g = d_head_g_;
        a.wl_bias = d_wl_bias_;
        a.k_scale = k_scale_;
        a.dz1_epi = ws.dz1_epi;
        a.geo_epi = ws.geo_epi;
        a.dproj = ws.dproj;
        a.nproj_ld = nproj_ld();
        a.dz1 = dz1;
        a.dz2 = dz2;
        a.drot = drot;
        a.dt_c = ws.dt_c;
        a.dg = ws.red;
        a.dwlb = ws.red + H;
        a.B = int(B);
        a.L = int(L);
        launch_bwd_unpack(d, a, stream);
    }
    mark(7);
    if (shard != nullptr) launch_centroid_sums(ws.dt_c, mask, shard->dt_sums, int(B), int(L), stream);
    }  // stage 2
    if (st3 && (parts & 2)) {
    if (dtrans != nullptr) {
        if (shard != nullptr) {  // dt = mask (dt_c - mean over the valid rows of ALL shards)
            launch_recenter_with_sums(ws.dt_c, shard->dt_sums, dtrans, int(B), int(L), stream,
                                      mask != nullptr ? mask : nullptr);
        } else {
            launch_bwd_recenter(ws.dt_c, mask, dtrans, int(B), int(L), stream);
        }
    }
    mark(8);
    {  // ds = dproj . W^T
        GemmArgs g;
        g.A = ws.dproj;
        g.lda = nproj_ld();
        g.B = d_wproj_t_;
        g.ldb = d.din_ld;
        g.b_mn_major = true;
        g.C = ds;
        g.ldc = d.d_in;
        g.M = BL;
        g.N = d.d_in;
        g.K = d.n_proj;
        launch_gemm_bf16(g, stream);
    }
    mark(9);
    {  // dW = s^T . dproj  [d_in, n_proj]
        GemmArgs g;
        g.A = ws.s_bf16;
        g.lda = d.din_ld;
        g.a_mn_major = true;
        g.B = ws.dproj;
        g.ldb = nproj_ld();
        g.b_mn_major = true;
        g.C = ws.dwproj;
        g.ldc = d.n_proj;
        g.M = d.d_in;
        g.N = d.n_proj;
        g.K = BL;
        const int bn = (d.n_proj >= 2048) ? 256 : 128;
        const int tiles = ((d.d_in + 127) / 128) * ((d.n_proj + bn - 1) / bn);
        g.split_k = std::max(chunked ? 2 : 1, std::min(148 / std::max(tiles, 1), std::max(1, BL / 512)));
        launch_gemm_bf16(g, stream);
    }
    mark(10);
    }
    if (st3 && (parts & 4)) {
    {  // scatter the fused projection gradient into w_q .. w_vp (one kernel)
        ScatterCols seg{};
        int col0 = 0;
        for (int i = 0; i < 6; ++i) {
            seg.col0[i] = col0;
            seg.width[i] = int(shapes[i][1]);
            seg.dst_off[i] = std::int64_t(woff[i]);
            col0 += seg.width[i];
        }
        seg.dst_off[6] = std::int64_t(woff[6]);
        launch_finish_weight_grads(ws.dwproj, d.d_in, d.n_proj, seg, dweights, ws.red, d_bwd_scale_, H, d.d_z, dw_bias,
                                   dgamma, stream);
    }
    mark(11);
    }  // stage 3
    if (timing_) bwd_timed_once_ = true;
    cuda_check(cudaGetLastError(), "backward launch");
}

bool FlashIpaLayer::attention_impl_for_sharding() const {
    return attention_impl(dims_, tuning_.attn, true) == AttnImpl::pair;
}

// ------------------------------------------------------------ micro-batched capture
// Materialised attention backward for lifted rows wider than the fused kernels hold (z_factor_rank
// 3-4: D_qk / D_v up to ~700; attn_bwd.cu needs the 128 x D stationary tile in shared memory and the
// 128 x D accumulator next to S in TMEM).  Per group of att_samples whole samples, every product is
// one batched tcgen05 GEMM over the (sample, head) pairs and the softmax algebra is two streaming
// kernels -- the same arithmetic as the fused kernels (S in log2 units from the lifted rows, P
// rounded to bf16, dS = P (dP - D) rounded to bf16, fp32 accumulation), with [L, L] intermediates:
//   S = Q_hat K_hat^T ; P = 2^(S - lse2) ; O_hat = P V_hat (the training forward of these widths
//   saves no O_hat) ; prep (dO_hat, D, epilogue gradients) ; dP = dO_hat V_hat^T ;
//   dS = P (dP - D) ; dV = P^T dO_hat ; dK = dS^T Q_hat ; dQ = dS K_hat
// Workspace: 12 bytes per (sample, head, query, key) of one group -- quadratic in L, unlike the
// fused path (Tuning::ds_cap_mb bounds the group, one sample at least).
void FlashIpaLayer::dense_attention_backward(std::int64_t B, std::int64_t L, const float* z1, const float* rot,
                                             const Workspace& ws, cudaStream_t stream) {
    const LayerDims& d = dims_;
    const int H = d.heads, ld = ws.att_ld, acc = acc_ld(), Li = int(L);
    const std::int64_t rdz = std::int64_t(d.rank) * d.d_z;
    auto bf = [](const void* p) { return static_cast<const __nv_bfloat16*>(p); };
    for (std::int64_t b0 = 0; b0 < B; b0 += ws.att_samples) {
        const int nb = int(std::min<std::int64_t>(ws.att_samples, B - b0));
        const Workspace v = slice(ws, b0, L);
        const int Z = nb * H;
        // batched product over the group's (sample, head) pairs; C either [Z][L][ld] (square
        // intermediates) or the residue-major [nb, L, H, width] rows
        auto product = [&](const void* A, int64_t lda, bool a_mn, const void* Bm, int64_t ldb, bool b_mn, float* C,
                           bool residue_major, int width, int N, int K) {
            GemmArgs g;
            g.A = bf(A);
            g.lda = lda;
            g.a_mn_major = a_mn;
            g.B = bf(Bm);
            g.ldb = ldb;
            g.b_mn_major = b_mn;
            g.C = C;
            if (residue_major) {
                g.ldc = int64_t(H) * width;
                g.ldc_h = width;
                g.ldc_b = int64_t(L) * H * width;
                g.batch_h = H;
            } else {
                g.ldc = ld;
                g.ldc_h = ld;
                g.ldc_b = int64_t(L) * ld;
                g.batch_h = 1;
            }
            g.M = Li;
            g.N = N;
            g.K = K;
            g.batch = Z;
            launch_gemm_bf16(g, stream);
        };
        product(v.qhat, d.dqk_pad, false, v.khat, d.dqk_pad, false, ws.att_s, false, 0, Li, d.dqk_pad);  // S
        launch_dense_softmax(ws.att_s, ld, v.lse, int64_t(Z) * L, Li, ws.att_p, stream);                // P
        product(ws.att_p, ld, false, v.vhat, d.dv_pad, true, v.o_hat, true, d.dv_pad, d.dv_pad, Li);      // O_hat
        {
            BwdPrepArgs a{};
            a.dfeat = v.dfeat;
            a.ohat = v.o_hat;
            a.z1 = z1 + b0 * L * rdz;
            a.rot = rot + b0 * L * 9;
            a.trans_c = v.trans_c;
            a.dohat = v.do_hat;
            a.Dvec = v.Dvec;
            a.dz1_epi = v.dz1_epi;
            a.geo_epi = v.geo_epi;
            a.B = nb;
            a.L = Li;
            launch_bwd_prep(d, a, stream);
        }
        product(v.do_hat, d.dv_pad, false, v.vhat, d.dv_pad, false, ws.att_dp, false, 0, Li, d.dv_pad);  // dP
        launch_dense_ds(ws.att_p, ws.att_dp, ld, v.Dvec, int64_t(Z) * L, Li, ws.att_ds, stream);           // dS
        product(ws.att_p, ld, true, v.do_hat, d.dv_pad, true, v.dv_acc, true, acc, d.dv_mma, Li);          // dV
        product(ws.att_ds, ld, true, v.qhat, d.dqk_pad, true, v.dk_acc, true, acc, d.dqk_mma, Li);         // dK
        product(ws.att_ds, ld, false, v.khat, d.dqk_pad, true, v.dq_acc, true, acc, d.dqk_mma, Li);        // dQ
    }
}

int FlashIpaLayer::micro_chunks(std::int64_t B, std::int64_t L, bool forward) const {
    if (tuning_.micro < 2 || timing_ || cfg_.precision != Precision::bf16 || B < 2) return 1;
    // each chunk's weight-gradient GEMMs run split-K >= 2 over K = (B / chunks) * L
    if ((B / 2) * L < 256) return 1;
    int n = int(std::min<std::int64_t>(forward ? std::max(tuning_.micro, 4) : tuning_.micro, B));
    n = std::min(n, int(sizeof(side_streams_) / sizeof(side_streams_[0])) + 1);
    while (n > 2 && (B / n) * L < 256) --n;  // chunks of at least 256 residues
    return n;
}

void FlashIpaLayer::ensure_side_streams() {
    for (auto& st : side_streams_)
        if (!st) cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    if (!fork_ev_) cuda_check(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "event");
    for (auto& e : join_ev_)
        if (!e) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
}

void FlashIpaLayer::forward_micro(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                  const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                                  float* out, void* workspace, std::size_t workspace_bytes, cudaStream_t stream,
                                  bool train) {
    const Workspace full = carve(workspace, B, L, train);
    REQUIRE(workspace != nullptr && workspace_bytes >= full.bytes, "workspace too small: need ", full.bytes,
            " bytes, got ", workspace_bytes);
    ensure_side_streams();
    const int n = micro_chunks(B, L, true);
    const std::size_t rdz = std::size_t(dims_.rank) * dims_.d_z, din = dims_.d_in;
    cuda_check(cudaEventRecord(fork_ev_, stream), "event record");
    for (int c = 0; c < n; ++c) {
        const std::int64_t b0 = B * c / n, nb = B * (c + 1) / n - b0;
        const std::size_t r = std::size_t(b0) * L;
        cudaStream_t st = c == 0 ? stream : side_streams_[c - 1];
        if (c > 0) cuda_check(cudaStreamWaitEvent(st, fork_ev_, 0), "stream wait");
        const Workspace v = slice(full, b0, L);
        forward_impl(nb, L, s + r * din, z1 + r * rdz, z2 + r * rdz, rot + r * 9, trans + r * 3,
                     mask ? mask + r : nullptr, out + r * din, workspace, workspace_bytes, st, train, nullptr, &v);
    }
    for (int c = 1; c < n; ++c) {
        cuda_check(cudaEventRecord(join_ev_[c - 1], side_streams_[c - 1]), "event record");
        cuda_check(cudaStreamWaitEvent(stream, join_ev_[c - 1], 0), "stream wait");
    }
}

void FlashIpaLayer::backward_micro(std::int64_t B, std::int64_t L, const float* s, const float* z1,
                                   const float* z2, const float* rot, const float* trans, const std::uint8_t* mask,
                                   const float* dout, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                                   float* dweights, void* workspace, std::size_t workspace_bytes,
                                   cudaStream_t stream) {
    const Workspace full = carve(workspace, B, L, true);
    REQUIRE(workspace != nullptr && workspace_bytes >= full.bytes, "train workspace too small: need ", full.bytes,
            " bytes, got ", workspace_bytes);
    ensure_side_streams();
    const int n = micro_chunks(B, L);
    const std::size_t rdz = std::size_t(dims_.rank) * dims_.d_z, din = dims_.d_in;
    backward_impl(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
                  workspace_bytes, stream, nullptr, &full, 1);
    cuda_check(cudaEventRecord(fork_ev_, stream), "event record");
    for (int c = 0; c < n; ++c) {
        const std::int64_t b0 = B * c / n, nb = B * (c + 1) / n - b0;
        const std::size_t r = std::size_t(b0) * L;
        cudaStream_t st = c == 0 ? stream : side_streams_[c - 1];
        if (c > 0) cuda_check(cudaStreamWaitEvent(st, fork_ev_, 0), "stream wait");
        const Workspace v = slice(full, b0, L);
        backward_impl(nb, L, s + r * din, z1 + r * rdz, z2 + r * rdz, rot + r * 9, trans + r * 3,
                      mask ? mask + r : nullptr, dout + r * din, ds + r * din, dz1 + r * rdz, dz2 + r * rdz,
                      drot ? drot + r * 9 : nullptr, dtrans ? dtrans + r * 3 : nullptr, dweights, workspace,
                      workspace_bytes, st, nullptr, &v, 2);
    }
    for (int c = 1; c < n; ++c) {
        cuda_check(cudaEventRecord(join_ev_[c - 1], side_streams_[c - 1]), "event record");
        cuda_check(cudaStreamWaitEvent(stream, join_ev_[c - 1], 0), "stream wait");
    }
    backward_impl(B, L, s, z1, z2, rot, trans, mask, dout, ds, dz1, dz2, drot, dtrans, dweights, workspace,
                  workspace_bytes, stream, nullptr, &full, 4);
}

}  // namespace fipa_b200
