// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libfipa_ref.so).  It exposes the reference's own hot-path
// functions on plain double arrays so tests/ and bench.py's CPU-baseline leg
// can call them through ctypes:
//
//   IpaWeights::init            proj/src/ipa.cpp:172-193
//   flash_ipa_forward           proj/src/flash_ipa.cpp:141-218
//   reference_forward           proj/src/ipa.cpp:244-310
//   lift_qkv (+ w_l fold)       proj/src/flash_ipa.cpp:128-139, 161-167
//   flash_attention             proj/src/attention_kernel.cpp:213-243
//   save_weights / load_weights proj/src/model_io.cpp:121-196
//   random_rototranslation      proj/src/geometry.cpp:107-132
//   gaussian / Rng              proj/src/tensor.cpp:286-290, proj/src/rng.cpp:11-41
//   knn_distogram / positional_encoding / build_factors
//                               proj/src/pair_features.cpp:10-97
//   fit_polynomial              proj/src/bench.cpp:103-149
//   report_to_csv / report_to_json / parse_records_csv / load_config + config_to_json
//                               proj/src/model_io.cpp:198-405
//
// Status codes mirror the product C-ABI: 0 ok, 1 ValueError, 2 NumericError,
// 3 IoError, 9 other.

#include <cstdint>
#include <cstring>
#include <sstream>
#include <exception>
#include <string>
#include <vector>

#include "fipa/attention_kernel.hpp"
#include "fipa/bench.hpp"
#include "fipa/error.hpp"
#include "fipa/flash_ipa.hpp"
#include "fipa/geometry.hpp"
#include "fipa/ipa.hpp"
#include "fipa/model_io.hpp"
#include "fipa/pair_features.hpp"
#include "fipa/rng.hpp"
#include "fipa/tensor.hpp"

using namespace fipa;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ValueError& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

// cfg = [d_in, d_z, heads, c, n_query, n_value, rank, precision(0 f32 / 1 f64), enforce_cap]
IpaConfig make_cfg(const std::uint64_t* c) {
    IpaConfig cfg;
    cfg.d_in = c[0];
    cfg.d_z = c[1];
    cfg.heads = c[2];
    cfg.c = c[3];
    cfg.n_query = c[4];
    cfg.n_value = c[5];
    cfg.rank = c[6];
    cfg.precision = c[7] == 0 ? Precision::f32 : Precision::f64;
    cfg.enforce_head_cap = c[8] != 0;
    return cfg;
}

Tensor from_ptr(const double* p, std::vector<std::size_t> shape, Precision prec) {
    Tensor t(std::move(shape), prec);
    for (std::size_t i = 0; i < t.size(); ++i) t.set_flat(i, p[i]);
    return t;
}

void to_ptr(const Tensor& t, double* p) {
    for (std::size_t i = 0; i < t.size(); ++i) p[i] = t.get_flat(i);
}

// Weight order: w_q w_k w_v w_qp w_kp w_vp w_bias gamma_raw w_out b_out; scal = {w_l, w_c}.
struct Shapes {
    std::vector<std::vector<std::size_t>> s;
    explicit Shapes(const IpaConfig& c) {
        const std::size_t seg = c.d_z + c.c + 4 * c.n_value;
        s = {{c.d_in, c.heads * c.c},
             {c.d_in, c.heads * c.c},
             {c.d_in, c.heads * c.c},
             {c.d_in, c.heads * c.n_query * 3},
             {c.d_in, c.heads * c.n_query * 3},
             {c.d_in, c.heads * c.n_value * 3},
             {c.heads, c.d_z},
             {c.heads},
             {c.heads * seg, c.d_in},
             {c.d_in}};
    }
};

IpaWeights make_weights(const IpaConfig& cfg, double* const* w, const double* scal) {
    const Shapes sh(cfg);
    const Precision p = cfg.precision;
    IpaWeights out;
    Tensor* dst[10] = {&out.w_q, &out.w_k, &out.w_v, &out.w_qp, &out.w_kp,
                       &out.w_vp, &out.w_bias, &out.gamma_raw, &out.w_out, &out.b_out};
    for (int i = 0; i < 10; ++i) *dst[i] = from_ptr(w[i], sh.s[i], p);
    out.w_l = scal[0];
    out.w_c = scal[1];
    return out;
}

void export_weights(const IpaConfig& cfg, const IpaWeights& in, double* const* w, double* scal) {
    const Shapes sh(cfg);
    const Tensor* src[10] = {&in.w_q, &in.w_k, &in.w_v, &in.w_qp, &in.w_kp,
                             &in.w_vp, &in.w_bias, &in.gamma_raw, &in.w_out, &in.b_out};
    for (int i = 0; i < 10; ++i) {
        FIPA_REQUIRE(src[i]->shape() == sh.s[i], "weights tensor ", i,
                     " has a shape that disagrees with the configuration");
        to_ptr(*src[i], w[i]);
    }
    scal[0] = in.w_l;
    scal[1] = in.w_c;
}

FrameSet make_frames(std::size_t L, const double* rot, const double* trans,
                     const std::uint8_t* mask) {
    FrameSet f;
    f.frames.resize(L);
    for (std::size_t i = 0; i < L; ++i) {
        for (int k = 0; k < 9; ++k) f.frames[i].rotation[k] = rot[i * 9 + k];
        for (int k = 0; k < 3; ++k) f.frames[i].translation[k] = trans[i * 3 + k];
    }
    f.mask.assign(L, true);
    if (mask != nullptr) {
        for (std::size_t i = 0; i < L; ++i) f.mask[i] = mask[i] != 0;
    }
    return f;
}

FactorizedPair make_pair(const IpaConfig& cfg, std::size_t L, const double* z1,
                         const double* z2) {
    FactorizedPair fp;
    fp.z1 = from_ptr(z1, {L, cfg.rank, cfg.d_z}, cfg.precision);
    fp.z2 = from_ptr(z2, {L, cfg.rank, cfg.d_z}, cfg.precision);
    return fp;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_init_weights(const std::uint64_t* c, std::uint64_t seed, double* const* w, double* scal) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        Rng rng(seed);
        export_weights(cfg, IpaWeights::init(cfg, rng), w, scal);
    });
}

int ref_flash_forward(const std::uint64_t* c, double* const* w, const double* scal,
                      std::uint64_t L, const double* s, const double* z1, const double* z2,
                      const double* rot, const double* trans, const std::uint8_t* mask,
                      std::uint64_t tile_rows, std::uint64_t tile_cols, int threads,
                      double* out) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        const IpaWeights wt = make_weights(cfg, w, scal);
        const Tensor ts = from_ptr(s, {L, cfg.d_in}, cfg.precision);
        const FactorizedPair fp = make_pair(cfg, L, z1, z2);
        const FrameSet frames = make_frames(L, rot, trans, mask);
        TileSpec tiles;
        tiles.block_rows = tile_rows;
        tiles.block_cols = tile_cols;
        to_ptr(flash_ipa_forward(ts, fp, frames, cfg, wt, tiles, threads), out);
    });
}

int ref_reference_forward(const std::uint64_t* c, double* const* w, const double* scal,
                          std::uint64_t L, const double* s, const double* z1, const double* z2,
                          const double* rot, const double* trans, const std::uint8_t* mask,
                          double* out) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        const IpaWeights wt = make_weights(cfg, w, scal);
        const Tensor ts = from_ptr(s, {L, cfg.d_in}, cfg.precision);
        const FactorizedPair fp = make_pair(cfg, L, z1, z2);
        const FrameSet frames = make_frames(L, rot, trans, mask);
        PairRep pair;
        pair.factors = &fp;
        to_ptr(reference_forward(ts, pair, frames, cfg, wt), out);
    });
}

// The lifted rows exactly as flash_ipa_forward builds them (w_l folded into
// the bias weights first, flash_ipa.cpp:161-167).  q_hat/k_hat [H, L, qk_width],
// v_hat [H, L, v_width].
int ref_lift(const std::uint64_t* c, double* const* w, const double* scal, std::uint64_t L,
             const double* s, const double* z1, const double* z2, const double* rot,
             const double* trans, double* q_hat, double* k_hat, double* v_hat) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        const IpaWeights wt = make_weights(cfg, w, scal);
        const Tensor ts = from_ptr(s, {L, cfg.d_in}, cfg.precision);
        const FactorizedPair fp = make_pair(cfg, L, z1, z2);
        const FrameSet frames = make_frames(L, rot, trans, nullptr);
        Tensor scaled({cfg.heads, cfg.d_z}, cfg.precision);
        for (std::size_t e = 0; e < scaled.size(); ++e) {
            scaled.set_flat(e, wt.w_l * wt.w_bias.get_flat(e));
        }
        const auto [b1, b2] = bias_factors(fp, scaled);
        const Projections proj = project_inputs(ts, cfg, wt);
        const LiftedQKV lifted = lift_qkv(proj, frames, b1, b2, fp, cfg, wt);
        to_ptr(lifted.q_hat, q_hat);
        to_ptr(lifted.k_hat, k_hat);
        to_ptr(lifted.v_hat, v_hat);
    });
}

int ref_flash_attention(std::uint64_t H, std::uint64_t L, std::uint64_t dqk, std::uint64_t dv,
                        const double* q, const double* k, const double* v,
                        const std::uint8_t* mask, std::uint64_t tile_rows,
                        std::uint64_t tile_cols, int threads, double* out) {
    return guarded([&] {
        const Tensor tq = from_ptr(q, {H, L, dqk}, Precision::f64);
        const Tensor tk = from_ptr(k, {H, L, dqk}, Precision::f64);
        const Tensor tv = from_ptr(v, {H, L, dv}, Precision::f64);
        std::vector<bool> m;
        if (mask != nullptr) {
            m.resize(L);
            for (std::size_t i = 0; i < L; ++i) m[i] = mask[i] != 0;
        }
        TileSpec tiles;
        tiles.block_rows = tile_rows;
        tiles.block_cols = tile_cols;
        to_ptr(flash_attention(tq, tk, tv, m, tiles, threads), out);
    });
}

int ref_save_weights(const std::uint64_t* c, double* const* w, const double* scal,
                     const char* path) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        save_weights(make_weights(cfg, w, scal), path);
    });
}

int ref_load_weights(const std::uint64_t* c, const char* path, double* const* w, double* scal) {
    return guarded([&] {
        const IpaConfig cfg = make_cfg(c);
        export_weights(cfg, load_weights(path), w, scal);
    });
}

int ref_random_frames(std::uint64_t seed, std::uint64_t L, double scale, double* rot,
                      double* trans) {
    return guarded([&] {
        Rng rng(seed);
        for (std::size_t i = 0; i < L; ++i) {
            const RigidTransform t = random_rototranslation(rng, scale);
            for (int k = 0; k < 9; ++k) rot[i * 9 + k] = t.rotation[k];
            for (int k = 0; k < 3; ++k) trans[i * 3 + k] = t.translation[k];
        }
    });
}

int ref_gaussian(std::uint64_t seed, std::uint64_t n, double stddev, double* out) {
    return guarded([&] {
        Rng rng(seed);
        to_ptr(gaussian(rng, {n}, stddev), out);
    });
}

// translations [L,3] f64 -> features [L, k, n_bins + pe_dim]
int ref_knn_distogram(std::uint64_t L, const double* trans, std::uint64_t k, std::uint64_t n_bins, double d_min,
                      double d_max, std::uint64_t pe_dim, double* out) {
    return guarded([&] {
        DistogramSpec spec;
        spec.k = k;
        spec.n_bins = n_bins;
        spec.d_min = d_min;
        spec.d_max = d_max;
        spec.pe_dim = pe_dim;
        to_ptr(knn_distogram(from_ptr(trans, {L, 3}, Precision::f64), spec), out);
    });
}

// features [L, f] x w1, w2 [f, r*d_z] -> z1, z2 [L, r, d_z]
int ref_build_factors(std::uint64_t L, std::uint64_t f, const double* feat, std::uint64_t r, std::uint64_t d_z,
                      const double* w1, const double* w2, double* z1, double* z2) {
    return guarded([&] {
        const FactorizedPair fp = build_factors(from_ptr(feat, {L, f}, Precision::f64), r, d_z,
                                                from_ptr(w1, {f, r * d_z}, Precision::f64),
                                                from_ptr(w2, {f, r * d_z}, Precision::f64));
        to_ptr(fp.z1, z1);
        to_ptr(fp.z2, z2);
    });
}

// ---------------------------------------------------------------- report / fit schema (f4)
// Strings cross as '\n'-joined lists; text results are copied into buf (cap bytes, NUL-terminated)
// and *need receives the full length.

// y = a L^2 + b L least squares (bench.cpp:103-149): out = {a, b, r^2}
int ref_fit_polynomial(std::uint64_t n, const double* L, const double* y, double* out) {
    return guarded([&] {
        std::vector<std::pair<double, double>> pts;
        for (std::uint64_t i = 0; i < n; ++i) pts.emplace_back(L[i], y[i]);
        const FitCoefficients f = fit_polynomial(pts);
        out[0] = f.quadratic;
        out[1] = f.linear;
        out[2] = f.r_squared;
    });
}

namespace {
std::vector<std::string> split_lines(const char* s, std::uint64_t n) {
    std::vector<std::string> out;
    std::string cur;
    for (const char* p = s ? s : ""; *p; ++p) {
        if (*p == '\n') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur.push_back(*p);
        }
    }
    if (!cur.empty() || out.size() < n) out.push_back(cur);
    out.resize(n);
    return out;
}

void put_text(const std::string& t, char* buf, std::uint64_t cap, std::uint64_t* need) {
    *need = t.size();
    if (buf != nullptr && cap > 0) {
        const std::size_t m = std::min<std::size_t>(t.size(), cap - 1);
        std::memcpy(buf, t.data(), m);
        buf[m] = '\0';
    }
}

// records: arms '\n'-joined; prec 0 = f32, 1 = f64
RunReport make_report(const char* command, const char* config_echo, std::uint64_t n, const char* arms,
                      const std::uint64_t* lengths, const std::uint64_t* seeds, const int* prec,
                      const std::uint64_t* peak, const double* secs, std::uint64_t nf, const char* fit_arms,
                      const char* fit_metrics, const double* fit_vals, std::uint64_t nc, const char* check_names,
                      const double* check_vals, const int* check_pass, std::uint64_t nn, const char* notes) {
    RunReport r;
    r.command = command ? command : "";
    r.config_echo = config_echo ? config_echo : "";
    const auto a = split_lines(arms, n);
    for (std::uint64_t i = 0; i < n; ++i) {
        RunRecord rec;
        rec.arm = a[i];
        rec.length = lengths[i];
        rec.seed = seeds[i];
        rec.precision = prec[i] == 0 ? Precision::f32 : Precision::f64;
        rec.peak_bytes = peak[i];
        rec.seconds = secs[i];
        r.records.push_back(rec);
    }
    const auto fa = split_lines(fit_arms, nf), fm = split_lines(fit_metrics, nf);
    for (std::uint64_t i = 0; i < nf; ++i)
        r.fits.push_back(FitSummary{fa[i], fm[i], fit_vals[3 * i], fit_vals[3 * i + 1], fit_vals[3 * i + 2]});
    const auto cn = split_lines(check_names, nc);
    for (std::uint64_t i = 0; i < nc; ++i)
        r.checks.push_back(CheckOutcome{cn[i], check_vals[2 * i], check_vals[2 * i + 1], check_pass[i] != 0});
    r.notes = split_lines(notes, nn);
    return r;
}
}  // namespace

// format 0 = csv, 1 = json (model_io.cpp:200-243)
int ref_report_text(int format, const char* command, const char* config_echo, std::uint64_t n, const char* arms,
                    const std::uint64_t* lengths, const std::uint64_t* seeds, const int* prec,
                    const std::uint64_t* peak, const double* secs, std::uint64_t nf, const char* fit_arms,
                    const char* fit_metrics, const double* fit_vals, std::uint64_t nc, const char* check_names,
                    const double* check_vals, const int* check_pass, std::uint64_t nn, const char* notes, char* buf,
                    std::uint64_t cap, std::uint64_t* need) {
    return guarded([&] {
        const RunReport r = make_report(command, config_echo, n, arms, lengths, seeds, prec, peak, secs, nf, fit_arms,
                                        fit_metrics, fit_vals, nc, check_names, check_vals, check_pass, nn, notes);
        put_text(format == 0 ? report_to_csv(r) : report_to_json(r), buf, cap, need);
    });
}

// parse_records_csv (model_io.cpp:260-306) re-serialised as its CSV (records only)
int ref_parse_records_csv(const char* path, char* buf, std::uint64_t cap, std::uint64_t* need) {
    return guarded([&] {
        RunReport r;
        r.records = parse_records_csv(path);
        put_text(report_to_csv(r), buf, cap, need);
    });
}

// config_to_json(load_config(path)) (model_io.cpp:308-405); path "" = defaults
int ref_config_json(const char* path, char* buf, std::uint64_t cap, std::uint64_t* need) {
    return guarded([&] { put_text(config_to_json(load_config(path ? path : "")), buf, cap, need); });
}

}  // extern "C"
