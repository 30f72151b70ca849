// pybind11 module `_fipa_b200`: the reference Python surface (proj/python/bindings.cpp:171-195,
// proj/python/fipa/__init__.py) rebuilt over the C ABI in include/fipa_b200.h.  Only C-ABI calls
// are made from here; numpy arrays are accepted as float64 (other dtypes cast) and results come
// back as float64, like the reference (bindings.cpp:26-45).
#include <pybind11/numpy.h>
#include <sys/mman.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <new>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fipa_b200.h"

namespace py = pybind11;

namespace {
// Large output arrays of the host entry points come from a recycling pool of 2 MB-aligned buffers,
// handed back when Python frees the array: the allocator otherwise maps fresh pages for each
// call's outputs and the first touch costs ~7 ms per 68 MB gradient set (the float64 flash_grad
// measured 14 ms per call at B=8 L=1024 against 8 ms with recycled pages).  Bounded: at most
// kMaxHeld bytes wait in the pool.
class HostBufPool {
public:
    static HostBufPool& get() {
        static HostBufPool* pool = new HostBufPool();  // never destroyed: arrays may outlive statics
        return *pool;
    }
    void* take(size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = free_.find(bytes);
            if (it != free_.end() && !it->second.empty()) {
                void* p = it->second.back();
                it->second.pop_back();
                held_ -= bytes;
                return p;
            }
        }
        void* p = std::aligned_alloc(size_t(2) << 20, bytes);
        if (p == nullptr) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);
        return p;
    }
    void give(void* p, size_t bytes) {
        std::lock_guard<std::mutex> lk(mu_);
        if (held_ + bytes > kMaxHeld) {
            std::free(p);
            return;
        }
        free_[bytes].push_back(p);
        held_ += bytes;
    }

private:
    static constexpr size_t kMaxHeld = size_t(1) << 30;
    std::mutex mu_;
    std::map<size_t, std::vector<void*>> free_;
    size_t held_ = 0;
};

// C-contiguous output array: pooled when >= 1 MB, a plain numpy allocation otherwise.
template <class T>
py::array_t<T> host_out(const std::vector<py::ssize_t>& shape) {
    size_t n = 1;
    for (auto d : shape) n *= size_t(d);
    if (n * sizeof(T) < (size_t(1) << 20)) return py::array_t<T>(shape);
    const size_t huge = size_t(2) << 20, bytes = (n * sizeof(T) + huge - 1) / huge * huge;
    void* p = HostBufPool::get().take(bytes);
    auto* info = new std::pair<void*, size_t>(p, bytes);
    py::capsule owner(info, [](void* v) {
        auto* i = static_cast<std::pair<void*, size_t>*>(v);
        HostBufPool::get().give(i->first, i->second);
        delete i;
    });
    return py::array_t<T>(shape, static_cast<T*>(p), owner);
}
}  // namespace

namespace {

using DArr = py::array_t<double, py::array::c_style | py::array::forcecast>;
using FArr = py::array_t<float, py::array::c_style | py::array::forcecast>;

// Additive float32 host API: when every array argument is a float32 numpy array the host path
// skips the float64 round trip (float32 in, float32 out); anything else takes the reference's
// float64 convention (proj/python/bindings.cpp:26-45).
bool all_f32(std::initializer_list<py::handle> xs) {
    for (py::handle h : xs) {
        if (!py::isinstance<py::array>(h)) return false;
        if (!py::reinterpret_borrow<py::array>(h).dtype().is(py::dtype::of<float>())) return false;
    }
    return true;
}

struct FipaValueError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FipaNumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FipaIoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FipaCudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FipaCommError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void check(int rc) {
    if (rc == FIPA_OK) return;
    const std::string msg = fipa_last_error();
    switch (rc) {
        case FIPA_ERR_VALUE: throw FipaValueError(msg);
        case FIPA_ERR_NUMERIC: throw FipaNumericError(msg);
        case FIPA_ERR_IO: throw FipaIoError(msg);
        case FIPA_ERR_CUDA: throw FipaCudaError(msg);
        case FIPA_ERR_COMM: throw FipaCommError(msg);
        default: throw std::runtime_error(msg);
    }
}

int parse_precision(const std::string& name) {
    if (name == "bf16") return FIPA_PREC_BF16;
    if (name == "f32") return FIPA_PREC_F32;
    if (name == "f64") return FIPA_PREC_F64;
    throw FipaValueError("unknown precision '" + name + "' (expected f32, f64 or bf16)");
}

const char* kNames[10] = {"w_q", "w_k", "w_v", "w_qp", "w_kp", "w_vp", "w_bias", "gamma_raw", "w_out", "b_out"};


// flash_attention / naive_attention (python/bindings.cpp:153-165, 202-220): q, k [L, d] or
// [H, L, d], v [L, d_v] or [H, L, d_v]; the output matches v's leading shape.
py::array_t<double> py_attention(const DArr& q, const DArr& k, const DArr& v, const py::object& mask, bool naive) {
    if (q.ndim() != k.ndim() || q.ndim() != v.ndim()) throw FipaValueError("attention operands must share rank");
    if (q.ndim() != 2 && q.ndim() != 3) throw FipaValueError("attention operands are [L, d] or [H, L, d]");
    const bool heads = q.ndim() == 3;
    const int a0 = heads ? 1 : 0;
    const int64_t H = heads ? q.shape(0) : 1, L = q.shape(a0), dqk = q.shape(a0 + 1), dv = v.shape(a0 + 1);
    if (heads && (k.shape(0) != H || v.shape(0) != H)) throw FipaValueError("attention operands must share the head count");
    if (k.shape(a0) != L || v.shape(a0) != L) throw FipaValueError("attention operands must share the sequence length");
    if (k.shape(a0 + 1) != dqk) throw FipaValueError("Q and K widths differ");
    std::vector<uint8_t> m;
    if (!mask.is_none()) {
        py::array_t<uint8_t, py::array::c_style | py::array::forcecast> ma(mask);
        if (ma.size() != L) throw FipaValueError("mask length must equal the sequence length");
        m.assign(ma.data(), ma.data() + ma.size());
        for (auto& x : m) x = x ? 1 : 0;
    }
    std::vector<py::ssize_t> shape = heads ? std::vector<py::ssize_t>{H, L, dv} : std::vector<py::ssize_t>{L, dv};
    py::array_t<double> out(shape);
    if (L == 0 || dv == 0) return out;
    double* op = out.mutable_data();
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = fipa_attention_host(H, L, dqk, dv, q.data(), k.data(), v.data(), m.empty() ? nullptr : m.data(), op,
                                 naive ? 1 : 0, 0);
    }
    check(rc);
    return out;
}

// NCCL communicator for query-row sharding (one per process / GPU).
class Comm {
public:
    Comm(int world, int rank, const py::bytes& uid, int device) {
        const std::string id = uid;
        if (id.size() != 128) throw FipaValueError("NCCL unique id must be 128 bytes");
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_comm_create(world, rank, reinterpret_cast<const uint8_t*>(id.data()), device, &comm_);
        }
        check(rc);
        world_ = world;
        rank_ = rank;
    }
    ~Comm() { fipa_comm_destroy(comm_); }
    Comm(const Comm&) = delete;
    Comm& operator=(const Comm&) = delete;
    fipa_comm* get() const { return comm_; }
    void all_reduce_sum_f32(uintptr_t buf, size_t n, uintptr_t stream) {
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_comm_all_reduce_f32(comm_, reinterpret_cast<float*>(buf), n, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    int world() const { return world_; }
    int rank() const { return rank_; }

private:
    fipa_comm* comm_ = nullptr;
    int world_ = 1, rank_ = 0;
};

py::bytes comm_unique_id() {
    uint8_t id[128];
    check(fipa_comm_unique_id(id));
    return py::bytes(reinterpret_cast<const char*>(id), 128);
}

class Model {
public:
    Model(uint64_t d_in, uint64_t d_z, uint64_t heads, uint64_t c, uint64_t n_query,
          uint64_t n_value, uint64_t rank, const std::string& precision, uint64_t seed,
          bool enforce_head_cap)
        : precision_name_(precision) {
        cfg_.d_in = d_in;
        cfg_.d_z = d_z;
        cfg_.heads = heads;
        cfg_.c = c;
        cfg_.n_query = n_query;
        cfg_.n_value = n_value;
        cfg_.rank = rank;
        cfg_.precision = parse_precision(precision);
        cfg_.enforce_head_cap = enforce_head_cap ? 1 : 0;
        check(fipa_config_validate(&cfg_));
        check(fipa_layer_create(&cfg_, &layer_));
        check(fipa_layer_init_weights(layer_, seed));
    }
    // Borrowed view of a trunk layer (fipa_trunk_layer); destroying it is a no-op in the C ABI.
    Model(fipa_layer* borrowed, const fipa_config& cfg, const std::string& precision)
        : cfg_(cfg), layer_(borrowed), precision_name_(precision) {}
    ~Model() { fipa_layer_destroy(layer_); }
    Model(const Model&) = delete;
    Model& operator=(const Model&) = delete;

    std::vector<std::vector<size_t>> shapes() const {
        const size_t seg = cfg_.d_z + cfg_.c + 4 * cfg_.n_value;
        return {{cfg_.d_in, cfg_.heads * cfg_.c},          {cfg_.d_in, cfg_.heads * cfg_.c},
                {cfg_.d_in, cfg_.heads * cfg_.c},          {cfg_.d_in, cfg_.heads * cfg_.n_query * 3},
                {cfg_.d_in, cfg_.heads * cfg_.n_query * 3}, {cfg_.d_in, cfg_.heads * cfg_.n_value * 3},
                {cfg_.heads, cfg_.d_z},                    {cfg_.heads},
                {cfg_.heads * seg, cfg_.d_in},             {cfg_.d_in}};
    }

    // flash(s, z1, z2, rotations, translations, mask=None, tile_rows=64, tile_cols=64, threads=1)
    // Unbatched [L, ...] inputs return [L, d_in]; a leading batch axis [B, L, ...] is accepted
    // additively (mask then [B][L]).  Tiling/thread arguments are accepted and ignored: the
    // GPU result does not depend on them (reference guarantee, attention_kernel.hpp:34-37).
    py::array flash(const py::object& s, const py::object& z1, const py::object& z2, const py::object& rotations,
                    const py::object& translations, const py::object& mask, size_t tile_rows, size_t tile_cols,
                    int threads) {
        if (tile_rows == 0 || tile_cols == 0) throw FipaValueError("tile sizes must be positive");
        (void)threads;
        if (all_f32({s, z1, z2, rotations, translations}))
            return run_host<float>(FArr(s), FArr(z1), FArr(z2), FArr(rotations), FArr(translations), mask, false);
        return run_host<double>(DArr(s), DArr(z1), DArr(z2), DArr(rotations), DArr(translations), mask, false);
    }

    // Quadratic-memory forward (python/bindings.cpp:187-189 `reference`), on the GPU in fp32.
    py::array reference(const DArr& s, const DArr& z1, const DArr& z2, const DArr& rotations,
                        const DArr& translations, const py::object& mask) {
        return run_host<double>(s, z1, z2, rotations, translations, mask, true);
    }
    size_t reference_workspace_size(int64_t B, int64_t L) const {
        return fipa_layer_reference_workspace_size(layer_, B, L);
    }
    void reference_device(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                          uintptr_t trans, uintptr_t mask, uintptr_t out, uintptr_t ws, size_t ws_bytes,
                          uintptr_t stream) {
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_reference_forward(layer_, B, L, reinterpret_cast<const float*>(s),
                                              reinterpret_cast<const float*>(z1), reinterpret_cast<const float*>(z2),
                                              reinterpret_cast<const float*>(rot), reinterpret_cast<const float*>(trans),
                                              reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(out),
                                              reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }

    template <class T>
    py::array run_host(const py::array_t<T, py::array::c_style | py::array::forcecast>& s,
                       const py::array_t<T, py::array::c_style | py::array::forcecast>& z1,
                       const py::array_t<T, py::array::c_style | py::array::forcecast>& z2,
                       const py::array_t<T, py::array::c_style | py::array::forcecast>& rotations,
                       const py::array_t<T, py::array::c_style | py::array::forcecast>& translations,
                       const py::object& mask, bool dense) {
        using Arr = py::array_t<T, py::array::c_style | py::array::forcecast>;
        const bool batched = s.ndim() == 3;
        if (s.ndim() != 2 && s.ndim() != 3)
            throw FipaValueError("single representation must be [L, d_in] or [B, L, d_in]");
        const int64_t B = batched ? s.shape(0) : 1;
        const int64_t L = batched ? s.shape(1) : s.shape(0);
        const int o = batched ? 1 : 0;
        if (L < 1) throw FipaValueError("empty frame set");
        if (batched && s.shape(0) < 1) throw FipaValueError("batch must be >= 1");
        if (s.shape(o + 1) != int64_t(cfg_.d_in))
            throw FipaValueError("single representation must be [L, " + std::to_string(cfg_.d_in) + "]");
        auto lead_ok = [&](const Arr& a, int nd) {
            if (a.ndim() != nd + o) return false;
            if (batched && a.shape(0) != B) return false;
            return a.shape(o) == L;
        };
        if (!lead_ok(rotations, 3) || rotations.shape(o + 1) != 3 || rotations.shape(o + 2) != 3)
            throw FipaValueError("rotations must have shape [L, 3, 3]");
        if (!lead_ok(translations, 2) || translations.shape(o + 1) != 3)
            throw FipaValueError("translations must have shape [L, 3]");
        for (const Arr* z : {&z1, &z2}) {
            if (!lead_ok(*z, 3) || z->shape(o + 1) != int64_t(cfg_.rank) ||
                z->shape(o + 2) != int64_t(cfg_.d_z))
                throw FipaValueError("factor shapes disagree with the configuration");
        }
        std::vector<uint8_t> m;
        const uint8_t* mp = nullptr;
        if (!mask.is_none()) {
            py::array_t<uint8_t, py::array::c_style | py::array::forcecast> ma(mask);
            if (ma.size() != B * L) throw FipaValueError("mask length must equal L");
            m.assign(ma.data(), ma.data() + ma.size());
            for (auto& v : m) v = v ? 1 : 0;
            mp = m.data();
        }
        std::vector<py::ssize_t> shape = batched ? std::vector<py::ssize_t>{B, L, (py::ssize_t)cfg_.d_in}
                                                 : std::vector<py::ssize_t>{L, (py::ssize_t)cfg_.d_in};
        py::array_t<T> out = host_out<T>(shape);
        T* op = out.mutable_data();
        int rc;
        {
            py::gil_scoped_release nogil;
            if constexpr (std::is_same_v<T, float>) {
                rc = fipa_layer_forward_host_f32(layer_, B, L, s.data(), z1.data(), z2.data(), rotations.data(),
                                                 translations.data(), mp, op);
            } else {
                rc = dense ? fipa_layer_reference_host(layer_, B, L, s.data(), z1.data(), z2.data(), rotations.data(),
                                                       translations.data(), mp, op)
                           : fipa_layer_forward_host(layer_, B, L, s.data(), z1.data(), z2.data(), rotations.data(),
                                                     translations.data(), mp, op);
            }
        }
        check(rc);
        return out;
    }

    void save(const std::string& path) const { check(fipa_layer_save_weights(layer_, path.c_str())); }
    void load(const std::string& path) { check(fipa_layer_load_weights(layer_, path.c_str())); }

    py::dict weights() const {
        const auto sh = shapes();
        std::vector<py::array_t<double>> arrs;
        double* ptrs[10];
        for (int i = 0; i < 10; ++i) {
            arrs.emplace_back(std::vector<py::ssize_t>(sh[i].begin(), sh[i].end()));
            ptrs[i] = arrs.back().mutable_data();
        }
        double scal[2];
        check(fipa_layer_get_weights(layer_, ptrs, scal));
        py::dict d;
        for (int i = 0; i < 10; ++i) d[kNames[i]] = arrs[i];
        d["w_l"] = scal[0];
        d["w_c"] = scal[1];
        return d;
    }

    void set_weights(const py::dict& d) {
        const auto sh = shapes();
        std::vector<DArr> keep;
        fipa_host_weights w{};
        const double** dst[10] = {&w.w_q,  &w.w_k,    &w.w_v,         &w.w_qp,   &w.w_kp,
                                  &w.w_vp, &w.w_bias, &w.gamma_raw,   &w.w_out,  &w.b_out};
        for (int i = 0; i < 10; ++i) {
            DArr a(d[kNames[i]]);
            size_t n = 1;
            for (auto v : sh[i]) n *= v;
            if (size_t(a.size()) != n)
                throw FipaValueError(std::string("weights tensor '") + kNames[i] + "' has the wrong size");
            keep.push_back(a);
            *dst[i] = keep.back().data();
        }
        w.w_l = d["w_l"].cast<double>();
        w.w_c = d["w_c"].cast<double>();
        check(fipa_layer_set_weights(layer_, &w));
    }

    size_t workspace_size(int64_t B, int64_t L) const { return fipa_layer_workspace_size(layer_, B, L); }

    // Device-pointer forward for benchmarks / tests that own device memory (e.g. torch tensors).
    void forward_device(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                        uintptr_t trans, uintptr_t mask, uintptr_t out, uintptr_t ws, size_t ws_bytes,
                        uintptr_t stream) {
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_forward(layer_, B, L, reinterpret_cast<const float*>(s),
                                    reinterpret_cast<const float*>(z1), reinterpret_cast<const float*>(z2),
                                    reinterpret_cast<const float*>(rot), reinterpret_cast<const float*>(trans),
                                    reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(out),
                                    reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }

    py::tuple workspace_layout(int64_t B, int64_t L) const {
        int64_t off[9], dims[4];
        const int n = fipa_layer_workspace_layout(layer_, B, L, off, dims);
        if (n != 9) throw FipaValueError("invalid batch shape");
        return py::make_tuple(std::vector<int64_t>(off, off + 9), std::vector<int64_t>(dims, dims + 4));
    }

    int forward_launches() const { return fipa_layer_forward_launches(layer_); }
    int step_launches(int64_t B, int64_t L, bool train) const {
        return fipa_layer_step_launches(layer_, B, L, train ? 1 : 0);
    }
    int backward_launches() const { return fipa_layer_backward_launches(layer_); }
    size_t sharded_workspace_size(int64_t B, int64_t L, int world) const {
        return fipa_layer_sharded_workspace_size(layer_, B, L, world);
    }
    void forward_sharded_device(Comm& comm, int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2,
                                uintptr_t rot, uintptr_t trans, uintptr_t mask, uintptr_t out, uintptr_t ws,
                                size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<const float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_forward_sharded(layer_, comm.get(), B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                            reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(out),
                                            reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    void shard_centroid_sums(int64_t B, int64_t L, uintptr_t trans, uintptr_t mask, uintptr_t sums, uintptr_t stream) {
        check(fipa_layer_shard_centroid_sums(layer_, B, L, reinterpret_cast<const float*>(trans),
                                             reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(sums),
                                             reinterpret_cast<void*>(stream)));
    }
    py::tuple shard_pack(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                         uintptr_t trans, uintptr_t mask, uintptr_t sums, uintptr_t ws, size_t ws_bytes,
                         uintptr_t stream, bool train) {
        auto f = [](uintptr_t p) { return reinterpret_cast<const float*>(p); };
        void *k = nullptr, *v = nullptr;
        size_t kb = 0, vb = 0;
        check((train ? fipa_layer_shard_pack_train : fipa_layer_shard_pack)(layer_, B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                    reinterpret_cast<const uint8_t*>(mask), f(sums), reinterpret_cast<void*>(ws),
                                    ws_bytes, reinterpret_cast<void*>(stream), &k, &kb, &v, &vb));
        return py::make_tuple(reinterpret_cast<uintptr_t>(k), kb, reinterpret_cast<uintptr_t>(v), vb);
    }
    void shard_attend(int64_t B, int64_t L, int world, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                      uintptr_t trans, uintptr_t mask, uintptr_t k_all, uintptr_t v_all, uintptr_t out, uintptr_t ws,
                      size_t ws_bytes, uintptr_t stream, bool train) {
        auto f = [](uintptr_t p) { return reinterpret_cast<const float*>(p); };
        check((train ? fipa_layer_shard_attend_train : fipa_layer_shard_attend)(layer_, B, L, world, f(s), f(z1), f(z2), f(rot), f(trans),
                                      reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<const void*>(k_all),
                                      reinterpret_cast<const void*>(v_all), reinterpret_cast<float*>(out),
                                      reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream)));
    }
    void shard_backward(int stage, int world, int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2,
                        uintptr_t rot, uintptr_t trans, uintptr_t mask, uintptr_t dout, uintptr_t k_all,
                        uintptr_t v_all, uintptr_t dk_part, uintptr_t dv_part, uintptr_t dk_own, uintptr_t dv_own,
                        uintptr_t dt_sums, uintptr_t ds, uintptr_t dz1, uintptr_t dz2, uintptr_t drot,
                        uintptr_t dtrans, uintptr_t dweights, uintptr_t ws, size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_shard_backward(layer_, stage, world, B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                           reinterpret_cast<const uint8_t*>(mask), f(dout),
                                           reinterpret_cast<const void*>(k_all), reinterpret_cast<const void*>(v_all),
                                           f(dk_part), f(dv_part), f(dk_own), f(dv_own), f(dt_sums), f(ds), f(dz1),
                                           f(dz2), f(drot), f(dtrans), f(dweights), reinterpret_cast<void*>(ws),
                                           ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    size_t sharded_train_workspace_size(int64_t B, int64_t L, int world) const {
        return fipa_layer_sharded_train_workspace_size(layer_, B, L, world);
    }
    void forward_train_sharded_device(Comm& comm, int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2,
                                      uintptr_t rot, uintptr_t trans, uintptr_t mask, uintptr_t out, uintptr_t ws,
                                      size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<const float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_forward_train_sharded(layer_, comm.get(), B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                                  reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(out),
                                                  reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    void backward_sharded_device(Comm& comm, int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2,
                                 uintptr_t rot, uintptr_t trans, uintptr_t mask, uintptr_t dout, uintptr_t ds,
                                 uintptr_t dz1, uintptr_t dz2, uintptr_t drot, uintptr_t dtrans, uintptr_t dweights,
                                 uintptr_t ws, size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_backward_sharded(layer_, comm.get(), B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                             reinterpret_cast<const uint8_t*>(mask), f(dout), f(ds), f(dz1), f(dz2),
                                             f(drot), f(dtrans), f(dweights), reinterpret_cast<void*>(ws), ws_bytes,
                                             reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    size_t train_workspace_size(int64_t B, int64_t L) const { return fipa_layer_train_workspace_size(layer_, B, L); }
    uint64_t num_weights() const { return fipa_layer_num_weights(layer_); }
    void forward_train_device(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                              uintptr_t trans, uintptr_t mask, uintptr_t out, uintptr_t ws, size_t ws_bytes,
                              uintptr_t stream) {
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_forward_train(layer_, B, L, reinterpret_cast<const float*>(s),
                                          reinterpret_cast<const float*>(z1), reinterpret_cast<const float*>(z2),
                                          reinterpret_cast<const float*>(rot), reinterpret_cast<const float*>(trans),
                                          reinterpret_cast<const uint8_t*>(mask), reinterpret_cast<float*>(out),
                                          reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    void backward_device(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot,
                         uintptr_t trans, uintptr_t mask, uintptr_t dout, uintptr_t ds, uintptr_t dz1,
                         uintptr_t dz2, uintptr_t drot, uintptr_t dtrans, uintptr_t dweights, uintptr_t ws,
                         size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_layer_backward(layer_, B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                     reinterpret_cast<const uint8_t*>(mask), f(dout), f(ds), f(dz1), f(dz2),
                                     f(drot), f(dtrans), f(dweights), reinterpret_cast<void*>(ws), ws_bytes,
                                     reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    py::tuple train_workspace_layout(int64_t B, int64_t L) const {
        int64_t off[FIPA_TRAIN_LAYOUT_SLOTS], dims[3];
        if (fipa_layer_train_workspace_layout(layer_, B, L, off, dims) != FIPA_TRAIN_LAYOUT_SLOTS)
            throw FipaValueError("invalid batch shape");
        return py::make_tuple(std::vector<int64_t>(off, off + FIPA_TRAIN_LAYOUT_SLOTS),
                              std::vector<int64_t>(dims, dims + 3));
    }
    // flash_grad(s, z1, z2, rotations, translations, dout, mask=None) -> (out, grads)
    // Forward + backward of sum(out * dout) through the host-buffer C ABI; grads is a dict with
    // s, z1, z2, rotations, translations and every weight tensor (reference names).
    py::tuple flash_grad(const py::object& s, const py::object& z1, const py::object& z2,
                         const py::object& rotations, const py::object& translations, const py::object& dout,
                         const py::object& mask) {
        if (all_f32({s, z1, z2, rotations, translations, dout}))
            return grad_host<float>(FArr(s), FArr(z1), FArr(z2), FArr(rotations), FArr(translations), FArr(dout), mask);
        return grad_host<double>(DArr(s), DArr(z1), DArr(z2), DArr(rotations), DArr(translations), DArr(dout), mask);
    }
    template <class T>
    py::tuple grad_host(const py::array_t<T, py::array::c_style | py::array::forcecast>& s,
                        const py::array_t<T, py::array::c_style | py::array::forcecast>& z1,
                        const py::array_t<T, py::array::c_style | py::array::forcecast>& z2,
                        const py::array_t<T, py::array::c_style | py::array::forcecast>& rotations,
                        const py::array_t<T, py::array::c_style | py::array::forcecast>& translations,
                        const py::array_t<T, py::array::c_style | py::array::forcecast>& dout, const py::object& mask) {
        using Arr = py::array_t<T, py::array::c_style | py::array::forcecast>;
        const bool batched = s.ndim() == 3;
        if (s.ndim() != 2 && s.ndim() != 3)
            throw FipaValueError("single representation must be [L, d_in] or [B, L, d_in]");
        const int64_t B = batched ? s.shape(0) : 1;
        const int64_t L = batched ? s.shape(1) : s.shape(0);
        if (dout.size() != s.size()) throw FipaValueError("dout must have the output's shape");
        if (z1.size() != B * L * int64_t(cfg_.rank * cfg_.d_z) || z2.size() != z1.size() ||
            rotations.size() != B * L * 9 || translations.size() != B * L * 3 ||
            s.size() != B * L * int64_t(cfg_.d_in))
            throw FipaValueError("input shapes disagree with the configuration");
        std::vector<uint8_t> m;
        const uint8_t* mp = nullptr;
        if (!mask.is_none()) {
            py::array_t<uint8_t, py::array::c_style | py::array::forcecast> ma(mask);
            if (ma.size() != B * L) throw FipaValueError("mask length must equal L");
            m.assign(ma.data(), ma.data() + ma.size());
            for (auto& v : m) v = v ? 1 : 0;
            mp = m.data();
        }
        auto like = [](const Arr& a) { return host_out<T>(std::vector<py::ssize_t>(a.shape(), a.shape() + a.ndim())); };
        py::array_t<T> out = like(s), gs = like(s), gz1 = like(z1), gz2 = like(z2), gr = like(rotations),
                       gt = like(translations);
        const uint64_t nw = fipa_layer_num_weights(layer_);
        py::array_t<T> gw(static_cast<py::ssize_t>(nw));  // weight grads land here directly
        T* gwp = gw.mutable_data();
        int rc;
        {
            py::gil_scoped_release nogil;
            if constexpr (std::is_same_v<T, float>) {
                rc = fipa_layer_grad_host_f32(layer_, B, L, s.data(), z1.data(), z2.data(), rotations.data(),
                                              translations.data(), mp, dout.data(), out.mutable_data(),
                                              gs.mutable_data(), gz1.mutable_data(), gz2.mutable_data(),
                                              gr.mutable_data(), gt.mutable_data(), gwp);
            } else {
                rc = fipa_layer_grad_host(layer_, B, L, s.data(), z1.data(), z2.data(), rotations.data(),
                                          translations.data(), mp, dout.data(), out.mutable_data(), gs.mutable_data(),
                                          gz1.mutable_data(), gz2.mutable_data(), gr.mutable_data(), gt.mutable_data(),
                                          gwp);
            }
        }
        check(rc);
        py::dict g;
        g["s"] = gs;
        g["z1"] = gz1;
        g["z2"] = gz2;
        g["rotations"] = gr;
        g["translations"] = gt;
        const auto sh = shapes();
        py::ssize_t o = 0;
        for (int i = 0; i < 10; ++i) {
            py::ssize_t n = 1;
            for (auto v : sh[i]) n *= static_cast<py::ssize_t>(v);
            py::object view = gw[py::slice(o, o + n, 1)];
            g[kNames[i]] = view.attr("reshape")(py::cast(std::vector<py::ssize_t>(sh[i].begin(), sh[i].end())));
            o += n;
        }
        return py::make_tuple(out, g);
    }
    void set_timing(bool on) { check(fipa_layer_set_timing(layer_, on ? 1 : 0)); }
    py::dict tuning() const {
        fipa_tuning t{};
        check(fipa_layer_get_tuning(layer_, &t));
        static const char* attn[4] = {"auto", "pair", "pass", "1sm"};
        py::dict d;
        d["attn_impl"] = attn[t.attn_impl];
        d["fused_pack"] = t.fused_pack != 0;
        d["bwd_ds"] = t.bwd_ds;
        std::vector<int> ring(t.bwd_ring, t.bwd_ring + 4);
        ring.push_back(t.bwd_slice);
        d["bwd_ring"] = ring;
        d["pass_ring"] = std::vector<int>(t.pass_ring, t.pass_ring + 4);
        d["f32_tc"] = t.f32_tc != 0;
        d["graphs"] = t.graphs != 0;
        d["micro"] = t.micro;
        d["shard_chunks"] = t.shard_chunks;
        d["ds_cap_mb"] = t.ds_cap_mb;
        return d;
    }
    // Keyword-wise update of the layer's tuning knobs (fipa_layer_set_tuning); None keeps a value.
    void set_tuning(py::object attn_impl, py::object fused_pack, py::object bwd_ds, py::object bwd_ring,
                    py::object pass_ring, py::object f32_tc, py::object graphs, py::object micro,
                    py::object shard_chunks, py::object ds_cap_mb) {
        fipa_tuning t{};
        check(fipa_layer_get_tuning(layer_, &t));
        if (!attn_impl.is_none()) {
            const std::string v = attn_impl.cast<std::string>();
            if (v == "auto") t.attn_impl = 0;
            else if (v == "pair") t.attn_impl = 1;
            else if (v == "pass") t.attn_impl = 2;
            else if (v == "1sm") t.attn_impl = 3;
            else throw py::value_error("attn_impl must be 'auto', 'pair', 'pass' or '1sm'");
        }
        if (!fused_pack.is_none()) t.fused_pack = fused_pack.cast<bool>() ? 1 : 0;
        if (!bwd_ds.is_none()) t.bwd_ds = bwd_ds.cast<int>();
        if (!f32_tc.is_none()) t.f32_tc = f32_tc.cast<bool>() ? 1 : 0;
        if (!graphs.is_none()) t.graphs = graphs.cast<bool>() ? 1 : 0;
        if (!micro.is_none()) t.micro = micro.cast<int>();
        if (!shard_chunks.is_none()) t.shard_chunks = shard_chunks.cast<int>();
        if (!ds_cap_mb.is_none()) t.ds_cap_mb = ds_cap_mb.cast<int>();
        auto ring = [](py::object o, int32_t* dst, int32_t* extra) {
            if (o.is_none()) return;
            const auto v = o.cast<std::vector<int>>();
            if (v.size() != 4 && !(extra && v.size() == 5)) throw py::value_error("ring plans have 4 entries (5 with the slice)");
            for (int i = 0; i < 4; ++i) dst[i] = v[i];
            if (extra) *extra = v.size() == 5 ? v[4] : 0;
        };
        ring(bwd_ring, t.bwd_ring, &t.bwd_slice);
        ring(pass_ring, t.pass_ring, nullptr);
        check(fipa_layer_set_tuning(layer_, &t));
    }
    std::vector<float> stage_times() const {
        std::vector<float> t(16);
        t.resize(fipa_layer_stage_times(layer_, t.data(), 16));
        return t;
    }
    std::vector<float> bwd_stage_times() const {
        std::vector<float> t(16);
        t.resize(fipa_layer_bwd_stage_times(layer_, t.data(), 16));
        return t;
    }
    std::string precision() const { return precision_name_; }
    py::dict config() const {
        py::dict d;
        d["d_in"] = cfg_.d_in;
        d["d_z"] = cfg_.d_z;
        d["heads"] = cfg_.heads;
        d["c"] = cfg_.c;
        d["n_query"] = cfg_.n_query;
        d["n_value"] = cfg_.n_value;
        d["rank"] = cfg_.rank;
        d["precision"] = precision_name_;
        d["enforce_head_cap"] = bool(cfg_.enforce_head_cap);
        return d;
    }

private:
    fipa_config cfg_{};
    fipa_layer* layer_ = nullptr;
    std::string precision_name_;
};

}  // namespace

// BASELINE cfg3 trunk: n_layers layers + residual + backbone frame update (fipa_trunk_* C ABI).
class Trunk {
public:
    Trunk(uint64_t d_in, uint64_t d_z, uint64_t heads, uint64_t c, uint64_t n_query, uint64_t n_value, uint64_t rank,
          const std::string& precision, uint64_t seed, bool enforce_head_cap, int n_layers)
        : precision_name_(precision) {
        cfg_.d_in = d_in;
        cfg_.d_z = d_z;
        cfg_.heads = heads;
        cfg_.c = c;
        cfg_.n_query = n_query;
        cfg_.n_value = n_value;
        cfg_.rank = rank;
        cfg_.precision = parse_precision(precision);
        cfg_.enforce_head_cap = enforce_head_cap ? 1 : 0;
        check(fipa_config_validate(&cfg_));
        check(fipa_trunk_create(&cfg_, n_layers, seed, &trunk_));
    }
    ~Trunk() { fipa_trunk_destroy(trunk_); }
    Trunk(const Trunk&) = delete;
    Trunk& operator=(const Trunk&) = delete;
    int n_layers() const { return fipa_trunk_num_layers(trunk_); }
    Model* layer(int l) {
        fipa_layer* v = fipa_trunk_layer(trunk_, l);
        if (v == nullptr) throw FipaValueError("layer index out of range");
        return new Model(v, cfg_, precision_name_);
    }
    py::tuple backbone(int l) const {
        py::array_t<double> w(std::vector<py::ssize_t>{(py::ssize_t)cfg_.d_in, 6}), b(6);
        check(fipa_trunk_get_backbone(trunk_, l, w.mutable_data(), b.mutable_data()));
        return py::make_tuple(w, b);
    }
    void set_backbone(int l, const DArr& w, const DArr& b) {
        if (w.size() != int64_t(cfg_.d_in * 6) || b.size() != 6) throw FipaValueError("backbone must be [d_in, 6] and [6]");
        check(fipa_trunk_set_backbone(trunk_, l, w.data(), b.data()));
    }
    size_t workspace_size(int64_t B, int64_t L) const { return fipa_trunk_workspace_size(trunk_, B, L); }
    void forward_device(int64_t B, int64_t L, uintptr_t s, uintptr_t z1, uintptr_t z2, uintptr_t rot, uintptr_t trans,
                        uintptr_t mask, uintptr_t s_out, uintptr_t rot_out, uintptr_t trans_out, uintptr_t ws,
                        size_t ws_bytes, uintptr_t stream) {
        auto f = [](uintptr_t p) { return reinterpret_cast<float*>(p); };
        int rc;
        {
            py::gil_scoped_release nogil;
            rc = fipa_trunk_forward(trunk_, B, L, f(s), f(z1), f(z2), f(rot), f(trans),
                                    reinterpret_cast<const uint8_t*>(mask), f(s_out), f(rot_out), f(trans_out),
                                    reinterpret_cast<void*>(ws), ws_bytes, reinterpret_cast<void*>(stream));
        }
        check(rc);
    }
    int forward_launches() const { return fipa_trunk_forward_launches(trunk_); }
    int step_launches(int64_t B, int64_t L) const { return fipa_trunk_step_launches(trunk_, B, L); }

private:
    fipa_config cfg_{};
    fipa_trunk* trunk_ = nullptr;
    std::string precision_name_;
};

// fully_masked(mask [L] or [B, L]) -> bool array of the same shape: the reference's
// flash_ipa_forward `fully_masked` output (proj/src/flash_ipa.cpp:156-158), on the GPU.
py::array_t<bool> fully_masked(const py::object& mask_obj) {
    py::array_t<uint8_t, py::array::c_style | py::array::forcecast> mask(mask_obj);
    if (mask.ndim() != 1 && mask.ndim() != 2) throw FipaValueError("mask must be [L] or [B, L]");
    const int64_t B = mask.ndim() == 2 ? mask.shape(0) : 1;
    const int64_t L = mask.shape(mask.ndim() - 1);
    std::vector<uint8_t> flags(size_t(B) * size_t(L));
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = fipa_fully_masked_host(B, L, mask.data(), flags.data());
    }
    check(rc);
    py::array_t<bool> out(std::vector<py::ssize_t>(mask.shape(), mask.shape() + mask.ndim()));
    bool* o = out.mutable_data();
    for (size_t e = 0; e < flags.size(); ++e) o[e] = flags[e] != 0;
    return out;
}

// knn_distogram(translations, k=20, n_bins=22, d_min=2.0, d_max=22.0, pe_dim=16) -> [.., L, k, n_bins+pe_dim]
py::array_t<double> knn_distogram(const DArr& trans, uint64_t k, uint64_t n_bins, double d_min, double d_max,
                                  uint64_t pe_dim) {
    if ((trans.ndim() != 2 && trans.ndim() != 3) || trans.shape(trans.ndim() - 1) != 3)
        throw FipaValueError("knn_distogram expects [L, 3] translations");
    const bool batched = trans.ndim() == 3;
    const int64_t B = batched ? trans.shape(0) : 1, L = trans.shape(batched ? 1 : 0);
    std::vector<py::ssize_t> shape = {(py::ssize_t)L, (py::ssize_t)k, (py::ssize_t)(n_bins + pe_dim)};
    if (batched) shape.insert(shape.begin(), (py::ssize_t)B);
    py::array_t<double> out(shape);
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = fipa_knn_distogram_host(B, L, trans.data(), k, n_bins, d_min, d_max, pe_dim, out.mutable_data());
    }
    check(rc);
    return out;
}

// build_factors(features [rows, f], r, d_z, w1 [f, r*d_z], w2, precision="bf16") -> (z1, z2) [rows, r, d_z]
py::tuple build_factors(const DArr& features, uint64_t r, uint64_t d_z, const DArr& w1, const DArr& w2,
                        const std::string& precision) {
    if (features.ndim() != 2) throw FipaValueError("build_factors expects [L, f] features");
    const int64_t rows = features.shape(0);
    const uint64_t f = features.shape(1);
    for (const DArr* w : {&w1, &w2})
        if (w->ndim() != 2 || uint64_t(w->shape(0)) != f || uint64_t(w->shape(1)) != r * d_z)
            throw FipaValueError("factor projection weights must be [f, r*d_z]");
    const int prec = parse_precision(precision);
    py::array_t<double> z1({(py::ssize_t)rows, (py::ssize_t)r, (py::ssize_t)d_z}), z2({(py::ssize_t)rows, (py::ssize_t)r, (py::ssize_t)d_z});
    int rc;
    {
        py::gil_scoped_release nogil;
        rc = fipa_build_factors_host(rows, f, features.data(), r, d_z, w1.data(), w2.data(), z1.mutable_data(),
                                     z2.mutable_data(), prec);
    }
    check(rc);
    return py::make_tuple(z1, z2);
}

PYBIND11_MODULE(_fipa_b200, m) {
    m.doc() = "B200-native FlashIPA layer (tcgen05 sm_100a kernels behind the reference fipa.Model API)";

    py::register_exception<FipaValueError>(m, "FipaValueError", PyExc_ValueError);
    py::register_exception<FipaNumericError>(m, "FipaNumericError", PyExc_ArithmeticError);
    py::register_exception<FipaIoError>(m, "FipaIoError", PyExc_IOError);
    py::register_exception<FipaCudaError>(m, "FipaCudaError", PyExc_RuntimeError);
    py::register_exception<FipaCommError>(m, "FipaCommError", PyExc_RuntimeError);
    m.def("fully_masked", &fully_masked, py::arg("mask"),
          "Per-row flags of the reference flash_ipa_forward `fully_masked` output (rows of a sample with no valid "
          "residue), on the GPU");
    m.def("knn_distogram", &knn_distogram, py::arg("translations"), py::arg("k") = 20, py::arg("n_bins") = 22,
          py::arg("d_min") = 2.0, py::arg("d_max") = 22.0, py::arg("pe_dim") = 16,
          "k-NN distogram + offset encoding of each residue (reference knn_distogram), on the GPU");
    m.def("build_factors", &build_factors, py::arg("features"), py::arg("r"), py::arg("d_z"), py::arg("w1"),
          py::arg("w2"), py::arg("precision") = "bf16", "z1, z2 = features.w1, features.w2 on the GPU");
    m.def(
        "flash_attention",
        [](const DArr& q, const DArr& k, const DArr& v, const py::object& mask, size_t tile_rows, size_t tile_cols,
           int threads) {
            if (tile_rows == 0 || tile_cols == 0) throw FipaValueError("tile sizes must be positive");
            (void)threads;
            return py_attention(q, k, v, mask, false);
        },
        py::arg("q"), py::arg("k"), py::arg("v"), py::arg("mask") = py::none(), py::arg("tile_rows") = 64,
        py::arg("tile_cols") = 64, py::arg("threads") = 1,
        "Online-softmax attention on the GPU, O(L) memory (callers pre-scale their logits)");
    m.def(
        "naive_attention",
        [](const DArr& q, const DArr& k, const DArr& v, const py::object& mask) {
            return py_attention(q, k, v, mask, true);
        },
        py::arg("q"), py::arg("k"), py::arg("v"), py::arg("mask") = py::none(),
        "Dense softmax attention on the GPU (materialises the [H, L, L] logits)");
    m.def("comm_unique_id", &comm_unique_id, "128-byte NCCL unique id (rank 0 creates, all ranks share)");
    py::class_<Comm>(m, "Comm", "NCCL communicator for query-row sharding (one process per GPU)")
        .def(py::init<int, int, const py::bytes&, int>(), py::arg("world"), py::arg("rank"), py::arg("unique_id"),
             py::arg("device"))
        .def("all_reduce_sum_f32", &Comm::all_reduce_sum_f32, py::arg("buf"), py::arg("n"), py::arg("stream") = 0,
             "In-place sum of a device float buffer (pointer) over the ranks, on `stream`")
        .def_property_readonly("world", &Comm::world)
        .def_property_readonly("rank", &Comm::rank);

    py::class_<Model>(m, "Model", "One FlashIPA layer: hyper-parameters plus deterministic weights")
        .def(py::init<uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t,
                      const std::string&, uint64_t, bool>(),
             py::arg("d_in") = 32, py::arg("d_z") = 4, py::arg("heads") = 2, py::arg("c") = 8,
             py::arg("n_query") = 2, py::arg("n_value") = 2, py::arg("rank") = 2,
             py::arg("precision") = "f64", py::arg("seed") = 0, py::arg("enforce_head_cap") = true)
        .def("flash", &Model::flash, py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rotations"),
             py::arg("translations"), py::arg("mask") = py::none(), py::arg("tile_rows") = 64,
             py::arg("tile_cols") = 64, py::arg("threads") = 1,
             "Linear-memory FlashIPA forward on the GPU")
        .def("reference", &Model::reference, py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rotations"),
             py::arg("translations"), py::arg("mask") = py::none(),
             "Quadratic-memory forward pass (dense pair tensor, fp32 on the GPU)")
        .def("reference_workspace_size", &Model::reference_workspace_size, py::arg("B"), py::arg("L"))
        .def("reference_device", &Model::reference_device, py::arg("B"), py::arg("L"), py::arg("s"), py::arg("z1"),
             py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"), py::arg("out"), py::arg("workspace"),
             py::arg("workspace_bytes"), py::arg("stream") = 0)
        .def("save", &Model::save, py::arg("path"), "Write weights to a binary file")
        .def("load", &Model::load, py::arg("path"), "Replace weights from a binary file")
        .def("weights", &Model::weights, "Master weights as a dict of float64 arrays")
        .def("set_weights", &Model::set_weights, py::arg("weights"))
        .def("workspace_size", &Model::workspace_size, py::arg("B"), py::arg("L"))
        .def("forward_device", &Model::forward_device, py::arg("B"), py::arg("L"), py::arg("s"),
             py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("workspace_layout", &Model::workspace_layout, py::arg("B"), py::arg("L"))
        .def("forward_launches", &Model::forward_launches)
        .def("step_launches", &Model::step_launches, py::arg("B"), py::arg("L"), py::arg("train"))
        .def("backward_launches", &Model::backward_launches)
        .def("sharded_workspace_size", &Model::sharded_workspace_size, py::arg("B"), py::arg("L"), py::arg("world"))
        .def("forward_sharded_device", &Model::forward_sharded_device, py::arg("comm"), py::arg("B"), py::arg("L"),
             py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("shard_centroid_sums", &Model::shard_centroid_sums, py::arg("B"), py::arg("L"), py::arg("trans"),
             py::arg("mask"), py::arg("sums"), py::arg("stream"))
        .def("shard_pack", &Model::shard_pack, py::arg("B"), py::arg("L"), py::arg("s"), py::arg("z1"),
             py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"), py::arg("sums"), py::arg("workspace"),
             py::arg("workspace_bytes"), py::arg("stream"), py::arg("train") = false)
        .def("shard_attend", &Model::shard_attend, py::arg("B"), py::arg("L"), py::arg("world"), py::arg("s"),
             py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"), py::arg("k_all"),
             py::arg("v_all"), py::arg("out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"),
             py::arg("train") = false)
        .def("shard_backward", &Model::shard_backward, py::arg("stage"), py::arg("world"), py::arg("B"), py::arg("L"),
             py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("dout"), py::arg("k_all"), py::arg("v_all"), py::arg("dk_part"), py::arg("dv_part"),
             py::arg("dk_own"), py::arg("dv_own"), py::arg("dt_sums"), py::arg("ds"), py::arg("dz1"), py::arg("dz2"),
             py::arg("drot"), py::arg("dtrans"), py::arg("dweights"), py::arg("workspace"),
             py::arg("workspace_bytes"), py::arg("stream"))
        .def("sharded_train_workspace_size", &Model::sharded_train_workspace_size, py::arg("B"), py::arg("L"),
             py::arg("world"))
        .def("forward_train_sharded_device", &Model::forward_train_sharded_device, py::arg("comm"), py::arg("B"),
             py::arg("L"), py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("backward_sharded_device", &Model::backward_sharded_device, py::arg("comm"), py::arg("B"), py::arg("L"),
             py::arg("s"), py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("dout"), py::arg("ds"), py::arg("dz1"), py::arg("dz2"), py::arg("drot"), py::arg("dtrans"),
             py::arg("dweights"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("train_workspace_size", &Model::train_workspace_size, py::arg("B"), py::arg("L"))
        .def("num_weights", &Model::num_weights)
        .def("forward_train_device", &Model::forward_train_device, py::arg("B"), py::arg("L"), py::arg("s"),
             py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"),
             py::arg("out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("backward_device", &Model::backward_device, py::arg("B"), py::arg("L"), py::arg("s"),
             py::arg("z1"), py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"), py::arg("dout"),
             py::arg("ds"), py::arg("dz1"), py::arg("dz2"), py::arg("drot"), py::arg("dtrans"),
             py::arg("dweights"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("train_workspace_layout", &Model::train_workspace_layout, py::arg("B"), py::arg("L"))
        .def("flash_grad", &Model::flash_grad, py::arg("s"), py::arg("z1"), py::arg("z2"),
             py::arg("rotations"), py::arg("translations"), py::arg("dout"), py::arg("mask") = py::none(),
             "Forward + backward (gradient of sum(out * dout)) on the GPU")
        .def("set_timing", &Model::set_timing, py::arg("enable"))
        .def("tuning", &Model::tuning)
        .def("set_tuning", &Model::set_tuning, py::arg("attn_impl") = py::none(), py::arg("fused_pack") = py::none(),
             py::arg("bwd_ds") = py::none(), py::arg("bwd_ring") = py::none(), py::arg("pass_ring") = py::none(),
             py::arg("f32_tc") = py::none(), py::arg("graphs") = py::none(), py::arg("micro") = py::none(),
             py::arg("shard_chunks") = py::none(), py::arg("ds_cap_mb") = py::none())
        .def("stage_times", &Model::stage_times)
        .def("bwd_stage_times", &Model::bwd_stage_times)
        .def_property_readonly("precision", &Model::precision)
        .def_property_readonly("config", &Model::config);
    py::class_<Trunk>(m, "Trunk", "FlashIPA trunk: layers + residual + per-layer backbone frame update (cfg3)")
        .def(py::init<uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, const std::string&, uint64_t,
                      bool, int>(),
             py::arg("d_in") = 32, py::arg("d_z") = 4, py::arg("heads") = 2, py::arg("c") = 8, py::arg("n_query") = 2,
             py::arg("n_value") = 2, py::arg("rank") = 2, py::arg("precision") = "bf16", py::arg("seed") = 0,
             py::arg("enforce_head_cap") = true, py::arg("n_layers") = 6)
        .def_property_readonly("n_layers", &Trunk::n_layers)
        .def("layer", &Trunk::layer, py::arg("index"), py::keep_alive<0, 1>(), py::return_value_policy::take_ownership)
        .def("backbone", &Trunk::backbone, py::arg("index"))
        .def("set_backbone", &Trunk::set_backbone, py::arg("index"), py::arg("w"), py::arg("b"))
        .def("workspace_size", &Trunk::workspace_size, py::arg("B"), py::arg("L"))
        .def("forward_device", &Trunk::forward_device, py::arg("B"), py::arg("L"), py::arg("s"), py::arg("z1"),
             py::arg("z2"), py::arg("rot"), py::arg("trans"), py::arg("mask"), py::arg("s_out"), py::arg("rot_out"),
             py::arg("trans_out"), py::arg("workspace"), py::arg("workspace_bytes"), py::arg("stream"))
        .def("forward_launches", &Trunk::forward_launches)
        .def("step_launches", &Trunk::step_launches, py::arg("B"), py::arg("L"));
}
