// Host-buffer entry points of the layer (the reference calling convention: float64 arrays in,
// float64 arrays out -- proj/python/bindings.cpp:26-45, 122-135), pipelined over the batch.
//
// The batch is cut into chunks of whole samples.  Two pinned staging slots and two device slots
// rotate so that, while the GPU runs chunk k, the host converts chunk k+1's inputs (float64 ->
// float32, fork-join over the host cores) and chunk k-1's outputs (float32 -> float64), and the
// copy engines move chunk k+1 in (H2D stream) and chunk k out (D2H stream):
//
//   host   : cvt_in(k+1) ........ cvt_out(k-1)
//   H2D    :        [copy k+1]
//   compute:  [ forward / forward+backward k ]
//   D2H    :                               [copy k]
//
// Weight gradients (grad_host) are summed over the chunks on the device.  float32 host arrays
// are accepted as well (no conversion: a parallel copy into the pinned slot).  One pipeline per
// layer, serialised by host_mu_ (the entry points release the GIL).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "layer.hpp"

namespace fipa_b200 {

namespace {

// Fork-join pool over the host cores for the conversions (persistent workers: spawning threads
// per call cost tens of microseconds per tensor).
class Pool {
public:
    static Pool& get() {
        static Pool pool;
        return pool;
    }
    // f(begin, end) over [0, n) split into size() contiguous parts; the caller runs part 0.
    void run(std::size_t n, const std::function<void(std::size_t, std::size_t)>& f) {
        const std::size_t parts = n < (std::size_t(1) << 15) ? 1 : std::min<std::size_t>(size(), n >> 14);
        if (parts <= 1) {
            f(0, n);
            return;
        }
        std::lock_guard<std::mutex> one_job(run_mu_);  // layers on other threads share the pool
        std::unique_lock<std::mutex> lk(mu_);
        job_ = &f;
        n_ = n;
        parts_ = parts;
        pending_ = parts - 1;
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        f(0, n / parts);
        lk.lock();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }
    std::size_t size() const { return workers_.size() + 1; }

private:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(16u, hw) - 1;
        for (unsigned t = 0; t < n; ++t) workers_.emplace_back([this, t] { loop(t + 1); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    void loop(std::size_t id) {
        std::uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            if (id >= parts_) continue;
            const auto* f = job_;
            const std::size_t a = n_ * id / parts_, b = n_ * (id + 1) / parts_;
            lk.unlock();
            (*f)(a, b);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(std::size_t, std::size_t)>* job_ = nullptr;
    std::size_t n_ = 0, parts_ = 0, pending_ = 0;
    std::uint64_t gen_ = 0;
    bool stop_ = false;
};

template <class D, class S>
void convert(D* dst, const S* src, std::size_t n) {
    Pool::get().run(n, [dst, src](std::size_t a, std::size_t b) {
        if constexpr (std::is_same_v<D, S>) {
            std::memcpy(dst + a, src + a, (b - a) * sizeof(D));
        } else {
            for (std::size_t i = a; i < b; ++i) dst[i] = static_cast<D>(src[i]);
        }
    });
}

std::size_t up256(std::size_t x) { return (x + 255) / 256 * 256; }

__attribute__((unused)) void check(cudaError_t e, const char* what) { cuda_check(e, what); }

}  // namespace

struct FlashIpaLayer::HostPipe {
    cudaStream_t comp = nullptr, h2d = nullptr, d2h = nullptr;
    cudaEvent_t h2d_done[2] = {}, comp_done[2] = {}, d2h_done[2] = {};
    void* pin[2] = {};
    void* dev[2] = {};
    std::size_t slot_bytes = 0;
    void* ws = nullptr;
    std::size_t ws_bytes = 0;
    float* dw = nullptr;  // per-chunk weight gradients | their sum
    std::size_t dw_n = 0;
    int device = 0;

    ~HostPipe() {
        cudaSetDevice(device);
        for (int k = 0; k < 2; ++k) {
            if (pin[k]) cudaFreeHost(pin[k]);
            if (dev[k]) cudaFree(dev[k]);
            for (cudaEvent_t e : {h2d_done[k], comp_done[k], d2h_done[k]})
                if (e) cudaEventDestroy(e);
        }
        if (ws) cudaFree(ws);
        if (dw) cudaFree(dw);
        for (cudaStream_t s : {comp, h2d, d2h})
            if (s) cudaStreamDestroy(s);
    }
    void init(int dev_id) {
        if (comp) return;
        device = dev_id;
        check(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking), "stream");
        check(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "stream");
        check(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "stream");
        for (int k = 0; k < 2; ++k)
            for (cudaEvent_t* e : {&h2d_done[k], &comp_done[k], &d2h_done[k]})
                check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
    void reserve(std::size_t slot, std::size_t wsb, std::size_t dwn) {
        if (slot > slot_bytes) {
            for (int k = 0; k < 2; ++k) {
                if (pin[k]) cudaFreeHost(pin[k]);
                if (dev[k]) cudaFree(dev[k]);
                pin[k] = dev[k] = nullptr;
            }
            slot_bytes = 0;
            for (int k = 0; k < 2; ++k) {
                check(cudaMallocHost(&pin[k], slot), "cudaMallocHost");
                check(cudaMalloc(&dev[k], slot), "cudaMalloc");
            }
            slot_bytes = slot;
        }
        if (wsb > ws_bytes) {
            if (ws) cudaFree(ws);
            ws = nullptr;
            ws_bytes = 0;
            check(cudaMalloc(&ws, wsb), "cudaMalloc");
            ws_bytes = wsb;
        }
        if (dwn > dw_n) {
            if (dw) cudaFree(dw);
            dw = nullptr;
            dw_n = 0;
            check(cudaMalloc(reinterpret_cast<void**>(&dw), 2 * dwn * sizeof(float)), "cudaMalloc");
            dw_n = dwn;
        }
    }
};

FlashIpaLayer::HostPipe& FlashIpaLayer::host_pipe() {
    if (pipe_ == nullptr) pipe_ = new HostPipe();
    pipe_->init(device_);
    return *pipe_;
}

void FlashIpaLayer::release_host_pipe() {
    delete pipe_;
    pipe_ = nullptr;
}

namespace {
// Samples per chunk: at least ~2k residues per chunk (smaller batches leave the GPU idle) and,
// when B allows, four or more chunks so the conversions and copies overlap the kernels.
std::int64_t chunk_samples(std::int64_t B, std::int64_t L, int forced) {
    if (forced > 0) return std::min<std::int64_t>(B, forced);
    const std::int64_t by_size = std::max<std::int64_t>(1, (2048 + L - 1) / L);
    const std::int64_t by_count = std::max<std::int64_t>(1, B / 4);
    return std::min(B, std::max<std::int64_t>(1, std::min(by_size, by_count)));
}
}  // namespace

template <class T, class O>
void FlashIpaLayer::host_forward(std::int64_t B, std::int64_t L, const T* s, const T* z1, const T* z2, const T* rot,
                                 const T* trans, const std::uint8_t* mask, O* out, bool dense) {
    if (B < 1) throw ValueError("batch must be >= 1");
    if (L < 1) throw ValueError("empty frame set");
    std::lock_guard<std::mutex> host_lock(host_mu_);  // one pipeline per layer
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    HostPipe& hp = host_pipe();
    const std::size_t din = cfg_.d_in, rdz = cfg_.rank * cfg_.d_z;
    const std::int64_t nb = chunk_samples(B, L, tuning_.host_chunk);
    const std::size_t R = std::size_t(nb) * L;  // residues per chunk (max)
    // slot layout (floats): s | z1 | z2 | rot | trans | out | mask bytes
    const std::size_t o_s = 0, o_z1 = R * din, o_z2 = o_z1 + R * rdz, o_r = o_z2 + R * rdz, o_t = o_r + R * 9,
                      o_out = o_t + R * 3, n_f = o_out + R * din;
    const std::size_t slot = up256(n_f * 4 + R);
    const std::size_t wsb = dense ? reference_workspace_size(nb, L) : workspace_size(nb, L);
    hp.reserve(slot, wsb, 0);
    const std::int64_t nchunks = (B + nb - 1) / nb;
    auto rows = [&](std::int64_t k) { return std::min(nb, B - k * nb); };
    auto convert_out = [&](std::int64_t k) {
        const int sl = int(k & 1);
        check(cudaEventSynchronize(hp.d2h_done[sl]), "D2H");
        const std::size_t r = std::size_t(rows(k)) * L;
        convert(out + std::size_t(k * nb) * L * din, static_cast<const float*>(hp.pin[sl]) + o_out, r * din);
    };
    for (std::int64_t k = 0; k < nchunks; ++k) {
        const int sl = int(k & 1);
        const std::size_t r = std::size_t(rows(k)) * L, r0 = std::size_t(k * nb) * L;
        float* h = static_cast<float*>(hp.pin[sl]);
        float* d = static_cast<float*>(hp.dev[sl]);
        std::uint8_t* hm = reinterpret_cast<std::uint8_t*>(h + n_f);
        std::uint8_t* dm = reinterpret_cast<std::uint8_t*>(d + n_f);
        if (k >= 2) check(cudaEventSynchronize(hp.h2d_done[sl]), "H2D");  // the slot's last copy-in is done
        convert(h + o_s, s + r0 * din, r * din);
        convert(h + o_z1, z1 + r0 * rdz, r * rdz);
        convert(h + o_z2, z2 + r0 * rdz, r * rdz);
        convert(h + o_r, rot + r0 * 9, r * 9);
        convert(h + o_t, trans + r0 * 3, r * 3);
        if (mask) std::memcpy(hm, mask + r0, r);
        if (k >= 2) check(cudaStreamWaitEvent(hp.h2d, hp.comp_done[sl]), "wait");  // device slot consumed
        for (auto [off, n] : {std::pair{o_s, r * din}, std::pair{o_z1, r * rdz}, std::pair{o_z2, r * rdz},
                              std::pair{o_r, r * 9}, std::pair{o_t, r * 3}})
            check(cudaMemcpyAsync(d + off, h + off, n * 4, cudaMemcpyHostToDevice, hp.h2d), "H2D");
        if (mask) check(cudaMemcpyAsync(dm, hm, r, cudaMemcpyHostToDevice, hp.h2d), "H2D");
        check(cudaEventRecord(hp.h2d_done[sl], hp.h2d), "event");
        check(cudaStreamWaitEvent(hp.comp, hp.h2d_done[sl]), "wait");
        if (k >= 2) check(cudaStreamWaitEvent(hp.comp, hp.d2h_done[sl]), "wait");  // output slot read back
        const std::int64_t bk = rows(k);
        if (dense) {
            reference_forward(bk, L, d + o_s, d + o_z1, d + o_z2, d + o_r, d + o_t, mask ? dm : nullptr, d + o_out,
                              hp.ws, hp.ws_bytes, hp.comp);
        } else {
            forward(bk, L, d + o_s, d + o_z1, d + o_z2, d + o_r, d + o_t, mask ? dm : nullptr, d + o_out, hp.ws,
                    hp.ws_bytes, hp.comp);
        }
        check(cudaEventRecord(hp.comp_done[sl], hp.comp), "event");
        check(cudaStreamWaitEvent(hp.d2h, hp.comp_done[sl]), "wait");
        check(cudaMemcpyAsync(h + o_out, d + o_out, r * din * 4, cudaMemcpyDeviceToHost, hp.d2h), "D2H");
        check(cudaEventRecord(hp.d2h_done[sl], hp.d2h), "event");
        if (k >= 1) convert_out(k - 1);  // overlaps chunk k on the GPU
    }
    convert_out(nchunks - 1);
}

template <class T, class O>
void FlashIpaLayer::host_grad(std::int64_t B, std::int64_t L, const T* s, const T* z1, const T* z2, const T* rot,
                              const T* trans, const std::uint8_t* mask, const T* dout, O* out, O* ds, O* dz1, O* dz2,
                              O* drot, O* dtrans, O* dweights) {
    if (B < 1) throw ValueError("batch must be >= 1");
    if (L < 1) throw ValueError("empty frame set");
    std::lock_guard<std::mutex> host_lock(host_mu_);
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    HostPipe& hp = host_pipe();
    const std::size_t din = cfg_.d_in, rdz = cfg_.rank * cfg_.d_z, nw = num_weights();
    const std::int64_t nb = chunk_samples(B, L, tuning_.host_chunk);
    const std::size_t R = std::size_t(nb) * L;
    // slot (floats): inputs s | z1 | z2 | rot | trans | dout, outputs out | ds | dz1 | dz2 | drot | dtrans, mask
    const std::size_t sz_in[6] = {R * din, R * rdz, R * rdz, R * 9, R * 3, R * din};
    const std::size_t sz_out[6] = {R * din, R * din, R * rdz, R * rdz, R * 9, R * 3};
    std::size_t oin[6], oout[6], n_f = 0;
    for (int i = 0; i < 6; ++i) {
        oin[i] = n_f;
        n_f += sz_in[i];
    }
    for (int i = 0; i < 6; ++i) {
        oout[i] = n_f;
        n_f += sz_out[i];
    }
    const std::size_t slot = up256(n_f * 4 + R);
    hp.reserve(slot, train_workspace_size(nb, L), nw);
    float* dw_chunk = hp.dw;
    float* dw_sum = hp.dw + nw;
    check(cudaMemsetAsync(dw_sum, 0, nw * 4, hp.comp), "memset");
    const std::int64_t nchunks = (B + nb - 1) / nb;
    auto rows = [&](std::int64_t k) { return std::min(nb, B - k * nb); };
    const std::size_t per_res_in[6] = {din, rdz, rdz, 9, 3, din};
    const std::size_t per_res_out[6] = {din, din, rdz, rdz, 9, 3};
    O* dsts[6] = {out, ds, dz1, dz2, drot, dtrans};
    const T* srcs[6] = {s, z1, z2, rot, trans, dout};
    auto convert_out = [&](std::int64_t k) {
        const int sl = int(k & 1);
        check(cudaEventSynchronize(hp.d2h_done[sl]), "D2H");
        const std::size_t r = std::size_t(rows(k)) * L, r0 = std::size_t(k * nb) * L;
        const float* h = static_cast<const float*>(hp.pin[sl]);
        for (int i = 0; i < 6; ++i)
            if (dsts[i] != nullptr) convert(dsts[i] + r0 * per_res_out[i], h + oout[i], r * per_res_out[i]);
    };
    for (std::int64_t k = 0; k < nchunks; ++k) {
        const int sl = int(k & 1);
        const std::size_t r = std::size_t(rows(k)) * L, r0 = std::size_t(k * nb) * L;
        float* h = static_cast<float*>(hp.pin[sl]);
        float* d = static_cast<float*>(hp.dev[sl]);
        std::uint8_t* hm = reinterpret_cast<std::uint8_t*>(h + n_f);
        std::uint8_t* dm = reinterpret_cast<std::uint8_t*>(d + n_f);
        if (k >= 2) check(cudaEventSynchronize(hp.h2d_done[sl]), "H2D");
        for (int i = 0; i < 6; ++i) convert(h + oin[i], srcs[i] + r0 * per_res_in[i], r * per_res_in[i]);
        if (mask) std::memcpy(hm, mask + r0, r);
        if (k >= 2) check(cudaStreamWaitEvent(hp.h2d, hp.comp_done[sl]), "wait");
        for (int i = 0; i < 6; ++i)
            check(cudaMemcpyAsync(d + oin[i], h + oin[i], r * per_res_in[i] * 4, cudaMemcpyHostToDevice, hp.h2d),
                  "H2D");
        if (mask) check(cudaMemcpyAsync(dm, hm, r, cudaMemcpyHostToDevice, hp.h2d), "H2D");
        check(cudaEventRecord(hp.h2d_done[sl], hp.h2d), "event");
        check(cudaStreamWaitEvent(hp.comp, hp.h2d_done[sl]), "wait");
        if (k >= 2) check(cudaStreamWaitEvent(hp.comp, hp.d2h_done[sl]), "wait");
        const std::int64_t bk = rows(k);
        const std::uint8_t* mk = mask ? dm : nullptr;
        forward(bk, L, d + oin[0], d + oin[1], d + oin[2], d + oin[3], d + oin[4], mk, d + oout[0], hp.ws, hp.ws_bytes,
                hp.comp, true);
        backward(bk, L, d + oin[0], d + oin[1], d + oin[2], d + oin[3], d + oin[4], mk, d + oin[5], d + oout[1],
                 d + oout[2], d + oout[3], d + oout[4], d + oout[5], dw_chunk, hp.ws, hp.ws_bytes, hp.comp);
        launch_add_inplace(dw_sum, dw_chunk, static_cast<std::int64_t>(nw), hp.comp);  // weight grads sum over B
        check(cudaEventRecord(hp.comp_done[sl], hp.comp), "event");
        check(cudaStreamWaitEvent(hp.d2h, hp.comp_done[sl]), "wait");
        for (int i = 0; i < 6; ++i)
            if (dsts[i] != nullptr)
                check(cudaMemcpyAsync(h + oout[i], d + oout[i], r * per_res_out[i] * 4, cudaMemcpyDeviceToHost, hp.d2h),
                      "D2H");
        check(cudaEventRecord(hp.d2h_done[sl], hp.d2h), "event");
        if (k >= 1) convert_out(k - 1);
    }
    convert_out(nchunks - 1);
    if (dweights != nullptr) {
        std::vector<float> w(nw);
        check(cudaMemcpyAsync(w.data(), dw_sum, nw * 4, cudaMemcpyDeviceToHost, hp.comp), "D2H");
        check(cudaStreamSynchronize(hp.comp), "grad");
        for (std::size_t i = 0; i < nw; ++i) dweights[i] = static_cast<O>(w[i]);
    } else {
        check(cudaStreamSynchronize(hp.comp), "grad");
    }
}

void FlashIpaLayer::forward_host(std::int64_t B, std::int64_t L, const double* s, const double* z1, const double* z2,
                                 const double* rot, const double* trans, const std::uint8_t* mask, double* out) {
    host_forward(B, L, s, z1, z2, rot, trans, mask, out, false);
}

void FlashIpaLayer::forward_host_f32(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                                     const float* rot, const float* trans, const std::uint8_t* mask, float* out) {
    host_forward(B, L, s, z1, z2, rot, trans, mask, out, false);
}

void FlashIpaLayer::reference_host(std::int64_t B, std::int64_t L, const double* s, const double* z1,
                                   const double* z2, const double* rot, const double* trans,
                                   const std::uint8_t* mask, double* out) {
    host_forward(B, L, s, z1, z2, rot, trans, mask, out, true);
}

void FlashIpaLayer::grad_host(std::int64_t B, std::int64_t L, const double* s, const double* z1, const double* z2,
                              const double* rot, const double* trans, const std::uint8_t* mask, const double* dout,
                              double* out, double* ds, double* dz1, double* dz2, double* drot, double* dtrans,
                              double* dweights) {
    host_grad(B, L, s, z1, z2, rot, trans, mask, dout, out, ds, dz1, dz2, drot, dtrans, dweights);
}

void FlashIpaLayer::grad_host_f32(std::int64_t B, std::int64_t L, const float* s, const float* z1, const float* z2,
                                  const float* rot, const float* trans, const std::uint8_t* mask, const float* dout,
                                  float* out, float* ds, float* dz1, float* dz2, float* drot, float* dtrans,
                                  float* dweights) {
    host_grad(B, L, s, z1, z2, rot, trans, mask, dout, out, ds, dz1, dz2, drot, dtrans, dweights);
}

}  // namespace fipa_b200
