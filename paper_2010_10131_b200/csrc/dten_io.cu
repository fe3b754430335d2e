// dten_io.cu — the reference's .dten tensor file (tensor_io.hpp:15-99)
// streamed straight to / from device memory.
//
// Format (tensor_io.hpp:15-16): "DTEN", u32 LE version = 1, u32 LE order N,
// N x u64 LE dims, prod(dims) f64 LE payload in column-major order — the
// engine's own device layout, so a file maps 1:1 onto an atk_tensor.
//
// Read: the payload is pulled through two pinned host chunks; while the host
// reads chunk c+1 from the file, chunk c is in flight over PCIe, and for an
// fp32 tensor a kernel narrows the staged fp64 chunk into place on the device
// (the 8-byte payload never exists whole in host or device memory).  Write:
// the mirror image (widen on the device, D2H, fwrite while the next chunk
// copies).  Header validation and messages follow read_dten
// (tensor_io.hpp:62-91): bad magic, unsupported version, empty header, zero
// dimension, implausible product (> 2^40 elements), truncated payload -> the
// reference's IoFailure (ATK_IO_FAILURE).
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "atk_driver.cuh"

namespace atk {

namespace {

constexpr size_t kChunkElems = size_t(8) << 20;  // 8 Mi doubles = 64 MB per chunk

__global__ void narrow_f64(const double* __restrict__ s, float* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = float(s[i]);
}
__global__ void widen_f32(const float* __restrict__ s, double* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = double(s[i]);
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

struct Pinned {
    void* p = nullptr;
    explicit Pinned(size_t bytes) { ATK_CUDA(cudaMallocHost(&p, bytes)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct Event {
    cudaEvent_t e = nullptr;
    Event() { ATK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    ~Event() {
        if (e) cudaEventDestroy(e);
    }
};

[[noreturn]] void io_fail(const std::string& m) { fail(ATK_IO_FAILURE, m); }

}  // namespace

DtenHeader dten_header(const char* path, FILE** keep) {
    const std::string p = path ? path : "";
    FILE* f = std::fopen(p.c_str(), "rb");
    if (!f) io_fail("cannot open " + p);
    File guard{f};
    DtenHeader h;
    char magic[4] = {};
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "DTEN", 4) != 0)
        io_fail(p + ": not a .dten file (bad magic)");
    uint32_t version = 0, order = 0;
    if (std::fread(&version, 4, 1, f) != 1 || version != 1)
        io_fail(p + ": unsupported .dten version " + std::to_string(version));
    if (std::fread(&order, 4, 1, f) != 1 || order == 0) io_fail(p + ": truncated or empty header");
    if (order > ATK_MAX_ORDER) io_fail(p + ": order " + std::to_string(order) + " exceeds ATK_MAX_ORDER");
    h.order = int(order);
    if (std::fread(h.dims, 8, order, f) != order) io_fail(p + ": truncated dims block");
    uint64_t total = 1;
    for (uint32_t m = 0; m < order; ++m) {
        const uint64_t d = h.dims[m];
        if (d == 0) io_fail(p + ": zero dimension in header");
        if (d > (uint64_t(1) << 40) / total) io_fail(p + ": dims product is implausibly large");
        total *= d;
    }
    h.numel = total;
    if (keep) {
        *keep = f;
        guard.f = nullptr;
    }
    return h;
}

atk_tensor* dten_read(atk_ctx* ctx, const char* path, atk_dtype dt) {
    FILE* raw = nullptr;
    const DtenHeader h = dten_header(path, &raw);
    File file{raw};
    atk_tensor* t = new_tensor(ctx, dt, h.order, h.dims);
    try {
        const size_t chunk = std::min<size_t>(kChunkElems, h.numel);
        Pinned host(2 * chunk * sizeof(double));
        DevBuf<double> stage(ctx, dt == ATK_F32 ? 2 * chunk : 0);
        Event done[2];
        auto* hbuf = static_cast<double*>(host.p);
        size_t off = 0;
        for (int c = 0; off < h.numel; ++c) {
            const int b = c & 1;
            const size_t n = std::min(chunk, h.numel - off);
            ATK_CUDA(cudaEventSynchronize(done[b].e));  // the copy that last used buffer b has landed
            const size_t got = std::fread(hbuf + b * chunk, sizeof(double), n, file.f);
            if (got != n)
                io_fail(std::string(path) + ": truncated payload, expected " +
                        std::to_string(h.numel * sizeof(double)) + " bytes but read " +
                        std::to_string((off + got) * sizeof(double)));
            if (dt == ATK_F64) {
                ATK_CUDA(cudaMemcpyAsync(static_cast<double*>(t->data) + off, hbuf + b * chunk, n * sizeof(double),
                                         cudaMemcpyHostToDevice, ctx->stream));
            } else {
                double* s = stage.get() + b * chunk;
                ATK_CUDA(cudaMemcpyAsync(s, hbuf + b * chunk, n * sizeof(double), cudaMemcpyHostToDevice,
                                         ctx->stream));
                narrow_f64<<<unsigned(std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0,
                             ctx->stream>>>(s, static_cast<float*>(t->data) + off, n);
                ATK_LAUNCHED(ctx);
            }
            ATK_CUDA(cudaEventRecord(done[b].e, ctx->stream));
            off += n;
        }
        ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        atk_tensor_free(t);
        throw;
    }
    return t;
}

void dten_write(atk_ctx* ctx, const atk_tensor* t, const char* path) {
    check_tensor(t, "write_dten tensor");
    const std::string p = path ? path : "";
    File file{std::fopen(p.c_str(), "wb")};
    if (!file.f) io_fail("cannot open " + p + " for writing");
    const uint32_t version = 1, order = uint32_t(t->order);
    bool ok = std::fwrite("DTEN", 1, 4, file.f) == 4 && std::fwrite(&version, 4, 1, file.f) == 1 &&
              std::fwrite(&order, 4, 1, file.f) == 1 && std::fwrite(t->dims, 8, order, file.f) == order;
    const size_t total = t->numel();
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(kChunkElems, total));
    Pinned host(2 * chunk * sizeof(double));
    DevBuf<double> stage(ctx, t->dtype == ATK_F32 ? 2 * chunk : 0);
    Event done[2];
    auto* hbuf = static_cast<double*>(host.p);
    size_t pend_n[2] = {0, 0};
    auto drain = [&](int b) {
        if (!pend_n[b]) return;
        ATK_CUDA(cudaEventSynchronize(done[b].e));
        ok = ok && std::fwrite(hbuf + b * chunk, sizeof(double), pend_n[b], file.f) == pend_n[b];
        pend_n[b] = 0;
    };
    size_t off = 0;
    for (int c = 0; off < total; ++c) {
        const int b = c & 1;
        drain(b);
        const size_t n = std::min(chunk, total - off);
        const double* src = static_cast<const double*>(t->data) + off;
        if (t->dtype == ATK_F32) {
            double* s = stage.get() + b * chunk;
            widen_f32<<<unsigned(std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0, ctx->stream>>>(
                static_cast<const float*>(t->data) + off, s, n);
            ATK_LAUNCHED(ctx);
            src = s;
        }
        ATK_CUDA(cudaMemcpyAsync(hbuf + b * chunk, src, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        ATK_CUDA(cudaEventRecord(done[b].e, ctx->stream));
        pend_n[b] = n;
        off += n;
        if (c > 0) drain(b ^ 1);  // write chunk c-1 while chunk c copies
    }
    drain(0);
    drain(1);
    if (!ok || std::fflush(file.f) != 0) io_fail("failed writing " + p);
}

}  // namespace atk
