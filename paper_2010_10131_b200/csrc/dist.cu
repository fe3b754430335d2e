// dist.cu — multi-GPU st-HOSVD plumbing: NCCL over NVLink 5 / NVSwitch, one
// process per GPU.
//
// The input is sharded along the LAST mode: in column-major order each rank's
// slab [I_1 .. I_{N-1}, I_N / g] is one contiguous block of the flat buffer,
// so the same kernels run on a smaller O.  For modes n < N-1 the local Gram
// is a partial sum -> ONE ncclAllReduce(sum, fp64) per mode; the replicated
// eigensolver is deterministic, so every rank holds bit-identical factors and
// the TTM stays local (no data-path collective).  Before the shard mode the
// shrunk tensor is small (C5: 64 x 64 x 2048 fp32 = 33.5 MB) and is
// all-gathered once; that mode then runs replicated.
//
// NCCL is loaded with dlopen("libnccl.so.2") on first use, so single-GPU
// processes carry no NCCL dependency and share torch's copy when present.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "atk_driver.cuh"

namespace atk {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        // Prefer (1) an explicit ATK_NCCL_PATH (the Python layer points it at
        // torch's bundled NCCL), (2) a libnccl already in the process, (3) the
        // system one.  Loading an older system NCCL first would shadow the
        // newer symbols a later `import torch` needs.
        void* h = nullptr;
        if (const char* env = std::getenv("ATK_NCCL_PATH")) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) fail(ATK_NCCL_ERROR, std::string("cannot load libnccl.so.2: ") + dlerror());
        auto get = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) fail(ATK_NCCL_ERROR, std::string("NCCL symbol missing: ") + n);
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))get("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))get("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))get("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))get("ncclAllReduce");
        api.Broadcast = (decltype(api.Broadcast))get("ncclBroadcast");
        api.AllGather = (decltype(api.AllGather))get("ncclAllGather");
        api.CommGetAsyncError = (decltype(api.CommGetAsyncError))get("ncclCommGetAsyncError");
        api.GroupStart = (decltype(api.GroupStart))get("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))get("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))get("ncclGetErrorString");
        api.h = h;
    }
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(ATK_NCCL_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace


struct Comm {
    ncclComm_t comm = nullptr;  // NCCL backend
    bool host = false;          // host-staged backend (atk_comm_init_host)
    atk_host_collectives coll{};
    int rank = 0, world = 1;
    // per-rank last-mode slab sizes of the current sthosvd (one exchange up
    // front, reused by the last-mode all-gather; cleared when the call ends)
    std::vector<uint64_t> last_sizes;
    atk_comm_stats stats{};
};

namespace {

// A peer that died or a network error surfaces asynchronously: poll the
// communicator after every enqueue and after every synchronisation, so a
// failed collective becomes ATK_NCCL_ERROR instead of a hang on the next one.
void nccl_poll(const Comm* c, const char* what) {
    if (!c || !c->comm) return;
    ncclResult_t a = ncclSuccess;
    nccl_check(nccl().CommGetAsyncError(c->comm, &a), "ncclCommGetAsyncError");
    if (a != ncclSuccess && a != ncclInProgress)
        fail(ATK_NCCL_ERROR, std::string(what) + " (async): " + nccl().GetErrorString(a));
}

void count(Comm* c, int kind, uint64_t bytes) {  // 0 allreduce, 1 broadcast / all-gather
    if (kind == 0) {
        c->stats.allreduce_calls += 1;
        c->stats.allreduce_bytes += bytes;
    } else {
        c->stats.gather_calls += 1;
        c->stats.gather_bytes += bytes;
    }
}

// Gram symmetry: only the upper triangle (column-major j >= i) crosses the
// wire, I(I+1)/2 doubles instead of I^2 (C5: 16.8 instead of 33.5 MB per mode)
__global__ void pack_upper(const double* __restrict__ s, uint64_t n, double* __restrict__ p) {
    const uint64_t tot = n * (n + 1) / 2;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        // column j holds j + 1 entries starting at j (j + 1) / 2
        uint64_t j = uint64_t((sqrt(8.0 * double(e) + 1.0) - 1.0) * 0.5);
        while (j * (j + 1) / 2 > e) --j;
        while ((j + 1) * (j + 2) / 2 <= e) ++j;
        const uint64_t i = e - j * (j + 1) / 2;
        p[e] = s[i + n * j];
    }
}

__global__ void unpack_sym(const double* __restrict__ p, uint64_t n, double* __restrict__ s) {
    const uint64_t tot = n * n;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e % n, j = e / n;
        const uint64_t a = i <= j ? i : j, b = i <= j ? j : i;
        s[e] = p[a + b * (b + 1) / 2];
    }
}

}  // namespace

namespace {

void host_check(int rc, const char* what) {
    if (rc != 0) fail(ATK_NCCL_ERROR, std::string("host collective ") + what + " failed (" +
                                          std::to_string(rc) + ")");
}

// In-place sum of device doubles through host memory (host backend).
void host_allreduce(atk_ctx* ctx, double* dev, uint64_t count) {
    std::vector<double> h(count);
    ATK_CUDA(cudaMemcpyAsync(h.data(), dev, count * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    host_check(ctx->comm->coll.allreduce_f64(ctx->comm->coll.user, h.data(), count), "allreduce");
    ATK_CUDA(cudaMemcpyAsync(dev, h.data(), count * sizeof(double), cudaMemcpyHostToDevice,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void comm_init(atk_ctx* ctx, const void* unique_id, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(ATK_INVALID_ARGUMENT, "bad rank/world");
    comm_destroy(ctx);
    auto* c = new Comm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ATK_CUDA(cudaSetDevice(ctx->device));
    nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    ctx->comm = c;
}

void comm_init_host(atk_ctx* ctx, const atk_host_collectives* coll, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(ATK_INVALID_ARGUMENT, "bad rank/world");
    if (!coll || !coll->allreduce_f64 || !coll->broadcast)
        fail(ATK_INVALID_ARGUMENT, "host collectives need allreduce_f64 and broadcast");
    comm_destroy(ctx);
    auto* c = new Comm();
    c->host = true;
    c->coll = *coll;
    c->rank = rank;
    c->world = world;
    ctx->comm = c;
}

void comm_destroy(atk_ctx* ctx) {
    if (!ctx->comm) return;
    if (ctx->comm->comm) nccl().CommDestroy(ctx->comm->comm);
    delete ctx->comm;
    ctx->comm = nullptr;
}

void allreduce_sum(atk_ctx* ctx, double* buf, uint64_t n, double* comm_ms) {
    if (!ctx->comm || ctx->comm->world == 1) return;
    StageTimer t(ctx);
    t.start();
    count(ctx->comm, 0, n * sizeof(double));
    if (ctx->comm->host) {
        host_allreduce(ctx, buf, n);
    } else {
        nccl_check(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, ctx->comm->comm, ctx->stream),
                   "ncclAllReduce");
        nccl_poll(ctx->comm, "ncclAllReduce");
    }
    const double ms = t.stop_ms(kStageComm);
    if (comm_ms) *comm_ms += ms;
}

void allreduce_sym(atk_ctx* ctx, double* s, uint64_t n, double* comm_ms) {
    if (!ctx->comm || ctx->comm->world == 1) return;
    const uint64_t np = n * (n + 1) / 2;
    DevBuf<double> p(ctx, np);
    const int grid = int(std::min<uint64_t>((np + 255) / 256, uint64_t(ctx->num_sms) * 8));
    pack_upper<<<grid, 256, 0, ctx->stream>>>(s, n, p.get());
    ATK_LAUNCHED(ctx);
    allreduce_sum(ctx, p.get(), np, comm_ms);
    unpack_sym<<<int(std::min<uint64_t>((n * n + 255) / 256, uint64_t(ctx->num_sms) * 8)), 256, 0, ctx->stream>>>(
        p.get(), n, s);
    ATK_LAUNCHED(ctx);
}

void allreduce_sum2(atk_ctx* ctx, double* a, uint64_t na, double* b, uint64_t nb,
                    double* comm_ms) {
    if (!ctx->comm || ctx->comm->world == 1) return;
    StageTimer t(ctx);
    t.start();
    count(ctx->comm, 0, na * sizeof(double));
    count(ctx->comm, 0, nb * sizeof(double));
    if (ctx->comm->host) {
        host_allreduce(ctx, a, na);
        host_allreduce(ctx, b, nb);
    } else {
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        nccl_check(nccl().AllReduce(a, a, na, ncclFloat64, ncclSum, ctx->comm->comm, ctx->stream),
                   "ncclAllReduce");
        nccl_check(nccl().AllReduce(b, b, nb, ncclFloat64, ncclSum, ctx->comm->comm, ctx->stream),
                   "ncclAllReduce");
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
        nccl_poll(ctx->comm, "ncclAllReduce(YR, GR)");
    }
    const double ms = t.stop_ms(kStageComm);
    if (comm_ms) *comm_ms += ms;
}

static std::vector<uint64_t> gather_last(atk_ctx* ctx, const atk_tensor* local) {
    const int w = ctx->comm->world;
    if (ctx->comm->host) {  // sizes are < 2^53: exact in an fp64 sum
        std::vector<double> v(w, 0.0);
        v[ctx->comm->rank] = double(local->dims[local->order - 1]);
        count(ctx->comm, 0, w * sizeof(double));
        host_check(ctx->comm->coll.allreduce_f64(ctx->comm->coll.user, v.data(), w), "allreduce");
        std::vector<uint64_t> h(w);
        for (int r = 0; r < w; ++r) h[r] = uint64_t(v[r]);
        return h;
    }
    DevBuf<uint64_t> d(ctx, w);
    ATK_CUDA(cudaMemsetAsync(d.get(), 0, w * sizeof(uint64_t), ctx->stream));
    const uint64_t mine = local->dims[local->order - 1];
    ATK_CUDA(cudaMemcpyAsync(d.get() + ctx->comm->rank, &mine, sizeof(uint64_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    count(ctx->comm, 0, w * sizeof(uint64_t));
    nccl_check(nccl().AllReduce(d.get(), d.get(), w, ncclUint64, ncclSum, ctx->comm->comm, ctx->stream),
               "ncclAllReduce(sizes)");
    std::vector<uint64_t> h(w);
    ATK_CUDA(cudaMemcpyAsync(h.data(), d.get(), w * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    ATK_CUDA(cudaStreamSynchronize(ctx->stream));
    nccl_poll(ctx->comm, "ncclAllReduce(sizes)");
    return h;
}

uint64_t comm_global_last(atk_ctx* ctx, const atk_tensor* local) {
    if (!ctx->comm || ctx->comm->world == 1) return local->dims[local->order - 1];
    ctx->comm->last_sizes = gather_last(ctx, local);
    uint64_t s = 0;
    for (uint64_t v : ctx->comm->last_sizes) s += v;
    return s;
}

void comm_end_call(atk_ctx* ctx) {
    if (ctx->comm) ctx->comm->last_sizes.clear();
}

void comm_stats(const atk_ctx* ctx, atk_comm_stats* out) {
    *out = ctx->comm ? ctx->comm->stats : atk_comm_stats{};
}

void comm_stats_reset(atk_ctx* ctx) {
    if (ctx->comm) ctx->comm->stats = atk_comm_stats{};
}

atk_tensor* allgather_last_mode(atk_ctx* ctx, const atk_tensor* local) {
    const int order = local->order;
    const bool cached = ctx->comm && ctx->comm->world > 1 && int(ctx->comm->last_sizes.size()) == ctx->comm->world &&
                        ctx->comm->last_sizes[ctx->comm->rank] == local->dims[order - 1];
    std::vector<uint64_t> sizes = cached ? ctx->comm->last_sizes
                                  : (ctx->comm && ctx->comm->world > 1) ? gather_last(ctx, local)
                                                                        : std::vector<uint64_t>{local->dims[order - 1]};
    uint64_t total = 0;
    for (uint64_t v : sizes) total += v;
    uint64_t dims[ATK_MAX_ORDER];
    for (int m = 0; m < order; ++m) dims[m] = local->dims[m];
    dims[order - 1] = total;
    atk_tensor* out = new_tensor(ctx, local->dtype, order, dims);
    const uint64_t slab = local->numel() / std::max<uint64_t>(1, local->dims[order - 1]);
    if (!ctx->comm || ctx->comm->world == 1) {
        ATK_CUDA(cudaMemcpyAsync(out->data, local->data, local->bytes(), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
        return out;
    }
    if (ctx->comm->host) {
        const size_t es = local->elem_bytes();
        std::vector<char> h(out->bytes());
        uint64_t off = 0;
        for (int r = 0; r < ctx->comm->world; ++r) {
            char* dst = h.data() + off * slab * es;
            const uint64_t nb = sizes[r] * slab * es;
            if (r == ctx->comm->rank) {
                ATK_CUDA(cudaMemcpyAsync(dst, local->data, nb, cudaMemcpyDeviceToHost, ctx->stream));
                ATK_CUDA(cudaStreamSynchronize(ctx->stream));
            }
            count(ctx->comm, 1, nb);
            host_check(ctx->comm->coll.broadcast(ctx->comm->coll.user, dst, nb, r), "broadcast");
            off += sizes[r];
        }
        ATK_CUDA(cudaMemcpyAsync(out->data, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
        ATK_CUDA(cudaStreamSynchronize(ctx->stream));
        return out;
    }
    const ncclDataType_t dt = local->dtype == ATK_F32 ? ncclFloat32 : ncclFloat64;
    const size_t es = local->elem_bytes();
    bool even = true;
    for (uint64_t v : sizes) even = even && v == sizes[0];
    if (even) {  // equal slabs: one all-gather, rank-major blocks = the last-mode order
        count(ctx->comm, 1, sizes[0] * slab * es * ctx->comm->world);
        nccl_check(nccl().AllGather(local->data, out->data, sizes[0] * slab, dt, ctx->comm->comm, ctx->stream),
                   "ncclAllGather");
        nccl_poll(ctx->comm, "ncclAllGather");
        return out;
    }
    uint64_t off = 0;
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < ctx->comm->world; ++r) {
        char* dst = static_cast<char*>(out->data) + off * slab * es;
        const void* src = (r == ctx->comm->rank) ? local->data : dst;
        count(ctx->comm, 1, sizes[r] * slab * es);
        nccl_check(nccl().Broadcast(src, dst, sizes[r] * slab, dt, r, ctx->comm->comm, ctx->stream),
                   "ncclBroadcast");
        off += sizes[r];
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    nccl_poll(ctx->comm, "ncclBroadcast");
    return out;
}

}  // namespace atk
