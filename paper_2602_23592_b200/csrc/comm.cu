// comm.cu -- the collectives of KV-head sharding.
//
// Per layer, G ranks (one process and one B200 each) exchange:
//   * the fp64 segment summary: a sum over ranks in which every rank must
//     receive IDENTICAL bits, because `converge` then runs replicated
//     (recompute.hpp:130-138).  NCCL: reduce-scatter + all-gather, so each
//     element is reduced at exactly one place and then copied.
//   * attention context, head-sharded -> row-sharded: all-to-all.
//   * the fp32 residual rows after Wo + MLP: all-gather.
//
// NcclComm drives NCCL over NVLink/NVSwitch.  libnccl is dlopen'ed (soname
// libnccl.so.2, or $KEEP_NCCL_LIB): when torch has already loaded its NCCL the
// same library instance is used, and a single-GPU process never needs NCCL.
//
// LoopbackComm is a test double for the SAME code path with G logical ranks
// on one GPU inside one process (one host thread per rank): collectives are
// stream-ordered device copies between the ranks' buffers, synchronised by a
// host barrier and CUDA events.  It lets the sharded arithmetic run, and be
// checked against the single-GPU result, on a one-GPU box.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "engine.hpp"

namespace keep_b200 {

// ------------------------------------------------------------------ NCCL --
namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        const char* env = std::getenv("KEEP_NCCL_LIB");
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            if (!n || !*n) continue;
            a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return a;
        auto sym = [&](auto& fp, const char* name) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(a.h, name)); };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.AllGather, "ncclAllGather");
        sym(a.ReduceScatter, "ncclReduceScatter");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.h || !api.CommInitRank || !api.AllGather || !api.ReduceScatter || !api.Send || !api.GroupStart)
        raise(KEEP_ERR_CUDA, "NCCL (libnccl.so.2) is not loadable; set KEEP_NCCL_LIB");
    return api;
}

#define KEEP_NCCL(expr)                                                                                  \
    do {                                                                                                 \
        ncclResult_t r_ = (expr);                                                                        \
        if (r_ != ncclSuccess) raise(KEEP_ERR_CUDA, std::string(#expr) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

class NcclComm final : public Comm {
  public:
    NcclComm(int world_, int rank_, const uint8_t* id, void* external) {
        world = world_;
        rank = rank_;
        if (external) {
            comm_ = static_cast<ncclComm_t>(external);
            owned_ = false;
        } else {
            ncclUniqueId uid;
            std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
            KEEP_NCCL(nccl().CommInitRank(&comm_, world, uid, rank));
            owned_ = true;
        }
    }
    ~NcclComm() override {
        if (owned_ && comm_) nccl().CommDestroy(comm_);
    }
    void allreduce_f64(double* buf, size_t n, cudaStream_t st) override {
        const size_t chunk = size_t(ceil_div(int64_t(n), world));
        scratch_.ensure(sizeof(double) * chunk * world);
        double* s = scratch_.as<double>();
        KEEP_CUDA(cudaMemcpyAsync(s, buf, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        if (chunk * world > n) KEEP_CUDA(cudaMemsetAsync(s + n, 0, sizeof(double) * (chunk * world - n), st));
        // in place: recv = send + rank * chunk
        KEEP_NCCL(nccl().ReduceScatter(s, s + rank * chunk, chunk, ncclFloat64, ncclSum, comm_, st));
        KEEP_NCCL(nccl().AllGather(s + rank * chunk, s, chunk, ncclFloat64, comm_, st));
        KEEP_CUDA(cudaMemcpyAsync(buf, s, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        KEEP_NCCL(nccl().AllGather(send, recv, bytes, ncclChar, comm_, st));
    }
    void alltoall(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        KEEP_NCCL(nccl().GroupStart());
        for (int q = 0; q < world; ++q) {
            KEEP_NCCL(nccl().Send(static_cast<const uint8_t*>(send) + q * bytes, bytes, ncclChar, q, comm_, st));
            KEEP_NCCL(nccl().Recv(static_cast<uint8_t*>(recv) + q * bytes, bytes, ncclChar, q, comm_, st));
        }
        KEEP_NCCL(nccl().GroupEnd());
    }

  private:
    ncclComm_t comm_ = nullptr;
    bool owned_ = false;
    DevBuf scratch_;
};

// -------------------------------------------------------------- loopback --
__global__ void sum_ranks_f64(const double* __restrict__ parts, int world, size_t n, double* __restrict__ out) {
    for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
        double acc = parts[e];
        for (int r = 1; r < world; ++r) acc += parts[r * n + e];  // rank order on every rank
        out[e] = acc;
    }
}

}  // namespace

struct LoopbackHub {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void*> send;
    std::vector<cudaEvent_t> ready, done;
    explicit LoopbackHub(int w) : world(w), send(w, nullptr), ready(w, nullptr), done(w, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {

class LoopbackComm final : public Comm {
  public:
    LoopbackComm(LoopbackHub* hub, int rank_) : hub_(hub) {
        world = hub->world;
        rank = rank_;
        KEEP_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
        KEEP_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    }
    ~LoopbackComm() override {
        cudaEventDestroy(ready_);
        cudaEventDestroy(done_);
    }
    void allreduce_f64(double* buf, size_t n, cudaStream_t st) override {
        gather_.ensure(sizeof(double) * n * world);
        exchange(buf, st, [&](int q, const void* peer) {
            KEEP_CUDA(cudaMemcpyAsync(gather_.as<double>() + q * n, peer, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        });
        sum_ranks_f64<<<unsigned(std::min<int64_t>(ceil_div(int64_t(n), 256), kNumSMs * 4)), 256, 0, st>>>(
            gather_.as<double>(), world, n, buf);
        KEEP_LAUNCH_CHECK();
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        exchange(send, st, [&](int q, const void* peer) {
            uint8_t* dst = static_cast<uint8_t*>(recv) + q * bytes;
            if (dst != peer) KEEP_CUDA(cudaMemcpyAsync(dst, peer, bytes, cudaMemcpyDeviceToDevice, st));
        });
    }
    void alltoall(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        exchange(send, st, [&](int q, const void* peer) {
            KEEP_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + q * bytes,
                                      static_cast<const uint8_t*>(peer) + rank * bytes, bytes,
                                      cudaMemcpyDeviceToDevice, st));
        });
    }

  private:
    // publish my send buffer (ready after the work queued on st), copy from
    // every peer's, and do not let anyone overwrite a send buffer before all
    // readers' copies have executed (stream-ordered, like NCCL)
    template <class F>
    void exchange(const void* mine, cudaStream_t st, F&& copy_from) {
        KEEP_CUDA(cudaEventRecord(ready_, st));
        {
            std::lock_guard<std::mutex> lk(hub_->mu);
            hub_->send[rank] = mine;
            hub_->ready[rank] = ready_;
            hub_->done[rank] = done_;
        }
        hub_->barrier();
        for (int q = 0; q < world; ++q) {
            if (q != rank) KEEP_CUDA(cudaStreamWaitEvent(st, hub_->ready[q], 0));
            copy_from(q, hub_->send[q]);
        }
        KEEP_CUDA(cudaEventRecord(done_, st));
        hub_->barrier();
        for (int q = 0; q < world; ++q)
            if (q != rank) KEEP_CUDA(cudaStreamWaitEvent(st, hub_->done[q], 0));
        hub_->barrier();
    }

    LoopbackHub* hub_;
    cudaEvent_t ready_ = nullptr, done_ = nullptr;
    DevBuf gather_;
};

}  // namespace

std::unique_ptr<Comm> make_comm(const keep_config& cfg) {
    if (cfg.world_size <= 1) return nullptr;
    if (cfg.loopback) {
        auto* hub = static_cast<LoopbackHub*>(cfg.loopback);
        if (hub->world != cfg.world_size) raise(KEEP_ERR_CONFIG, "loopback group size != world_size");
        return std::unique_ptr<Comm>(new LoopbackComm(hub, cfg.rank));
    }
    if (!cfg.nccl_comm && !cfg.nccl_id) raise(KEEP_ERR_CONFIG, "world_size > 1 needs nccl_id, nccl_comm or loopback");
    return std::unique_ptr<Comm>(new NcclComm(cfg.world_size, cfg.rank, cfg.nccl_id, cfg.nccl_comm));
}

}  // namespace keep_b200

extern "C" {

int keep_comm_unique_id(uint8_t* id_out) {
    try {
        ncclUniqueId uid;
        const ncclResult_t r = keep_b200::nccl().GetUniqueId(&uid);
        if (r != ncclSuccess) keep_b200::raise(KEEP_ERR_CUDA, "ncclGetUniqueId failed");
        std::memcpy(id_out, uid.internal, NCCL_UNIQUE_ID_BYTES);
        return KEEP_OK;
    } catch (const keep_b200::KeepError& e) {
        keep_b200::set_last_error(e.what());
        return e.code;
    }
}

int keep_loopback_create(int32_t world, void** hub_out) {
    if (world < 1 || !hub_out) {
        keep_b200::set_last_error("bad loopback group size");
        return KEEP_ERR_CONFIG;
    }
    *hub_out = new keep_b200::LoopbackHub(world);
    return KEEP_OK;
}

int keep_loopback_destroy(void* hub) {
    delete static_cast<keep_b200::LoopbackHub*>(hub);
    return KEEP_OK;
}

}  // extern "C"
