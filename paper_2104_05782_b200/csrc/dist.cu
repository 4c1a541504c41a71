// dist.cu -- the blocked randUTV sharded over a 2D block-cyclic P x Q grid of GPUs.
//
// The reference's distributed version is ScaLAPACK over MPI
// with the layout of proj/src/block_cyclic.cpp:26-38: block (br, bc) of b x b
// lives on rank (br mod P) * Q + (bc mod Q), at local block (br div P, bc div Q).
// Here one rank = one GPU, T, U, V are distributed identically with the
// distribution block equal to the step width b, and every step of
// randutv_blocked.cpp:122-155 (s = n - i b) becomes local DMMA products plus
// one collective per product over NVLink (NCCL):
//
//   sketch   G (s x b) is replicated by construction -- the counter RNG
//            (rng.hpp:9-17) lets each rank draw exactly its own rows, no traffic.
//            Y = T22' G: local T22_loc' G_loc, all-reduce over the process COLUMN;
//            each power iteration Z = T22 Y (all-reduce over the process ROW) and
//            Y = T22' Z (column).
//   QR(Y)    all-gather Y's column-block slices over the row, factor redundantly
//            on every rank (deterministic kernels + bit-identical all-reduce
//            results => identical W_v, Twy_v everywhere, nothing broadcast).
//   V-apply  [V; T](:, r0:) Q_v = X - (X W_v) M_v': Zx = X_loc W_v[my cols],
//            all-reduce over the row, local rank-b update.  T22's rows are the
//            critical chain (stream A); V and the finished rows of T go to the
//            low-priority stream B with their OWN row communicator.
//   U-QR     block column i lives in process column i mod Q: it is all-gathered
//            there, factored by the owner of the diagonal block (i, i), and the
//            packed panel + tau are broadcast to every rank.
//   Qu'      T22(:, b:) <- Q_u' T22(:, b:): Zl = W_u[my rows]' B_loc, all-reduce
//            over the column, local update.
//   U-apply  like the V-apply, on stream B.
//   beta     deferred exactly as on one GPU (randutv.cu): each diagonal owner
//            SVDs its R_i in ONE batched Jacobi launch, the [Us | Vs | sigma]
//            factors are all-gathered once, then diagonal writes, row strips and
//            right-multiplies are local.
//
// Communication backends (struct Group): NCCL communicators (world, row, column,
// row-side, split from one world communicator; algorithm/protocol pinned to
// Ring/Simple unless the caller set them, for run-to-run determinism), or an
// in-process exchange for P x Q ranks run as host threads on ONE device
// (grid_sim): the same driver code, collectives done by device copies between
// the ranks' buffers behind host barriers -- how the sharded path is validated
// on a single-GPU box.  Kernels never wait on each other on the device.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rutv_common.cuh"

#include <dlfcn.h>

namespace rutv {
namespace dist {

// NCCL is bound at first use, not at load: a process that imports torch after
// this library must get torch's own libnccl.so.2 (a newer NCCL than the
// system's), so an already-loaded libnccl.so.2 is preferred (RTLD_NOLOAD) and
// the system one is opened only when none is.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && err.empty()) err = std::string("NCCL symbol missing: ") + name;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommSplit, "ncclCommSplit");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.Broadcast, "ncclBroadcast");
        sym(api.AllGather, "ncclAllGather");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    if (!err.empty()) throw Error(RUTV_ERR_NCCL, err);
    return api;
}

#define RUTV_NCCL(call)                                                                                    \
    do {                                                                                                   \
        ncclResult_t r_ = ::rutv::dist::nccl().call;                                                       \
        if (r_ != ncclSuccess)                                                                             \
            throw ::rutv::Error(RUTV_ERR_NCCL, std::string("NCCL error ") +                                \
                                                   ::rutv::dist::nccl().GetErrorString(r_) + " at " +      \
                                                   __FILE__ + ":" + std::to_string(__LINE__));             \
    } while (0)

// ------------------------------------------------------------------ layout
// One dimension of the block-cyclic layout (block_cyclic.cpp:26-38): n indices in
// blocks of b over p processes.  Only the last global block can be ragged, so the
// local offset of an owned block k is (k / p) * b.
struct Axis {
    int64_t n = 0, b = 1;
    int p = 1;
    int64_t nblk() const { return (n + b - 1) / b; }
    int64_t width(int64_t k) const { return std::min(b, n - k * b); }
    int64_t loc(int64_t k) const { return (k / p) * b; }
    int64_t length(int c) const {
        const int64_t nb = nblk();
        if (c >= nb) return 0;
        const int64_t cnt = (nb - 1 - c) / p + 1;
        int64_t len = cnt * b;
        if ((nb - 1) % p == c) len -= b - width(nb - 1);
        return len;
    }
    int64_t first_from(int64_t i, int c) const {
        const int64_t k = i + (((c - i) % p) + p) % p;
        return k < nblk() ? k : -1;
    }
    // (local offset, block count) of the owned blocks >= i
    std::pair<int64_t, int64_t> suffix(int64_t i, int c) const {
        const int64_t k = first_from(i, c);
        if (k < 0) return {length(c), 0};
        return {loc(k), (nblk() - 1 - k) / p + 1};
    }
};

// ----------------------------------------------------------- communication
struct Group {
    int size = 1, index = 0;
    virtual ~Group() = default;
    virtual void allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
    virtual void broadcast(double* buf, size_t count, int root, cudaStream_t st) = 0;
    // recv holds size * count doubles, member r's contribution at r * count
    virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
};

struct SelfGroup : Group {
    void allreduce_sum(double*, size_t, cudaStream_t) override {}
    void broadcast(double*, size_t, int, cudaStream_t) override {}
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        if (send != recv && count) RUTV_CUDA(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, st));
    }
};

struct NcclGroup : Group {
    ncclComm_t comm = nullptr;
    explicit NcclGroup(ncclComm_t c) : comm(c) {
        RUTV_NCCL(CommCount(c, &size));
        RUTV_NCCL(CommUserRank(c, &index));
    }
    ~NcclGroup() override {
        if (comm) nccl().CommDestroy(comm);
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        if (count) RUTV_NCCL(AllReduce(buf, buf, count, ncclDouble, ncclSum, comm, st));
    }
    void broadcast(double* buf, size_t count, int root, cudaStream_t st) override {
        if (count) RUTV_NCCL(Broadcast(buf, buf, count, ncclDouble, root, comm, st));
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        if (count) RUTV_NCCL(AllGather(send, recv, count, ncclDouble, comm, st));
    }
};

__global__ void add_into_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] += x[i];
}

// In-process exchange between ranks that are host threads on one device.
struct SimHub {
    struct State {
        int arrived = 0;
        uint64_t gen = 0;
        std::vector<const void*> ptrs, snapshot;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::string, State> states;

    std::vector<const void*> exchange(const std::string& key, int size, int index, const void* p) {
        std::unique_lock<std::mutex> lk(mu);
        State& s = states[key];
        if (s.ptrs.size() != static_cast<size_t>(size)) s.ptrs.assign(static_cast<size_t>(size), nullptr);
        s.ptrs[static_cast<size_t>(index)] = p;
        const uint64_t gen = s.gen;
        if (++s.arrived == size) {
            s.arrived = 0;
            s.snapshot = s.ptrs;
            ++s.gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return s.gen != gen; });
        }
        return s.snapshot;
    }
};

struct SimGroup : Group {
    SimHub* hub;
    std::string key;
    double* tmp = nullptr;  // plain cudaMalloc: outlives the streams of any one call
    size_t tmp_elems = 0;
    SimGroup(SimHub* h, std::string k, int sz, int idx) : hub(h), key(std::move(k)) {
        size = sz;
        index = idx;
    }
    ~SimGroup() override {
        if (tmp) cudaFree(tmp);
    }
    void sync_exchange_done(cudaStream_t st) {
        RUTV_CUDA(cudaStreamSynchronize(st));
        hub->exchange(key, size, index, nullptr);  // nobody re-reads a peer's buffer after this
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        if (!count) return;
        RUTV_CUDA(cudaStreamSynchronize(st));
        auto ptrs = hub->exchange(key, size, index, buf);
        if (tmp_elems < count) {
            if (tmp) RUTV_CUDA(cudaFree(tmp));
            tmp = nullptr;
            RUTV_CUDA(cudaMalloc(reinterpret_cast<void**>(&tmp), count * 8));
            tmp_elems = count;
        }
        // fixed rank order: identical bits on every member
        RUTV_CUDA(cudaMemcpyAsync(tmp, ptrs[0], count * 8, cudaMemcpyDeviceToDevice, st));
        const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 4 * kNumSMs));
        for (int r = 1; r < size; ++r) {
            add_into_kernel<<<blocks, 256, 0, st>>>(tmp, static_cast<const double*>(ptrs[static_cast<size_t>(r)]),
                                                    static_cast<int64_t>(count));
            note_launch();
            RUTV_CHECK_LAUNCH();
        }
        sync_exchange_done(st);
        RUTV_CUDA(cudaMemcpyAsync(buf, tmp, count * 8, cudaMemcpyDeviceToDevice, st));
        RUTV_CUDA(cudaStreamSynchronize(st));
    }
    void broadcast(double* buf, size_t count, int root, cudaStream_t st) override {
        if (!count) return;
        RUTV_CUDA(cudaStreamSynchronize(st));
        auto ptrs = hub->exchange(key, size, index, buf);
        if (index != root)
            RUTV_CUDA(cudaMemcpyAsync(buf, ptrs[static_cast<size_t>(root)], count * 8, cudaMemcpyDeviceToDevice, st));
        sync_exchange_done(st);
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        if (!count) return;
        RUTV_CUDA(cudaStreamSynchronize(st));
        auto ptrs = hub->exchange(key, size, index, send);
        for (int r = 0; r < size; ++r)
            RUTV_CUDA(cudaMemcpyAsync(recv + static_cast<size_t>(r) * count, ptrs[static_cast<size_t>(r)], count * 8,
                                      cudaMemcpyDeviceToDevice, st));
        sync_exchange_done(st);
    }
};

// One rank of the grid: its device and communicators.
struct Ctx {
    int P = 1, Q = 1, rank = 0, device = 0;
    std::unique_ptr<Group> world, row, col, row_side;
    int pr() const { return rank / Q; }
    int pc() const { return rank % Q; }
    int owner2(int64_t br, int64_t bc) const { return static_cast<int>((br % P) * Q + (bc % Q)); }
};

std::unique_ptr<Group> wrap(ncclComm_t c) {
    int n = 0;
    RUTV_NCCL(CommCount(c, &n));
    if (n == 1) {
        nccl().CommDestroy(c);
        return std::make_unique<SelfGroup>();
    }
    return std::make_unique<NcclGroup>(c);
}

void pin_nccl_env() {
    // Fixed algorithm and protocol: reductions are bit-reproducible run to run
    // (SURVEY.md section 8e).  A caller's own settings win.
    setenv("NCCL_ALGO", "Ring", 0);
    setenv("NCCL_PROTO", "Simple", 0);
}

// World communicator -> row / column / row-side groups (every rank calls this).
void split_groups(Ctx& cx, ncclComm_t world) {
    ncclComm_t row = nullptr, col = nullptr, side = nullptr;
    RUTV_NCCL(CommSplit(world, cx.pr(), cx.pc(), &row, nullptr));
    RUTV_NCCL(CommSplit(world, cx.pc(), cx.pr(), &col, nullptr));
    RUTV_NCCL(CommSplit(world, cx.pr(), cx.pc(), &side, nullptr));
    cx.world = wrap(world);
    cx.row = wrap(row);
    cx.col = wrap(col);
    cx.row_side = wrap(side);
    // One tiny collective per communicator, in a fixed order, synchronously: NCCL sets up
    // its buffers and connections lazily at a communicator's first collective, and that
    // must not happen later while the other communicator has a kernel in flight on
    // another stream of this rank.
    double* one = nullptr;
    cudaStream_t s = nullptr;
    RUTV_CUDA(cudaMalloc(reinterpret_cast<void**>(&one), 8));
    RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    RUTV_CUDA(cudaMemsetAsync(one, 0, 8, s));
    for (Group* g : {cx.world.get(), cx.row.get(), cx.col.get(), cx.row_side.get()}) {
        g->allreduce_sum(one, 1, s);
        RUTV_CUDA(cudaStreamSynchronize(s));
    }
    cudaStreamDestroy(s);
    cudaFree(one);
}

void sim_groups(Ctx& cx, SimHub* hub) {
    const int W = cx.P * cx.Q;
    auto mk = [&](const std::string& key, int size, int index) -> std::unique_ptr<Group> {
        if (size == 1) return std::make_unique<SelfGroup>();
        return std::make_unique<SimGroup>(hub, key, size, index);
    };
    cx.world = mk("world", W, cx.rank);
    cx.row = mk("row" + std::to_string(cx.pr()), cx.Q, cx.pc());
    cx.col = mk("col" + std::to_string(cx.pc()), cx.P, cx.pr());
    cx.row_side = mk("side" + std::to_string(cx.pr()), cx.Q, cx.pc());
}

// ------------------------------------------------------------------ driver
struct Args {
    int64_t n, b;
    int q;
    bool bu, bv;
    uint64_t seed;
    int max_steps;
    const double* dG;  // full explicit stream (replicated) or null
    const double* A;
    int64_t lda;
    double *T, *U, *V;
    int64_t ldt, ldu, ldv;
    bool overlap;
};

inline int64_t rup4(int64_t x) { return std::max<int64_t>((x + 3) / 4 * 4, 1); }

void factorize_rank(Ctx& cx, const Args& fa, cudaStream_t st_in) {
    NvtxRange range("rutv/factorize_dist");
    const int64_t n = fa.n, b = fa.b;
    const int P = cx.P, Q = cx.Q, pr = cx.pr(), pc = cx.pc(), me = cx.rank;
    const Axis RA{n, b, P}, CA{n, b, Q};
    const int64_t mr = RA.length(pr), mc = CA.length(pc), nblk = RA.nblk();
    const bool bu = fa.bu, bv = fa.bv;
    const int64_t vr = bv ? mr : 0;
    // in place when V sits on top of T in one caller buffer, or V is not built
    const bool vt_inplace = mr > 0 && mc > 0 && (!bv || (fa.V && fa.T == fa.V + mr && fa.ldt == fa.ldv));
    const int64_t ldvt = vt_inplace ? (bv ? fa.ldv : fa.ldt) : rup4(vr + mr);
    const bool u_inplace = bu && fa.U;
    const int64_t ldu = u_inplace ? fa.ldu : rup4(mr);

    // streams: critical chain on a high-priority stream A, V/U accumulation on B
    const bool overlap = fa.overlap;
    // C: the panel-first look-ahead's remaining columns (one priority level below A)
    cudaStream_t sA = st_in, sB = st_in, sC = st_in, sD = st_in;
    int lo = 0, hi = 0;
    RUTV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (overlap) {
        RUTV_CUDA(cudaStreamCreateWithPriority(&sA, cudaStreamNonBlocking, hi));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sB, cudaStreamNonBlocking, lo));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sC, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
        RUTV_CUDA(cudaStreamCreateWithPriority(&sD, cudaStreamNonBlocking, hi));
        cudaEvent_t e;
        RUTV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        RUTV_CUDA(cudaEventRecord(e, st_in));
        RUTV_CUDA(cudaStreamWaitEvent(sA, e, 0));
        cudaEventDestroy(e);
    }
    struct StreamGuard {
        cudaStream_t s;
        bool own;
        ~StreamGuard() {
            if (own) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        }
    } gA{sA, overlap}, gB{sB, overlap}, gC{sC, overlap}, gD{sD, overlap};
    std::vector<cudaEvent_t> events;
    struct EventGuard {
        std::vector<cudaEvent_t>& ev;
        ~EventGuard() {
            for (auto e : ev) cudaEventDestroy(e);
        }
    } eg{events};
    auto record = [&](cudaStream_t s) {
        cudaEvent_t e;
        RUTV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        RUTV_CUDA(cudaEventRecord(e, s));
        events.push_back(e);
        return e;
    };
    auto wait = [&](cudaStream_t s, cudaEvent_t e) {
        if (overlap && e) RUTV_CUDA(cudaStreamWaitEvent(s, e, 0));
    };

    DevBuf VTb(vt_inplace ? 1 : ldvt * std::max<int64_t>(mc, 1), sA), Ub(bu && !u_inplace ? ldu * std::max<int64_t>(mc, 1) : 1, sA);
    DView vt(vr + mr, mc, ldvt, vt_inplace ? (bv ? fa.V : fa.T) : VTb.p);
    DView tl(mr, mc, ldvt, vt.data + vr);
    DView ul(mr, mc, ldu, u_inplace ? fa.U : Ub.p);
    if (mr * mc > 0 && (tl.data != fa.A || tl.ld != fa.lda))
        copy_view(sA, tl, DView(mr, mc, fa.lda, const_cast<double*>(fa.A)));
    // U, V := I (randutv_blocked.cpp:114-120): zeros, identity on my diagonal blocks
    if (mr * mc > 0) {
        if (bv) RUTV_CUDA(cudaMemset2DAsync(vt.data, ldvt * 8, 0, mr * 8, mc, sA));
        if (bu) RUTV_CUDA(cudaMemset2DAsync(ul.data, ldu * 8, 0, mr * 8, mc, sA));
        for (int64_t k = pr; k < nblk; k += P) {
            if (k % Q != pc) continue;
            const int64_t w = RA.width(k), ro = RA.loc(k), co = CA.loc(k);
            if (bv) set_identity(sA, vt.block(ro, co, w, w));
            if (bu) set_identity(sA, ul.block(ro, co, w, w));
        }
    }

    // ---- workspace (largest step sizes)
    const int64_t cntR = (nblk + P - 1) / P, cntC = (nblk + Q - 1) / Q;
    const int64_t slabR = cntR * b, slabC = cntC * b;
    const int64_t nb = std::max<int64_t>(n * b, 1);
    DevBuf Gl(std::max<int64_t>(mr, 1) * b, sA), Yl(slabC * b, sA), Zr(std::max<int64_t>(mr, 1) * b, sA);
    DevBuf Yf(nb, sA), SlabY(slabC * b, sA), SlabsY(static_cast<int64_t>(Q) * slabC * b, sA);
    DevBuf Wv(nb, sA), Mv(nb, sA), Pan(nb, sA), SlabP(slabR * b, sA), SlabsP(static_cast<int64_t>(P) * slabR * b, sA);
    DevBuf Wu(nb, sA), Mu(nb, sA), Gram(b * b, sA), Twy(b * b, sA), TauV(b + 1, sA), TauU(b + 1, sA);
    DevBuf WlA(std::max<int64_t>(mc, 1) * b, sA), MlA(std::max<int64_t>(mc, 1) * b, sA);
    DevBuf WrA(std::max<int64_t>(mr, 1) * b, sA), MrA(std::max<int64_t>(mr, 1) * b, sA);
    DevBuf ZxA(std::max<int64_t>(mr, 1) * b, sA), ZlA(b * std::max<int64_t>(mc, 1), sA);
    // stream B private, double-buffered hand-off from A (slot = step parity)
    DevBuf WvB0(std::max<int64_t>(mc, 1) * b, sA), WvB1(std::max<int64_t>(mc, 1) * b, sA);
    DevBuf MvB0(std::max<int64_t>(mc, 1) * b, sA), MvB1(std::max<int64_t>(mc, 1) * b, sA);
    DevBuf WuB0(std::max<int64_t>(mc, 1) * b, sA), WuB1(std::max<int64_t>(mc, 1) * b, sA);
    DevBuf MuB0(std::max<int64_t>(mc, 1) * b, sA), MuB1(std::max<int64_t>(mc, 1) * b, sA);
    double* WvB[2] = {WvB0.p, WvB1.p};
    double* MvB[2] = {MvB0.p, MvB1.p};
    double* WuB[2] = {WuB0.p, WuB1.p};
    double* MuB[2] = {MuB0.p, MuB1.p};
    DevBuf ZxB(std::max<int64_t>(vr + mr, 1) * b, sA), ZuB(std::max<int64_t>(mr, 1) * b, sA);
    const int64_t gwe = std::max<int64_t>({gemm_work_elems(std::max(vr + mr, n), b, std::max(mr, mc)),
                                           gemm_work_elems(b, std::max<int64_t>(mc, 1), std::max<int64_t>(mr, 1)),
                                           gemm_work_elems(n, b, b), gemm_work_elems(b, b, n), int64_t(1)});
    DevBuf GWA(gwe, sA), GWB(gwe, sA), GWC(gwe, sA), GWD(gwe, sA);
    const int64_t hqw = hqr_work_elems(n, b);
    DevBuf HQ(hqw, sA);
    // deferred beta: my diagonal steps' R, and the factor slots
    std::vector<int64_t> my_steps;
    for (int64_t k = 0; k < nblk; ++k)
        if (cx.owner2(k, k) == me) my_steps.push_back(k);
    int slots = 0;
    for (int r = 0; r < P * Q; ++r) {
        int c = 0;
        for (int64_t k = 0; k < nblk; ++k) c += cx.owner2(k, k) == r;
        slots = std::max(slots, c);
    }
    const int64_t fslot = 2 * b * b + b;  // [Us | Vs | sigma] of one step
    DevBuf Rm(std::max<int64_t>(static_cast<int64_t>(my_steps.size()), 1) * b * b, sA);
    DevBuf Fac(std::max<int64_t>(slots, 1) * fslot, sA), FacAll(std::max<int64_t>(slots, 1) * fslot * P * Q, sA);
    const int64_t svdw = svd_work_elems(b, 30);
    DevBuf SvdW(std::max<int64_t>(static_cast<int64_t>(my_steps.size()), 1) * svdw, sA);
    DevBuf Jst(std::max<int64_t>(static_cast<int64_t>(my_steps.size()), 1) * 4, sA);
    DevBuf Desc((static_cast<int64_t>(sizeof(SvdDesc)) * std::max<int64_t>(static_cast<int64_t>(my_steps.size()), 1) + 7) / 8, sA);
    RUTV_CUDA(cudaMemsetAsync(Jst.p, 0, std::max<size_t>(my_steps.size(), 1) * 32, sA));
    RUTV_CUDA(cudaMemsetAsync(Fac.p, 0, static_cast<size_t>(std::max(slots, 1) * fslot) * 8, sA));
    {
        const cudaEvent_t ev = record(sA);
        wait(sB, ev);
        wait(sC, ev);
        wait(sD, ev);
    }
    struct Join {
        cudaStream_t a, b, c, d;
        bool own;
        ~Join() {
            if (own) {
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
                cudaStreamSynchronize(c);
                cudaStreamSynchronize(d);
            }
        }
    } join{sA, sB, sC, sD, overlap};

    auto gemmA = [&](double al, Op ta, const DView& x, Op tb, const DView& y, double be, const DView& c) {
        gemm(sA, al, ta, x, tb, y, be, c, GWA.p, gwe);
    };
    auto gemmB = [&](double al, Op ta, const DView& x, Op tb, const DView& y, double be, const DView& c) {
        gemm(sB, al, ta, x, tb, y, be, c, GWB.p, gwe);
    };
    // my blocks >= i of an axis, as rows of the s x w matrix `full` (global block order from i)
    auto pick = [&](cudaStream_t s, const Axis& ax, int c, int64_t i, int64_t srows, const double* full, int64_t w,
                    double* out, int64_t ldo) {
        const auto sf = ax.suffix(i, c);
        if (sf.second == 0) return;
        block_rows(s, out, ldo, const_cast<double*>(full), srows, srows, w, b, ax.first_from(i, c) - i, ax.p,
                   sf.second, false);
    };
    // all-gather the slices `loc` (my blocks >= i of `ax`, m rows) over `grp` and assemble
    // the s x b matrix `full` (ld s) in global block order
    auto gather = [&](Group& grp, const Axis& ax, int64_t i, int64_t s, const double* loc, int64_t ldloc, int64_t m,
                      int64_t slab_rows, double* slab, double* slabs, double* full) {
        if (m > 0) copy_view(sA, DView(m, b, slab_rows, slab), DView(m, b, ldloc, const_cast<double*>(loc)));
        grp.allgather(slab, slabs, static_cast<size_t>(slab_rows * b), sA);
        for (int c = 0; c < grp.size; ++c) {
            const int64_t k0 = ax.first_from(i, c);
            if (k0 < 0) continue;
            const int64_t cnt = (ax.nblk() - 1 - k0) / ax.p + 1;
            block_rows(sA, slabs + static_cast<int64_t>(c) * slab_rows * b, slab_rows, full, s, s, b, b, k0 - i, ax.p,
                       cnt, true);
        }
    };
    // W (unit lower), Twy, M = W Twy' of a packed s x b panel
    // W (unit lower) on A; Twy (Gram + form_wy_t) and M = W Twy' on stream D, while A
    // already runs the W-only half of the apply (X W, resp. W' B) -- as randutv.cu.
    // Returns D's event (M ready).
    auto form_wy = [&](const double* qr, int64_t s, const double* tau, double* W, double* M) {
        DView Wv_(s, b, s, W), Mv_(s, b, s, M);
        make_w(sA, DView(s, b, s, const_cast<double*>(qr)), b, Wv_);
        wait(sD, record(sA));
        gemm(sD, 1.0, Op::T, Wv_, Op::N, Wv_, 0.0, DView(b, b, b, Gram.p), GWD.p, gwe);
        form_t(sD, Gram.p, b, tau, b, Twy.p, b);
        gemm(sD, 1.0, Op::N, Wv_, Op::T, DView(b, b, b, Twy.p), 0.0, Mv_, GWD.p, gwe);
        return record(sD);
    };

    uint64_t pos = 0;
    int64_t steps = 0, tail_w = 0;
    std::vector<cudaEvent_t> evB;
    // Sketch hoisting (as randutv.cu): the next step's first sketch product is formed
    // from B = (T22 Q_v)(my rows >= i+1, my cols >= i+1) -- final once the V-apply is
    // done -- on stream C beside the panel QR: P = B' G'_loc, corrected after Q_u' by
    // - Zl' (M_u(my rows >= i+1)' G'_loc), since T22' = B - M_u Zl on those rows.  The
    // corrected partial is what the next step all-reduces (mathematically T22'^T G').
    const char* hoist_env = std::getenv("RUTV_HOIST");
    const bool hoist = overlap && !(hoist_env && std::strcmp(hoist_env, "0") == 0);
    bool have_y = false;
    DevBuf G2(std::max<int64_t>(mr, 1) * b, sA), Mh(std::max<int64_t>(mr, 1) * b, sA), Hh(b * b, sA);
    for (int64_t i = 0; i < nblk; ++i) {
        if (fa.max_steps >= 0 && steps >= fa.max_steps) break;
        const int64_t s = n - i * b;
        const int64_t ri = RA.suffix(i, pr).first, ci = CA.suffix(i, pc).first;
        const int64_t m_r = mr - ri, m_c = mc - ci;
        const int downer = cx.owner2(i, i);
        ++steps;
        DView T22 = m_r > 0 && m_c > 0 ? tl.block(ri, ci, m_r, m_c) : DView(m_r, m_c, tl.ld, tl.data);
        if (s <= b) {  // ragged tail: the dense s x s block lives on the diagonal owner (:129-137)
            tail_w = s;
            if (me == downer) {
                const size_t slot = std::find(my_steps.begin(), my_steps.end(), i) - my_steps.begin();
                copy_view(sA, DView(s, s, b, Rm.p + slot * b * b), T22.block(0, 0, s, s));
            }
            break;
        }
        const int par = static_cast<int>(i & 1);
        if (i >= 2) wait(sA, evB[static_cast<size_t>(i - 2)]);  // B done with slot `par`
        // ---- sketch (build_v_alpha, :41-50)
        DView G(m_r, b, std::max<int64_t>(m_r, 1), Gl.p), Y(m_c, b, std::max<int64_t>(m_c, 1), Yl.p), Z(m_r, b, std::max<int64_t>(m_r, 1), Zr.p);
        if (m_r > 0 && !have_y) {
            const int64_t k0 = RA.first_from(i, pr);
            if (fa.dG)
                block_rows(sA, G.data, G.ld, const_cast<double*>(fa.dG) + pos, s, s, b, b, k0 - i, P,
                           RA.suffix(i, pr).second, false);
            else
                normal_fill_cyclic(sA, fa.seed, pos, s, b, k0 - i, P, G);
        }
        pos += static_cast<uint64_t>(s * b);
        if (m_c > 0) {
            // hoisted: Yl already holds this rank's partial of T22' G (formed during the
            // previous step beside its panel QR); otherwise the plain product
            if (!have_y) gemmA(1.0, Op::T, T22, Op::N, G, 0.0, Y);
            cx.col->allreduce_sum(Yl.p, static_cast<size_t>(m_c * b), sA);
        }
        have_y = false;
        for (int it = 0; it < fa.q; ++it) {
            if (m_r > 0) {
                gemmA(1.0, Op::N, T22, Op::N, Y, 0.0, Z);
                cx.row->allreduce_sum(Zr.p, static_cast<size_t>(std::max<int64_t>(m_r, 1) * b), sA);
            }
            if (m_c > 0) {
                gemmA(1.0, Op::T, T22, Op::N, Z, 0.0, Y);
                cx.col->allreduce_sum(Yl.p, static_cast<size_t>(m_c * b), sA);
            }
        }
        // ---- QR(Y), redundantly on every rank (:52-53)
        gather(*cx.row, CA, i, s, Yl.p, std::max<int64_t>(m_c, 1), m_c, slabC, SlabY.p, SlabsY.p, Yf.p);
        hqr_panel(sA, DView(s, b, s, Yf.p), TauV.p, nullptr, 0, HQ.p, hqw);
        const cudaEvent_t evMv = form_wy(Yf.p, s, TauV.p, Wv.p, Mv.p);
        // ---- V-apply (:140-143): T22 rows on A; V and finished T rows on B
        if (m_c > 0) pick(sA, CA, pc, i, s, Wv.p, b, WlA.p, std::max<int64_t>(m_c, 1));
        if (m_r > 0) {  // Zx = X W_v[my cols]: needs only W (D forms Twy_v, M_v meanwhile)
            DView X = vt.block(vr + ri, ci, m_r, m_c), Zx(m_r, b, std::max<int64_t>(m_r, 1), ZxA.p);
            if (m_c > 0) gemmA(1.0, Op::N, X, Op::N, DView(m_c, b, std::max<int64_t>(m_c, 1), WlA.p), 0.0, Zx);
            else RUTV_CUDA(cudaMemsetAsync(ZxA.p, 0, static_cast<size_t>(m_r * b) * 8, sA));
            cx.row->allreduce_sum(ZxA.p, static_cast<size_t>(m_r * b), sA);
        }
        wait(sA, evMv);
        if (m_c > 0) {
            pick(sA, CA, pc, i, s, Mv.p, b, MlA.p, std::max<int64_t>(m_c, 1));
            copy_view(sA, DView(m_c, b, std::max<int64_t>(mc, 1), WvB[par]), DView(m_c, b, std::max<int64_t>(m_c, 1), WlA.p));
            copy_view(sA, DView(m_c, b, std::max<int64_t>(mc, 1), MvB[par]), DView(m_c, b, std::max<int64_t>(m_c, 1), MlA.p));
        }
        const cudaEvent_t evV = record(sA);
        if (m_r > 0) {
            DView X = vt.block(vr + ri, ci, m_r, m_c), Zx(m_r, b, std::max<int64_t>(m_r, 1), ZxA.p);
            DView Ml(m_c, b, std::max<int64_t>(m_c, 1), MlA.p);
            // Panel-first look-ahead (as randutv.cu): the process column that holds block
            // column i updates those b columns first on A -- all the panel QR needs --
            // and every other column on C, beside the panel gather / QR / broadcast.
            const int64_t c_first = (static_cast<int>(i % Q) == pc) ? std::min<int64_t>(b, m_c) : 0;
            if (c_first > 0) gemmA(-1.0, Op::N, Zx, Op::T, Ml.block(0, 0, c_first, b), 1.0, X.block(0, 0, m_r, c_first));
            if (m_c > c_first) {
                wait(sC, record(sA));
                gemm(sC, -1.0, Op::N, Zx, Op::T, Ml.block(c_first, 0, m_c - c_first, b), 1.0,
                     X.block(0, c_first, m_r, m_c - c_first), GWC.p, gwe);
            }
        }
        const cudaEvent_t evRest = record(sC);  // the columns Q_u' needs besides the panel
        // ---- sketch hoisting: P = B' G'_loc on stream C, beside the panel QR
        const bool hoist_next =
            hoist && i + 1 < nblk && n - (i + 1) * b > b && (fa.max_steps < 0 || steps < fa.max_steps);
        cudaEvent_t evP = nullptr;
        const int64_t ri1 = RA.suffix(i + 1, pr).first, ci1 = CA.suffix(i + 1, pc).first;
        const int64_t mr1 = mr - ri1, nc1 = mc - ci1;
        if (hoist_next) {
            const int64_t s1 = s - b;
            wait(sC, record(sA));
            if (mr1 > 0) {
                const int64_t k1 = RA.first_from(i + 1, pr);
                if (fa.dG)
                    block_rows(sC, G2.p, mr1, const_cast<double*>(fa.dG) + pos, s1, s1, b, b, k1 - (i + 1), P,
                               RA.suffix(i + 1, pr).second, false);
                else
                    normal_fill_cyclic(sC, fa.seed, pos, s1, b, k1 - (i + 1), P, DView(mr1, b, mr1, G2.p));
            }
            if (nc1 > 0) {
                const DView Bl = mr1 > 0 ? tl.block(ri1, ci1, mr1, nc1) : DView(0, nc1, tl.ld, tl.data);
                gemm(sC, 1.0, Op::T, Bl, Op::N, DView(mr1, b, std::max<int64_t>(mr1, 1), G2.p), 0.0,
                     DView(nc1, b, nc1, Yl.p), GWC.p, gwe);
            }
            evP = record(sC);
        }
        // ---- U-side panel QR (build_u_alpha, :58-64)
        const int pan_pc = static_cast<int>(i % Q);
        if (pc == pan_pc) gather(*cx.col, RA, i, s, T22.data, tl.ld, m_r, slabR, SlabP.p, SlabsP.p, Pan.p);
        if (me == downer) {
            hqr_panel(sA, DView(s, b, s, Pan.p), TauU.p, nullptr, 0, HQ.p, hqw);
            const size_t slot = std::find(my_steps.begin(), my_steps.end(), i) - my_steps.begin();
            copy_upper(sA, DView(b, b, b, Rm.p + slot * b * b), DView(b, b, s, Pan.p));  // beta_stage's R (:73-75)
        }
        cx.world->broadcast(Pan.p, static_cast<size_t>(s * b), downer, sA);
        cx.world->broadcast(TauU.p, static_cast<size_t>(b), downer, sA);
        const cudaEvent_t evMu = form_wy(Pan.p, s, TauU.p, Wu.p, Mu.p);
        // ---- Q_u' on T22(:, b:) (:147): Zl = W_u' B needs only W (D forms M_u meanwhile)
        wait(sA, evRest);
        {
            const int64_t c0 = pc == pan_pc ? b : 0;
            const int64_t nc = m_c - c0;
            if (nc > 0) {
                DView Zl(b, nc, b, ZlA.p);
                if (m_r > 0) {
                    pick(sA, RA, pr, i, s, Wu.p, b, WrA.p, std::max<int64_t>(m_r, 1));
                    gemmA(1.0, Op::T, DView(m_r, b, std::max<int64_t>(m_r, 1), WrA.p), Op::N, T22.block(0, c0, m_r, nc),
                          0.0, Zl);
                } else {
                    RUTV_CUDA(cudaMemsetAsync(ZlA.p, 0, static_cast<size_t>(b * nc) * 8, sA));
                }
                cx.col->allreduce_sum(ZlA.p, static_cast<size_t>(b * nc), sA);
                wait(sA, evMu);
                wait(sA, evP);  // the hoisted P read B before this update
                if (m_r > 0) {
                    pick(sA, RA, pr, i, s, Mu.p, b, MrA.p, std::max<int64_t>(m_r, 1));
                    gemmA(-1.0, Op::N, DView(m_r, b, std::max<int64_t>(m_r, 1), MrA.p), Op::N, Zl, 1.0,
                          T22.block(0, c0, m_r, nc));
                }
            }
        }
        wait(sA, evMu);
        if (hoist_next) {  // Y'_partial = P - Zl' (M_u(my rows >= i+1)' G'_loc)
            wait(sA, evP);
            if (nc1 > 0) {
                if (mr1 > 0) {
                    const int64_t k1 = RA.first_from(i + 1, pr);
                    block_rows(sA, Mh.p, mr1, Mu.p + b, s, s - b, b, b, k1 - (i + 1), P, RA.suffix(i + 1, pr).second,
                               false);
                }
                gemmA(1.0, Op::T, DView(mr1, b, std::max<int64_t>(mr1, 1), Mh.p), Op::N,
                      DView(mr1, b, std::max<int64_t>(mr1, 1), G2.p), 0.0, DView(b, b, b, Hh.p));
                gemmA(-1.0, Op::T, DView(b, nc1, b, ZlA.p), Op::N, DView(b, b, b, Hh.p), 1.0,
                      DView(nc1, b, nc1, Yl.p));
            }
            have_y = true;
        }
        if (m_c > 0 && bu) {
            pick(sA, CA, pc, i, s, Wu.p, b, WuB[par], std::max<int64_t>(mc, 1));
            pick(sA, CA, pc, i, s, Mu.p, b, MuB[par], std::max<int64_t>(mc, 1));
        }
        const cudaEvent_t evU = record(sA);

        // ======== stream B: V / finished-T and U accumulation of step i ========
        wait(sB, evV);
        if (vr + ri > 0) {
            DView X = vt.block(0, ci, vr + ri, m_c), Zx(vr + ri, b, vr + ri, ZxB.p);
            if (m_c > 0) gemmB(1.0, Op::N, X, Op::N, DView(m_c, b, std::max<int64_t>(mc, 1), WvB[par]), 0.0, Zx);
            else RUTV_CUDA(cudaMemsetAsync(ZxB.p, 0, static_cast<size_t>((vr + ri) * b) * 8, sB));
            cx.row_side->allreduce_sum(ZxB.p, static_cast<size_t>((vr + ri) * b), sB);
            if (m_c > 0) gemmB(-1.0, Op::N, Zx, Op::T, DView(m_c, b, std::max<int64_t>(mc, 1), MvB[par]), 1.0, X);
        }
        wait(sB, evU);
        if (bu && mr > 0) {
            DView X = ul.block(0, ci, mr, m_c), Zu(mr, b, mr, ZuB.p);
            if (m_c > 0) gemmB(1.0, Op::N, X, Op::N, DView(m_c, b, std::max<int64_t>(mc, 1), WuB[par]), 0.0, Zu);
            else RUTV_CUDA(cudaMemsetAsync(ZuB.p, 0, static_cast<size_t>(mr * b) * 8, sB));
            cx.row_side->allreduce_sum(ZuB.p, static_cast<size_t>(mr * b), sB);
            if (m_c > 0) gemmB(-1.0, Op::N, Zu, Op::T, DView(m_c, b, std::max<int64_t>(mc, 1), MuB[par]), 1.0, X);
        }
        evB.push_back(record(sB));
    }
    wait(sA, record(sB));  // join

    // ======== deferred beta stage (:66-82, :129-137, :150-154) ========
    const int64_t nmine = static_cast<int64_t>(std::count_if(my_steps.begin(), my_steps.end(),
                                                             [&](int64_t k) { return k < steps; }));
    auto wstep = [&](int64_t k) { return (tail_w > 0 && k == steps - 1) ? tail_w : b; };
    if (nmine > 0) {
        std::vector<SvdDesc> d(static_cast<size_t>(nmine));
        int nmax = 0;
        for (int64_t t = 0; t < nmine; ++t) {
            const int64_t k = my_steps[static_cast<size_t>(t)], w = wstep(k);
            double* f = Fac.p + t * fslot;
            d[static_cast<size_t>(t)] = SvdDesc{Rm.p + t * b * b, b, static_cast<int>(w), 0, f, f + 2 * b * b, f + b * b,
                                                SvdW.p + t * svdw, Jst.p + 4 * t};
            nmax = std::max<int>(nmax, static_cast<int>(w));
        }
        RUTV_CUDA(cudaMemcpyAsync(Desc.p, d.data(), sizeof(SvdDesc) * d.size(), cudaMemcpyHostToDevice, sA));
        svd_batch(sA, reinterpret_cast<const SvdDesc*>(Desc.p), static_cast<int>(nmine), nmax, 1e-15, 30);
    }
    // every rank learns of a ConvergenceError before anyone leaves the collectives
    std::vector<double> hs(static_cast<size_t>(std::max<int64_t>(nmine, 1)) * 4, 0.0);
    if (nmine > 0)
        RUTV_CUDA(cudaMemcpyAsync(hs.data(), Jst.p, static_cast<size_t>(nmine) * 32, cudaMemcpyDeviceToHost, sA));
    RUTV_CUDA(cudaStreamSynchronize(sA));
    double flag[2] = {0.0, 0.0};
    for (int64_t t = 0; t < nmine; ++t)
        if (hs[static_cast<size_t>(4 * t)] == RUTV_ERR_CONVERGENCE) {
            flag[0] = 1.0;
            flag[1] = std::max(flag[1], hs[static_cast<size_t>(4 * t + 1)]);
        }
    RUTV_CUDA(cudaMemcpyAsync(Gram.p, flag, 16, cudaMemcpyHostToDevice, sA));
    cx.world->allreduce_sum(Gram.p, 2, sA);
    RUTV_CUDA(cudaMemcpyAsync(flag, Gram.p, 16, cudaMemcpyDeviceToHost, sA));
    RUTV_CUDA(cudaStreamSynchronize(sA));
    if (flag[0] > 0.0) throw Error(RUTV_ERR_CONVERGENCE, "jacobi sweeps exhausted after 30 sweeps", flag[1]);
    if (steps > 0) cx.world->allgather(Fac.p, FacAll.p, static_cast<size_t>(std::max(slots, 1) * fslot), sA);
    // step k's factors: rank owner2(k, k), slot = rank of k among that owner's diagonal steps
    auto fac_of = [&](int64_t k) {
        const int r = cx.owner2(k, k);
        int64_t t = 0;
        for (int64_t j = 0; j < k; ++j) t += cx.owner2(j, j) == r;
        return FacAll.p + (static_cast<int64_t>(r) * std::max(slots, 1) + t) * fslot;
    };
    DevBuf Tmp(std::max<int64_t>({(vr + mr) * b, b * std::max<int64_t>(mc, 1), mr * b, int64_t(1)}), sA);
    for (int64_t k = 0; k < steps; ++k) {  // diagonal writes: block column k, rows >= r0 (the finished panel)
        if (k % Q != pc) continue;
        const int64_t ro = RA.suffix(k, pr).first, w = wstep(k), co = CA.loc(k);
        if (mr - ro <= 0) continue;
        const double* f = fac_of(k);
        write_rect_diag(sA, tl.block(ro, co, mr - ro, w), f + 2 * b * b, cx.owner2(k, k) == me ? w : 0);
    }
    for (int64_t k = 0; k < steps; ++k) {  // strips T(r0:r0+b, r0+b:) <- Us_k' (...)
        if (n - k * b <= b || k % P != pr) continue;
        const int64_t c1 = CA.suffix(k + 1, pc).first;
        if (c1 >= mc) continue;
        const int64_t ro = RA.loc(k);
        DView strip = tl.block(ro, c1, b, mc - c1), tv(b, mc - c1, b, Tmp.p);
        gemmA(1.0, Op::T, DView(b, b, b, const_cast<double*>(fac_of(k))), Op::N, strip, 0.0, tv);
        copy_view(sA, strip, tv);
    }
    for (int64_t k = 0; k < steps; ++k) {  // right-multiplies of block column k: [V; T(0:r0)] Vs, U Us
        if (k % Q != pc) continue;
        const int64_t w = wstep(k), co = CA.loc(k);
        const double* f = fac_of(k);
        const int64_t above = vr + RA.suffix(k, pr).first;
        if (above > 0) {
            DView X = vt.block(0, co, above, w), tv(above, w, above, Tmp.p);
            gemmA(1.0, Op::N, X, Op::N, DView(w, w, w, const_cast<double*>(f + b * b)), 0.0, tv);
            copy_view(sA, X, tv);
        }
        if (bu && mr > 0) {
            DView X = ul.block(0, co, mr, w), tv(mr, w, mr, Tmp.p);
            gemmA(1.0, Op::N, X, Op::N, DView(w, w, w, const_cast<double*>(f)), 0.0, tv);
            copy_view(sA, X, tv);
        }
    }
    if (!vt_inplace && mr * mc > 0) {
        copy_view(sA, DView(mr, mc, fa.ldt, fa.T), tl);
        if (bv && fa.V) copy_view(sA, DView(mr, mc, fa.ldv, fa.V), vt.block(0, 0, mr, mc));
    }
    if (bu && fa.U && !u_inplace && mr * mc > 0) copy_view(sA, DView(mr, mc, fa.ldu, fa.U), ul);
    RUTV_CUDA(cudaStreamSynchronize(sA));
}

// Copy the (kr, kc) blocks of a full n x n column-major matrix to / from a rank's
// local block layout (cudaMemcpy2D per block pair; any memory kinds).
void grid_copy(const Ctx& cx, int64_t n, int64_t b, double* full, int64_t ldf, double* loc, int64_t ldl,
               bool to_local, cudaStream_t st) {
    const Axis RA{n, b, cx.P}, CA{n, b, cx.Q};
    for (int64_t kc = cx.pc(); kc < CA.nblk(); kc += cx.Q)
        for (int64_t kr = cx.pr(); kr < RA.nblk(); kr += cx.P) {
            const int64_t wr = RA.width(kr), wc = CA.width(kc);
            double* f = full + kr * b + kc * b * ldf;
            double* l = loc + RA.loc(kr) + CA.loc(kc) * ldl;
            if (to_local)
                RUTV_CUDA(cudaMemcpy2DAsync(l, ldl * 8, f, ldf * 8, wr * 8, wc, cudaMemcpyDefault, st));
            else
                RUTV_CUDA(cudaMemcpy2DAsync(f, ldf * 8, l, ldl * 8, wr * 8, wc, cudaMemcpyDefault, st));
        }
}

}  // namespace dist
}  // namespace rutv

// ------------------------------------------------------------------------ C ABI
using rutv::DevBuf;
using rutv::Error;
using rutv::dist::Axis;
using rutv::dist::Ctx;

struct rutv_dist_ctx {
    Ctx cx;
};

namespace {

int dstatus(rutv_status* st, int code, const char* msg, double residual = 0.0) {
    if (st) {
        st->code = code;
        st->reserved = 0;
        st->residual = residual;
        std::snprintf(st->message, sizeof st->message, "%s", msg ? msg : "");
    }
    return code;
}

template <class F>
int drun(rutv_status* st, F&& f) {
    int rc;
    try {
        f();
        rc = dstatus(st, RUTV_OK, "");
    } catch (const Error& e) {
        rc = dstatus(st, e.code, e.what(), e.residual);
    } catch (const std::bad_alloc&) {
        rc = dstatus(st, RUTV_ERR_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        rc = dstatus(st, RUTV_ERR_INTERNAL, e.what());
    }
    rutv::pool_trim();
    return rc;
}

void check_grid(int P, int Q) {
    if (P < 1 || Q < 1) throw Error(RUTV_ERR_CONFIG, "process grid must be at least 1 x 1");
}

rutv::dist::Args args_of(const rutv_opts* o, int64_t n, const double* A, int64_t lda, const double* G, double* T,
                         int64_t ldt, double* U, int64_t ldu, double* V, int64_t ldv) {
    return rutv::dist::Args{n,   o->b, o->q, o->build_u != 0, o->build_v != 0, o->seed, o->max_steps, G, A, lda,
                            T,   U,    V,    ldt,             ldu,             ldv,     o->overlap != 0};
}

void check_opts_dist(const rutv_opts* o) {
    if (!o) throw Error(RUTV_ERR_CONFIG, "null options");
    if (o->b < 1) throw Error(RUTV_ERR_CONFIG, "block size must be >= 1, got " + std::to_string(o->b));
    if (o->q < 0) throw Error(RUTV_ERR_CONFIG, "power iteration count must be >= 0, got " + std::to_string(o->q));
}

}  // namespace

namespace rutv {

// Single-process grid run from HOST buffers (rutv_b200_factorize with
// grid_p * grid_q > 1): one host thread per rank; NCCL clique over devices
// 0 .. P*Q-1, or (grid_sim) every rank on o->device with the in-process exchange.
void factorize_grid_host(const rutv_opts* o, const double* A, int64_t n, int64_t lda, const double* G, int64_t glen,
                         double* T, int64_t ldt, double* U, int64_t ldu, double* V, int64_t ldv) {
    check_opts_dist(o);
    const int P = std::max(o->grid_p, 1), Q = std::max(o->grid_q, 1), W = P * Q;
    const bool sim = o->grid_sim != 0;
    std::vector<ncclComm_t> worlds(static_cast<size_t>(W), nullptr);
    std::vector<int> devs(static_cast<size_t>(W), o->device);
    if (!sim) {
        int ndev = 0;
        RUTV_CUDA(cudaGetDeviceCount(&ndev));
        if (ndev < W)
            throw Error(RUTV_ERR_CONFIG, "a " + std::to_string(P) + " x " + std::to_string(Q) + " grid needs " +
                                             std::to_string(W) + " GPUs, " + std::to_string(ndev) + " visible");
        for (int r = 0; r < W; ++r) devs[static_cast<size_t>(r)] = r;
        dist::pin_nccl_env();
        RUTV_NCCL(CommInitAll(worlds.data(), W, devs.data()));
    }
    dist::SimHub hub;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(W));
    auto body = [&](int r) {
        try {
            RUTV_CUDA(cudaSetDevice(devs[static_cast<size_t>(r)]));
            Ctx cx;
            cx.P = P;
            cx.Q = Q;
            cx.rank = r;
            cx.device = devs[static_cast<size_t>(r)];
            if (sim) dist::sim_groups(cx, &hub);
            else dist::split_groups(cx, worlds[static_cast<size_t>(r)]);
            const Axis RA{n, o->b, P}, CA{n, o->b, Q};
            const int64_t mr = RA.length(cx.pr()), mc = CA.length(cx.pc());
            const int64_t ld = std::max<int64_t>((2 * mr + 3) / 4 * 4, 1), ldu4 = std::max<int64_t>((mr + 3) / 4 * 4, 1);
            cudaStream_t st;
            RUTV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            struct SG {
                cudaStream_t s;
                ~SG() {
                    cudaStreamSynchronize(s);
                    cudaStreamDestroy(s);
                }
            } sg{st};
            {
                const int64_t vr = o->build_v ? mr : 0;
                DevBuf vt(std::max<int64_t>(ld, 1) * std::max<int64_t>(mc, 1), st);
                DevBuf du(o->build_u ? ldu4 * std::max<int64_t>(mc, 1) : 1, st);
                DevBuf dg(G ? std::max<int64_t>(glen, 1) : 1, st);
                if (G && glen > 0) RUTV_CUDA(cudaMemcpyAsync(dg.p, G, static_cast<size_t>(glen) * 8, cudaMemcpyHostToDevice, st));
                double* dT = vt.p + vr;
                if (mr * mc > 0) dist::grid_copy(cx, n, o->b, const_cast<double*>(A), lda, dT, ld, true, st);
                auto fa = args_of(o, n, dT, ld, G ? dg.p : nullptr, dT, ld, o->build_u ? du.p : nullptr, ldu4,
                                  o->build_v ? vt.p : nullptr, ld);
                dist::factorize_rank(cx, fa, st);
                if (mr * mc > 0) {
                    dist::grid_copy(cx, n, o->b, T, ldt, dT, ld, false, st);
                    if (o->build_u && U) dist::grid_copy(cx, n, o->b, U, ldu, du.p, ldu4, false, st);
                    if (o->build_v && V) dist::grid_copy(cx, n, o->b, V, ldv, vt.p, ld, false, st);
                }
                RUTV_CUDA(cudaStreamSynchronize(st));
            }
        } catch (...) {
            errs[static_cast<size_t>(r)] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int r = 0; r < W; ++r) th.emplace_back(body, r);
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

}  // namespace rutv

extern "C" {

int rutv_b200_grid_local_shape(int64_t n, int64_t b, int P, int Q, int rank, int64_t* rows, int64_t* cols) {
    if (n < 0 || b < 1 || P < 1 || Q < 1 || rank < 0 || rank >= P * Q) return RUTV_ERR_CONFIG;
    const Axis RA{n, b, P}, CA{n, b, Q};
    if (rows) *rows = RA.length(rank / Q);
    if (cols) *cols = CA.length(rank % Q);
    return RUTV_OK;
}

int rutv_b200_grid_copy(int device, int64_t n, int64_t b, int P, int Q, int rank, double* full, int64_t ldf,
                        double* loc, int64_t ldl, int to_local, rutv_status* st) {
    return drun(st, [&] {
        check_grid(P, Q);
        if (rank < 0 || rank >= P * Q) throw Error(RUTV_ERR_CONFIG, "rank outside the grid");
        RUTV_CUDA(cudaSetDevice(device));
        Ctx cx;
        cx.P = P;
        cx.Q = Q;
        cx.rank = rank;
        cudaStream_t s;
        RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        rutv::dist::grid_copy(cx, n, b, full, ldf, loc, ldl, to_local != 0, s);
        RUTV_CUDA(cudaStreamSynchronize(s));
        cudaStreamDestroy(s);
    });
}

int rutv_b200_nccl_unique_id(unsigned char* id, rutv_status* st) {
    return drun(st, [&] {
        static_assert(sizeof(ncclUniqueId) == RUTV_NCCL_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        RUTV_NCCL(GetUniqueId(&u));
        std::memcpy(id, &u, sizeof u);
    });
}

int rutv_b200_dist_create(const unsigned char* id, int P, int Q, int rank, int device, rutv_dist_ctx** out,
                          rutv_status* st) {
    return drun(st, [&] {
        check_grid(P, Q);
        if (!out) throw Error(RUTV_ERR_SHAPE, "null output handle");
        *out = nullptr;
        if (rank < 0 || rank >= P * Q) throw Error(RUTV_ERR_CONFIG, "rank outside the grid");
        RUTV_CUDA(cudaSetDevice(device));
        auto h = std::make_unique<rutv_dist_ctx>();
        h->cx.P = P;
        h->cx.Q = Q;
        h->cx.rank = rank;
        h->cx.device = device;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        rutv::dist::pin_nccl_env();
        ncclComm_t world = nullptr;
        RUTV_NCCL(CommInitRank(&world, P * Q, u, rank));
        rutv::dist::split_groups(h->cx, world);
        *out = h.release();
    });
}

int rutv_b200_dist_destroy(rutv_dist_ctx* h, rutv_status* st) {
    return drun(st, [&] {
        if (h) {
            RUTV_CUDA(cudaSetDevice(h->cx.device));
            delete h;
        }
    });
}

int rutv_b200_factorize_dist(rutv_dist_ctx* h, const rutv_opts* o, int64_t n, const double* A_loc, int64_t lda,
                             const double* G, int64_t g_len, double* T_loc, int64_t ldt, double* U_loc, int64_t ldu,
                             double* V_loc, int64_t ldv, rutv_status* st) {
    return drun(st, [&] {
        if (!h) throw Error(RUTV_ERR_CONFIG, "null distributed context");
        check_opts_dist(o);
        RUTV_CUDA(cudaSetDevice(h->cx.device));
        const Axis RA{n, o->b, h->cx.P};
        const int64_t mr = RA.length(h->cx.pr());
        if (lda < std::max<int64_t>(mr, 1) || ldt < std::max<int64_t>(mr, 1))
            throw Error(RUTV_ERR_SHAPE, "leading dimension smaller than the local row count");
        if (o->build_u && (!U_loc || ldu < std::max<int64_t>(mr, 1))) throw Error(RUTV_ERR_SHAPE, "U buffer");
        if (o->build_v && (!V_loc || ldv < std::max<int64_t>(mr, 1))) throw Error(RUTV_ERR_SHAPE, "V buffer");
        if (G && g_len < rutv_b200_stream_length(n, n, o->b) && o->max_steps < 0)
            throw Error(RUTV_ERR_SHAPE, "explicit G shorter than the stream the factorization draws");
        cudaStream_t s = reinterpret_cast<cudaStream_t>(o->stream);
        bool own = false;
        if (!s) {
            RUTV_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            own = true;
        }
        struct SG {
            cudaStream_t s;
            bool own;
            ~SG() {
                if (own) {
                    cudaStreamSynchronize(s);
                    cudaStreamDestroy(s);
                }
            }
        } sg{s, own};
        rutv::dist::factorize_rank(h->cx, args_of(o, n, A_loc, lda, G, T_loc, ldt, U_loc, ldu, V_loc, ldv), s);
        RUTV_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
