// usp_api.cu -- the C-ABI of include/usp.h: plan, workspace, setup and the
// iteration driver.  All arithmetic of the method runs in the kernels
// (kernels*.cu); this file only sequences launches and collectives,
// validates, and moves bytes.
//
// Slab decomposition: a 3-D grid is split into P z-slabs.
// The x pass (K_A) and the y passes (K_B, K_D) are local to a slab; the z
// pass (K_C) needs whole z-lines, so K_B stores its output in the "send
// layout" [q][z_loc][y_loc][x] (block q = the y-range of slab q), an
// all-to-all turns it into y-slabs [z][y_loc][x] on which K_C runs, and the
// reverse all-to-all brings the blocks back for K_D, which reads them through
// a 5-D tensor map.  The residual is one all-gather of P doubles summed in
// rank order, so every rank takes the same stop decision.
//   * NCCL mode (desc.nccl_comm): one GPU per rank, the all-to-alls are
//     grouped ncclSend/ncclRecv over NVLink.
//   * virtual mode (desc.virtual_ranks = P): all P slabs on one GPU, the
//     all-to-alls are device copies -- the same kernels, layouts and index
//     arithmetic, so the decomposition is testable on a single GPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nccl_device.h>   // ncclGetPeerPointer (device side of the NCCL 2.28 window API)
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <complex>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "usp.h"
#include "usp_internal.h"

using namespace usp;

namespace {

thread_local std::string g_err;

usp_status fail(usp_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(USP_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                             \
    } while (0)

// ------------------------------------------------------------ NCCL shim --
// libnccl.so.2 is opened at run time (the torch wheel's copy when torch has
// loaded it, else the path in USP_NCCL_LIB), so single-GPU use of libusp
// needs no NCCL at all.  nccl.h supplies the types only.
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommCount)(const ncclComm_t, int *);
    ncclResult_t (*CommUserRank)(const ncclComm_t, int *);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
    // NCCL >= 2.28 (optional): symmetric memory and windows
    bool win = false;
    ncclResult_t (*MemAlloc)(void **, size_t);
    ncclResult_t (*MemFree)(void *);
    ncclResult_t (*CommWindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int);
    ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t);
    bool devcomm = false;   // device communicators (LSA barrier)
    ncclResult_t (*DevCommCreate)(ncclComm_t, const ncclDevCommRequirements_t *, ncclDevComm_t *);
    ncclResult_t (*DevCommDestroy)(ncclComm_t, const ncclDevComm_t *);
};

Nccl &nccl_api() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        const char *path = std::getenv("USP_NCCL_LIB");
        if (path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
        n.why = "libnccl.so.2 not found (set USP_NCCL_LIB)";
        return n;
    }
    bool all = true;
    auto sym = [&](const char *name) {
        void *f = dlsym(h, name);
        if (!f) all = false;
        return f;
    };
    n.GetUniqueId = (decltype(n.GetUniqueId))sym("ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))sym("ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))sym("ncclCommDestroy");
    n.CommCount = (decltype(n.CommCount))sym("ncclCommCount");
    n.CommUserRank = (decltype(n.CommUserRank))sym("ncclCommUserRank");
    n.GroupStart = (decltype(n.GroupStart))sym("ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))sym("ncclGroupEnd");
    n.Send = (decltype(n.Send))sym("ncclSend");
    n.Recv = (decltype(n.Recv))sym("ncclRecv");
    n.AllGather = (decltype(n.AllGather))sym("ncclAllGather");
    n.AllReduce = (decltype(n.AllReduce))sym("ncclAllReduce");
    n.GetErrorString = (decltype(n.GetErrorString))sym("ncclGetErrorString");
    n.MemAlloc = (decltype(n.MemAlloc))dlsym(h, "ncclMemAlloc");
    n.MemFree = (decltype(n.MemFree))dlsym(h, "ncclMemFree");
    n.CommWindowRegister = (decltype(n.CommWindowRegister))dlsym(h, "ncclCommWindowRegister");
    n.CommWindowDeregister = (decltype(n.CommWindowDeregister))dlsym(h, "ncclCommWindowDeregister");
    n.win = n.MemAlloc && n.MemFree && n.CommWindowRegister && n.CommWindowDeregister;
    n.DevCommCreate = (decltype(n.DevCommCreate))dlsym(h, "ncclDevCommCreate");
    n.DevCommDestroy = (decltype(n.DevCommDestroy))dlsym(h, "ncclDevCommDestroy");
    n.devcomm = n.DevCommCreate && n.DevCommDestroy;
    n.ok = all;
    if (!all) n.why = "libnccl.so.2 lacks an entry point";
    return n;
}

#define NC(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            return fail(USP_ERR_NCCL, "%s failed: %s (%s:%d)", #call, nccl_api().GetErrorString(r_), __FILE__, \
                        __LINE__);                                                                 \
    } while (0)

// usp_shared_alloc's allocations: base -> (bytes, from ncclMemAlloc)
struct SharedAlloc {
    size_t bytes;
    bool nccl;
};
std::mutex g_shared_mu;
std::map<char *, SharedAlloc> g_shared;

// the ncclMemAlloc allocation holding [p, p + bytes), if any
bool shared_range(const void *p, size_t bytes, char **base, size_t *size) {
    std::lock_guard<std::mutex> g(g_shared_mu);
    auto it = g_shared.upper_bound((char *)p);
    if (it == g_shared.begin()) return false;
    --it;
    if (!it->second.nccl || (char *)p + bytes > it->first + it->second.bytes) return false;
    *base = it->first;
    *size = it->second.bytes;
    return true;
}

// peer q's address of the window's byte 0, for q < P (the window spans one
// LSA team: every rank of a single-node communicator)
__global__ void k_win_peers(ncclWindow_t w, int P, void **out) {
    const int q = threadIdx.x;
    if (q < P) out[q] = ncclGetPeerPointer(w, 0, q);
}
// cross-rank barrier of the fused transposes over the LSA team (NVLink peers):
// one CTA; acq_rel at system scope orders this rank's earlier peer stores
// (performed by the preceding kernels, which end with a system fence) before
// the peers' later reads, and theirs before ours
__global__ void k_lsa_barrier(ncclDevComm dc) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// window self-test on a one-rank communicator: write through the window's
// mapping, read through the plain pointer
__global__ void k_win_write(float2 *dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = make_float2((float)i, -(float)(i & 1023));
    __threadfence_system();
}
__global__ void k_win_check(const float2 *src, long long n, unsigned *bad) {
    unsigned b = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float2 v = src[i];
        b += (v.x != (float)i || v.y != -(float)(i & 1023)) ? 1u : 0u;
    }
    if (b) atomicAdd(bad, b);
}

enum KClass { KC_XPASS = 0, KC_YFWD, KC_ZMUL, KC_YINV, KC_YMUL2D, KC_SOLVE1D, KC_POTENTIAL,
              KC_FARTHEST, KC_SETSTATE, KC_XSETUP, KC_A2A, KC_FINISH, KC_ALLGATHER, KC_BARRIER, KC_XOP,
              KC_KUPD, KC_SOLVE2D, KC_SADD, KC_PLANE, KC_N };
const char *kc_names[KC_N] = {"xpass", "y_fwd", "z_fwd_mul_inv", "y_inv", "y_fwd_mul_inv",
                              "solve1d", "potential", "farthest", "set_state", "xpass_setup",
                              "all_to_all", "finish", "allgather", "rank_barrier", "krylov_xop",
                              "krylov_update", "solve2d", "sparse_source_add", "plane_dab"};

struct Timed {
    int cls;
    cudaEvent_t a, b;
};

}  // namespace

constexpr size_t kHostMapBytes = 1024 * 1024;   // mapped pinned scratch for small read-backs

struct usp_plan_s {
    usp_plan_desc d{};
    int ndim = 0;
    long long nx = 1, ny = 1, nz = 1, nvox = 0;   // global grid
    cudaStream_t stream = nullptr;
    int nsm = 148;
    // slab decomposition
    int P = 1, rank = 0;          // slabs, this rank
    bool virt = false;            // all P slabs on this GPU (device-copy transposes)
    ncclComm_t comm = nullptr;    // NCCL mode
    long long nzs = 1;            // z planes per slab (nz / P)
    long long nzh = 1;            // z planes this plan holds (nzs, or nz in virtual / 1-GPU mode)
    long long nyl = 1;            // y rows per y block (ny / P)
    long long nloc = 0;           // voxels this plan holds
    // real path (diffusion with float32 data, kernels_real.cu): x, Delta, B
    // are float32 and `work` holds the half spectrum in rows of rp complex
    bool real = false;
    long long rp = 1;             // row pitch of `work` in complex64 (nx, or nx/2 + 16 on the real path)
    float2 *twr = nullptr;        // real path: W_nx^k, k < nx/2
    // workspace
    char *ws = nullptr;
    size_t ws_bytes = 0;
    float2 *x = nullptr, *delta = nullptr, *B = nullptr, *work = nullptr;
    float2 *sendb = nullptr, *recvb = nullptr;   // P > 1
    // separate transposes, pipelined over x-chunks: chunk c of
    // width chunk_w owns a contiguous region of the send / receive buffers
    // ([c][r][q][z_loc][y_loc][chunk_w]); K_B(c) -> all-to-all(c) -> K_C(c) ->
    // all-to-all back(c) -> K_D(c), the all-to-alls on xstream overlapping the
    // other chunks' passes
    int nchunk = 1;
    long long chunk_w = 0;
    std::vector<CUtensorMap> smap_zc, smap_kdc;
    cudaStream_t xstream = nullptr;
    std::vector<cudaEvent_t> ev_b, ev_x, ev_c, ev_y;
    // transposes fused into the K_B / K_C stores (peer memory; desc.separate_transposes -> NCCL all-to-all)
    bool fused = false;
    float2 *peer_recv[kMaxPeers] = {}, *peer_send[kMaxPeers] = {};
    std::vector<void *> ipc_bases;   // peer allocations mapped with cudaIpcOpenMemHandle
    // NCCL window over the workspace (ncclMemAlloc'd by usp_shared_alloc): the
    // peers' send / receive buffers through ncclGetPeerPointer (NEXT-1)
    ncclWindow_t win = nullptr;
    int transport = USP_TRANSPORT_NONE;
    // device communicator with one LSA barrier: the cross-rank barrier after
    // K_B / K_C (else an ncclAllReduce of one double)
    ncclDevComm_t devcomm{};
    bool lsa = false;
    // BiCGSTAB (caller-owned Krylov workspace: rhat, p, v, s, t)
    float2 *k_rh = nullptr, *k_p = nullptr, *k_v = nullptr, *k_s = nullptr, *k_t = nullptr;
    KState *ks = nullptr;
    // GMRES(m) (caller-owned workspace: b, U_0 .. U_m; plan-owned partials)
    int gm_m = 0;
    float2 *gm_b = nullptr;
    std::vector<float2 *> gm_U;
    double *gm_part = nullptr;
    int gm_grid = 0;
    // antisymmetrised system (Eq. 9-10; desc.antisymmetric): two-component x,
    // Delta, work (component-major) and v = (w - sigma)/c in place of B
    bool anti = false;
    // first-order tensor diffusion (§3.2 Eqs. 16-18; desc.tensor_diffusion): d + 1
    // component fields x, Delta, work; V and D^-1 per voxel (float32)
    bool tdiff = false;
    int ncomp = 1;                 // components of the fields (1; 2 anti; d + 1 tdiff)
    float *td_vu = nullptr, *td_vf = nullptr, *td_dinv = nullptr, *td_red = nullptr;
    int td_pipe = 0;   // lines per unit of the fused x pass (k_tdiff_pipe), 0: k_xfft + k_tdiff_upd
    TDParams td{};
    // persistent 2-D solve (kernels_small.cu; desc.launch_per_pass disables)
    bool solve2d = false;
    // plane-chained pass (kernels_plane.cu, NEXT-4; desc.plane_chain enables): an
    // iteration is K_C + one persistent K_D -> K_A -> K_B kernel; unit counter,
    // per-plane done counters, per-unit residual partials
    bool plane = false;
    unsigned long long *pl_ctr = nullptr;
    unsigned *pl_done = nullptr;
    double *pl_part = nullptr;
    // x-form passes while r >= r_sw (reading R-30; desc.delta_form disables,
    // desc.r_switch sets r_sw): s = S / c kept in its own field
    bool xform_cap = false, xform = false, probe_needed = false;
    bool force_finish = false;   // desc.test_hooks & USP_HOOK_RANK_FINISH (see rank_finish)
    // sparse source (R-31; desc.dense_source disables): <= kSparseMaxLines x-lines carry
    // the source; their x-transforms live in the s field (list, then lines)
    unsigned char *s_flag = nullptr;
    unsigned *s_ctr = nullptr;
    bool s_sparse = false;
    int s_count = 0;
    // expect_x: the host's view of the device-side form (x-form or not),
    // refreshed at call start and batch boundaries; it picks the x-pass
    // instance (lean 3-slot pass for sparse-source x-form passes, general
    // body, Delta-form body) and whether the sparse source lines are added
    // after a pass
    bool expect_x = false;
    // mapped pinned scratch for small read-backs (see readback) and the
    // device view of st_host
    void *hmap = nullptr, *hmap_dev = nullptr, *st_host_dev = nullptr;
    // asynchronous input staging (usp_stage_inputs): caller-owned area, copy
    // streams, "copies done" event
    char *stg = nullptr;
    size_t stg_bytes = 0;
    cudaStream_t cstream = nullptr, dstream = nullptr;   // H2D staging, D2H results
    // per slot "consumed by the plan stream" events: the copy stream refills a
    // slot only after them; medium_taken = set_potential(STAGED) ran, its
    // source not yet consumed (usp_stage_inputs refuses meanwhile)
    cudaEvent_t ev_staged = nullptr, ev_med_used = nullptr, ev_src_used = nullptr, ev_snap = nullptr,
                ev_out = nullptr;
    bool staged = false, med_used_rec = false, src_used_rec = false, medium_taken = false, out_pending = false;
    bool stg_result = false;   // the staging area has the read-back slot
    double r_sw = 1e-2;
    // after a converged stop of usp_iterate the final iterate's own residual
    // is not computed (reading R-5): the history then holds r_0 .. r_{k-1}
    bool hist_conv = false;
    float2 *s = nullptr;
    unsigned *bar = nullptr;   // [0] count, [1] generation
    // plan-owned small device memory
    IterState *st = nullptr;
    double *partials = nullptr;
    int partials_cap = 0;
    double *hist = nullptr;
    int hist_cap = 65536;
    float2 *tw[3] = {nullptr, nullptr, nullptr};
    unsigned int *red_u = nullptr;  // [0] max|V| bits, [1] non-accretive, [2] non-finite
    double *far_d = nullptr;
    long long *far_i = nullptr;
    int far_cap = 0;
    double *coll = nullptr;         // collective scratch: [0] local x-pass total, [8..15]
                                    // all-gathered totals, [16..] IPC records, [64..] / [128..] host gathers
    IterState *st_host = nullptr;   // pinned mirror
    // split
    usp_c128 sigma{}, c{}, centre{};
    double radius = 0.0, vmax = 0.0;
    bool have_potential = false, have_source = false;
    // launch configuration: the TMA-pipelined x pass (one CTA per SM), the
    // TMA-prefetched strided passes (kernels_stile.cu, lines of 64..2048;
    // shorter lines take the register-staged k_strided)
    int gridp_x = 0;
    int grid_y = 0, grid_z = 0;   // k_strided (N = 16, 32)
    bool stile_y = false, stile_z = false;
    int grids_y = 0, grids_z = 0;
    CUtensorMap smap_y{}, smap_z{}, smap_kd{};
    // z-pair chain buffer of the z pass (usp_internal.h; desc.flat_work
    // disables): work2 (one more field of workspace), smap_z on it, smap_yp =
    // K_D's map of its [nz/2][ny][2 nx] view
    bool wpair = false;
    float2 *work2 = nullptr;
    CUtensorMap smap_yp{};
    // profiling
    bool prof = false;
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[KC_N] = {0};
    long long prof_n[KC_N] = {0};
    long long launches = 0;
};

namespace {

bool multi_rank(const usp_plan_s *p) { return p->P > 1 && !p->virt; }

cudaEvent_t get_event(usp_plan_s *p) {
    if (!p->ev_pool.empty()) {
        cudaEvent_t e = p->ev_pool.back();
        p->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// NVTX range over a host-side scope (an ABI call, a launch): a timeline tool
// (nsys, ncu --nvtx) shows which call / kernel class issued what; without a
// tool attached a push/pop is a no-op call.
struct Range {
    explicit Range(const char *name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};

struct Tick {   // brackets one launch with events when profiling, and with an NVTX range
    usp_plan_s *p;
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    Tick(usp_plan_s *pl, int c, bool count = true, cudaStream_t st = nullptr) : p(pl), cls(c), s(st ? st : pl->stream) {
        nvtxRangePushA(kc_names[c]);
        if (count) ++p->launches;
        if (p->prof) {
            a = get_event(p);
            cudaEventRecord(a, s);
        }
    }
    ~Tick() {
        nvtxRangePop();
        if (p->prof) {
            cudaEvent_t b = get_event(p);
            cudaEventRecord(b, s);
            p->timed.push_back({cls, a, b});
        }
    }
};

void drain_timing(usp_plan_s *p) {
    if (p->timed.empty()) return;
    cudaStreamSynchronize(p->stream);
    if (p->xstream) cudaStreamSynchronize(p->xstream);
    for (auto &t : p->timed) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.a, t.b);
        p->prof_ms[t.cls] += ms;
        p->prof_n[t.cls] += 1;
        p->ev_pool.push_back(t.a);
        p->ev_pool.push_back(t.b);
    }
    p->timed.clear();
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

int log2ll(long long n) {
    int l = 0;
    while ((1LL << l) < n) ++l;
    return l;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// Tensor map over a complex64 field viewed with 8-byte elements.
bool make_map(CUtensorMap *m, void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides_bytes,
              const cuuint32_t *box) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUtensorMapL2promotion promo = (box[0] * 8 >= 128) ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                              : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, base, dims, strides_bytes, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

std::vector<float2> twiddle_table(int n) {
    // tw[k2*N1 + j] = W_n^(j*k2) = exp(-2 pi i j k2 / n), computed in double
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    const int n1 = 1 << (lg / 2), n2 = n / n1;
    std::vector<float2> t((size_t)n);
    for (int k2 = 0; k2 < n2; ++k2)
        for (int j = 0; j < n1; ++j) {
            const long long e = ((long long)j * k2) % n;
            const double a = -2.0 * M_PI * (double)e / (double)n;
            double cr = std::cos(a), ci = std::sin(a);
            if (4 * e == n) { cr = 0.0; ci = -1.0; }
            if (2 * e == n) { cr = -1.0; ci = 0.0; }
            if (4 * e == 3 * n) { cr = 0.0; ci = 1.0; }
            if (e == 0) { cr = 1.0; ci = 0.0; }
            t[(size_t)k2 * n1 + j] = make_float2((float)cr, (float)ci);
        }
    return t;
}

int occ_grid(usp_plan_s *p, long long units, int per_sm) {
    long long g = (long long)p->nsm * per_sm;
    return (int)std::max(1LL, std::min(units, g));
}

// ------------------------------------------------------- collectives --
// Gather `n` host doubles from every rank (rank order) into out[P*n].
usp_status readback(usp_plan_s *p, void *host, const void *dev, size_t bytes);

usp_status gather_host(usp_plan_s *p, const double *mine, int n, std::vector<double> &out) {
    out.assign((size_t)p->P * n, 0.0);
    if (!multi_rank(p)) {
        std::copy(mine, mine + n, out.begin());
        return USP_OK;
    }
    if (n > 64 || (size_t)p->P * n > 1920) return fail(USP_ERR_ARG, "gather of %d doubles x %d ranks too large", n, p->P);
    double *snd = p->coll + 64, *rcv = p->coll + 128;
    CU(launch_put_bytes(snd, mine, sizeof(double) * n, p->stream));
    NC(nccl_api().AllGather(snd, rcv, (size_t)n, ncclDouble, p->comm, p->stream));
    return readback(p, out.data(), rcv, sizeof(double) * n * p->P);
}

// ---------------------------------------------------------------- MEC --
struct P2 { double x, y; };

bool in_circle(P2 q, P2 c, double r) {
    const double sc = std::fabs(c.x) + std::fabs(c.y) + r + 1e-300;
    return std::hypot(q.x - c.x, q.y - c.y) <= r + 1e-13 * sc;
}

void circ2(P2 a, P2 b, P2 &c, double &r) {
    c = {0.5 * (a.x + b.x), 0.5 * (a.y + b.y)};
    r = 0.5 * std::hypot(a.x - b.x, a.y - b.y);
}

void circ3(P2 a, P2 b, P2 q, P2 &c, double &r) {
    const double bx = b.x - a.x, by = b.y - a.y, cx = q.x - a.x, cy = q.y - a.y;
    const double d = 2.0 * (bx * cy - by * cx);
    const double sc = (std::fabs(bx) + std::fabs(by)) * (std::fabs(cx) + std::fabs(cy));
    if (d == 0.0 || std::fabs(d) <= 1e-14 * sc) {   // collinear: farthest pair's diameter
        const double ab = std::hypot(bx, by), aq = std::hypot(cx, cy), bq = std::hypot(q.x - b.x, q.y - b.y);
        if (ab >= aq && ab >= bq) circ2(a, b, c, r);
        else if (aq >= bq) circ2(a, q, c, r);
        else circ2(b, q, c, r);
        return;
    }
    const double b2 = bx * bx + by * by, c2 = cx * cx + cy * cy;
    const double ux = (cy * b2 - by * c2) / d, uy = (bx * c2 - cx * b2) / d;
    c = {a.x + ux, a.y + uy};
    r = std::hypot(ux, uy);
}

// Smallest circle of a small support set (incremental construction with
// two / three boundary points; exact for the handful of support points the
// device-side farthest-point loop collects).
void mec_small(const std::vector<P2> &pts, P2 &c, double &r) {
    c = pts[0];
    r = 0.0;
    for (size_t i = 1; i < pts.size(); ++i) {
        if (in_circle(pts[i], c, r)) continue;
        c = pts[i];
        r = 0.0;
        for (size_t j = 0; j < i; ++j) {
            if (in_circle(pts[j], c, r)) continue;
            circ2(pts[i], pts[j], c, r);
            for (size_t k = 0; k < j; ++k) {
                if (in_circle(pts[k], c, r)) continue;
                circ3(pts[i], pts[j], pts[k], c, r);
            }
        }
    }
}

// Small device -> host read-backs through mapped pinned memory, copied by
// an SM kernel on the plan stream: they never wait behind bulk transfers on
// the copy engines (usp_stage_inputs / usp_get_field_async).
usp_status readback(usp_plan_s *p, void *host, const void *dev, size_t bytes) {
    if (bytes > kHostMapBytes) return fail(USP_ERR_ARG, "read-back of %zu bytes exceeds the mapped scratch", bytes);
    CU(launch_copy_bytes(p->hmap_dev, dev, bytes, bytes > 65536 ? 64 : 4, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    std::memcpy(host, p->hmap, bytes);
    return USP_OK;
}

usp_status read_point(usp_plan_s *p, const void *medium_dev, long long idx, P2 &out) {
    if (p->d.dtype == USP_R32) {
        float v = 0.f;
        usp_status s = readback(p, &v, (const float *)medium_dev + idx, sizeof(float));
        if (s) return s;
        out = {v, 0.0};
    } else {
        float2 v{};
        usp_status s = readback(p, &v, (const float2 *)medium_dev + idx, sizeof(float2));
        if (s) return s;
        out = {v.x, v.y};
    }
    return USP_OK;
}

// Smallest enclosing circle of all medium values: grow a
// support set with the farthest point from the current circle (one device
// pass each; across ranks the farthest of the ranks' farthest points, ties
// to the lowest rank) until every value is inside.  The result is the MEC of
// a subset that encloses all points, i.e. the MEC of the full set, and it is
// identical on every rank.
usp_status device_mec(usp_plan_s *p, const void *medium_dev, P2 &centre, double &radius) {
    std::vector<P2> sup;
    P2 q;
    usp_status s = read_point(p, medium_dev, 0, q);
    if (s) return s;
    std::vector<double> g;
    {
        const double mine[3] = {0.0, q.x, q.y};
        if ((s = gather_host(p, mine, 3, g))) return s;
        q = {g[1], g[2]};   // rank 0's first value
    }
    sup.push_back(q);
    centre = q;
    radius = 0.0;
    const int grid = farthest_grid(std::min(p->far_cap, occ_grid(p, (p->nloc + 255) / 256, 8)));
    std::vector<double> bd(grid);
    std::vector<long long> bi(grid);
    for (int it = 0; it < 200; ++it) {
        FarParams fp{medium_dev, p->d.dtype == USP_R32, p->nloc, centre.x, centre.y, p->far_d, p->far_i};
        {
            Tick t(p, KC_FARTHEST);
            CU(launch_farthest(fp, grid, p->stream));
        }
        if ((s = readback(p, bd.data(), p->far_d, sizeof(double) * grid))) return s;
        if ((s = readback(p, bi.data(), p->far_i, sizeof(long long) * grid))) return s;
        int b = 0;
        for (int i = 1; i < grid; ++i)
            if (bd[i] > bd[b] || (bd[i] == bd[b] && bi[i] < bi[b])) b = i;
        s = read_point(p, medium_dev, bi[b], q);
        if (s) return s;
        {
            const double mine[3] = {bd[b], q.x, q.y};
            if ((s = gather_host(p, mine, 3, g))) return s;
            int best = 0;
            for (int r = 1; r < p->P && multi_rank(p); ++r)
                if (g[3 * r] > g[3 * best]) best = r;
            q = {g[3 * best + 1], g[3 * best + 2]};
        }
        if (in_circle(q, centre, radius)) return USP_OK;
        sup.push_back(q);
        mec_small(sup, centre, radius);
    }
    return fail(USP_ERR_CUDA, "smallest-circle search did not converge");
}

// Copy a caller's input into the workspace.  Device inputs are copied by an
// SM kernel (not a copy engine, so the plan stream never queues behind bulk
// staging transfers); a pointer the device cannot dereference is refused
// here instead of faulting in the kernel.
usp_status stage(usp_plan_s *p, void *dst, const void *src, size_t bytes, usp_where where) {
    if (where == USP_HOST) {
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, p->stream));
        return USP_OK;
    }
    if (where != USP_DEVICE) return fail(USP_ERR_ARG, "bad where (%d)", (int)where);
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, src) != cudaSuccess) {
        cudaGetLastError();
        return fail(USP_ERR_ARG, "input pointer is not device memory (where = USP_DEVICE)");
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged &&
        !(at.type == cudaMemoryTypeHost && at.devicePointer))
        return fail(USP_ERR_ARG, "input pointer is not device memory (where = USP_DEVICE)");
    const void *dsrc = at.type == cudaMemoryTypeHost ? at.devicePointer : src;   // mapped pinned host memory
    CU(launch_copy_bytes(dst, dsrc, bytes, 4 * p->nsm, p->stream));
    return USP_OK;
}

// Write the device iteration state from the host without a copy engine (the
// state travels as a kernel argument).
usp_status put_state(usp_plan_s *p, const IterState &h) {
    CU(launch_put_state(p->st, h, p->stream));
    return USP_OK;
}

size_t elem_bytes(const usp_plan_s *p) { return p->d.dtype == USP_R32 ? 4 : 8; }

MulParams mul_params(const usp_plan_s *p) {
    MulParams mp{};
    const double cr = p->c.re / (double)p->nvox, ci = p->c.im / (double)p->nvox;   // 1/N_vox of the global F^-1
    mp.cn = make_float2((float)cr, (float)ci);
    mp.sc = make_float2((float)(p->sigma.re + p->c.re), (float)(p->sigma.im + p->c.im));
    mp.D = (float)p->d.D;
    mp.sqrtD = (float)std::sqrt(p->d.D);
    mp.kx = (float)(2.0 * M_PI / ((double)p->nx * p->d.h[0]));
    mp.ky = (float)(2.0 * M_PI / ((double)p->ny * p->d.h[1]));
    mp.kz = (float)(2.0 * M_PI / ((double)p->nz * p->d.h[2]));
    mp.nx = (int)p->nx;
    mp.ny = (int)p->ny;
    mp.nz = (int)p->nz;
    mp.rowc = (int)p->rp;
    return mp;
}

// The x pass's residual goes through the all-gather + k_finish path: with
// P > 1 ranks, or (desc.test_hooks & USP_HOOK_RANK_FINISH) on a one-rank
// communicator, so the rank-ordered finish is exercised on one GPU.
bool rank_finish(const usp_plan_s *p) { return multi_rank(p) || (p->comm && p->force_finish); }

Red red_params(usp_plan_s *p) {
    Red r{p->partials, p->hist, p->hist_cap, nullptr};
    if (rank_finish(p)) r.local_sum = p->coll;
    return r;
}

XParams x_params(usp_plan_s *p) {
    XParams xp{};
    xp.work = p->work;
    xp.delta = p->delta;
    xp.x = p->x;
    xp.B = p->B;
    xp.tw = p->tw[0];
    xp.twr = p->twr;
    xp.nlines = p->ny * p->nzh;
    xp.src_real = p->d.dtype == USP_R32;
    const double m = p->c.re * p->c.re + p->c.im * p->c.im;
    xp.inv_c = make_float2((float)(p->c.re / m), (float)(-p->c.im / m));
    xp.st = p->st;
    xp.red = red_params(p);
    xp.s = p->xform ? p->s : nullptr;
    xp.s_sparse = p->s_sparse ? 1 : 0;
    return xp;
}

// x pass; with P ranks the CTA total is all-gathered and k_finish sums the
// ranks' totals in rank order (X_SRC_FWD reduces nothing).
usp_status run_xpass(usp_plan_s *p, XMode mode, const XParams &xp) {
    {
        Tick t(p, mode == X_ITER ? KC_XPASS : KC_XSETUP);
        if (p->real) CU(launch_xpass_real((int)p->nx, mode, xp, p->gridp_x, p->stream));
        else
            CU(launch_xpass_pipe((int)p->nx, mode, xp, p->gridp_x, p->stream,
                                 mode == X_ITER && p->s_sparse && p->expect_x, p->xform && p->expect_x));
    }
    if (mode != X_SRC_FWD && rank_finish(p)) {
        {
            Tick t(p, KC_ALLGATHER, false);
            NC(nccl_api().AllGather(p->coll, p->coll + 8, 1, ncclDouble, p->comm, p->stream));
        }
        Tick t(p, KC_FINISH);
        CU(launch_finish(p->st, p->coll + 8, p->P, mode == X_SRC_EPI, red_params(p), p->stream));
    }
    return USP_OK;
}

constexpr int kSparseMaxLines = 64;

// sparse source: after an x pass of the iteration, add the x-transformed
// source lines if that pass formed u = B x (k_sparse_add checks st->add_s)
usp_status sparse_add(usp_plan_s *p) {
    // (once the host has seen the Delta-form, no x-form pass can follow in this call)
    if (!p->s_sparse || !p->expect_x) return USP_OK;
    SAddParams sa{};
    sa.work = p->work;
    sa.list = reinterpret_cast<const int *>(p->s);
    sa.comp = p->s + 256;   // list: kSparseMaxLines ints in the first 2 KiB
    sa.count = p->s_count;
    sa.n = (int)p->nx;
    sa.st = p->st;
    Tick t(p, KC_SADD);
    CU(launch_sparse_add(sa, p->stream));
    return USP_OK;
}

SParams sparams(usp_plan_s *p, float2 *data, float2 *dst, const float2 *tw, long long stride, long long ncols,
                long long nouter, long long ostride, int line_axis, int check_state, int map_rank);
usp_status run_strided(usp_plan_s *p, int cls, int n, SMode mode, const SParams &sp, const CUtensorMap &map,
                       bool use_stile, int grid_short, const CUtensorMap *smap = nullptr);

// plane-chained schedule: K_C over the volume (z forward, g(p), z inverse),
// then the persistent K_D -> K_A -> K_B kernel (kernels_plane.cu)
usp_status plane_iteration(usp_plan_s *p) {
    SParams zm = sparams(p, p->work, p->work, p->tw[2], p->rp * p->ny, p->rp * p->ny, 1, 0, 2, 1, 2);
    usp_status s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zm, p->smap_z, p->stile_z, p->grid_z);
    if (s) return s;
    PParams pp{};
    pp.work = p->work;
    pp.x = p->x;
    pp.delta = p->delta;
    pp.B = p->B;
    pp.s = p->xform ? p->s : nullptr;
    pp.tw = p->tw[0];
    pp.nz = p->nz;
    pp.s_sparse = p->s_sparse ? 1 : 0;
    pp.s_list = reinterpret_cast<const int *>(p->s);
    pp.s_comp = p->s ? p->s + 256 : nullptr;
    pp.s_count = p->s_count;
    pp.ctr = p->pl_ctr;
    pp.d_done = p->pl_done;
    pp.a_done = p->pl_done + p->nz;
    pp.upart = p->pl_part;
    // y role : x role CTAs (USP_PLANE_Y64 / 64 of the SMs run the y role;
    // a build-time constant, tools/gpu/kab.py compares builds)
#ifndef USP_PLANE_Y64
#define USP_PLANE_Y64 27
#endif
    pp.ny_ctas = (p->nsm * USP_PLANE_Y64 + 32) / 64;
    pp.st = p->st;
    pp.red = red_params(p);
    Tick t(p, KC_PLANE);
    CU(launch_plane(p->smap_y, pp, p->nsm, p->stream, p->s_sparse && p->expect_x, p->xform && p->expect_x));
    return USP_OK;
}

usp_status run_strided(usp_plan_s *p, int cls, int n, SMode mode, const SParams &sp, const CUtensorMap &map,
                       bool use_stile, int grid_short, const CUtensorMap *smap) {
    Tick t(p, cls);
    if (use_stile) {
        // half-tile tensor-map stores (the upper half of each tile through the
        // exchange buffer) where a map describes the destination (the load map of
        // an in-place pass, or smap), in the z pass and the y-inverse pass: K_C
        // 4.59 -> 4.48 ms, K_D 2.90 -> 2.70 ms at 1024^3; the y-forward pass
        // measured slower with them (2.69 -> 2.94 ms)
        SParams q = sp;
        q.tma_store = (mode == S_FWD_MUL_INV || mode == S_INV) && (sp.dst == sp.data || smap) &&
                      (sp.map_rank == 2 || sp.map_rank == 3) && !sp.peer_mode && !sp.send_layout;
        CU(launch_stile(n, mode, map, smap ? *smap : map, q, cls == KC_ZMUL ? p->grids_z : p->grids_y, p->stream));
        return USP_OK;
    }
    // register-staged passes for the short lines (N = 16, 32) the TMA tiles do not take
    CU(launch_strided(n, mode, sp, grid_short, p->stream));
    return USP_OK;
}

SParams sparams(usp_plan_s *p, float2 *data, float2 *dst, const float2 *tw, long long stride, long long ncols,
                long long nouter, long long ostride, int line_axis, int check_state, int map_rank) {
    SParams sp{};
    sp.data = data;
    sp.dst = dst;
    sp.tw = tw;
    sp.stride = stride;
    sp.ncols = ncols;
    sp.nouter = nouter;
    sp.ostride = ostride;
    sp.line_axis = line_axis;
    sp.check_state = check_state;
    sp.mp = mul_params(p);
    sp.st = p->st;
    sp.map_rank = map_rank;
    sp.send_layout = 0;
    sp.P = p->P;
    sp.nz_loc = (int)p->nzs;
    sp.nyl_lg = log2ll(p->nyl);
    sp.y0 = 0;
    return sp;
}

typedef CUresult (*AddrRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddrRangeFn>(ptr);
    }
    return fn;
}

void close_peers(usp_plan_s *p) {
    for (void *b : p->ipc_bases) cudaIpcCloseMemHandle(b);
    p->ipc_bases.clear();
    if (p->lsa) {   // collective, like the creation
        nccl_api().DevCommDestroy(p->comm, &p->devcomm);
        p->lsa = false;
    }
    if (p->win) {   // collective, like the registration
        nccl_api().CommWindowDeregister(p->comm, p->win);
        p->win = nullptr;
    }
    p->fused = false;
    p->transport = USP_TRANSPORT_NONE;
}

// every rank's flag (1/0) -> the minimum over the ranks (on the plan stream)
usp_status all_agree(usp_plan_s *p, bool mine, bool *all) {
    double good = mine ? 1.0 : 0.0;
    CU(cudaMemcpyAsync(p->coll + 2, &good, sizeof(double), cudaMemcpyHostToDevice, p->stream));
    NC(nccl_api().AllReduce(p->coll + 2, p->coll + 2, 1, ncclDouble, ncclMin, p->comm, p->stream));
    CU(cudaMemcpyAsync(&good, p->coll + 2, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    *all = good == 1.0;
    return USP_OK;
}

// NCCL window over the workspace allocation (collective): on success the P
// ranks' addresses of byte 0 of that allocation in peer[0..P)
usp_status window_peers(usp_plan_s *p, char *base, size_t size, char **peer) {
    Nccl &n = nccl_api();
    NC(n.CommWindowRegister(p->comm, base, size, &p->win, NCCL_WIN_COLL_SYMMETRIC));
    void **d = reinterpret_cast<void **>(p->coll + 176);   // scratch: 8 pointers (past the IPC records)
    k_win_peers<<<1, 32, 0, p->stream>>>(p->win, p->P, d);
    CU(cudaGetLastError());
    return readback(p, peer, d, sizeof(void *) * p->P);
}

// device communicator with one LSA barrier (collective; p->lsa on success on
// every rank, decided by consensus)
usp_status setup_lsa(usp_plan_s *p) {
    Nccl &n = nccl_api();
    bool mine = false;
    if (n.devcomm) {
        ncclDevCommRequirements_t req{};
        req.lsaBarrierCount = 1;
        mine = n.DevCommCreate(p->comm, &req, &p->devcomm) == ncclSuccess;
    }
    bool all = false;
    usp_status s = all_agree(p, mine, &all);
    if (s) return s;
    if (all) {
        p->lsa = true;
    } else if (mine) {
        n.DevCommDestroy(p->comm, &p->devcomm);
    }
    return USP_OK;
}

// Map every rank's send / receive buffer for the fused transposes (collective
// in NCCL mode: CUDA IPC handles of the workspace allocations are
// all-gathered; every rank takes the same decision, falling back to the NCCL
// all-to-alls if any rank cannot map its peers).
usp_status setup_peers(usp_plan_s *p) {
    close_peers(p);
    const bool want = p->P > 1 && p->P <= kMaxPeers && !p->d.separate_transposes;
    const long long bk = p->nzs * p->nyl * p->rp;
    if (!want) return USP_OK;
    if (p->virt) {   // rank q's region of the one-GPU buffers
        for (int q = 0; q < p->P; ++q) {
            p->peer_recv[q] = p->recvb + (long long)q * p->P * bk;
            p->peer_send[q] = p->sendb + (long long)q * p->P * bk;
        }
        p->fused = true;
        p->transport = USP_TRANSPORT_VIRTUAL;
        return USP_OK;
    }
    // 1. NCCL window (the workspace came from usp_shared_alloc = ncclMemAlloc on
    //    every rank): peers' buffers through ncclGetPeerPointer
    {
        char *base = nullptr;
        size_t size = 0;
        const bool can = nccl_api().win && shared_range(p->ws, p->ws_bytes, &base, &size);
        bool all = false;
        usp_status s = all_agree(p, can, &all);
        if (s) return s;
        if (all) {
            char *peer[kMaxPeers] = {};
            s = window_peers(p, base, size, peer);
            bool ok = s == USP_OK;
            for (int q = 0; ok && q < p->P; ++q) ok = peer[q] != nullptr;
            if ((s = all_agree(p, ok, &all))) return s;
            if (all) {
                for (int q = 0; q < p->P; ++q) {
                    p->peer_recv[q] = (float2 *)(peer[q] + ((char *)p->recvb - base));
                    p->peer_send[q] = (float2 *)(peer[q] + ((char *)p->sendb - base));
                }
                p->fused = true;
                p->transport = USP_TRANSPORT_NCCL_WINDOW;
                return setup_lsa(p);
            }
            close_peers(p);
        }
    }
    // 2. CUDA IPC handles of the workspace allocations, all-gathered
    struct Rec {
        cudaIpcMemHandle_t h;
        long long off_recv, off_send;
        long long ok;
    } mine{};
    CUdeviceptr base = 0;
    size_t sz = 0;
    AddrRangeFn ar = addr_range_fn();
    if (ar && ar(&base, &sz, (CUdeviceptr)p->ws) == CUDA_SUCCESS &&
        cudaIpcGetMemHandle(&mine.h, (void *)base) == cudaSuccess) {
        mine.off_recv = (long long)((char *)p->recvb - (char *)base);
        mine.off_send = (long long)((char *)p->sendb - (char *)base);
        mine.ok = 1;
    }
    cudaGetLastError();   // clear a failed IPC query
    Rec *d = reinterpret_cast<Rec *>(p->coll + 16);   // scratch: 8 x 88 bytes fits the 192 doubles
    CU(cudaMemcpyAsync(d, &mine, sizeof(Rec), cudaMemcpyHostToDevice, p->stream));
    NC(nccl_api().AllGather(d, d + 1, sizeof(Rec), ncclChar, p->comm, p->stream));
    std::vector<Rec> all(p->P);
    CU(cudaMemcpyAsync(all.data(), d + 1, sizeof(Rec) * p->P, cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    bool ok = true;
    for (auto &r : all) ok = ok && r.ok;
    double good = 1.0;
    if (ok) {
        for (int q = 0; q < p->P; ++q) {
            if (q == p->rank) {
                p->peer_recv[q] = p->recvb;
                p->peer_send[q] = p->sendb;
                continue;
            }
            void *pb = nullptr;
            if (cudaIpcOpenMemHandle(&pb, all[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                good = 0.0;
                break;
            }
            p->ipc_bases.push_back(pb);
            p->peer_recv[q] = (float2 *)((char *)pb + all[q].off_recv);
            p->peer_send[q] = (float2 *)((char *)pb + all[q].off_send);
        }
    } else {
        good = 0.0;
    }
    // consensus: fused only if every rank mapped every peer
    CU(cudaMemcpyAsync(p->coll + 2, &good, sizeof(double), cudaMemcpyHostToDevice, p->stream));
    NC(nccl_api().AllReduce(p->coll + 2, p->coll + 2, 1, ncclDouble, ncclMin, p->comm, p->stream));
    CU(cudaMemcpyAsync(&good, p->coll + 2, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    if (good == 1.0) {
        p->fused = true;
        p->transport = USP_TRANSPORT_CUDA_IPC;
        return setup_lsa(p);
    } else {
        close_peers(p);
    }
    return USP_OK;
}

// Cross-rank barrier on the plan stream (fused transposes: the peers' stores
// into this rank's buffers are complete before the next kernel reads them).
usp_status rank_barrier(usp_plan_s *p) {
    if (!multi_rank(p)) return USP_OK;
    Tick t(p, KC_BARRIER, false);
    if (p->lsa) {   // LSA barrier of the device communicator (NCCL 2.28 device API)
        k_lsa_barrier<<<1, 32, 0, p->stream>>>(p->devcomm);
        CU(cudaGetLastError());
        return USP_OK;
    }
    NC(nccl_api().AllReduce(p->coll + 3, p->coll + 3, 1, ncclDouble, ncclSum, p->comm, p->stream));
    return USP_OK;
}

// The two transposes of the slab decomposition.  Block (r, q) of the send
// layout holds slab r's rows for y block q; block (r, q) of the receive
// layout holds y block r's planes of slab q.  forward: recv(r,q) <- send(q,r);
// back: send(q,r) <- recv(r,q).
// The whole exchange (nchunk = 1) or that of x-chunk `chunk` (blocks of
// width chunk_w in the chunk's region), on stream `st`.
usp_status exchange(usp_plan_s *p, bool forward, int chunk = 0, cudaStream_t st = nullptr) {
    if (!st) st = p->stream;
    const long long w = p->nchunk > 1 ? p->chunk_w : p->rp;
    const long long bk = p->nzs * p->nyl * w;   // elements per block
    const long long pv = p->virt ? p->P : 1;
    const long long base = (long long)chunk * pv * p->P * bk;
    const size_t bytes = (size_t)bk * sizeof(float2);
    Tick t(p, KC_A2A, false, st);
    if (p->virt) {
        for (int r = 0; r < p->P; ++r)
            for (int q = 0; q < p->P; ++q) {
                float2 *rv = p->recvb + base + ((long long)r * p->P + q) * bk;
                float2 *sd = p->sendb + base + ((long long)q * p->P + r) * bk;
                if (forward) CU(cudaMemcpyAsync(rv, sd, bytes, cudaMemcpyDeviceToDevice, st));
                else CU(cudaMemcpyAsync(sd, rv, bytes, cudaMemcpyDeviceToDevice, st));
            }
        return USP_OK;
    }
    Nccl &n = nccl_api();
    float2 *from = (forward ? p->sendb : p->recvb) + base, *to = (forward ? p->recvb : p->sendb) + base;
    NC(n.GroupStart());
    for (int q = 0; q < p->P; ++q) {
        NC(n.Send(from + q * bk, (size_t)bk * 2, ncclFloat, q, p->comm, st));
        NC(n.Recv(to + q * bk, (size_t)bk * 2, ncclFloat, q, p->comm, st));
    }
    NC(n.GroupEnd());
    return USP_OK;
}

// ---- antisymmetrised system (Eq. 9-10): component-major two-component chain
AParams anti_params(usp_plan_s *p) {
    AParams a{};
    a.work = p->work;
    a.delta = p->delta;
    a.x = p->x;
    a.v = p->B;
    a.tw = p->tw[0];
    a.nlines = p->ny * p->nz;
    a.nvox = p->nloc;
    a.inv_c = (float)(1.0 / p->c.re);
    a.sigma = make_float2((float)p->sigma.re, (float)p->sigma.im);
    a.inv_n = (float)(1.0 / (double)p->nvox);
    a.mp = mul_params(p);
    a.st = p->st;
    a.red = Red{p->partials, p->hist, p->hist_cap, nullptr};
    return a;
}

usp_status run_anti_x(usp_plan_s *p, XMode mode) {
    Tick t(p, mode == X_ITER ? KC_XPASS : KC_XSETUP);
    if (mode == X_ITER) {   // TMA-pipelined, one CTA per SM
        const long long units = p->ny * p->nz / anti_pipe_units((int)p->nx);
        CU(launch_anti_pipe((int)p->nx, anti_params(p), occ_grid(p, units, 1), p->stream));
        return USP_OK;
    }
    const int grid = occ_grid(p, (p->ny * p->nz + anti_lines_per_cta((int)p->nx) - 1) / anti_lines_per_cta((int)p->nx), 4);
    CU(launch_anti_x((int)p->nx, mode, anti_params(p), grid, p->stream));
    return USP_OK;
}

// forward FFT (y, z) of both components, the 2x2 symbol, inverse FFT (z, y)
usp_status chain_anti(usp_plan_s *p, int check_state) {
    usp_status s;
    const long long plane = p->nx * p->ny;
    if (p->ndim == 2) {
        SParams yf = sparams(p, p->work, p->work, p->tw[1], p->nx, p->nx, 2, plane, 1, check_state, 2);
        if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, true, 0))) return s;
        {
            Tick t(p, KC_ZMUL);
            CU(launch_anti_mul(anti_params(p), check_state, occ_grid(p, (p->nloc + 255) / 256, 8), p->stream));
        }
        return run_strided(p, KC_YINV, (int)p->ny, S_INV, yf, p->smap_y, true, 0);
    }
    SParams yf = sparams(p, p->work, p->work, p->tw[1], p->nx, p->nx, 2 * p->nz, plane, 1, check_state, 3);
    SParams zf = sparams(p, p->work, p->work, p->tw[2], plane, plane, 2, p->nz * plane, 2, check_state, 2);
    if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, true, 0))) return s;
    if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD, zf, p->smap_z, true, 0))) return s;
    {
        Tick t(p, KC_ZMUL);
        CU(launch_anti_mul(anti_params(p), check_state, occ_grid(p, (p->nloc + 255) / 256, 8), p->stream));
    }
    if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_INV, zf, p->smap_z, true, 0))) return s;
    return run_strided(p, KC_YINV, (int)p->ny, S_INV, yf, p->smap_y, true, 0);
}

// ---- first-order tensor diffusion (§3.2): (d + 1)-component chain
TDParams td_params(usp_plan_s *p) {
    TDParams t = p->td;
    t.d = p->ndim;
    t.n = p->nloc;
    t.work = p->work;
    t.delta = p->delta;
    t.x = p->x;
    t.vu = p->td_vu;
    t.vf = p->td_vf;
    t.dinv = p->td_dinv;
    t.red = p->td_red;
    t.inv_n = (float)(1.0 / (double)p->nvox);
    t.mp = mul_params(p);
    t.twx = p->tw[0];
    t.st = p->st;
    t.red_d = Red{p->partials, p->hist, p->hist_cap, nullptr};
    return t;
}

usp_status td_xfft(usp_plan_s *p, bool inv) {
    Tick t(p, inv ? KC_XPASS : KC_XSETUP);
    const long long lines = (long long)p->ncomp * p->ny * p->nz;
    const int lpc = 128 / (1 << (log2ll(p->nx) / 2));
    CU(launch_xfft((int)p->nx, inv, p->work, p->tw[0], lines, occ_grid(p, (lines + lpc - 1) / lpc, 8), p->stream));
    return USP_OK;
}

usp_status chain_tdiff(usp_plan_s *p, int check_state) {
    usp_status s;
    const long long plane = p->nx * p->ny, nc = p->ncomp;
    const int ge = occ_grid(p, (p->nloc + 255) / 256, 8);
    if (p->ndim == 2) {
        SParams yf = sparams(p, p->work, p->work, p->tw[1], p->nx, p->nx, nc, plane, 1, check_state, 2);
        if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, true, 0))) return s;
        {
            Tick t(p, KC_ZMUL);
            CU(launch_tdiff_mul(td_params(p), check_state, ge, p->stream));
        }
        return run_strided(p, KC_YINV, (int)p->ny, S_INV, yf, p->smap_y, true, 0);
    }
    SParams yf = sparams(p, p->work, p->work, p->tw[1], p->nx, p->nx, nc * p->nz, plane, 1, check_state, 3);
    SParams zf = sparams(p, p->work, p->work, p->tw[2], plane, plane, nc, p->nz * plane, 2, check_state, 2);
    if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, true, 0))) return s;
    if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD, zf, p->smap_z, true, 0))) return s;
    {
        Tick t(p, KC_ZMUL);
        CU(launch_tdiff_mul(td_params(p), check_state, ge, p->stream));
    }
    if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_INV, zf, p->smap_z, true, 0))) return s;
    return run_strided(p, KC_YINV, (int)p->ny, S_INV, yf, p->smap_y, true, 0);
}

usp_status td_upd(usp_plan_s *p, XMode mode) {
    Tick t(p, mode == X_ITER ? KC_XPASS : KC_XSETUP);
    if (mode == X_ITER && p->td_pipe) {   // x inverse FFT + update + x forward FFT in one TMA-pipelined pass
        const long long units = p->ny * p->nz / p->td_pipe;
        CU(launch_tdiff_pipe((int)p->nx, td_params(p), occ_grid(p, units, 1), p->stream));
        return USP_OK;
    }
    CU(launch_tdiff_upd(mode, td_params(p), occ_grid(p, (p->nloc + 255) / 256, 8), p->stream));
    return USP_OK;
}

// Separate transposes pipelined over x-chunks: the compute
// stream runs B0 B1 C0 B2 C1 D0 ... (K_B(c), K_C(c - 1), K_D(c - 2)), the
// exchange stream F0 F1 R0 F2 R1 ... (forward all-to-all of chunk c once
// K_B(c) is done, the return of chunk c once K_C(c) is done), so each chunk's
// transfer overlaps the other chunks' FFT passes.  Per element the same
// arithmetic as the unchunked path (bit-identical results).
usp_status chain_mid_chunked(usp_plan_s *p, int check_state) {
    usp_status s;
    const int C = p->nchunk;
    const long long W = p->chunk_w, pv = p->virt ? p->P : 1;
    const long long bkc = p->nzs * p->nyl * W, creg = pv * p->P * bkc;   // elements per block / chunk region
    for (int st = 0; st < C + 2; ++st) {
        if (st < C) {   // K_B(st): y forward of columns [st W, st W + W) into the chunk's send layout
            SParams yb = sparams(p, p->work, p->sendb + st * creg, p->tw[1], W, W, p->nzh, p->rp * p->ny, 1,
                                 check_state, 3);
            yb.send_layout = 1;
            yb.col0 = (int)(st * W);
            if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yb, p->smap_y, true, 0))) return s;
            CU(cudaEventRecord(p->ev_b[st], p->stream));
            CU(cudaStreamWaitEvent(p->xstream, p->ev_b[st], 0));
            if ((s = exchange(p, true, st, p->xstream))) return s;
            CU(cudaEventRecord(p->ev_x[st], p->xstream));
        }
        const int c = st - 1;
        if (c >= 0 && c < C) {   // K_C(c) on the chunk's y-slab blocks, then the return transpose
            CU(cudaStreamWaitEvent(p->stream, p->ev_x[c], 0));
            SParams zm = sparams(p, p->recvb + c * creg, p->recvb + c * creg, p->tw[2], p->nyl * W, p->nyl * W, pv,
                                 p->nz * p->nyl * W, 2, check_state, 2);
            zm.y0 = p->virt ? 0 : (long long)p->rank * p->nyl;
            zm.x0 = (int)(c * W);
            zm.mp.rowc = (int)W;
            if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zm, p->smap_zc[c], true, 0))) return s;
            CU(cudaEventRecord(p->ev_c[c], p->stream));
            CU(cudaStreamWaitEvent(p->xstream, p->ev_c[c], 0));
            if ((s = exchange(p, false, c, p->xstream))) return s;
            CU(cudaEventRecord(p->ev_y[c], p->xstream));
        }
        const int d = st - 2;
        if (d >= 0 && d < C) {   // K_D(d): y inverse from the chunk's send layout into work columns [d W, d W + W)
            CU(cudaStreamWaitEvent(p->stream, p->ev_y[d], 0));
            SParams yd = sparams(p, p->sendb + d * creg, p->work + d * W, p->tw[1], p->rp, W, p->nzh,
                                 p->rp * p->ny, 1, check_state, 5);
            if ((s = run_strided(p, KC_YINV, (int)p->ny, S_INV, yd, p->smap_kdc[d], true, 0))) return s;
        }
    }
    return USP_OK;
}

// The middle of the chain: every FFT pass between the x forward and the x
// inverse, with the (L+1)^-1 multiplier on the last axis (Eq. 12).
usp_status chain_mid(usp_plan_s *p, int check_state) {
    if (p->ndim == 2) {
        SParams sp = sparams(p, p->work, p->work, p->tw[1], p->rp, p->rp, 1, 0, 1, check_state, 2);
        return run_strided(p, KC_YMUL2D, (int)p->ny, S_FWD_MUL_INV, sp, p->smap_y, p->stile_y, p->grid_y);
    }
    usp_status s;
    if (p->P == 1) {
        SParams yf = sparams(p, p->work, p->work, p->tw[1], p->rp, p->rp, p->nz, p->rp * p->ny, 1, check_state, 3);
        SParams zm = sparams(p, p->work, p->work, p->tw[2], p->rp * p->ny, p->rp * p->ny, 1, 0, 2, check_state, 2);
        if (p->wpair) {
            // z-pair buffer (usp_internal.h): K_B stores work -> work2 (planes 2zp, 2zp+1
            // interleaved), K_C runs on work2's 256-byte pair rows, K_D reads work2
            // through the [nz/2][ny][2 nx] view and stores work back in [z][y][x]
            const long long nx = p->rp, ny = p->ny;   // row pitch (nx; nx/2 + 16 on the real path)
            SParams yb = sparams(p, p->work, p->work2, p->tw[1], 2 * nx, nx, p->nz, 2 * nx * ny, 1, check_state, 3);
            yb.pair_dst = 1;
            SParams zp = sparams(p, p->work2, p->work2, p->tw[2], 2 * nx * ny, nx * ny, 1, 0, 2, check_state, 2);
            zp.zpair = 1;
            SParams yd = sparams(p, p->work2, p->work, p->tw[1], nx, nx, p->nz, nx * ny, 1, check_state, 3);
            yd.pair_src = 1;
            if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yb, p->smap_y, true, 0))) return s;
            if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zp, p->smap_z, true, 0))) return s;
            return run_strided(p, KC_YINV, (int)p->ny, S_INV, yd, p->smap_yp, true, 0, &p->smap_y);
        }
        if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, p->stile_y, p->grid_y))) return s;
        if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zm, p->smap_z, p->stile_z, p->grid_z))) return s;
        return run_strided(p, KC_YINV, (int)p->ny, S_INV, yf, p->smap_y, p->stile_y, p->grid_y);
    }
    // slab decomposition: K_B -> transpose -> K_C -> transpose -> K_D
    const long long pv = p->virt ? p->P : 1;   // y blocks held here
    if (p->fused) {   // transposes fused into the K_B / K_C stores (peer memory)
        const int rank0 = p->virt ? 0 : p->rank;
        SParams yb = sparams(p, p->work, p->work, p->tw[1], p->rp, p->rp, p->nzh, p->rp * p->ny, 1, check_state, 3);
        yb.peer_mode = 1;
        yb.rank0 = rank0;
        yb.bk = p->nzs * p->nyl * p->rp;
        for (int q = 0; q < p->P; ++q) yb.peer[q] = p->peer_recv[q];
        SParams zm = sparams(p, p->recvb, p->recvb, p->tw[2], p->nyl * p->rp, p->nyl * p->rp, pv,
                             p->nz * p->nyl * p->rp, 2, check_state, 2);
        zm.y0 = p->virt ? 0 : (long long)p->rank * p->nyl;
        zm.peer_mode = 2;
        zm.rank0 = rank0;
        zm.bk = yb.bk;
        for (int q = 0; q < p->P; ++q) zm.peer[q] = p->peer_send[q];
        SParams yd = sparams(p, p->sendb, p->work, p->tw[1], p->rp, p->rp, p->nzh, p->rp * p->ny, 1, check_state, 5);
        if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yb, p->smap_y, true, 0))) return s;
        if ((s = rank_barrier(p))) return s;
        if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zm, p->smap_z, true, 0))) return s;
        if ((s = rank_barrier(p))) return s;
        return run_strided(p, KC_YINV, (int)p->ny, S_INV, yd, p->smap_kd, true, 0);
    }
    if (p->nchunk > 1) return chain_mid_chunked(p, check_state);
    SParams yb = sparams(p, p->work, p->sendb, p->tw[1], p->rp, p->rp, p->nzh, p->rp * p->ny, 1, check_state, 3);
    yb.send_layout = 1;
    SParams zm = sparams(p, p->recvb, p->recvb, p->tw[2], p->nyl * p->rp, p->nyl * p->rp, pv,
                         p->nz * p->nyl * p->rp, 2, check_state, 2);
    zm.y0 = p->virt ? 0 : (long long)p->rank * p->nyl;
    SParams yd = sparams(p, p->sendb, p->work, p->tw[1], p->rp, p->rp, p->nzh, p->rp * p->ny, 1, check_state, 5);
    if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yb, p->smap_y, true, 0))) return s;
    if ((s = exchange(p, true))) return s;
    if ((s = run_strided(p, KC_ZMUL, (int)p->nz, S_FWD_MUL_INV, zm, p->smap_z, true, 0))) return s;
    if ((s = exchange(p, false))) return s;
    return run_strided(p, KC_YINV, (int)p->ny, S_INV, yd, p->smap_kd, true, 0);
}

usp_status chain_mid(usp_plan_s *p, int check_state);
usp_status run_xpass(usp_plan_s *p, XMode mode, const XParams &xp);

// x-form state after iterations (reading R-30): one probe pass computes
// Delta_k = B(y_k - x_k) of the current x_k (x and the x-form chain input
// unchanged), so r_k, Delta_k and the history r_0..r_k are as after a
// Delta-form iteration.  Runs only when a query needs them.
usp_status probe_xform(usp_plan_s *p);

usp_status sync_state(usp_plan_s *p) {
    // (st_host is mapped pinned memory: an SM copy, see readback)
    CU(launch_copy_bytes(p->st_host_dev, p->st, sizeof(IterState), 1, p->stream));
    CU(cudaStreamSynchronize(p->stream));
    if (p->st_host->err)
        return fail(USP_ERR_CUDA, "pipeline watchdog: a kernel gave up waiting (code %d, unit %d)",
                    p->st_host->err, p->st_host->err_info);
    return USP_OK;
}

// Tensor maps of the strided passes (they embed the workspace addresses).
void build_maps(usp_plan_s *p) {
    p->stile_y = p->stile_z = false;
    if (p->ndim < 2) return;
    const cuuint32_t cy = (cuuint32_t)stile_cols((int)p->ny), by = (cuuint32_t)stile_box((int)p->ny);
    if (p->ndim == 2) {
        if (!stile_supported(p->ny)) return;
        const cuuint64_t dims[2] = {(cuuint64_t)p->rp, (cuuint64_t)(p->ny * p->ncomp)};
        const cuuint64_t str[1] = {(cuuint64_t)p->rp * 8};
        const cuuint32_t box[2] = {cy, by};
        p->stile_y = make_map(&p->smap_y, p->work, 2, dims, str, box);
        return;
    }
    const long long comps = p->ncomp;   // multi-component fields: the components as extra planes
    if (stile_supported(p->ny)) {   // y pass over the planes held here: {x, y, z}
        const cuuint64_t dims[3] = {(cuuint64_t)p->rp, (cuuint64_t)p->ny, (cuuint64_t)(p->nzh * comps)};
        const cuuint64_t str[2] = {(cuuint64_t)p->rp * 8, (cuuint64_t)(p->rp * p->ny) * 8};
        const cuuint32_t box[3] = {cy, by, 1};
        p->stile_y = make_map(&p->smap_y, p->work, 3, dims, str, box);
    }
    if (!stile_supported(p->nz)) return;
    const cuuint32_t cz = (cuuint32_t)stile_cols((int)p->nz), bz = (cuuint32_t)stile_box((int)p->nz);
    if (p->wpair) {
        // z-pair buffer (usp_internal.h): K_C on pair rows {2 nx ny, nz/2} with {32, BP}
        // boxes, K_D on the [nz/2][ny][2 nx] view with {16, by, 1} boxes (K_B loads work
        // through the plain y map above)
        const long long nx = p->rp, ny = p->ny, nz = p->nz;   // row pitch: nx, or nx/2 + 16 (real path)
        const cuuint64_t dz[2] = {(cuuint64_t)(2 * nx * ny), (cuuint64_t)(nz / 2)};
        const cuuint64_t sz[1] = {(cuuint64_t)(2 * nx * ny) * 8};
        const cuuint32_t bxz[2] = {32, (cuuint32_t)std::min<long long>(256, nz / 4)};
        const cuuint64_t dy[3] = {(cuuint64_t)(2 * nx), (cuuint64_t)ny, (cuuint64_t)(nz / 2)};
        const cuuint64_t sy[2] = {(cuuint64_t)(2 * nx) * 8, (cuuint64_t)(2 * nx * ny) * 8};
        const cuuint32_t bxy[3] = {cy, by, 1};
        if (p->stile_y && make_map(&p->smap_z, p->work2, 2, dz, sz, bxz) &&
            make_map(&p->smap_yp, p->work2, 3, dy, sy, bxy)) {
            p->stile_z = true;
            return;
        }
        p->wpair = false;   // (plain chain then)
    }
    if (p->P == 1) {   // z pass: {x*y columns, z}
        const cuuint64_t dims[2] = {(cuuint64_t)(p->rp * p->ny), (cuuint64_t)(p->nz * comps)};
        const cuuint64_t str[1] = {(cuuint64_t)(p->rp * p->ny) * 8};
        const cuuint32_t box[2] = {cz, bz};
        p->stile_z = make_map(&p->smap_z, p->work, 2, dims, str, box);
        return;
    }
    const long long pv = p->virt ? p->P : 1;
    bool ok;
    {   // z pass on the y-slabs of the receive buffer: {x*y_loc columns, z * (y blocks)}
        const cuuint64_t dims[2] = {(cuuint64_t)(p->nyl * p->rp), (cuuint64_t)(p->nz * pv)};
        const cuuint64_t str[1] = {(cuuint64_t)(p->nyl * p->rp) * 8};
        const cuuint32_t box[2] = {cz, bz};
        ok = make_map(&p->smap_z, p->recvb, 2, dims, str, box);
    }
    {   // K_D reads the send layout [r][q][z_loc][y_loc][x]: {x, y_loc, z_loc, q, r}
        const cuuint64_t dims[5] = {(cuuint64_t)p->rp, (cuuint64_t)p->nyl, (cuuint64_t)p->nzs, (cuuint64_t)p->P,
                                    (cuuint64_t)pv};
        const cuuint64_t bk = (cuuint64_t)(p->nzs * p->nyl * p->rp) * 8;
        const cuuint64_t str[4] = {(cuuint64_t)p->rp * 8, (cuuint64_t)(p->nyl * p->rp) * 8, bk, bk * p->P};
        const cuuint32_t box[5] = {cy, std::min<cuuint32_t>(by, (cuuint32_t)p->nyl), 1, 1, 1};
        ok = ok && make_map(&p->smap_kd, p->sendb, 5, dims, str, box);
    }
    if (p->nchunk > 1) {   // the x-chunked separate transposes: one pair of maps per chunk region
        const long long W = p->chunk_w, bkc = p->nzs * p->nyl * W, creg = pv * p->P * bkc;
        p->smap_zc.assign(p->nchunk, CUtensorMap{});
        p->smap_kdc.assign(p->nchunk, CUtensorMap{});
        for (int c = 0; c < p->nchunk && ok; ++c) {
            const cuuint64_t dz[2] = {(cuuint64_t)(p->nyl * W), (cuuint64_t)(p->nz * pv)};
            const cuuint64_t sz[1] = {(cuuint64_t)(p->nyl * W) * 8};
            const cuuint32_t bxz[2] = {cz, bz};
            ok = make_map(&p->smap_zc[c], p->recvb + c * creg, 2, dz, sz, bxz);
            const cuuint64_t dd[5] = {(cuuint64_t)W, (cuuint64_t)p->nyl, (cuuint64_t)p->nzs, (cuuint64_t)p->P,
                                      (cuuint64_t)pv};
            const cuuint64_t sd[4] = {(cuuint64_t)W * 8, (cuuint64_t)(p->nyl * W) * 8, (cuuint64_t)bkc * 8,
                                      (cuuint64_t)bkc * p->P * 8};
            const cuuint32_t bxd[5] = {cy, std::min<cuuint32_t>(by, (cuuint32_t)p->nyl), 1, 1, 1};
            ok = ok && make_map(&p->smap_kdc[c], p->sendb + c * creg, 5, dd, sd, bxd);
        }
    }
    p->stile_z = ok;
    p->stile_y = p->stile_y && ok;
}

}  // namespace

// =================================================================== ABI ==
extern "C" {

const char *usp_last_error(void) { return g_err.c_str(); }

const char *usp_version(void) { return "0.4 sm_100a"; }

usp_status usp_comm_unique_id(unsigned char id[128]) {
    if (!id) return fail(USP_ERR_ARG, "NULL argument");
    Nccl &n = nccl_api();
    if (!n.ok) return fail(USP_ERR_NCCL, "%s", n.why.c_str());
    ncclUniqueId u;
    NC(n.GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return USP_OK;
}

usp_status usp_comm_init(const unsigned char id[128], int nranks, int rank, void **comm) {
    if (!id || !comm) return fail(USP_ERR_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(USP_ERR_ARG, "bad rank %d of %d", rank, nranks);
    Nccl &n = nccl_api();
    if (!n.ok) return fail(USP_ERR_NCCL, "%s", n.why.c_str());
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    NC(n.CommInitRank(&c, nranks, u, rank));
    *comm = c;
    return USP_OK;
}

usp_status usp_comm_destroy(void *comm) {
    if (!comm) return USP_OK;
    Nccl &n = nccl_api();
    if (!n.ok) return fail(USP_ERR_NCCL, "%s", n.why.c_str());
    NC(n.CommDestroy((ncclComm_t)comm));
    return USP_OK;
}

usp_status usp_plan_create(const usp_plan_desc *desc, usp_plan_t *out) {
    if (!desc || !out) return fail(USP_ERR_ARG, "NULL argument");
    *out = nullptr;
    if (desc->ndim < 1 || desc->ndim > 3) return fail(USP_ERR_ARG, "ndim must be 1..3 (got %d)", desc->ndim);
    if (!(desc->D > 0.0)) return fail(USP_ERR_ARG, "D must be > 0");
    if (desc->dtype != USP_C64 && desc->dtype != USP_R32) return fail(USP_ERR_ARG, "bad dtype");
    if (desc->medium != USP_MEDIUM_K2 && desc->medium != USP_MEDIUM_W) return fail(USP_ERR_ARG, "bad medium");
    for (int a = 0; a < desc->ndim; ++a) {
        if (!supported_n(desc->n[a]))
            return fail(USP_ERR_UNSUPPORTED, "extent n[%d]=%lld must be a power of two in [16, 2048]", a,
                        (long long)desc->n[a]);
        if (!(desc->h[a] > 0.0)) return fail(USP_ERR_ARG, "h[%d] must be > 0", a);
    }
    int P = 1, rank = 0;
    bool virt = false;
    if (desc->nccl_comm && desc->virtual_ranks > 1)
        return fail(USP_ERR_ARG, "nccl_comm and virtual_ranks are exclusive");
    if (desc->nccl_comm) {
        Nccl &n = nccl_api();
        if (!n.ok) return fail(USP_ERR_NCCL, "%s", n.why.c_str());
        NC(n.CommCount((ncclComm_t)desc->nccl_comm, &P));
        NC(n.CommUserRank((ncclComm_t)desc->nccl_comm, &rank));
    } else if (desc->virtual_ranks > 1) {
        P = desc->virtual_ranks;
        virt = true;
    }
    if (P > 1) {
        // z-slabs over P ranks: 3-D, P | nz, P | ny, and the
        // TMA-tiled strided passes for both y and z
        if (desc->ndim != 3) return fail(USP_ERR_UNSUPPORTED, "slab decomposition needs a 3-D grid");
        if (P & (P - 1)) return fail(USP_ERR_UNSUPPORTED, "rank count %d must be a power of two", P);
        if (desc->n[2] % P || desc->n[1] % P)
            return fail(USP_ERR_UNSUPPORTED, "rank count %d must divide ny and nz", P);
        if (!stile_supported(desc->n[1]) || !stile_supported(desc->n[2]))
            return fail(USP_ERR_UNSUPPORTED, "slab decomposition needs ny, nz in [64, 2048]");
    }
    if (desc->tensor_diffusion) {
        if (desc->ndim < 2 || desc->dtype != USP_R32 || P > 1 || desc->antisymmetric)
            return fail(USP_ERR_UNSUPPORTED, "tensor diffusion runs on 2-D / 3-D float32 plans on one GPU");
        for (int a = 0; a < desc->ndim; ++a)
            if (desc->n[a] < 64 || desc->n[a] > 1024)
                return fail(USP_ERR_UNSUPPORTED, "tensor diffusion needs extents in [64, 1024]");
    }
    if (desc->antisymmetric) {
        if (desc->ndim < 2 || desc->dtype != USP_C64 || P > 1)
            return fail(USP_ERR_UNSUPPORTED, "the antisymmetrised system runs on 2-D / 3-D complex64 plans on one GPU");
        for (int a = 0; a < desc->ndim; ++a)
            if (desc->n[a] < 64 || desc->n[a] > 1024)
                return fail(USP_ERR_UNSUPPORTED, "the antisymmetrised system needs extents in [64, 1024]");
    }
    usp_plan_s *p = new usp_plan_s();
    p->d = *desc;
    p->anti = desc->antisymmetric != 0;
    p->tdiff = desc->tensor_diffusion != 0;
    p->ncomp = p->anti ? 2 : (p->tdiff ? desc->ndim + 1 : 1);
    p->td_pipe = p->tdiff ? tdiff_pipe_units((int)desc->n[0], desc->ndim) : 0;
    p->ndim = desc->ndim;
    p->nx = desc->n[0];
    p->ny = desc->ndim >= 2 ? desc->n[1] : 1;
    p->nz = desc->ndim >= 3 ? desc->n[2] : 1;
    for (int a = desc->ndim; a < 3; ++a) p->d.h[a] = 1.0;
    p->nvox = p->nx * p->ny * p->nz;
    p->P = P;
    p->rank = rank;
    p->virt = virt;
    p->comm = (ncclComm_t)desc->nccl_comm;
    p->nzs = p->nz / P;
    p->nzh = (P > 1 && !virt) ? p->nzs : p->nz;
    p->nyl = p->ny / P;
    p->nloc = p->nx * p->ny * p->nzh;
    p->real = !p->anti && !p->tdiff && !desc->complex_path && desc->dtype == USP_R32 &&
              desc->medium == USP_MEDIUM_W && desc->ndim == 3 && xreal_supported(p->nx) && stile_supported(p->ny) &&
              stile_supported(p->nz);
    p->rp = p->real ? xreal_row_pitch((int)p->nx) : p->nx;
    if (P > 1 && !p->real) {   // x-chunks of the separate transposes: 4 chunks of >= 16 columns
        p->nchunk = (int)std::min<long long>(4, p->rp / 16);
        p->chunk_w = p->rp / p->nchunk;
    }
    p->stream = (cudaStream_t)desc->stream;
    p->sigma = desc->sigma;
    p->c = desc->c;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) {
        delete p;
        return fail(USP_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    }
    // launch grids: one resident wave, persistent grid-stride loops
    {
        const long long xl = p->ny * p->nzh;
        // short strided lines (k_strided, 16-column tiles of 64 threads, 2 CTAs per SM)
        if (p->ndim >= 2) p->grid_y = occ_grid(p, (p->nx / 16) * p->nzh * p->ncomp, 2);
        if (p->ndim >= 3) p->grid_z = occ_grid(p, (p->nx * p->ny) / 16 * p->ncomp, 2);
        const long long comps = p->ncomp;
        if (p->ndim >= 2 && stile_supported(p->ny))
            p->grids_y = occ_grid(p, (p->rp / stile_cols((int)p->ny)) * p->nzh * comps, stile_ctas_per_sm((int)p->ny));
        if (p->ndim >= 3 && stile_supported(p->nz)) {
            const long long zcols = (P > 1) ? p->nyl * p->rp * (virt ? P : 1) : p->rp * p->ny * comps;
            p->grids_z = occ_grid(p, zcols / stile_cols((int)p->nz), stile_ctas_per_sm((int)p->nz));
        }
        const int u = p->real ? xreal_lines_per_unit((int)p->nx) : 32 / (1 << (log2ll(p->nx) / 2));
        p->gridp_x = occ_grid(p, xl / u, 1);   // one CTA per SM, persistent over the warp units
    }
    // reduction partials: <= 3 doubles per CTA of the largest reducing grid
    p->partials_cap = 3 * std::max(p->gridp_x, p->nsm * 8);
    p->far_cap = p->nsm * 8;
    std::vector<float2> twh[3];
    const long long ext[3] = {p->nx, p->ny, p->nz};
#define TRY(call)                                                                         \
    do {                                                                                  \
        cudaError_t e2 = (call);                                                          \
        if (e2 != cudaSuccess) {                                                          \
            usp_plan_destroy(p);                                                          \
            return fail(USP_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e2));          \
        }                                                                                 \
    } while (0)
    TRY(cudaMalloc(&p->st, sizeof(IterState)));
    TRY(cudaMalloc(&p->partials, sizeof(double) * p->partials_cap));
    TRY(cudaMalloc(&p->hist, sizeof(double) * p->hist_cap));
    TRY(cudaMalloc(&p->red_u, sizeof(unsigned) * 4));
    TRY(cudaMalloc(&p->far_d, sizeof(double) * p->far_cap));
    TRY(cudaMalloc(&p->far_i, sizeof(long long) * p->far_cap));
    TRY(cudaMalloc(&p->coll, sizeof(double) * 2048));
    TRY(cudaMalloc(&p->ks, sizeof(KState)));
    TRY(cudaMalloc(&p->bar, sizeof(unsigned) * 2));
    TRY(cudaMemset(p->bar, 0, sizeof(unsigned) * 2));
    p->solve2d = !p->anti && !p->tdiff && p->ndim == 2 && solve2d_supported(p->nx, p->ny) && !desc->launch_per_pass;
    p->plane = desc->plane_chain && P == 1 && p->ndim == 3 && !p->real && !p->anti && !p->tdiff && p->nx == kPlaneN &&
               p->ny == kPlaneN && stile_supported(p->nz);
    if (p->plane) {
        TRY(cudaMalloc(&p->pl_ctr, sizeof(unsigned long long)));
        TRY(cudaMemset(p->pl_ctr, 0, sizeof(unsigned long long)));
        TRY(cudaMalloc(&p->pl_done, sizeof(unsigned) * 2 * p->nz));
        TRY(cudaMemset(p->pl_done, 0, sizeof(unsigned) * 2 * p->nz));
        TRY(cudaMalloc(&p->pl_part, sizeof(double) * kPlaneN * p->nz));
    }
    // the z pass on the z-pair buffer where the passes around it support it (one
    // GPU, 3-D, one component, 16-column TMA tiles on y and z)
    p->wpair = !desc->flat_work && P == 1 && p->ndim == 3 && !p->anti && !p->tdiff && !p->plane &&
               stile_supported(p->ny) && p->ny <= 1024 && stile_supported(p->nz) && p->nz <= 1024;
    p->xform_cap = !p->anti && !p->tdiff && p->ndim >= 2 && !p->solve2d && !desc->delta_form;
    if (desc->r_switch > 0.0) p->r_sw = desc->r_switch;
    p->force_finish = (desc->test_hooks & USP_HOOK_RANK_FINISH) != 0;
    TRY(cudaHostAlloc(&p->st_host, sizeof(IterState), cudaHostAllocMapped));
    TRY(cudaHostGetDevicePointer(&p->st_host_dev, p->st_host, 0));
    TRY(cudaHostAlloc(&p->hmap, kHostMapBytes, cudaHostAllocMapped));
    TRY(cudaHostGetDevicePointer(&p->hmap_dev, p->hmap, 0));
    if (p->real) {   // M-point four-step table for x, plus W_nx^k for the split/merge steps
        const int n = (int)p->nx, m = n / 2;
        std::vector<float2> tr(m);
        for (int k = 0; k < m; ++k) {
            const double a = -2.0 * M_PI * (double)k / (double)n;
            double c_ = std::cos(a), s_ = std::sin(a);
            if (4 * k == n) { c_ = 0.0; s_ = -1.0; }
            if (k == 0) { c_ = 1.0; s_ = 0.0; }
            tr[k] = make_float2((float)c_, (float)s_);
        }
        TRY(cudaMalloc(&p->twr, sizeof(float2) * m));
        TRY(cudaMemcpy(p->twr, tr.data(), sizeof(float2) * m, cudaMemcpyHostToDevice));
    }
    for (int a = 0; a < p->ndim; ++a) {
        twh[a] = twiddle_table((int)((a == 0 && p->real) ? ext[a] / 2 : ext[a]));
        TRY(cudaMalloc(&p->tw[a], sizeof(float2) * twh[a].size()));
        TRY(cudaMemcpy(p->tw[a], twh[a].data(), sizeof(float2) * twh[a].size(), cudaMemcpyHostToDevice));
    }
    IterState s0{};
    s0.status = ST_NO_SOURCE;
    TRY(cudaMemcpy(p->st, &s0, sizeof s0, cudaMemcpyHostToDevice));
#undef TRY
    *out = p;
    return USP_OK;
}

usp_status usp_plan_workspace_size(usp_plan_t p, size_t *bytes) {
    if (!p || !bytes) return fail(USP_ERR_ARG, "NULL argument");
    const size_t f = align256((size_t)p->nloc * (p->real ? sizeof(float) : sizeof(float2)));
    const size_t w = align256((size_t)p->nzh * p->ny * p->rp * sizeof(float2));
    if (p->anti) {   // x, Delta, work: two components each; v
        *bytes = 7 * f;
        return USP_OK;
    }
    if (p->tdiff) {  // x, Delta, work: d + 1 components each; v_u, V_F, D^-1 (float32)
        const int np = p->ndim * (p->ndim + 1) / 2;
        *bytes = 3 * (size_t)p->ncomp * f + align256((size_t)p->nloc * 4) * (1 + 2 * np);
        return USP_OK;
    }
    *bytes = 3 * f + w * (p->P > 1 ? 3 : 1) + (p->xform_cap ? f : 0)   // + s for the x-form
             + (p->wpair ? w : 0);                                        // + the z-pair buffer
    return USP_OK;
}

usp_status usp_plan_set_workspace(usp_plan_t p, void *dev, size_t bytes) {
    if (!p || !dev) return fail(USP_ERR_ARG, "NULL argument");
    if (((uintptr_t)dev) & 255) return fail(USP_ERR_ARG, "workspace must be 256-byte aligned");
    size_t need = 0;
    usp_plan_workspace_size(p, &need);
    if (bytes < need) return fail(USP_ERR_NOMEM, "workspace %zu bytes < required %zu", bytes, need);
    const size_t f = align256((size_t)p->nloc * (p->real ? sizeof(float) : sizeof(float2)));
    const size_t w = align256((size_t)p->nzh * p->ny * p->rp * sizeof(float2));
    p->ws = (char *)dev;
    p->ws_bytes = bytes;
    p->x = (float2 *)(p->ws);
    p->delta = (float2 *)(p->ws + f);
    p->B = (float2 *)(p->ws + 2 * f);
    p->work = (float2 *)(p->ws + 3 * f);
    if (p->anti) {   // [x x'] [Delta Delta'] [work work'] [v]
        p->x = (float2 *)(p->ws);
        p->delta = (float2 *)(p->ws + 2 * f);
        p->work = (float2 *)(p->ws + 4 * f);
        p->B = (float2 *)(p->ws + 6 * f);
    }
    if (p->tdiff) {  // [x]*(d+1) [Delta]*(d+1) [work]*(d+1) [v_u] [V_F]*np [D^-1]*np
        const int nc = p->ncomp, np = p->ndim * (p->ndim + 1) / 2;
        const size_t fr = align256((size_t)p->nloc * 4);
        p->x = (float2 *)(p->ws);
        p->delta = (float2 *)(p->ws + nc * f);
        p->work = (float2 *)(p->ws + 2 * nc * f);
        p->B = nullptr;
        p->td_vu = (float *)(p->ws + 3 * nc * f);
        p->td_vf = (float *)(p->ws + 3 * nc * f + fr);
        p->td_dinv = (float *)(p->ws + 3 * nc * f + fr + np * fr);
    }
    if (p->P > 1) {
        p->sendb = (float2 *)(p->ws + 3 * f + w);
        p->recvb = (float2 *)(p->ws + 3 * f + 2 * w);
    }
    p->s = p->xform_cap ? (float2 *)(p->ws + 3 * f + w * (p->P > 1 ? 3 : 1)) : nullptr;
    p->work2 = p->wpair ? (float2 *)(p->ws + 3 * f + w * (p->P > 1 ? 3 : 1) + (p->xform_cap ? f : 0)) : nullptr;
    if (p->real)   // the spectrum rows' padding columns are never written by the x pass: keep them 0
        CU(cudaMemsetAsync(p->work, 0, w * (p->P > 1 ? 3 : 1), p->stream));
    p->have_potential = p->have_source = false;
    build_maps(p);
    if (p->P > 1 && !(p->stile_y && p->stile_z))
        return fail(USP_ERR_CUDA, "could not encode the tensor maps of the slab decomposition");
    usp_status s = setup_peers(p);
    if (s) return s;
    if (p->P > 1 && !p->fused) p->transport = p->virt ? USP_TRANSPORT_VIRTUAL_COPY : USP_TRANSPORT_NCCL_ALLTOALL;
    if (p->comm && p->P == 1 && (p->d.test_hooks & USP_HOOK_WINDOW)) {
        // the window machinery on one GPU: register, resolve rank 0's mapping,
        // write through it, check through the plain pointer
        char *base = nullptr, *peer[kMaxPeers] = {};
        size_t size = 0;
        if (!nccl_api().win || !shared_range(p->ws, p->ws_bytes, &base, &size))
            return fail(USP_ERR_UNSUPPORTED, "window test: NCCL >= 2.28 and a usp_shared_alloc workspace needed");
        if ((s = window_peers(p, base, size, peer))) return s;
        if (!peer[0]) return fail(USP_ERR_NCCL, "ncclGetPeerPointer returned NULL");
        const long long n = std::min<long long>(p->nloc, 1LL << 22);
        unsigned *bad = reinterpret_cast<unsigned *>(p->coll + 184);
        CU(cudaMemsetAsync(bad, 0, sizeof(unsigned), p->stream));
        k_win_write<<<p->nsm, 256, 0, p->stream>>>((float2 *)(peer[0] + ((char *)p->work - base)), n);
        k_win_check<<<p->nsm, 256, 0, p->stream>>>(p->work, n, bad);
        CU(cudaGetLastError());
        unsigned nbad = 0;
        if ((s = readback(p, &nbad, bad, sizeof nbad))) return s;
        if (nbad) return fail(USP_ERR_NCCL, "window test: %u of %lld values differ", nbad, n);
        p->transport = USP_TRANSPORT_NCCL_WINDOW;
        // and the device communicator's LSA barrier (one rank: returns at once)
        if ((s = setup_lsa(p))) return s;
        if (!p->lsa) return fail(USP_ERR_NCCL, "window test: ncclDevCommCreate failed");
        k_lsa_barrier<<<1, 32, 0, p->stream>>>(p->devcomm);
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(p->stream));
    }
    if (p->P > 1 && !p->fused && p->nchunk > 1 && !p->xstream) {
        CU(cudaStreamCreateWithFlags(&p->xstream, cudaStreamNonBlocking));
        for (auto *v : {&p->ev_b, &p->ev_x, &p->ev_c, &p->ev_y}) {
            v->assign(p->nchunk, nullptr);
            for (auto &e : *v) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    return USP_OK;
}

usp_status usp_local_extent(usp_plan_t p, int64_t *z0, int64_t *nz_local) {
    if (!p || !z0 || !nz_local) return fail(USP_ERR_ARG, "NULL argument");
    if (p->ndim == 3) {
        *z0 = (p->P > 1 && !p->virt) ? (int64_t)p->rank * p->nzs : 0;
        *nz_local = p->nzh;
    } else {
        *z0 = 0;
        *nz_local = p->ndim == 2 ? p->ny : p->nx;
    }
    return USP_OK;
}

usp_status usp_set_potential(usp_plan_t p, const void *medium, usp_where where, double target_norm) {
    Range nvtx_range("usp_set_potential");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    bool from_stage = false;
    if (where == USP_STAGED) {   // the medium staged by usp_stage_inputs
        if (!p->staged || p->medium_taken) return fail(USP_ERR_STATE, "no staged medium (usp_stage_inputs)");
        CU(cudaStreamWaitEvent(p->stream, p->ev_staged, 0));
        medium = p->stg;
        where = USP_DEVICE;
        from_stage = true;
    }
    if (!medium) return fail(USP_ERR_ARG, "NULL argument");
    if (p->tdiff) return fail(USP_ERR_STATE, "tensor-diffusion plans take usp_set_tensor_medium");
    if (!p->ws) return fail(USP_ERR_STATE, "workspace not set");
    if (where != USP_HOST && where != USP_DEVICE) return fail(USP_ERR_ARG, "bad where");
    // stage the medium in the chain buffer (the source resets it later)
    usp_status s = stage(p, p->work, medium, (size_t)p->nloc * elem_bytes(p), where);
    if (s) return s;
    if (from_stage) {   // the medium slot may be refilled once this copy has run
        CU(cudaEventRecord(p->ev_med_used, p->stream));
        p->med_used_rec = true;
        p->medium_taken = true;
    }
    p->have_source = false;
    p->have_potential = false;
    if (target_norm > 0.0) {
        if (!(target_norm < 1.0)) return fail(USP_ERR_ARG, "target_norm must be in (0, 1)");
        P2 cen;
        double r;
        s = device_mec(p, p->work, cen, r);
        if (s) return s;
        if (!(r > 0.0))
            return fail(USP_ERR_ARG, "homogeneous medium: smallest circle has radius 0; give sigma and c explicitly");
        p->centre = {cen.x, cen.y};
        p->radius = r;
        if (p->anti) {                        // Eq. 9-10: REAL scale, ||V|| = r / c (L100-128)
            p->sigma = {cen.x, cen.y};
            if (p->d.medium == USP_MEDIUM_K2) p->sigma = {-cen.x, -cen.y};
            p->c = {r / target_norm, 0.0};
        } else if (p->d.medium == USP_MEDIUM_K2) {   // sigma = -kbar^2, c = -i r / 0.95 (R-1)
            p->sigma = {-cen.x, -cen.y};
            p->c = {0.0, -r / target_norm};
        } else {                              // diffusion: sigma = centre, c = r / 0.95 (R-15)
            p->sigma = {cen.x, cen.y};
            p->c = {r / target_norm, 0.0};
        }
    } else {
        p->sigma = p->d.sigma;
        p->c = p->d.c;
        p->centre = {0.0, 0.0};
        p->radius = 0.0;
    }
    if (p->c.re == 0.0 && p->c.im == 0.0) return fail(USP_ERR_ARG, "c must be non-zero");
    if (p->anti && !(p->c.im == 0.0 && p->c.re > 0.0))
        return fail(USP_ERR_ARG, "the antisymmetrised system needs a real scale c > 0 (Eq. 9-10)");
    if (!p->anti && p->d.D * p->c.re < 0.0)
        return fail(USP_ERR_NOT_ACCRETIVE, "D Re(c) < 0: -D lap / c is not accretive (Eq. 1)");
    CU(cudaMemsetAsync(p->red_u, 0, sizeof(unsigned) * 4, p->stream));
    if (p->real && (p->sigma.im != 0.0 || p->c.im != 0.0))
        return fail(USP_ERR_UNSUPPORTED, "the real (float32 diffusion) path needs real sigma and c");
    PotParams pp{p->work, p->d.dtype == USP_R32, p->d.medium == USP_MEDIUM_K2, p->B, p->nloc,
                 p->sigma.re, p->sigma.im, p->c.re, p->c.im, p->red_u, p->red_u + 1, p->red_u + 2};
    pp.b_real = p->real;
    pp.store_v = p->anti;
    {
        Tick t(p, KC_POTENTIAL);
        CU(launch_potential(pp, occ_grid(p, (p->nloc + 255) / 256, 8), p->stream));
    }
    if (multi_rank(p)) {   // the Theorem 1 checks over the whole grid
        NC(nccl_api().AllReduce(p->red_u, p->red_u, 1, ncclUint32, ncclMax, p->comm, p->stream));
        NC(nccl_api().AllReduce(p->red_u + 1, p->red_u + 1, 2, ncclUint32, ncclSum, p->comm, p->stream));
    }
    unsigned red[4];
    if ((s = readback(p, red, p->red_u, sizeof red))) return s;
    float vmax;
    std::memcpy(&vmax, &red[0], sizeof vmax);
    p->vmax = vmax;
    if (red[2]) return fail(USP_ERR_NONFINITE, "%u non-finite medium values", red[2]);
    if (!(vmax < 1.0f))
        return fail(USP_ERR_NOT_CONTRACTIVE, "max|V| = %g >= 1: Theorem 1 needs ||V|| < 1", (double)vmax);
    if (red[1])
        return fail(USP_ERR_NOT_ACCRETIVE, "Re(w/c) < 0 at %u voxels: A is not accretive (Eq. 1)", red[1]);
    p->have_potential = true;
    return USP_OK;
}

usp_status usp_set_tensor_medium(usp_plan_t p, const float *mu, const float *D, usp_where where, double target_norm) {
    Range nvtx_range("usp_set_tensor_medium");
    if (!p || !mu || !D) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->tdiff) return fail(USP_ERR_STATE, "the plan was not created with desc.tensor_diffusion");
    if (!p->ws) return fail(USP_ERR_STATE, "workspace not set");
    if (!(target_norm > 0.0 && target_norm < 1.0)) return fail(USP_ERR_ARG, "target_norm must be in (0, 1)");
    const int d = p->ndim, np = d * (d + 1) / 2;
    const size_t nb = (size_t)p->nloc * 4;
    usp_status s;
    p->have_source = p->have_potential = false;
    // stage: mu into v_u, D (packed) into V_F (both rewritten by the second pass)
    if ((s = stage(p, p->td_vu, mu, nb, where))) return s;
    if ((s = stage(p, p->td_vf, D, nb * np, where))) return s;
    const int grid = occ_grid(p, (p->nloc + 255) / 256, 4);
    if (!p->td_red) CU(cudaMalloc(&p->td_red, sizeof(float) * 16 * p->nsm * 4));
    TDParams t = td_params(p);
    t.mu = p->td_vu;
    t.Dpk = p->td_vf;
    t.red = p->td_red;
    CU(launch_tdiff_pot(t, 0, grid, p->stream));
    std::vector<float> red((size_t)16 * grid);
    if ((s = readback(p, red.data(), p->td_red, sizeof(float) * red.size()))) return s;
    double lo[7], hi[7], bad = 0.0;
    for (int q = 0; q < 7; ++q) { lo[q] = 3e38; hi[q] = -3e38; }
    for (int c = 0; c < grid; ++c) {
        for (int q = 0; q <= np; ++q) {
            lo[q] = std::min(lo[q], (double)red[(size_t)c * 16 + q]);
            hi[q] = std::max(hi[q], (double)red[(size_t)c * 16 + 7 + q]);
        }
        bad += red[(size_t)c * 16 + 15];
    }
    if (bad > 0) return fail(USP_ERR_NONFINITE, "%g voxels with non-finite mu or a D that is not positive definite", bad);
    // canonical form (reading R-29): mid-ranges into L, radii equilibrated by S
    const double mubar = 0.5 * (hi[0] + lo[0]), r_mu = 0.5 * (hi[0] - lo[0]);
    double dbar[6] = {0, 0, 0, 0, 0, 0}, r_d = 0.0;
    for (int q = 0; q < np; ++q) {
        dbar[q] = 0.5 * (hi[q + 1] + lo[q + 1]);
        r_d = std::max(r_d, 0.5 * (hi[q + 1] - lo[q + 1]));
    }
    const double s_u = r_mu > 0 ? r_mu : 1.0, s_F = r_d > 0 ? r_d : 1.0;
    t.mubar = (float)mubar;
    for (int q = 0; q < np; ++q) t.dbar[q] = (float)dbar[q];
    double c = 1.0;
    for (int pass = 0; pass < 2; ++pass) {   // pass 0: max |V| at c = 1; pass 1: V with c
        t.inv_cu = (float)(1.0 / (c * s_u));
        t.inv_cf = (float)(1.0 / (c * s_F));
        CU(launch_tdiff_pot(t, pass == 0 ? 1 : 2, grid, p->stream));
        if ((s = readback(p, red.data(), p->td_red, sizeof(float) * red.size()))) return s;
        double vmax = 0.0;
        for (int q = 0; q < grid; ++q) vmax = std::max(vmax, (double)red[(size_t)q * 16 + 14]);
        if (pass == 0) {
            if (!(vmax > 0.0)) return fail(USP_ERR_ARG, "homogeneous medium: give a heterogeneous mu or D");
            c = vmax / target_norm;
        } else {
            p->vmax = vmax;
        }
    }
    // (L + 1)^-1 symbol: a, q scale, (Dbar^-1 / (c s_F) + I)^-1
    double Dm[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    const int idx2[3][2] = {{0, 0}, {0, 1}, {1, 1}};
    const int idx3[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int q = 0; q < np; ++q) {
        const int i = d == 2 ? idx2[q][0] : idx3[q][0], j = d == 2 ? idx2[q][1] : idx3[q][1];
        Dm[i][j] = Dm[j][i] = dbar[q] / (c * s_F);
    }
    for (int k = 0; k < d; ++k) Dm[k][k] += 1.0;
    double R[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    if (d == 2) {
        const double det = Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0];
        R[0][0] = Dm[1][1] / det; R[1][1] = Dm[0][0] / det; R[0][1] = R[1][0] = -Dm[0][1] / det;
    } else {
        const double c00 = Dm[1][1] * Dm[2][2] - Dm[1][2] * Dm[2][1], c01 = Dm[1][2] * Dm[2][0] - Dm[1][0] * Dm[2][2];
        const double c02 = Dm[1][0] * Dm[2][1] - Dm[1][1] * Dm[2][0];
        const double det = Dm[0][0] * c00 + Dm[0][1] * c01 + Dm[0][2] * c02;
        R[0][0] = c00 / det; R[1][0] = c01 / det; R[2][0] = c02 / det;
        R[0][1] = (Dm[0][2] * Dm[2][1] - Dm[0][1] * Dm[2][2]) / det;
        R[1][1] = (Dm[0][0] * Dm[2][2] - Dm[0][2] * Dm[2][0]) / det;
        R[2][1] = (Dm[0][1] * Dm[2][0] - Dm[0][0] * Dm[2][1]) / det;
        R[0][2] = (Dm[0][1] * Dm[1][2] - Dm[0][2] * Dm[1][1]) / det;
        R[1][2] = (Dm[0][2] * Dm[1][0] - Dm[0][0] * Dm[1][2]) / det;
        R[2][2] = (Dm[0][0] * Dm[1][1] - Dm[0][1] * Dm[1][0]) / det;
    }
    for (int k = 0; k < 3; ++k)
        for (int m = 0; m < 3; ++m) t.dm_inv[k * 3 + m] = (float)R[k][m];
    t.a = (float)(mubar / (c * s_u) + 1.0);
    t.qs = (float)(1.0 / (c * std::sqrt(s_u * s_F)));
    t.s_scale = (float)(1.0 / (c * std::sqrt(s_u)));
    p->td = t;
    p->sigma = {mubar, 0.0};
    p->c = {c, 0.0};
    p->centre = {s_u, s_F};   // reported by usp_get_split: (s_u, s_F) of the equilibration S
    p->radius = r_mu;
    p->have_potential = true;
    return USP_OK;
}

usp_status usp_get_split(usp_plan_t p, usp_c128 *sigma, usp_c128 *c, usp_c128 *centre, double *radius,
                         double *max_abs_V) {
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (sigma) *sigma = p->sigma;
    if (c) *c = p->c;
    if (centre) *centre = p->centre;
    if (radius) *radius = p->radius;
    if (max_abs_V) *max_abs_V = p->vmax;
    return USP_OK;
}

usp_status usp_set_source(usp_plan_t p, const void *src, usp_where where) {
    Range nvtx_range("usp_set_source");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    const bool from_stage = where == USP_STAGED;
    if (where != USP_HOST && where != USP_DEVICE && !from_stage) return fail(USP_ERR_ARG, "bad where");
    if (from_stage) {   // the source staged by usp_stage_inputs
        if (!p->staged) return fail(USP_ERR_STATE, "nothing staged (usp_stage_inputs)");
        CU(cudaStreamWaitEvent(p->stream, p->ev_staged, 0));
        src = p->stg + align256((size_t)p->nloc * elem_bytes(p));
        where = USP_DEVICE;
    }
    if (!src) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->have_potential) return fail(USP_ERR_STATE, "set_potential must succeed first");
    usp_status s = stage(p, p->x, src, (size_t)p->nloc * elem_bytes(p), where);
    if (s) return s;
    if (from_stage) {   // the source slot may be refilled once this copy has run
        CU(cudaEventRecord(p->ev_src_used, p->stream));
        p->src_used_rec = true;
        p->staged = false;
        p->medium_taken = false;
    }
    IterState s0{};
    s0.status = ST_NO_SOURCE;
    s0.alpha = 0.75;
    p->xform = p->xform_cap;
    p->probe_needed = false;
    p->hist_conv = false;
    s0.xform = p->xform ? 1 : 0;
    s0.r_sw = p->r_sw;
    s0.form = FORM_DELTA;   // the source setup's finish sets FORM_X on x-form plans
    if ((s = put_state(p, s0))) return s;
    if (p->ndim == 1) {
        OneParams op{};
        op.delta = p->delta;
        op.x = p->x;
        op.B = p->B;
        op.tw = p->tw[0];
        op.src_real = p->d.dtype == USP_R32;
        const double m = p->c.re * p->c.re + p->c.im * p->c.im;
        op.inv_c = make_float2((float)(p->c.re / m), (float)(-p->c.im / m));
        op.mp = mul_params(p);
        op.st = p->st;
        op.red = Red{p->partials, p->hist, p->hist_cap, nullptr};
        Tick t(p, KC_SOLVE1D);
        CU(launch_solve1d((int)p->nx, O_SETUP, op, p->stream));
    } else if (p->tdiff) {
        p->td.Sraw = (const float *)p->x;   // the staged raw source (float32)
        if ((s = td_upd(p, X_SRC_FWD))) return s;
        if ((s = td_xfft(p, false))) return s;
        if ((s = chain_tdiff(p, 0))) return s;
        if ((s = td_xfft(p, true))) return s;
        if ((s = td_upd(p, X_SRC_EPI))) return s;
        if (p->td_pipe && (s = td_xfft(p, false))) return s;   // the fused pass expects x-transformed input
    } else if (p->anti) {
        if ((s = run_anti_x(p, X_SRC_FWD))) return s;
        if ((s = chain_anti(p, 0))) return s;
        if ((s = run_anti_x(p, X_SRC_EPI))) return s;
    } else {
        p->s_sparse = false;
        p->expect_x = false;
        XParams xp = x_params(p);
        const bool try_sparse = p->xform && !p->real && !p->d.dense_source;
        if (try_sparse) {
            if (!p->s_flag) CU(cudaMalloc(&p->s_flag, (size_t)p->ny * p->nzh));
            if (!p->s_ctr) CU(cudaMalloc(&p->s_ctr, sizeof(unsigned)));
            xp.s_flag = p->s_flag;
        }
        s = run_xpass(p, X_SRC_FWD, xp);
        if (s) return s;
        xp.s_flag = nullptr;
        s = chain_mid(p, 0);
        if (s) return s;
        s = run_xpass(p, X_SRC_EPI, xp);
        if (s) return s;
        if (try_sparse) {
            // reading R-31: few source lines -> keep FFT_x(s) of those lines only
            // (work holds FFT_x(u_0) = FFT_x(s) after the x-form setup)
            const long long nlines = p->ny * p->nzh;
            unsigned cnt = 0;
            CU(launch_sparse_count(p->s_flag, nlines, p->s_ctr, p->stream));
            if ((s = readback(p, &cnt, p->s_ctr, sizeof cnt))) return s;
            // the list (2 KiB) and the lines must fit in the s field
            const long long cap = std::min<long long>(kSparseMaxLines, ((long long)p->nloc - 256) / p->nx);
            if (cnt > 0 && (long long)cnt <= cap) {
                CU(launch_sparse_gather(p->s_flag, nlines, p->work, (int)p->nx, reinterpret_cast<int *>(p->s),
                                        p->s + 256, p->s_ctr, p->stream));
                p->s_sparse = true;
                p->s_count = (int)cnt;
                p->expect_x = true;
            }
        }
        if (p->plane) {   // the plane-chained invariant: work = FFT_y FFT_x (u_0)
            SParams yf = sparams(p, p->work, p->work, p->tw[1], p->rp, p->rp, p->nz, p->rp * p->ny, 1, 0, 3);
            if ((s = run_strided(p, KC_YFWD, (int)p->ny, S_FWD, yf, p->smap_y, p->stile_y, p->grid_y))) return s;
        }
    }
    s = sync_state(p);
    if (s) return s;
    p->have_source = true;
    return USP_OK;
}

}  // extern "C"

namespace {
usp_status probe_xform(usp_plan_s *p) {
    if (!p->probe_needed) return USP_OK;
    p->probe_needed = false;
    usp_status s = sync_state(p);
    if (s) return s;
    if (p->st_host->form != FORM_X || p->st_host->status != ST_RUNNING || p->st_host->k == 0) return USP_OK;
    p->expect_x = true;
    {
        Tick t(p, KC_SETSTATE);
        CU(launch_set_form(p->st, FORM_PROBE, p->stream));
    }
    if (p->plane) return plane_iteration(p);
    if ((s = chain_mid(p, 1))) return s;
    if ((s = run_xpass(p, X_ITER, x_params(p)))) return s;
    return sparse_add(p);
}
}  // namespace

extern "C" {

usp_status usp_iterate(usp_plan_t p, int64_t n_max, double alpha, double tol, int64_t *n_done, usp_term *term) {
    Range nvtx_range("usp_iterate");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (!p->have_source) return fail(USP_ERR_STATE, "set_source must succeed first");
    if (n_max < 0 || !(alpha > 0.0)) return fail(USP_ERR_ARG, "need n_max >= 0 and alpha > 0");
    usp_status s = sync_state(p);
    if (s) return s;
    p->expect_x = p->st_host->form != FORM_DELTA;
    const long long k0 = p->st_host->k;
    const long long kmax = k0 + n_max;
    {
        Tick t(p, KC_SETSTATE);
        CU(launch_set_state(p->st, alpha, tol, kmax, p->stream));
    }
    if (p->ndim == 1) {
        OneParams op{};
        op.delta = p->delta;
        op.x = p->x;
        op.B = p->B;
        op.tw = p->tw[0];
        op.mp = mul_params(p);
        op.st = p->st;
        op.red = Red{p->partials, p->hist, p->hist_cap, nullptr};
        Tick t(p, KC_SOLVE1D);
        CU(launch_solve1d((int)p->nx, O_ITER, op, p->stream));
    } else if (p->solve2d) {   // one cooperative launch runs every iteration
        S2Params sp{};
        sp.work = p->work;
        sp.delta = p->delta;
        sp.x = p->x;
        sp.B = p->B;
        sp.twx = p->tw[0];
        sp.twy = p->tw[1];
        sp.mp = mul_params(p);
        sp.st = p->st;
        sp.red = Red{p->partials, p->hist, p->hist_cap, nullptr};
        sp.partials = p->partials;
        sp.bar_count = p->bar;
        sp.bar_gen = p->bar + 1;
        Tick t(p, KC_SOLVE2D);
        CU(launch_solve2d((int)p->nx, (int)p->ny, sp, p->nsm, p->stream));
    } else {
        const XParams xp = x_params(p);
        const long long batch = 16;
        long long launched = 0;
        // with tol > 0 the device stops itself (every kernel checks the state);
        // the host looks once per batch.  x-form plans: one spare launch for
        // the pass that turns the x-form into the Delta-form (it does not
        // count as an iteration); spare launches skip themselves.
        const long long total = n_max + (p->xform ? 1 : 0);
        while (launched < total) {
            const long long nb = std::min(batch, total - launched);
            if (p->xform && launched > 0) {   // the x-form may have switched to the Delta-form
                s = sync_state(p);
                if (s) return s;
                p->expect_x = p->st_host->form != FORM_DELTA;
            }
            for (long long i = 0; i < nb; ++i) {
                if (p->tdiff) {
                    if (!p->td_pipe && (s = td_xfft(p, false))) return s;
                    if ((s = chain_tdiff(p, 1))) return s;
                    if (!p->td_pipe && (s = td_xfft(p, true))) return s;
                    if ((s = td_upd(p, X_ITER))) return s;
                    continue;
                }
                if (p->anti) {
                    if ((s = chain_anti(p, 1))) return s;
                    if ((s = run_anti_x(p, X_ITER))) return s;
                    continue;
                }
                if (p->plane) {
                    if ((s = plane_iteration(p))) return s;
                    continue;
                }
                s = chain_mid(p, 1);
                if (s) return s;
                s = run_xpass(p, X_ITER, xp);
                if (s) return s;
                if ((s = sparse_add(p))) return s;
            }
            launched += nb;
            if (tol > 0.0) {
                s = sync_state(p);
                if (s) return s;
                const int stt = p->st_host->status;
                if (stt == ST_DONE_CONV || stt == ST_DIVERGED) break;
            }
        }
        // still in the x-form: r_k / Delta_k of the current x_k are computed on
        // demand (usp_residual*, probe_xform) -- a resumed call continues in the x-form
        p->probe_needed = p->xform;
    }
    s = sync_state(p);
    if (s) return s;
    drain_timing(p);
    const IterState &h = *p->st_host;
    p->hist_conv = h.status == ST_DONE_CONV;
    if (n_done) *n_done = h.k - k0;
    if (term) {
        if (h.status == ST_DONE_CONV) *term = USP_CONVERGED;
        else if (h.status == ST_DIVERGED) *term = USP_DIVERGED;
        else *term = USP_MAX_ITER;
    }
    return USP_OK;
}

usp_status usp_residual(usp_plan_t p, double *rel, double *abs_norm, int64_t *k) {
    Range nvtx_range("usp_residual");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (!p->have_source) return fail(USP_ERR_STATE, "no source");
    usp_status s = probe_xform(p);
    if (s) return s;
    s = sync_state(p);
    if (s) return s;
    if (rel) *rel = p->st_host->r;
    if (abs_norm) *abs_norm = p->st_host->r * p->st_host->n0;
    if (k) *k = p->st_host->k;
    return USP_OK;
}

usp_status usp_residual_history(usp_plan_t p, double *host, int64_t cap, int64_t *n) {
    Range nvtx_range("usp_residual_history");
    if (!p || !n) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->have_source) return fail(USP_ERR_STATE, "no source");
    usp_status s = probe_xform(p);
    if (s) return s;
    s = sync_state(p);
    if (s) return s;
    // entries r_0 .. r_last: the last computed residual (after a converged
    // fixed-point stop, r_{k-1}: the residual of x_k itself is not computed)
    const long long last = p->st_host->k - ((p->hist_conv && p->st_host->k > 0) ? 1 : 0);
    const long long avail = std::min<long long>(last + 1, p->hist_cap);
    *n = avail;
    if (host && cap > 0) {
        std::vector<double> all(p->hist_cap);
        if ((s = readback(p, all.data(), p->hist, sizeof(double) * p->hist_cap))) return s;
        const long long first = last + 1 - avail;
        for (long long i = 0; i < std::min<long long>(cap, avail); ++i) host[i] = all[(first + i) % p->hist_cap];
    }
    return USP_OK;
}

usp_status usp_staging_size(usp_plan_t p, int with_readback, size_t *bytes) {
    if (!p || !bytes) return fail(USP_ERR_ARG, "NULL argument");
    *bytes = (with_readback ? 3 : 2) * align256((size_t)p->nloc * elem_bytes(p));   // medium, source[, result]
    return USP_OK;
}

usp_status usp_plan_set_staging(usp_plan_t p, void *dev, size_t bytes) {
    if (!p || !dev) return fail(USP_ERR_ARG, "NULL argument");
    if (((uintptr_t)dev) & 255) return fail(USP_ERR_ARG, "staging area must be 256-byte aligned");
    size_t need = 0, need_rb = 0;
    usp_staging_size(p, 0, &need);
    usp_staging_size(p, 1, &need_rb);
    if (bytes < need) return fail(USP_ERR_NOMEM, "staging area %zu bytes < required %zu", bytes, need);
    if (p->tdiff) return fail(USP_ERR_UNSUPPORTED, "tensor-diffusion plans do not stage inputs");
    if (!p->cstream) {
        CU(cudaStreamCreateWithFlags(&p->cstream, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&p->dstream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&p->ev_staged, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->ev_med_used, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->ev_src_used, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->ev_snap, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming));
    }
    CU(cudaStreamSynchronize(p->stream));   // nothing on the plan stream still reads the old area
    CU(cudaStreamSynchronize(p->cstream));
    CU(cudaStreamSynchronize(p->dstream));
    p->out_pending = false;
    p->stg = (char *)dev;
    p->stg_bytes = bytes;
    p->stg_result = bytes >= need_rb;
    p->staged = p->medium_taken = false;
    p->med_used_rec = p->src_used_rec = false;
    return USP_OK;
}

usp_status usp_stage_inputs(usp_plan_t p, const void *medium, const void *source) {
    Range nvtx_range("usp_stage_inputs");
    if (!p || !medium || !source) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->stg) return fail(USP_ERR_STATE, "usp_plan_set_staging must be called first");
    if (p->medium_taken)
        return fail(USP_ERR_STATE, "the staged medium was taken by set_potential; consume its source with "
                                   "set_source(USP_STAGED) before staging the next problem");
    const size_t nb = (size_t)p->nloc * elem_bytes(p);
    // each slot is refilled only after the plan stream has consumed its previous contents
    if (p->med_used_rec) CU(cudaStreamWaitEvent(p->cstream, p->ev_med_used, 0));
    CU(cudaMemcpyAsync(p->stg, medium, nb, cudaMemcpyHostToDevice, p->cstream));
    if (p->src_used_rec) CU(cudaStreamWaitEvent(p->cstream, p->ev_src_used, 0));
    CU(cudaMemcpyAsync(p->stg + align256(nb), source, nb, cudaMemcpyHostToDevice, p->cstream));
    CU(cudaEventRecord(p->ev_staged, p->cstream));
    p->staged = true;
    return USP_OK;
}

usp_status usp_get_field_async(usp_plan_t p, void *out) {
    Range nvtx_range("usp_get_field_async");
    if (!p || !out) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->stg) return fail(USP_ERR_STATE, "usp_plan_set_staging must be called first");
    if (!p->have_source) return fail(USP_ERR_STATE, "no source");
    if (p->tdiff || (p->d.dtype != USP_C64 && !p->real))
        return fail(USP_ERR_UNSUPPORTED, "asynchronous read-back of this field layout");
    if (!p->stg_result)
        return fail(USP_ERR_NOMEM, "staging area sized without the read-back slot (usp_staging_size(plan, 1, ..))");
    const size_t nb = (size_t)p->nloc * elem_bytes(p);
    char *res = p->stg + 2 * align256(nb);
    // the previous read-back must have left the result slot
    if (p->out_pending) CU(cudaStreamWaitEvent(p->stream, p->ev_out, 0));
    CU(launch_copy_bytes(res, p->x, nb, 4 * p->nsm, p->stream));   // SMs, not a copy engine
    CU(cudaEventRecord(p->ev_snap, p->stream));
    CU(cudaStreamWaitEvent(p->dstream, p->ev_snap, 0));
    CU(cudaMemcpyAsync(out, res, nb, cudaMemcpyDeviceToHost, p->dstream));
    CU(cudaEventRecord(p->ev_out, p->dstream));
    p->out_pending = true;
    return USP_OK;
}

usp_status usp_wait_field(usp_plan_t p) {
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (p->out_pending) CU(cudaEventSynchronize(p->ev_out));
    return USP_OK;
}

usp_status usp_get_field(usp_plan_t p, void *out, usp_where where) {
    Range nvtx_range("usp_get_field");
    if (!p || !out) return fail(USP_ERR_ARG, "NULL argument");
    if (!p->have_source) return fail(USP_ERR_STATE, "no source");
    const cudaMemcpyKind kind = where == USP_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (p->tdiff) {   // u = E_0 / sqrt(s_u), float32
        float *dst = (float *)out;
        float *tmp = nullptr;
        if (where == USP_HOST) {
            tmp = (float *)(p->work);   // scratch (overwritten by the next chain)
            dst = tmp;
        }
        CU(launch_tdiff_out(p->x, dst, (float)(1.0 / std::sqrt(p->centre.re)), p->nloc,
                            occ_grid(p, (p->nloc + 255) / 256, 8), p->stream));
        if (where == USP_HOST) CU(cudaMemcpyAsync(out, tmp, (size_t)p->nloc * 4, cudaMemcpyDeviceToHost, p->stream));
    } else if (p->d.dtype == USP_C64) {
        CU(cudaMemcpyAsync(out, p->x, (size_t)p->nloc * sizeof(float2), kind, p->stream));
    } else if (p->real) {
        CU(cudaMemcpyAsync(out, p->x, (size_t)p->nloc * sizeof(float), kind, p->stream));
    } else {
        // real field: take the real parts (strided copy, pitch 8 -> 4 bytes)
        CU(cudaMemcpy2DAsync(out, sizeof(float), p->x, sizeof(float2), sizeof(float), (size_t)p->nloc, kind,
                             p->stream));
    }
    if (where == USP_HOST) CU(cudaStreamSynchronize(p->stream));
    return USP_OK;
}

usp_status usp_krylov_workspace_size(usp_plan_t p, size_t *bytes) {
    if (!p || !bytes) return fail(USP_ERR_ARG, "NULL argument");
    *bytes = 5 * align256((size_t)p->nloc * sizeof(float2));
    return USP_OK;
}

usp_status usp_krylov_set_workspace(usp_plan_t p, void *dev, size_t bytes) {
    if (!p || !dev) return fail(USP_ERR_ARG, "NULL argument");
    if (((uintptr_t)dev) & 255) return fail(USP_ERR_ARG, "Krylov workspace must be 256-byte aligned");
    size_t need = 0;
    usp_krylov_workspace_size(p, &need);
    if (bytes < need) return fail(USP_ERR_NOMEM, "Krylov workspace %zu bytes < required %zu", bytes, need);
    const size_t f = align256((size_t)p->nloc * sizeof(float2));
    char *b = (char *)dev;
    p->k_rh = (float2 *)b;
    p->k_p = (float2 *)(b + f);
    p->k_v = (float2 *)(b + 2 * f);
    p->k_s = (float2 *)(b + 3 * f);
    p->k_t = (float2 *)(b + 4 * f);
    return USP_OK;
}

usp_status usp_bicgstab(usp_plan_t p, int64_t n_max, double tol, int64_t *n_done, usp_term *term) {
    Range nvtx_range("usp_bicgstab");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (!p->have_source) return fail(USP_ERR_STATE, "set_source must succeed first");
    if (!p->k_rh) return fail(USP_ERR_STATE, "usp_krylov_set_workspace must be called first");
    if (n_max < 0) return fail(USP_ERR_ARG, "need n_max >= 0");
    if (p->ndim < 2 || p->real || p->anti || p->tdiff || multi_rank(p))
        return fail(USP_ERR_UNSUPPORTED, "BiCGSTAB runs on 2-D / 3-D complex64 plans on one GPU");
    usp_status s = sync_state(p);
    if (s) return s;
    if (p->st_host->k != 0)
        return fail(USP_ERR_STATE, "BiCGSTAB starts from x_0 = 0: call usp_set_source again first");
    const long long nvb = (long long)p->nloc * sizeof(float2);
    // r = b = Delta_0 (the fixed-point setup left it in `delta`), rhat = r, p = v = 0
    CU(launch_copy_bytes(p->k_rh, p->delta, nvb, 4 * p->nsm, p->stream));
    CU(cudaMemsetAsync(p->k_p, 0, nvb, p->stream));
    CU(cudaMemsetAsync(p->k_v, 0, nvb, p->stream));
    KState k0{};
    const double nb = p->st_host->n0;
    k0.rho = make_double2(nb * nb, 0.0);
    k0.omega = make_double2(1.0, 0.0);
    k0.nb = nb;
    CU(launch_put_bytes(p->ks, &k0, sizeof k0, p->stream));
    {
        Tick t(p, KC_SETSTATE);
        CU(launch_set_state(p->st, 1.0, tol, n_max, p->stream));
    }
    KParams kp{};
    kp.work = p->work;
    kp.x = p->x;
    kp.r = p->delta;
    kp.rh = p->k_rh;
    kp.p = p->k_p;
    kp.v = p->k_v;
    kp.s = p->k_s;
    kp.t = p->k_t;
    kp.B = p->B;
    kp.tw = p->tw[0];
    kp.nlines = p->ny * p->nzh;
    kp.nvox = p->nloc;
    kp.st = p->st;
    kp.ks = p->ks;
    kp.partials = p->partials;
    kp.hist = p->hist;
    kp.hist_cap = p->hist_cap;
    const int gx = p->gridp_x, gu = occ_grid(p, (p->nloc + 255) / 256, 8);
    auto xop = [&](KMode m) -> usp_status {
        Tick t(p, KC_XOP);
        CU(launch_xop((int)p->nx, m, kp, gx, p->stream));
        return USP_OK;
    };
    const long long batch = 8;
    long long launched = 0;
    while (launched < n_max) {
        const long long nb_ = std::min(batch, n_max - launched);
        for (long long i = 0; i < nb_; ++i) {
            if ((s = xop(K_PFWD))) return s;
            if ((s = chain_mid(p, 1))) return s;
            if ((s = xop(K_VINV))) return s;
            if ((s = xop(K_SFWD))) return s;
            if ((s = chain_mid(p, 1))) return s;
            if ((s = xop(K_TINV))) return s;
            {
                Tick t(p, KC_KUPD);
                CU(launch_kupd(kp, gu, p->stream));
            }
        }
        launched += nb_;
        if (tol > 0.0) {
            if ((s = sync_state(p))) return s;
            const int stt = p->st_host->status;
            if (stt == ST_DONE_CONV || stt == ST_DIVERGED) break;
        }
    }
    if ((s = sync_state(p))) return s;
    drain_timing(p);
    const IterState &h = *p->st_host;
    if (n_done) *n_done = h.k;
    if (term) {
        if (h.status == ST_DONE_CONV) *term = USP_CONVERGED;
        else if (h.status == ST_DIVERGED) *term = USP_DIVERGED;
        else *term = USP_MAX_ITER;
    }
    return USP_OK;
}

usp_status usp_gmres_workspace_size(usp_plan_t p, int m, size_t *bytes) {
    if (!p || !bytes) return fail(USP_ERR_ARG, "NULL argument");
    if (m < 1 || m > 64) return fail(USP_ERR_ARG, "restart length m must be in [1, 64]");
    *bytes = (size_t)(m + 2) * align256((size_t)p->nloc * sizeof(float2));
    return USP_OK;
}

usp_status usp_gmres_set_workspace(usp_plan_t p, int m, void *dev, size_t bytes) {
    if (!p || !dev) return fail(USP_ERR_ARG, "NULL argument");
    if (((uintptr_t)dev) & 255) return fail(USP_ERR_ARG, "GMRES workspace must be 256-byte aligned");
    size_t need = 0;
    usp_status s = usp_gmres_workspace_size(p, m, &need);
    if (s) return s;
    if (bytes < need) return fail(USP_ERR_NOMEM, "GMRES workspace %zu bytes < required %zu", bytes, need);
    const size_t f = align256((size_t)p->nloc * sizeof(float2));
    p->gm_m = m;
    p->gm_b = (float2 *)dev;
    p->gm_U.assign(m + 1, nullptr);
    for (int j = 0; j <= m; ++j) p->gm_U[j] = (float2 *)((char *)dev + (size_t)(j + 1) * f);
    return USP_OK;
}

namespace {
typedef std::complex<double> zd;

// Gram-Schmidt over basis vectors U[0..nv) in blocks of 8: GS_DOT returns
// d_j = (U_j, z) (+ ||z||^2 in *nrm); GS_AXPY applies z <- scale (z - sum c_j U_j)
// and returns ||z||^2 of the result.  Partial rows summed on the host in CTA order.

usp_status gs_dots(usp_plan_s *p, int nv, float2 *z, std::vector<zd> &d, double *nrm) {
    d.assign(nv, zd(0.0, 0.0));
    // every block of 8 basis vectors writes its own partials region; one
    // read-back and one host sync for the whole round
    const int nblk = (nv + 7) / 8;
    const size_t region = (size_t)17 * p->gm_grid;
    for (int bi = 0; bi < nblk; ++bi) {
        const int b0 = 8 * bi, nb = std::min(8, nv - b0);
        GSParams g{};
        for (int q = 0; q < nb; ++q) g.U[q] = p->gm_U[b0 + q];
        g.z = z;
        g.n = p->nloc;
        g.partials = p->gm_part + bi * region;
        Tick t(p, KC_KUPD);
        CU(launch_gs(GS_DOT, nb, g, p->gm_grid, p->stream));
    }
    std::vector<double> h(region * nblk);
    usp_status rs = readback(p, h.data(), p->gm_part, sizeof(double) * region * nblk);
    if (rs) return rs;
    for (int bi = 0; bi < nblk; ++bi) {
        const int b0 = 8 * bi, nb = std::min(8, nv - b0);
        const int K = 2 * nb + 1;
        const double *hb = h.data() + bi * region;
        std::vector<double> loc(K, 0.0);
        for (int q = 0; q < K; ++q)
            for (int c = 0; c < p->gm_grid; ++c) loc[q] += hb[(size_t)c * K + q];
        // slab-decomposed: every rank's local sums, added in rank order
        std::vector<double> all;
        usp_status s = gather_host(p, loc.data(), K, all);
        if (s) return s;
        for (int q = 0; q < K; ++q) {
            double t = 0.0;
            for (int r = 0; r < (multi_rank(p) ? p->P : 1); ++r) t += all[(size_t)r * K + q];
            loc[q] = t;
        }
        for (int q = 0; q < nb; ++q) d[b0 + q] = zd(loc[2 * q], loc[2 * q + 1]);
        if (nrm && b0 == 0) *nrm = loc[2 * nb];
    }
    return USP_OK;
}

usp_status gs_axpy(usp_plan_s *p, int nv, const std::vector<float2 *> &U, const std::vector<zd> &c, float2 *z,
                   zd scale, double *nrm) {
    std::vector<double> h(p->gm_grid);
    double s2 = 0.0;
    for (int b0 = 0; b0 < std::max(nv, 1); b0 += 8) {
        const int nb = std::min(8, nv - b0);
        GSParams g{};
        for (int q = 0; q < nb; ++q) {
            g.U[q] = U[b0 + q];
            g.c[q] = make_float2((float)c[b0 + q].real(), (float)c[b0 + q].imag());
        }
        const bool last = b0 + 8 >= nv;
        g.scale = last ? make_float2((float)scale.real(), (float)scale.imag()) : make_float2(1.f, 0.f);
        g.z = z;
        g.n = p->nloc;
        g.partials = p->gm_part;
        {
            Tick t(p, KC_KUPD);
            CU(launch_gs(GS_AXPY, nb, g, p->gm_grid, p->stream));
        }
        if (last && nrm) {
            usp_status rs = readback(p, h.data(), p->gm_part, sizeof(double) * p->gm_grid);
            if (rs) return rs;
            for (int q = 0; q < p->gm_grid; ++q) s2 += h[q];
            std::vector<double> all;   // slab-decomposed: ranks' norms in rank order
            usp_status st = gather_host(p, &s2, 1, all);
            if (st) return st;
            s2 = 0.0;
            for (int r = 0; r < (multi_rank(p) ? p->P : 1); ++r) s2 += all[r];
        }
    }
    if (nrm) *nrm = s2;
    return USP_OK;
}

// z = M u (the operator of the fixed-point path: two x passes + the chain)
usp_status apply_M_dev(usp_plan_s *p, float2 *u, float2 *z) {
    KParams kp{};
    kp.work = p->work;
    kp.p = u;
    kp.v = z;
    kp.B = p->B;
    kp.tw = p->tw[0];
    kp.nlines = p->ny * p->nzh;
    kp.st = p->st;
    usp_status s;
    {
        Tick t(p, KC_XOP);
        CU(launch_xop((int)p->nx, K_OFWD, kp, p->gridp_x, p->stream));
    }
    if ((s = chain_mid(p, 0))) return s;
    Tick t(p, KC_XOP);
    CU(launch_xop((int)p->nx, K_OINV, kp, p->gridp_x, p->stream));
    return USP_OK;
}
}  // namespace

usp_status usp_gmres(usp_plan_t p, int64_t n_max, double tol, int64_t *n_done, usp_term *term) {
    Range nvtx_range("usp_gmres");
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    if (!p->have_source) return fail(USP_ERR_STATE, "set_source must succeed first");
    if (!p->gm_b) return fail(USP_ERR_STATE, "usp_gmres_set_workspace must be called first");
    if (n_max < 0) return fail(USP_ERR_ARG, "need n_max >= 0");
    if (p->ndim < 2 || p->real || p->anti || p->tdiff)
        return fail(USP_ERR_UNSUPPORTED, "GMRES runs on 2-D / 3-D complex64 plans");
    usp_status s = sync_state(p);
    if (s) return s;
    if (p->st_host->k != 0)
        return fail(USP_ERR_STATE, "GMRES starts from x_0 = 0: call usp_set_source again first");
    if (!p->gm_part) {
        p->gm_grid = p->nsm * kGsCtasPerSm;   // every CTA resident at once (k_gs)
        CU(cudaMalloc(&p->gm_part, sizeof(double) * 17 * p->gm_grid * 9));   // (m + 1 <= 65 vectors) / 8 blocks
    }
    const int m = p->gm_m;
    const long long nvb = (long long)p->nloc * sizeof(float2);
    const double nb = p->st_host->n0;   // ||b||, b = Delta_0 = B (L+1)^-1 s
    CU(launch_copy_bytes(p->gm_b, p->delta, nvb, 4 * p->nsm, p->stream));
    std::vector<double> hist;
    long long steps = 0;
    double est = nb > 0.0 ? 1.0 : 0.0;
    int status = nb > 0.0 ? ST_RUNNING : ST_DONE_CONV;
    std::vector<double> nu(m + 1);
    std::vector<zd> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), d, d2;
    bool first = true;
    while (status == ST_RUNNING && steps < n_max) {
        // r = b - M x  (x = 0 on the first cycle: r = b)
        double b2 = 0.0;
        if (first) {
            CU(launch_copy_bytes(p->gm_U[0], p->gm_b, nvb, 4 * p->nsm, p->stream));
            b2 = nb * nb;
        } else {
            if ((s = apply_M_dev(p, p->x, p->gm_U[0]))) return s;
            std::vector<float2 *> Ub{p->gm_b};
            if ((s = gs_axpy(p, 1, Ub, std::vector<zd>{zd(1.0, 0.0)}, p->gm_U[0], zd(-1.0, 0.0), &b2))) return s;
        }
        first = false;
        nu[0] = std::sqrt(b2);
        const double beta = nu[0];
        if (!(beta > 0.0)) { status = ST_DONE_CONV; break; }
        std::fill(g.begin(), g.end(), zd(0.0, 0.0));
        g[0] = beta;
        int k = 0;
        bool stop = false;
        for (int j = 0; j < m && steps < n_max; ++j) {
            // z = M U_j into U_{j+1}: the stored vectors are U_i = nu_i v_i
            if ((s = apply_M_dev(p, p->gm_U[j], p->gm_U[j + 1]))) return s;
            std::vector<zd> hcol(j + 2, zd(0.0, 0.0));
            double z2 = 0.0;
            // classical Gram-Schmidt with selective re-orthogonalisation (DGKS,
            // eta = 1/sqrt(2)): a second pass only when the first cancelled
            // more than half of ||w||^2 ("twice is enough")
            for (int round = 0; round < 2; ++round) {
                double w2 = 0.0;
                if ((s = gs_dots(p, j + 1, p->gm_U[j + 1], d, round == 0 ? &w2 : nullptr))) return s;
                std::vector<zd> c(j + 1);
                for (int i = 0; i <= j; ++i) {
                    c[i] = d[i] / (nu[i] * nu[i]);
                    hcol[i] += d[i] / (nu[i] * nu[j]);
                }
                std::vector<float2 *> Ub(p->gm_U.begin(), p->gm_U.begin() + j + 1);
                if ((s = gs_axpy(p, j + 1, Ub, c, p->gm_U[j + 1], zd(1.0, 0.0), &z2))) return s;
                if (round == 0 && z2 >= 0.5 * w2) break;
            }
            nu[j + 1] = std::sqrt(z2);
            hcol[j + 1] = nu[j + 1] / nu[j];
            for (int i = 0; i < j; ++i) {   // previous rotations
                const zd t = cs[i] * hcol[i] + sn[i] * hcol[i + 1];
                hcol[i + 1] = -std::conj(sn[i]) * hcol[i] + std::conj(cs[i]) * hcol[i + 1];
                hcol[i] = t;
            }
            const double den = std::sqrt(std::norm(hcol[j]) + std::norm(hcol[j + 1]));
            if (!(den > 0.0)) { status = ST_DIVERGED; break; }
            cs[j] = std::conj(hcol[j]) / den;
            sn[j] = hcol[j + 1] / den;
            hcol[j] = den;
            hcol[j + 1] = 0.0;
            for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hcol[i];
            g[j + 1] = -std::conj(sn[j]) * g[j];
            g[j] = cs[j] * g[j];
            ++steps;
            k = j + 1;
            est = std::abs(g[j + 1]) / nb;
            hist.push_back(est);
            if (!std::isfinite(est) || est > 1e6) { status = ST_DIVERGED; stop = true; break; }
            if ((tol > 0.0 && est < tol) || nu[j + 1] == 0.0) { status = ST_DONE_CONV; stop = true; break; }
        }
        if (status == ST_DIVERGED && !stop) break;
        // y = R^-1 g; x += sum y_i v_i = sum (y_i / nu_i) U_i
        for (int i = k - 1; i >= 0; --i) {
            zd acc = g[i];
            for (int q = i + 1; q < k; ++q) acc -= H[(size_t)i * m + q] * y[q];
            y[i] = acc / H[(size_t)i * m + i];
        }
        std::vector<zd> c(k);
        for (int i = 0; i < k; ++i) c[i] = -y[i] / nu[i];
        std::vector<float2 *> Ub(p->gm_U.begin(), p->gm_U.begin() + k);
        if (k > 0 && (s = gs_axpy(p, k, Ub, c, p->x, zd(1.0, 0.0), nullptr))) return s;
        if (stop) break;
    }
    // publish the state (k = Arnoldi steps, r = residual estimate, history)
    IterState h = *p->st_host;
    h.k = steps;
    h.r = est;
    h.status = status == ST_RUNNING ? ST_RUNNING : status;
    if ((s = put_state(p, h))) return s;
    // history r_1 .. r_steps into the ring through the mapped scratch (contiguous segments)
    for (size_t i0 = 0; i0 < hist.size();) {
        const long long pos = (long long)(i0 + 1) % p->hist_cap;
        const size_t seg = std::min<size_t>({hist.size() - i0, (size_t)(p->hist_cap - pos), kHostMapBytes / 8});
        CU(cudaStreamSynchronize(p->stream));   // the previous segment's copy has read the scratch
        std::memcpy(p->hmap, hist.data() + i0, seg * sizeof(double));
        CU(launch_copy_bytes(p->hist + pos, p->hmap_dev, seg * sizeof(double), 4, p->stream));
        i0 += seg;
    }
    if ((s = sync_state(p))) return s;
    drain_timing(p);
    if (n_done) *n_done = steps;
    if (term) *term = status == ST_DONE_CONV ? USP_CONVERGED : (status == ST_DIVERGED ? USP_DIVERGED : USP_MAX_ITER);
    return USP_OK;
}

usp_status usp_profile_enable(usp_plan_t p, int enable) {
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    drain_timing(p);
    p->prof = enable != 0;
    if (enable) {
        for (int i = 0; i < KC_N; ++i) {
            p->prof_ms[i] = 0.0;
            p->prof_n[i] = 0;
        }
    }
    return USP_OK;
}

usp_status usp_profile_read(usp_plan_t p, int cap, char (*names)[32], double *ms, int64_t *launches, int *n) {
    if (!p || !n) return fail(USP_ERR_ARG, "NULL argument");
    drain_timing(p);
    int k = 0;
    for (int i = 0; i < KC_N && k < cap; ++i) {
        if (!p->prof_n[i]) continue;
        if (names) std::snprintf(names[k], 32, "%s", kc_names[i]);
        if (ms) ms[k] = p->prof_ms[i];
        if (launches) launches[k] = p->prof_n[i];
        ++k;
    }
    *n = k;
    return USP_OK;
}

usp_status usp_launch_count(usp_plan_t p, int64_t *launches) {
    if (!p || !launches) return fail(USP_ERR_ARG, "NULL argument");
    *launches = p->launches;
    return USP_OK;
}

usp_status usp_iteration_form(usp_plan_t p, int *xform, int *form, double *r_switch, int *source_lines) {
    if (!p) return fail(USP_ERR_ARG, "NULL plan");
    usp_status s = sync_state(p);
    if (s) return s;
    if (source_lines) *source_lines = p->s_sparse ? p->s_count : 0;
    if (xform) *xform = p->xform_cap ? 1 : 0;
    if (form) *form = (p->st_host->form == FORM_DELTA) ? 0 : 1;
    if (r_switch) *r_switch = p->r_sw;
    return USP_OK;
}

usp_status usp_shared_alloc(size_t bytes, void **ptr) {
    if (!ptr || !bytes) return fail(USP_ERR_ARG, "NULL argument or zero size");
    *ptr = nullptr;
    Nccl &n = nccl_api();
    void *q = nullptr;
    bool via = false;
    if (n.ok && n.win && n.MemAlloc(&q, bytes) == ncclSuccess && q) {
        via = true;
    } else {
        cudaGetLastError();
        q = nullptr;
        if (cudaMalloc(&q, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(USP_ERR_NOMEM, "could not allocate %zu bytes", bytes);
        }
    }
    std::lock_guard<std::mutex> g(g_shared_mu);
    g_shared[(char *)q] = SharedAlloc{bytes, via};
    *ptr = q;
    return USP_OK;
}

usp_status usp_shared_free(void *ptr) {
    if (!ptr) return USP_OK;
    SharedAlloc a{};
    {
        std::lock_guard<std::mutex> g(g_shared_mu);
        auto it = g_shared.find((char *)ptr);
        if (it == g_shared.end()) return fail(USP_ERR_ARG, "not a usp_shared_alloc pointer");
        a = it->second;
        g_shared.erase(it);
    }
    if (a.nccl) {
        NC(nccl_api().MemFree(ptr));
    } else {
        CU(cudaFree(ptr));
    }
    return USP_OK;
}

usp_status usp_transport(usp_plan_t p, int *kind) {
    if (!p || !kind) return fail(USP_ERR_ARG, "NULL argument");
    *kind = p->transport;
    return USP_OK;
}

usp_status usp_work_layout(usp_plan_t p, int *zpair) {
    if (!p || !zpair) return fail(USP_ERR_ARG, "NULL argument");
    *zpair = p->wpair ? 1 : 0;
    return USP_OK;
}

void usp_plan_destroy(usp_plan_t p) {
    if (!p) return;
    cudaStreamSynchronize(p->stream);
    drain_timing(p);
    close_peers(p);
    for (auto e : p->ev_pool) cudaEventDestroy(e);
    cudaFree(p->st);
    cudaFree(p->partials);
    cudaFree(p->hist);
    if (p->cstream) {
        cudaStreamSynchronize(p->cstream);
        cudaStreamSynchronize(p->dstream);
        cudaStreamDestroy(p->cstream);
        cudaStreamDestroy(p->dstream);
        cudaEventDestroy(p->ev_staged);
        cudaEventDestroy(p->ev_med_used);
        cudaEventDestroy(p->ev_src_used);
        cudaEventDestroy(p->ev_snap);
        cudaEventDestroy(p->ev_out);
    }
    cudaFree(p->red_u);
    if (p->s_flag) cudaFree(p->s_flag);
    if (p->s_ctr) cudaFree(p->s_ctr);
    cudaFree(p->far_d);
    cudaFree(p->far_i);
    cudaFree(p->coll);
    cudaFree(p->ks);
    cudaFree(p->gm_part);
    cudaFree(p->td_red);
    cudaFree(p->bar);
    if (p->xstream) {
        cudaStreamSynchronize(p->xstream);
        cudaStreamDestroy(p->xstream);
        for (auto *v : {&p->ev_b, &p->ev_x, &p->ev_c, &p->ev_y})
            for (auto e : *v) cudaEventDestroy(e);
    }
    cudaFree(p->pl_ctr);
    cudaFree(p->pl_done);
    cudaFree(p->pl_part);
    for (int a = 0; a < 3; ++a) cudaFree(p->tw[a]);
    cudaFree(p->twr);
    cudaFreeHost(p->st_host);
    if (p->hmap) cudaFreeHost(p->hmap);
    delete p;
}

}  // extern "C"
