// hk_api.cu — sm_100a kernels and the C ABI (include/hankel_b200.h).
//
// Kernels are grid-stride loops of warp-sized work items (hk_items.cuh); each
// warp carves its own slice of dynamic shared memory as MP scratch.  The LDLT
// step loop (ldlt.cpp:91-135; parallel form 206-351) is recorded once per
// (n, limbs) into a CUDA graph and replayed: per step i
//     recip (1 warp)  ->  mulB (n-i-1 warps)  ->  trailing (~(n-i)^2/2 warps)
//     ->  storeL (n-i-1 warps)
// A non-positive pivot sets a device flag (first column wins); every later
// item sees it and returns, and the host maps it to HK_ERR_PRECISION.
#include "../../include/hankel_b200.h"
#include "hk_items.cuh"
#include "moments_dev.cuh"
#include "tc_bulk.cuh"
#include "tc_pair.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h> // types only; libnccl.so.2 is dlopen'ed (multi-GPU section)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

extern "C" int hk_moments_impl(unsigned, unsigned, int, int, uint32_t*, int32_t*, int32_t*, int*, const char**);
extern "C" int hk_block_eigs_impl(int, int, const uint32_t*, const int32_t*, const int32_t*, int, double*, double*,
                                  double*, const char**);

namespace {

using hk::Meta;
using hk::MpArr;

template <class F>
__global__ void __launch_bounds__(256) k_items(long long n, int ws_words, F f) {
    extern __shared__ uint32_t smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory"); // see launch_ex (no-op for ordinary launches)
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* ws = smem + (size_t)wib * ws_words;
    const long long nw = (long long)gridDim.x * wpb;
    for (long long it = (long long)blockIdx.x * wpb + wib; it < n; it += nw) f(it, ws);
}

struct HkError {
    int code;
    std::string msg;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw HkError{HK_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e)};
}

// Launch through cudaLaunchKernelEx, optionally with programmatic stream
// serialization (the kernel must begin with griddepcontrol.wait before it
// reads its same-stream predecessor's outputs).
template <class K, class... Args>
void launch_ex(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
    if (e != cudaSuccess) throw HkError{HK_ERR_RUNTIME, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

// Dynamic shared-memory limit (>= 48 KB) and the maximal carveout of kernel
// `fn`, set once per (device, kernel): the attribute belongs to the current
// device's context, so a process driving several GPUs sets it on each.
void func_smem(const void* fn, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    const size_t v = smem < 48 * 1024 ? 48 * 1024 : smem;
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[{dev, fn}];
    if (cur >= v) return;
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(v)), "cudaFuncSetAttribute");
    // every kernel asks for the same (maximal) shared-memory carveout, so the
    // critical-path CTAs can start on SMs busy with bulk work without an L1/smem
    // reconfiguration (which waits for the SM to drain)
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
    cur = v;
}

// Stream capture that always ends: if recording throws, the capture (and every
// stream forked into it) is closed and the partial graph dropped, so the
// context stays usable after a failed launch.
struct Capture {
    cudaStream_t st;
    bool open = false;
    explicit Capture(cudaStream_t s) : st(s) {
        ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
        open = true;
    }
    cudaGraph_t end() {
        cudaGraph_t g = nullptr;
        open = false;
        ck(cudaStreamEndCapture(st, &g), "end capture");
        return g;
    }
    ~Capture() {
        if (!open) return;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError(); // clear the sticky-free capture error
    }
};

cudaGraphExec_t instantiate(cudaGraph_t g, unsigned long long flags) {
    cudaGraphExec_t ge = nullptr;
    const cudaError_t e = cudaGraphInstantiateWithFlags(&ge, g, flags);
    cudaGraphDestroy(g);
    ck(e, "graph instantiate");
    return ge;
}

// D_i = S(i, i) of the jagged triangle -> contiguous out[0..N) (one copy back)
__global__ void k_gather_diag(MpArr S, MpArr out, int N, int L) {
    const long long e = hk::tri_idx(int(blockIdx.x), int(blockIdx.x), N);
    for (int q = threadIdx.x; q < L; q += blockDim.x) out.limbs(blockIdx.x, L)[q] = S.limbs(e, L)[q];
    if (threadIdx.x == 0) out.m[blockIdx.x] = S.m[e];
}

struct DevArr {
    uint32_t* d = nullptr;
    Meta* m = nullptr;
    long long cap = 0;
    int L = 0;
    void ensure(long long n, int limbs) {
        if (n <= cap && limbs == L) return;
        release();
        ck(cudaMalloc(&d, size_t(n) * limbs * sizeof(uint32_t)), "cudaMalloc limbs");
        ck(cudaMalloc(&m, size_t(n) * sizeof(Meta)), "cudaMalloc meta");
        cap = n;
        L = limbs;
    }
    void release() {
        if (d) cudaFree(d);
        if (m) cudaFree(m);
        d = nullptr;
        m = nullptr;
        cap = 0;
    }
    MpArr view() const { return MpArr{d, m}; }
};

} // namespace

struct hk_ctx {
    int device = 0;
    int L = 0;
    int n = 0, m = 0, k = 0;
    cudaStream_t st = nullptr;  // bulk / default stream of the context
    cudaStream_t st2 = nullptr; // high-priority look-ahead stream
    cudaStream_t st3 = nullptr; // high-priority: off-diagonal part of the look-ahead column
    cudaStream_t st4 = nullptr; // side stream: StoreL (L in place), off both critical streams
    cudaStream_t st5 = nullptr; // L^-1 steps interleaved with the LDLT (hk_ldlt_invert)
    cudaEvent_t evJoin4 = nullptr, evMid = nullptr; // its join; end of the LDLT proper (timing split)
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    std::vector<cudaEvent_t> evP, evR, evU, evD, evO, evC, evB1; // per-step dependencies (graph capture)
    cudaEvent_t evJoin2 = nullptr, evJoin3 = nullptr;
    DevArr mu, S, R, B, X, Y, T, T2, M, Dg, Vf; // Vf: unscaled columns of the dataflow LDLT
    int* d_err = nullptr;
    std::string err;
    int bad_col = -1;
    bool factored = false, inverted = false, assembled = false;
    bool dist_factored = false; // this rank took part in a sharded factorisation (all ranks)
    int sm_count = 148;
    size_t smem_optin = 227 * 1024;  // cudaDevAttrMaxSharedMemoryPerBlockOptin
    long long launches = 0;
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // LDLT graph cache keyed by n
    std::map<int, cudaGraphExec_t> graphs;
    std::map<int, long long> graph_launches;
    std::vector<const void*> graph_sig;                      // buffers / modes the graphs were captured on
    std::map<long long, cudaGraphExec_t> inv_graphs;         // L^{-1} step graphs keyed by (n, m)
    std::map<long long, long long> inv_graph_launches;
    std::vector<const void*> inv_sig;                        // buffers / modes they were captured on
    std::vector<uint32_t> h_limbs;
    std::vector<int32_t> h_e, h_s;
    // ---- kernel timing inside the captured graphs (external event-record nodes)
    bool kprof = false;                 // hk_set_kernel_timing: events around every step's bulk kernels
    std::vector<cudaEvent_t> kev;       // 3 per LDLT step: before products, after products, after rounding
    int kev_steps = 0;                  // steps recorded in the LDLT graph launched last
    std::map<int, int> kev_steps_by_n;  // ... per cached graph (keyed by n)
    std::vector<cudaEvent_t> cev;       // sharded: 2 per step around the pivot-column broadcast (always on)
    int cev_steps = 0;
    // ---- tensor-core bulk products (large p): scratch of short products
    uint32_t* tc_P = nullptr;
    size_t tc_P_words = 0;
    size_t tc_fb_cap = 0;         // fix-up list capacity (items)
    uint8_t* tc_A = nullptr;      // preformatted A operand of the current step
    int tc_A_n = 0;               // rows it was sized for
    uint64_t* tc_gcarry = nullptr; // L^-1 chunk-group carries
    cudaEvent_t prof_mid = nullptr; // hk_profile_ldlt: recorded between TC products and rounding
    int* tc_fb_count = nullptr;   // uncertified items: [0] / [1] by step parity, [2] sharded path
    long long* tc_fb = nullptr;
    int* flow_ready = nullptr;    // dataflow L^-1: per-entry flags + entry counter
    long long flow_cap = 0;
    // L^-1 tensor-core steps riding in the LDLT graph: their own A operand, redo list and counters
    uint8_t* inv_A = nullptr;
    int inv_A_n = 0;
    long long* inv_fb = nullptr;
    size_t inv_fb_cap = 0;
    int* inv_fb_count = nullptr;
    int* lflow = nullptr;         // dataflow LDLT: control words, per-entry flags, per-column counts
    long long lflow_cap = 0;      // entries it was sized for
    // ---- sharded (multi-GPU) state; world == 1 means the single-GPU path
    struct Shard {
        int rank = 0;
        std::vector<int> owned;       // global columns owned, ascending
        std::vector<long long> off;   // local entry offset of each owned column (+ total)
        std::vector<int> loc;         // global column -> local index, -1 if not owned
        DevArr S, panel, R, B;
        int* d_erow = nullptr;
        int* d_ecol = nullptr;
        int* d_err = nullptr;
        int* d_owned = nullptr;      // tensor-core path: owned columns / local offsets on the device
        long long* d_off = nullptr;
        int* d_fb = nullptr;         // uncertified-item counters of this shard, by step parity
        int setup_n = -1;            // order the maps / buffers were built for
        // sharded L^-1 / block (row blocks b % world == rank): X (all rows arrive, only
        // owned ones are computed here), block buffers, owned row tiles
        DevArr X, Y, T, T2;
        std::vector<int> otiles;
        int* d_otiles = nullptr;
        int rows_n = -1;
    };
    cudaGraphExec_t dist_graph = nullptr; // sharded LDLT step graph (look-ahead, NCCL captured)
    long long dist_graph_launches = 0;
    std::vector<const void*> dist_sig;    // buffers it was captured on
    int world = 1, rank = 0;
    bool virt = false;               // all `world` ranks emulated in this one context
    void* nccl_comm = nullptr;       // ncclComm_t (one rank per process)
    void* bcast_buf = nullptr;       // device staging of the root's result broadcast
    unsigned long long* dev_cnt = nullptr; // dev what-if counters (HK_DEV_TCB bit 64)
    unsigned long long* fix_total = nullptr; // items the certified rounding left to the exact redo (all steps)
    std::vector<Shard> shards;
    std::vector<int> owner;          // assign_columns(n, world), or a caller's map (hk_set_owner_map)
    bool owner_custom = false;
    long long owner_version = 0;     // bumped when the map changes (the step graph depends on it)
};

namespace {

int ws_op_words(int L) { return hk::opws_words(L); }
int ws_recip_words(int L) { return hk::recipws_words(L); }

// One warp per item, one short-lived block per `wpb` items (no grid-stride
// persistence), so blocks of the high-priority look-ahead stream are
// dispatched as soon as any bulk block retires.
template <class F>
void launch(hk_ctx* c, const F& f, long long n, int ws_words, cudaStream_t st = nullptr, bool pdl = false) {
    if (n <= 0) return;
    if (!st) st = c->st;
    const size_t per_warp = size_t(ws_words) * sizeof(uint32_t);
    int wpb = int((96 * 1024) / per_warp);
    if (wpb > 8) wpb = 8;
    if (wpb < 1) wpb = 1;
    if ((long long)wpb > n) wpb = int(n);
    const size_t smem = per_warp * wpb;
    // all of the unified L1/shared array as shared memory: residency is then
    // register-bound (5 x 256-thread blocks at <= 48 registers)
    func_smem((const void*)&k_items<F>, smem);
    long long blocks = (n + wpb - 1) / wpb;
    const long long cap = 1LL << 30;
    if (blocks > cap) blocks = cap;
    launch_ex(k_items<F>, dim3(unsigned(blocks)), dim3(unsigned(32 * wpb)), smem, st, pdl, n, ws_words, f);
    ck(cudaGetLastError(), "kernel launch");
    ++c->launches;
}

// The paired bulk update (hot kernel) with a residency bound on registers.
template <class F>
__global__ void __launch_bounds__(256, HK_TRAILING2_MINB) k_items_hot(long long n, int ws_words, F f) {
    extern __shared__ uint32_t smem[];
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* ws = smem + (size_t)wib * ws_words;
    const long long nw = (long long)gridDim.x * wpb;
    for (long long it = (long long)blockIdx.x * wpb + wib; it < n; it += nw) f(it, ws);
}

template <class F>
void launch_hot(hk_ctx* c, const F& f, long long n, int ws_words, cudaStream_t st = nullptr) {
    if (n <= 0) return;
    if (!st) st = c->st;
    const size_t per_warp = size_t(ws_words) * sizeof(uint32_t);
    int wpb = int((96 * 1024) / per_warp);
    if (wpb > 8) wpb = 8;
    if (wpb < 1) wpb = 1;
    if ((long long)wpb > n) wpb = int(n);
    const size_t smem = per_warp * wpb;
    func_smem((const void*)&k_items_hot<F>, smem);
    const long long blocks = (n + wpb - 1) / wpb;
    k_items_hot<F><<<unsigned(blocks), unsigned(32 * wpb), smem, st>>>(n, ws_words, f);
    ck(cudaGetLastError(), "kernel launch");
    ++c->launches;
}

// One item per CTA (all warps cooperate on it): the critical-path ops.
template <class F>
__global__ void __launch_bounds__(256) k_cta_items(long long n, F f) {
    extern __shared__ __align__(16) uint32_t cta_smem[];
    // programmatic dependent launch (the look-ahead chain): this grid may be
    // launched before its predecessor finishes; wait for it before any read
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (long long it = blockIdx.x; it < n; it += gridDim.x) {
        f(it, cta_smem);
        __syncthreads();
    }
}

constexpr int kCtaThreads = 256;

template <class F>
void launch_cta(hk_ctx* c, const F& f, long long n, int ws_words, cudaStream_t st = nullptr, bool pdl = false) {
    if (n <= 0) return;
    if (!st) st = c->st;
    const size_t smem = size_t(ws_words) * sizeof(uint32_t);
    func_smem((const void*)&k_cta_items<F>, smem);
    const long long blocks = n < (1LL << 30) ? n : (1LL << 30);
    if (pdl) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(blocks));
        cfg.blockDim = dim3(kCtaThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ck(cudaLaunchKernelEx(&cfg, k_cta_items<F>, n, f), "kernel launch (PDL)");
    } else {
        k_cta_items<F><<<unsigned(blocks), kCtaThreads, smem, st>>>(n, f);
    }
    ck(cudaGetLastError(), "kernel launch");
    ++c->launches;
}

int ws_cta_words(int L) { return hk::ctaws_words(L); }
int ws_cta_recip_words(int L) { return hk::ctarecipws_words(L); }

// R_i = RNE(1/S_ii) (+ the pivot test): the CTA-cooperative reciprocal (the
// critical path), or one warp's when its workspace does not fit a CTA's shared
// memory (p beyond ~114,900 bits)
void launch_recip(hk_ctx* c, int i, cudaStream_t st, bool pdl = false) {
    const int N = c->n, L = c->L;
    if (size_t(ws_cta_recip_words(L)) * 4 <= c->smem_optin)
        launch_cta(c, hk::CItemRecip{c->S.view(), c->R.view(), N, L, i, c->d_err}, 1, ws_cta_recip_words(L), st, pdl);
    else
        launch(c, hk::ItemRecip{c->S.view(), c->R.view(), N, L, i, c->d_err}, 1, ws_recip_words(L), st, pdl);
}

int fail(hk_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

template <class Fn>
int guarded(hk_ctx* c, Fn&& fn) {
    if (!c) return HK_ERR_INVALID;
    try {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        return fn();
    } catch (const HkError& e) {
        return fail(c, e.code, e.msg);
    } catch (const std::exception& e) {
        return fail(c, HK_ERR_RUNTIME, e.what());
    }
}

void h2d_soa(hk_ctx* c, DevArr& a, long long n, const uint32_t* l, const int32_t* e, const int32_t* s) {
    a.ensure(n, c->L);
    ck(cudaMemcpyAsync(a.d, l, size_t(n) * c->L * sizeof(uint32_t), cudaMemcpyHostToDevice, c->st), "H2D limbs");
    std::vector<Meta> hm(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) hm[size_t(i)] = Meta{e[i], s[i]};
    ck(cudaMemcpyAsync(a.m, hm.data(), size_t(n) * sizeof(Meta), cudaMemcpyHostToDevice, c->st), "H2D meta");
    ck(cudaStreamSynchronize(c->st), "sync");
}

void d2h_range(hk_ctx* c, const DevArr& a, long long first, long long n, uint32_t* l, int32_t* e, int32_t* s) {
    const int L = c->L;
    std::vector<Meta> hm(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(l, a.d + first * L, size_t(n) * L * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->st), "D2H");
    ck(cudaMemcpyAsync(hm.data(), a.m + first, size_t(n) * sizeof(Meta), cudaMemcpyDeviceToHost, c->st), "D2H meta");
    ck(cudaStreamSynchronize(c->st), "sync");
    for (long long i = 0; i < n; ++i) {
        e[i] = hm[size_t(i)].exp;
        s[i] = hm[size_t(i)].sign;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// B_i lives in buffer i % 3: B_{i+1} is produced while B_i is still read, and
// the copy of B_{i-1} into column i-1 (StoreL) trails one step behind.
MpArr b_buf(hk_ctx* c, int i) {
    const long long off = (long long)(i % 3) * c->n;
    return MpArr{c->B.d + off * c->L, c->B.m + off};
}

// Record the n LDLT steps with depth-1 look-ahead (ldlt.cpp:271-331) on two
// streams (captured into one graph):
//   LA   (high priority): P(i+1) = update column i+1 with step i, R_{i+1} = recip,
//                         B_{i+1} = column * R_{i+1}          — the latency chain
//   BULK (ctx stream)   : U(i) = step-i update of columns i+2..N-1, then
//                         STORE(i): column i <- B_i (L in place)
// U(i) needs B_i (end of P(i)); P(i+1) needs column i+1 after step i-1 (end of
// U(i-1)+STORE(i-1)); STORE(i) needs P(i+1) to have read S(i+1,i).  So P(i+1)
// overlaps U(i) and the critical path per step is max(U(i), P(i+1)).
// Tensor-core products for the bulk update?  Default: when p >= 4096 bits and
// the per-CTA shared memory fits; HK_TC=0/1 forces it off/on (tests, sweeps).
// L^-1 steps are narrower (b <= m columns per step): there the tensor cores pay
// from p >= 12288 bits (measured: C2 5.1 ms IMAD vs 7.4 ms TC, C3 459 vs 107 ms).
bool use_tc(const hk_ctx* c) {
    const int L = c->L;
    if (L % 4 != 0 || hk::tc_smem_bytes(L, hk::tc_ewin(L)) > 220 * 1024) return false;
    if (const char* e = getenv("HK_TC")) return e[0] == '1';
    return L >= 128;
}
// Dev-only what-if timing (tools/gpu_whatif.sh): HK_DEV_SKIP="recip,round,..."
// drops those launches from the captured LDLT graph (results are then wrong;
// no test or bench sets it) to see which stream bounds the step time.
bool dev_skip(const char* what) {
    static const char* e = getenv("HK_DEV_SKIP");
    return e && strstr(e, what);
}

// Tests only (HK_TC_FORCE_FIX=1): the rounding passes hand every 7th certified
// item to the exact fix-up kernel too, so that path is exercised and checked.
bool force_fix() {
    const char* e = getenv("HK_TC_FORCE_FIX");
    return e && e[0] == '1';
}

// The certified rounding fused into the product kernel's epilogue (LDLT bulk
// steps; tc_fused.cuh).  HK_TC_FUSE=0 keeps the separate rounding pass.
bool use_fuse(const hk_ctx* c) {
    if (!hk::tc_fusable(c->L)) return false;
    const char* e = getenv("HK_TC_FUSE");
    return !e || e[0] != '0';
}

// which fused stream: HK_TC_FUSE_WARP=1 the warp-cooperative one (tc_fused.cuh warp_row_*)
int fuse_mode() {
    const char* e = getenv("HK_TC_FUSE_WARP");
    return e && e[0] == '1' ? 2 : 1;
}

// The fused products on CTA pairs (tc_pair.cuh) — an experiment, off by default:
// a cta_group::2 TMEM kernel runs one CTA per SM, and measured 2x slower at C4
// than two single-CTA kernels per SM.  HK_TC_PAIR=1 selects it.
bool use_pair(const hk_ctx* c) {
    if (!use_fuse(c) || !hk::tcp_ok(c->L)) return false;
    const char* e = getenv("HK_TC_PAIR");
    return e && e[0] == '1';
}

bool use_tc_inv(const hk_ctx* c) {
    if (!use_tc(c)) return false;
    if (getenv("HK_TC")) return true;
    return c->L >= 384;
}

// A operand preformat + the tcgen05 product kernel (one CTA per SM: it owns all
// 512 TMEM columns).  `rows` is the row-operand source (ItemTcPrep).
void tc_products(hk_ctx* c, hk::TcBulkArgs a, hk::MpArr rows, unsigned gx, cudaStream_t st, bool pdl = false,
                 int gy = -1, int prep_panel = 0) {
    const int N = c->n, L = c->L;
    // Windowed x expansion (93-103 KB of shared memory for any p) and one TMEM
    // accumulator: two CTAs per SM, one CTA's prologue and epilogue overlap the
    // other's MMAs (LDLT and L^-1 alike; L^-1 splits each product's chunks into
    // groups to fill that one wave: C4 L^-1 288 -> 222 ms against one CTA per SM
    // with two accumulators).  HK_TC_EWIN / HK_TC_NACC force the other variants.
    a.ewin = 1;
    if (const char* e = getenv("HK_TC_EWIN")) a.ewin = e[0] == '1' ? 1 : 0;
    if (a.fuse) a.ewin = 1;
    if (a.fuse) a.stages = hk::tc_fused_stages(L); // 3 (2 when p is so large that 3 would not fit two CTAs)
    if (const char* e = getenv("HK_TC_STAGES")) a.stages = std::max(2, std::min(hk::kTcStages, atoi(e)));
    const size_t need = hk::tc_smem_bytes(L, a.ewin != 0, a.fuse != 0, a.stages);
    a.nacc = need <= 113 * 1024 ? 1 : 2;
    if (const char* e = getenv("HK_TC_NACC")) a.nacc = e[0] == '1' ? 1 : 2;
    const size_t smem = a.nacc == 1 ? need : std::max(need, size_t(120 * 1024));
    func_smem((const void*)hk::k_tc_bulk, 220 * 1024);
    func_smem((const void*)hk::k_tc_prep, 0);
    static const char* dv = getenv("HK_DEV_TCB"); // dev what-if (tools only): bits of TcBulkArgs::dev
    a.dev = dv ? atoi(dv) : 0;
    if (a.dev & 64) a.dev_cnt = c->dev_cnt; // dev: issuer wait-cycle counters (hk_create), printed by hk_destroy
    const char* sl = getenv("HK_TC_SLEEP"); // barrier-poll back-off (ns) of the non-issuing warps
    a.sleep_ns = sl ? atoi(sl) : 0;
    hk::ItemTcPrep prep{rows, const_cast<uint8_t*>(a.A), N, L, a.i, a.mode};
    prep.panel = prep_panel;
    const long long nprep = prep.count();
    launch_ex(hk::k_tc_prep, dim3(unsigned((nprep + 255) / 256)), dim3(256), 0, st, pdl, prep, nprep);
    ck(cudaGetLastError(), "tc prep launch");
    ++c->launches;
    if (a.fuse && a.mode != 1 && use_pair(c)) { // CTA pairs: cluster (1, 2, 1) over row-tile pairs
        a.stages = hk::tcp_stages(L);
        if (const char* e = getenv("HK_TC_PAIR_STAGES")) a.stages = std::max(2, std::min(hk::kTcStagesMax, atoi(e)));
        const size_t ps = hk::tcp_smem_bytes(L, a.stages);
        func_smem((const void*)hk::k_tc_pair, ps);
        const int first_row = a.jfirst;
        const int tiles = hk::tc_ntiles(N) - first_row / hk::kTcRows;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(2 * ((tiles + 1) / 2)), gx, 1);
        cfg.blockDim = dim3(hk::kTcThreads);
        cfg.dynamicSmemBytes = ps;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 2 : 1;
        if (a.dev & 128) { // dev: occupancy of the pair kernel, once
            static bool told = false;
            if (!told) {
                told = true;
                int ncl = -1;
                cudaLaunchConfig_t c2 = cfg;
                c2.numAttrs = 1;
                cudaOccupancyMaxActiveClusters(&ncl, hk::k_tc_pair, &c2);
                cudaFuncAttributes fa{};
                cudaFuncGetAttributes(&fa, hk::k_tc_pair);
                fprintf(stderr, "k_tc_pair: %d active clusters max, smem %zu + static %zu, regs %d, stages %d\n", ncl, ps,
                        fa.sharedSizeBytes, fa.numRegs, a.stages);
            }
        }
        const cudaError_t le = cudaLaunchKernelEx(&cfg, hk::k_tc_pair, a);
        if (le != cudaSuccess) {
            cudaGetLastError();
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, hk::k_tc_pair);
            int ncl = -1;
            cfg.numAttrs = 1;
            const cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, hk::k_tc_pair, &cfg);
            throw HkError{HK_ERR_RUNTIME,
                          std::string("tc pair launch: ") + cudaGetErrorString(le) + " (grid " +
                              std::to_string(cfg.gridDim.x) + "x" + std::to_string(cfg.gridDim.y) + ", smem " +
                              std::to_string(ps) + ", static " + std::to_string(fa.sharedSizeBytes) + ", regs " +
                              std::to_string(fa.numRegs) + ", maxdyn " + std::to_string(fa.maxDynamicSharedSizeBytes) +
                              ", reqcluster " + std::to_string(fa.requiredClusterWidth) + "x" +
                              std::to_string(fa.requiredClusterHeight) + ", occupancy " + std::to_string(ncl) + " " +
                              cudaGetErrorString(oe) + ")"};
        }
        ++c->launches;
        return;
    }
    const int first_row = a.mode != 1 ? a.jfirst : a.i + 1;
    const dim3 grid(gx, unsigned(gy >= 0 ? gy : hk::tc_ntiles(N) - first_row / hk::kTcRows), unsigned(a.groups));
    launch_ex(hk::k_tc_bulk, grid, dim3(hk::kTcThreads), smem, st, pdl, a);
    ck(cudaGetLastError(), "tc bulk launch");
    ++c->launches;
}

// Per-(column, row) items over `ncols` columns of at most `maxrows` rows (k_cols).
template <class F>
void launch_cols(hk_ctx* c, const F& f, int ncols, int maxrows, int ws_words, cudaStream_t st, bool pdl = false) {
    if (ncols <= 0 || maxrows <= 0) return;
    const size_t per_warp = size_t(ws_words) * sizeof(uint32_t);
    int wpb = int((96 * 1024) / per_warp);
    wpb = std::max(1, std::min(8, wpb));
    const size_t smem = per_warp * wpb;
    func_smem((const void*)hk::k_cols<F>, 96 * 1024);
    const unsigned gx = unsigned((maxrows + wpb - 1) / wpb);
    launch_ex(hk::k_cols<F>, dim3(gx, unsigned(ncols)), dim3(unsigned(32 * wpb)), smem, st, pdl, f, ws_words);
    ck(cudaGetLastError(), "cols launch");
    ++c->launches;
}

// Exact redo of the items the rounding pass could not certify (device-side count).
template <class F>
void launch_fix(hk_ctx* c, const F& f, cudaStream_t st, int* count, int* reset, bool pdl = false,
                const long long* fb = nullptr) {
    const int wo = ws_op_words(c->L);
    const int wpb = std::max(1, std::min(8, int((96 * 1024) / (wo * 4))));
    func_smem((const void*)hk::k_tc_fix<F>, 200 * 1024);
    launch_ex(hk::k_tc_fix<F>, dim3(unsigned(c->sm_count)), dim3(unsigned(32 * wpb)), size_t(wo) * 4 * wpb, st, pdl, f,
              (const int*)count, fb ? fb : (const long long*)c->tc_fb, wo, reset, c->fix_total);
    ck(cudaGetLastError(), "tc fix launch");
    ++c->launches;
}

void grow_events(std::vector<cudaEvent_t>& v, size_t n, unsigned flags) {
    while (v.size() < n) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, flags), "event");
        v.push_back(e);
    }
}

// an event-record node of the graph being captured on `st` (timing events)
void graph_event(cudaEvent_t e, cudaStream_t st) {
    ck(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "event record node");
}

float event_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, a, b), "elapsed");
    return ms;
}

// Step-i update of columns jfirst..N-1 (bulk): IMAD paired warp FMAs, or the
// tcgen05 product kernel followed by the certified rounding pass.  kslot >= 0:
// timing events kev[3 kslot ..] around the products and the rounding pass.
void enqueue_bulk(hk_ctx* c, int i, int jfirst, cudaStream_t st, bool pdl = false, int kslot = -1) {
    const int N = c->n, L = c->L;
    const int ncols = N - jfirst;
    if (ncols <= 0) return;
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot)], st);
    if (!use_tc(c)) {
        launch_hot(c, hk::ItemTrailing2{c->S.view(), b_buf(c, i), N, L, i, jfirst, c->d_err},
                   hk::trailing2_items(N, jfirst), hk::opws2_words(L), st);
        if (kslot >= 0) {
            graph_event(c->kev[size_t(3 * kslot + 1)], st);
            graph_event(c->kev[size_t(3 * kslot + 2)], st);
        }
        return;
    }
    // fallback counters alternate by step: the fix-up of step i clears the one step i+1 uses
    int* cnt = c->tc_fb_count + (i & 1);
    int* nxt = c->tc_fb_count + ((i + 1) & 1);
    hk::TcBulkArgs ta{c->S.view(), hk::MpArr{}, c->tc_A, c->tc_P, N, L, i, jfirst, 0, 0, 0, c->d_err};
    const bool fuse = use_fuse(c);
    if (fuse) {
        ta.fuse = fuse_mode();
        ta.Y = b_buf(c, i);
        ta.fb_count = cnt;
        ta.fb = c->tc_fb;
        ta.force_fb = force_fix();
        ta.viol = c->tc_fb_count + 3;
    }
    if (!dev_skip("prod")) tc_products(c, ta, b_buf(c, i), unsigned(ncols), st, pdl);
    if (c->prof_mid) ck(cudaEventRecord(c->prof_mid, st), "prof mid");
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot + 1)], st);
    hk::ItemTcRound ri{c->S.view(), b_buf(c, i), c->tc_P, N, L, i, jfirst, c->d_err, cnt, c->tc_fb};
    static const char* rd = getenv("HK_ROUND_DIRECT");
    ri.direct = !rd || rd[0] == '1';
    ri.force_fb = force_fix();
    if (!fuse && !dev_skip("round"))
        launch_cols(c, ri, ncols, ncols, ri.direct ? hk::align4(L + 16) : hk::tcround_words(L), st, pdl);
    if (!dev_skip("fix")) launch_fix(c, hk::FixLdlt{c->S.view(), b_buf(c, i), N, L, i, jfirst}, st, cnt, nxt, pdl);
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot + 2)], st);
}

// Where an L^-1 step reads and writes (one GPU: S and X; a sharded rank: the
// panel of column i, its X, its rows and row tiles)
struct InvTarget {
    hk::MpArr Lsrc;             // L(:, i): S (tri_idx) or the panel (j - i)
    int panel = 0;
    hk::MpArr X;
    int rw = 1, rr = 0;         // row blocks of this rank (hk::row_mine)
    const int* otiles = nullptr; // device list of this rank's row tiles with rows > i (tc path)
    int ntiles = -1;
    // steps riding in the LDLT graph: buffers of their own (the LDLT's are in use) and the error gate
    uint8_t* A = nullptr;
    int* fb_count = nullptr;
    long long* fb = nullptr;
    const int* err = nullptr;
};

// L^-1 step i on the tensor cores (same product kernel, mode 1).
void enqueue_inv_tc(hk_ctx* c, int i, cudaStream_t st, bool pdl = false, const InvTarget* tg = nullptr) {
    const int N = c->n, L = c->L, m = c->m;
    const int b = i < m ? i : m;
    if (i + 1 >= N) return;
    InvTarget one;
    if (!tg) {
        one.Lsrc = c->S.view();
        one.X = c->X.view();
        tg = &one;
    }
    // narrow step: split each product's output chunks over G CTAs (carries joined in the rounding pass)
    const int tiles = tg->ntiles >= 0 ? tg->ntiles : hk::tc_ntiles(N) - (i + 1) / hk::kTcRows;
    // two CTAs per SM (windowed expansion, one accumulator): keep the split to a
    // single wave — rounding the group count up made a second, mostly empty wave
    int G = b > 0 && tiles > 0 ? 2 * c->sm_count / (b * tiles) : 1;
    G = std::min(G, std::min(int(hk::kTcMaxGroups), hk::tc_nchunks(L) / 2));
    if (G < 1) G = 1;
    if (b > 0 && tiles > 0) {
        hk::TcBulkArgs a{hk::MpArr{}, tg->X, tg->A ? tg->A : c->tc_A, c->tc_P, N, L, i, i + 1, 1, m, b, c->d_err};
        a.groups = G;
        a.gcarry = c->tc_gcarry;
        a.otiles = tg->otiles;
        a.inv_gate = tg->err ? 1 : 0;
        tc_products(c, a, tg->Lsrc, unsigned(b), st, pdl, tg->ntiles, tg->panel);
    }
    int* fbc = tg->fb_count ? tg->fb_count : c->tc_fb_count;
    long long* fbl = tg->fb ? tg->fb : c->tc_fb;
    int* cnt = fbc + (i & 1);
    int* nxt = fbc + ((i + 1) & 1);
    const long long items = (long long)(N - i - 1) * b + (i < m ? N - i - 1 : 0);
    hk::ItemTcRoundInv ri{tg->Lsrc, tg->X, c->tc_P, N, L, m, i, b, cnt, fbl};
    ri.err = tg->err;
    ri.G = G;
    ri.gcarry = c->tc_gcarry;
    ri.force_fb = force_fix();
    ri.panel = tg->panel;
    ri.rw = tg->rw;
    ri.rr = tg->rr;
    launch(c, ri, items, hk::tcround_words(L), st, pdl);
    if (b > 0) {
        hk::FixInv fx{tg->Lsrc, tg->X, N, L, m, i, b};
        fx.panel = tg->panel;
        launch_fix(c, fx, st, cnt, nxt, pdl, fbl);
    } else {
        ck(cudaMemsetAsync(nxt, 0, sizeof(int), st), "memset fb");
    }
}

// ---- L^{-1} as a dataflow (small p, IMAD path): one CTA per entry X(j,c),
// c < min(j, m), runs that entry's whole chain of the reference's row
// elimination (inversion.cpp:93-102) in order:
//     X(j,c) = -L(j,c);  for i = c+1 .. j-1:  X(j,c) = RNE(X(j,c) - L(j,i) X(i,c))
// waiting for X(i,c) to be final (a per-entry flag, release/acquire at gpu
// scope).  The per-entry order of the roundings is the reference's, so the
// result is bit-identical to the N-step schedule; the N dependent launches
// (latency-bound: a few hundred FMAs per step at C2) become one kernel whose
// critical path is the c = 0 column, one FMA + one flag hand-off per row.
// Entries are taken from a global counter in increasing (row-major) order, so
// a CTA only ever waits on entries already held by running CTAs: no
// deadlock whatever the residency.
struct InvFlowArgs {
    MpArr S, X;
    int N, L, m;
    int* ready;                 // [N * m] 0 pending / 1 final (cleared per run)
    unsigned long long* next;   // entry counter (cleared per run)
    long long E;                // entries: sum_j min(j, m)
    int ws_words;
    int fstride;                // flag stride in ints (a 128-byte line per flag: no false sharing)
    int sleep_ns;               // poll back-off
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// entry e -> (j, c): rows 1..m-1 hold j entries, rows >= m hold m
__device__ __forceinline__ void inv_flow_decode(long long e, int m, int& j, int& c) {
    const long long t0 = (long long)m * (m - 1) / 2;
    if (e >= t0) {
        j = m + int((e - t0) / m);
        c = int((e - t0) % m);
        return;
    }
    int jj = int((1.0 + sqrt(1.0 + 8.0 * double(e))) * 0.5);
    while ((long long)jj * (jj - 1) / 2 > e) --jj;
    while ((long long)(jj + 1) * jj / 2 <= e) ++jj;
    j = jj;
    c = int(e - (long long)jj * (jj - 1) / 2);
}

// One CTA per entry (cta_fms: the products on all 8 warps — the per-entry chain
// is latency-bound, a warp per entry measured 2x slower at C2).
// 3 warps per entry (C2 invL: 256 threads 3.67 ms, 128 3.14, 96 2.99; capping
// registers so that every C2 entry is resident at once spilled: 4.31 ms)
constexpr int kFlowThreads = 96;
__global__ void __launch_bounds__(256) k_inv_flow_cta(InvFlowArgs a) {
    extern __shared__ __align__(16) uint32_t fsm2_[];
    __shared__ unsigned long long e_s;
    const int L = a.L, m = a.m, N = a.N, tid = int(threadIdx.x);
    uint32_t* acc = fsm2_;
    uint32_t* xs = acc + hk::align4(L);
    uint32_t* ws = xs + hk::align4(L);
    for (;;) {
        if (tid == 0) e_s = atomicAdd(a.next, 1ull);
        __syncthreads();
        const unsigned long long e = e_s;
        __syncthreads();
        if ((long long)e >= a.E) return;
        int j, c;
        inv_flow_decode((long long)e, m, j, c);
        const long long el = hk::tri_idx(j, c, N);
        for (int q = tid; q < L; q += blockDim.x) acc[q] = a.S.limbs(el, L)[q];
        Meta am = a.S.m[el];
        am.sign = -am.sign;
        __syncthreads();
        for (int i = c + 1; i < j; ++i) {
            const long long xi = (long long)i * m + c;
            if (tid == 0)
                while (ld_acquire_gpu(a.ready + xi * a.fstride) == 0) __nanosleep(a.sleep_ns);
            __syncthreads();
            for (int q = tid; q < L; q += blockDim.x) xs[q] = __ldcg(a.X.limbs(xi, L) + q);
            const int2 xm2 = __ldcg(reinterpret_cast<const int2*>(a.X.m + xi));
            __syncthreads();
            const long long eli = hk::tri_idx(j, i, N);
            am = hk::cta_fms(acc, am, a.S.limbs(eli, L), a.S.m[eli], xs, Meta{xm2.x, xm2.y}, acc, L,
                             hk::ctaws_carve(ws, L));
            __syncthreads();
        }
        const long long xd = (long long)j * m + c;
        for (int q = tid; q < L; q += blockDim.x) a.X.limbs(xd, L)[q] = acc[q];
        if (tid == 0) a.X.m[xd] = am;
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release_gpu(a.ready + xd * a.fstride, 1);
    }
}

constexpr int kFlowStride = 32; // one 128-byte line per flag

// flags + counter of the dataflow L^{-1}, (re)sized for n*m entries
void ensure_inv_flow(hk_ctx* c, long long nm) {
    if (c->flow_cap >= nm) return;
    if (c->flow_ready) cudaFree(c->flow_ready);
    c->flow_ready = nullptr;
    ck(cudaMalloc(&c->flow_ready, size_t(nm) * kFlowStride * sizeof(int) + 16), "cudaMalloc flow flags");
    c->flow_cap = nm;
}

void enqueue_inv_flow(hk_ctx* c, cudaStream_t st) {
    const int N = c->n, L = c->L, m = c->m;
    const long long nm = (long long)N * m;
    long long E = 0;
    for (int j = 1; j < N; ++j) E += j < m ? j : m;
    unsigned long long* next = reinterpret_cast<unsigned long long*>(c->flow_ready + nm * kFlowStride);
    ck(cudaMemsetAsync(c->flow_ready, 0, size_t(nm) * kFlowStride * sizeof(int) + 8, st), "memset flow flags");
    if (E == 0) return;
    const char* sl = getenv("HK_FLOW_SLEEP");
    const int sleep_ns = sl ? atoi(sl) : 100;
    const int wsw = 2 * hk::align4(L) + hk::ctaws_words(L);
    const size_t smem = size_t(wsw) * sizeof(uint32_t);
    func_smem((const void*)k_inv_flow_cta, 200 * 1024);
    const int threads = kFlowThreads;
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_inv_flow_cta, threads, smem), "occupancy");
    const unsigned grid = unsigned(std::max(1LL, std::min(E, (long long)std::max(1, per_sm) * c->sm_count)));
    InvFlowArgs a{c->S.view(), c->X.view(), N, L, m, c->flow_ready, next, E, wsw, kFlowStride, sleep_ns};
    k_inv_flow_cta<<<grid, threads, smem, st>>>(a);
    ck(cudaGetLastError(), "flow launch");
    ++c->launches;
}

// ---- LDLT as a dataflow (small p, IMAD path): the blocked rank-b update taken
// to its limit, b = j.  One CTA per entry (k, j) of the lower triangle applies
// ALL of that entry's rank-1 updates in the reference's order (ldlt.cpp:122-129,
// ascending step i) while the entry sits in shared memory:
//     acc = mu_{k+j};  for i = 0 .. j-1:  acc = RNE(acc - V(j,i) L(k,i))
// V(j,i) = the entry (j,i) before scaling, L(k,i) = B_i(k) = RNE(V(k,i) R_i).  Then
//     k == j:  D_j = acc (pivot test, ldlt.cpp:111), R_j = RNE(1/D_j)
//     k >  j:  V(k,j) = acc,  L(k,j) = RNE(acc R_j) into S in place (ldlt.cpp:113-120)
// Every operation and its order per entry are those of the N-step schedule, so
// the factors are bit-identical; the accumulator is read and written once per
// entry instead of once per step (N(N+1)/2 instead of N^3/6 passes over S), and
// the N dependent step launches (each a look-ahead chain of 5 kernels) become
// one kernel whose critical path per column is fms -> recip -> mul with a flag
// hand-off between them.  Entries are taken from a global counter in
// column-major order and wait only for entries of earlier columns (or their own
// column's diagonal, taken earlier), i.e. for entries already held by running
// CTAs: no deadlock whatever the residency.  A per-column completion count
// (cols_done: every column below it is final) saves the per-entry flag polls
// for all but the frontier columns.
struct LdltFlowArgs {
    MpArr S, V, R, mu;
    int N, L;
    int* ready;    // [N(N+1)/2 * fstride]: entry final (diagonal: R_j published)
    int* col_cnt;  // [N]: finished entries of each column
    int* ctl;      // [0] cols_done, [1] abort (1 pivot <= 0, 2 watchdog), [2..3] entry counter
    int* err;      // failing column (ldlt.cpp:83-87)
    int fstride, sleep_ns;
};

// false: the run was aborted (a pivot failed elsewhere) or the watchdog fired
__device__ __forceinline__ bool flow_wait(const int* flag, int* abort_flag, int sleep_ns, int want = 2) {
    long long spins = 0;
    while (ld_acquire_gpu(flag) < want) {
        if (*(volatile const int*)abort_flag != 0) return false;
        if (++spins > (1LL << 26)) { // > 6 s on one flag: never in a healthy run
            atomicCAS(abort_flag, 0, 2);
            return false; // (the caller reports it through err = -2)
        }
        __nanosleep(sleep_ns);
    }
    return true;
}

// out-of-line copies of the three CTA ops: inlined together they cost the kernel
// 128 registers and spills, and with them its residency
__device__ __noinline__ Meta flow_fms(uint32_t* acc, Meta am, const uint32_t* xs, Meta xm, const uint32_t* ys, Meta ym,
                                      int L, uint32_t* ws) {
    return hk::cta_fms(acc, am, xs, xm, ys, ym, acc, L, hk::ctaws_carve(ws, L));
}
__device__ __noinline__ Meta flow_mulr(const uint32_t* acc, Meta am, const uint32_t* xs, Meta xm, uint32_t* out, int L,
                                       uint32_t* ws) {
    return hk::cta_mulr(acc, am, xs, xm, out, L, hk::ctaws_carve(ws, L));
}
__device__ __noinline__ Meta flow_recip(const uint32_t* acc, Meta am, uint32_t* out, int L, uint32_t* ws) {
    return hk::cta_recip(acc, am, out, L, ws);
}

__global__ void __launch_bounds__(256) k_ldlt_flow(LdltFlowArgs a) {
    extern __shared__ __align__(16) uint32_t lfs_[];
    __shared__ unsigned long long e_s;
    __shared__ int stop_s, done_s;
    const int L = a.L, N = a.N, tid = int(threadIdx.x), nt = int(blockDim.x);
    uint32_t* acc = lfs_;
    uint32_t* xs = acc + hk::align4(L);
    uint32_t* ys = xs + hk::align4(L);
    uint32_t* zs = ys + hk::align4(L);
    uint32_t* ws = zs + hk::align4(L);
    const long long E = (long long)N * (N + 1) / 2;
    int* cols_done = a.ctl;
    int* abort_flag = a.ctl + 1;
    unsigned long long* next = reinterpret_cast<unsigned long long*>(a.ctl + 2);
    int known = 0; // columns < known are final (block-uniform)
    // publish entry (k, j) as final (flag 2): flag, column count, and the prefix of finished columns
    auto publish = [&](long long e, int j) {
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            st_release_gpu(a.ready + e * a.fstride, 2);
            if (atomicAdd(a.col_cnt + j, 1) == N - j - 1) {
                __threadfence();
                int c = j;
                while (c < N && atomicCAS(cols_done, c, c + 1) == c) {
                    ++c;
                    __threadfence();
                    if (c >= N || *(volatile int*)(a.col_cnt + c) != N - c) break;
                }
            }
        }
    };
    for (;;) {
        if (tid == 0) {
            e_s = atomicAdd(next, 1ull);
            stop_s = 0;
        }
        __syncthreads();
        const long long e = (long long)e_s;
        if (e >= E) return;
        int j, k;
        hk::tri_decode(e, N, j, k);
        for (int q = tid; q < L; q += nt) acc[q] = a.mu.limbs(k + j, L)[q];
        Meta am = a.mu.m[k + j];
        __syncthreads();
        for (int i = 0; i < j; ++i) {
            const long long exi = hk::tri_idx(j, i, N), eyi = hk::tri_idx(k, i, N);
            // The diagonal's last update D_j -= V(j,j-1) L(j,j-1) sits on the critical
            // path (R_{j-1} -> L(j,j-1) -> D_j -> R_j): this CTA forms L(j,j-1) =
            // RNE(V(j,j-1) R_{j-1}) itself (the same value entry (j,j-1) stores) instead
            // of waiting for that entry's publication: one flag hand-off less per column.
            const bool own_l = k == j && i == j - 1;
            if (i >= known) {
                if (tid == 0) {
                    const int cd = ld_acquire_gpu(cols_done);
                    done_s = cd;
                    // x = V(j,i) needs flag >= 1; y = L(k,i) needs 2 (k == j: the same entry)
                    if (cd <= i && !flow_wait(a.ready + exi * a.fstride, abort_flag, a.sleep_ns, k == j && !own_l ? 2 : 1))
                        stop_s = 1;
                }
                if (tid == 32 && k != j && !flow_wait(a.ready + eyi * a.fstride, abort_flag, a.sleep_ns)) stop_s = 1;
                if (tid == 32 && own_l && !flow_wait(a.ready + hk::tri_idx(i, i, N) * a.fstride, abort_flag, a.sleep_ns))
                    stop_s = 1;
                __syncthreads();
                if (stop_s) {
                    if (tid == 0 && *(volatile int*)abort_flag == 2) atomicCAS(a.err, -1, -2);
                    return;
                }
                known = done_s;
            }
            const uint32_t* ysrc = own_l ? a.R.limbs(i, L) : a.S.limbs(eyi, L);
            for (int q = tid; q < L; q += nt) {
                xs[q] = __ldcg(a.V.limbs(exi, L) + q);
                ys[q] = __ldcg(ysrc + q);
            }
            const int2 xm2 = __ldcg(reinterpret_cast<const int2*>(a.V.m + exi));
            int2 ym2 = __ldcg(reinterpret_cast<const int2*>(own_l ? a.R.m + i : a.S.m + eyi));
            __syncthreads();
            const uint32_t* yop = ys;
            if (own_l) {
                const Meta lm = flow_mulr(xs, Meta{xm2.x, xm2.y}, ys, Meta{ym2.x, ym2.y}, zs, L, ws);
                ym2 = make_int2(lm.exp, lm.sign);
                yop = zs;
                __syncthreads();
            }
            am = flow_fms(acc, am, xs, Meta{xm2.x, xm2.y}, yop, Meta{ym2.x, ym2.y}, L, ws);
            __syncthreads();
        }
        if (k == j) {
            if (am.sign <= 0) { // ldlt.cpp:111: pivot must be positive
                if (tid == 0) {
                    atomicCAS(a.err, -1, j);
                    __threadfence();
                    atomicCAS(abort_flag, 0, 1);
                }
                return;
            }
            const Meta rm = flow_recip(acc, am, a.R.limbs(j, L), L, ws);
            if (tid == 0) a.R.m[j] = rm;
            for (int q = tid; q < L; q += nt) a.S.limbs(e, L)[q] = acc[q];
            if (tid == 0) a.S.m[e] = am;
            publish(e, j);
        } else {
            for (int q = tid; q < L; q += nt) a.V.limbs(e, L)[q] = acc[q];
            if (tid == 0) a.V.m[e] = am;
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                st_release_gpu(a.ready + e * a.fstride, 1); // V(k,j) is final (x operand of row k's entries)
                if (!flow_wait(a.ready + hk::tri_idx(j, j, N) * a.fstride, abort_flag, a.sleep_ns)) stop_s = 1;
            }
            __syncthreads();
            if (stop_s) {
                if (tid == 0 && *(volatile int*)abort_flag == 2) atomicCAS(a.err, -1, -2);
                return;
            }
            for (int q = tid; q < L; q += nt) xs[q] = __ldcg(a.R.limbs(j, L) + q);
            const int2 rm2 = __ldcg(reinterpret_cast<const int2*>(a.R.m + j));
            __syncthreads();
            const Meta bm = flow_mulr(acc, am, xs, Meta{rm2.x, rm2.y}, a.S.limbs(e, L), L, ws);
            if (tid == 0) a.S.m[e] = bm;
            publish(e, j);
        }
    }
}

constexpr int kLdltFlowStride = 8; // one 32-byte sector per flag
constexpr long long kLdltFlowMaxWork = 1LL << 21; // n^2 L bound of the default selection

int ldlt_flow_ws_words(int L) { return std::max(hk::ctaws_words(L), hk::ctarecipws_words(L)); }

int ldlt_flow_threads() {
    static const char* e = getenv("HK_LDLT_FLOW_THREADS");
    const int t = e ? atoi(e) : 128;
    return std::max(64, std::min(256, t / 32 * 32));
}

// The dataflow LDLT is for the IMAD path (p below the tensor-core threshold):
// past a few thousand entries of a few thousand MACs each the N-step schedule's
// paired warp FMAs have the better throughput.  HK_LDLT_FLOW=0/1 forces it.
bool use_ldlt_flow(const hk_ctx* c) {
    if (c->world > 1 || c->virt || c->nccl_comm) return false;
    const size_t smem = (4 * size_t(hk::align4(c->L)) + ldlt_flow_ws_words(c->L)) * sizeof(uint32_t);
    if (smem > c->smem_optin) return false;
    if (const char* e = getenv("HK_LDLT_FLOW")) return e[0] == '1';
    if (use_tc(c)) return false;
    return (long long)c->n * c->n * c->L <= kLdltFlowMaxWork;
}

// [8 control ints][flags][column counts]; n <= ntri
size_t ldlt_flow_ints(long long ntri, int n) { return 8 + size_t(ntri) * kLdltFlowStride + size_t(n); }

void ensure_ldlt_flow(hk_ctx* c, long long ntri) {
    c->Vf.ensure(ntri, c->L);
    if (c->lflow_cap >= ntri) return;
    if (c->lflow) cudaFree(c->lflow);
    c->lflow = nullptr;
    c->lflow_cap = 0;
    ck(cudaMalloc(&c->lflow, ldlt_flow_ints(ntri, c->n) * sizeof(int)), "cudaMalloc ldlt flow");
    c->lflow_cap = ntri;
}

void enqueue_ldlt_flow(hk_ctx* c, cudaStream_t st) {
    const int N = c->n, L = c->L;
    const long long ntri = (long long)N * (N + 1) / 2;
    int* ctl = c->lflow;
    int* ready = ctl + 8;
    int* col_cnt = ready + ntri * kLdltFlowStride;
    ck(cudaMemsetAsync(c->lflow, 0, ldlt_flow_ints(ntri, N) * sizeof(int), st), "memset ldlt flow");
    const char* sl = getenv("HK_FLOW_SLEEP");
    const int sleep_ns = sl ? atoi(sl) : 100;
    const size_t smem = (4 * size_t(hk::align4(L)) + ldlt_flow_ws_words(L)) * sizeof(uint32_t);
    func_smem((const void*)k_ldlt_flow, smem);
    const int threads = ldlt_flow_threads();
    int per_sm = 0;
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ldlt_flow, threads, smem), "occupancy");
    const unsigned grid = unsigned(std::max(1LL, std::min(ntri, (long long)std::max(1, per_sm) * c->sm_count)));
    LdltFlowArgs a{c->S.view(), c->Vf.view(), c->R.view(), c->mu.view(), N, L, ready, col_cnt, ctl, c->d_err,
                   kLdltFlowStride, sleep_ns};
    k_ldlt_flow<<<grid, threads, smem, st>>>(a);
    ck(cudaGetLastError(), "ldlt flow launch");
    ++c->launches;
}

// Tensor-core buffers: the A operand of N rows, product scratch for `p_items`
// products (the unfused rounding pass and L^-1 steps; the fused LDLT needs
// none) and the fix-up list for `fb_items` items per step.
void ensure_tc_items(hk_ctx* c, size_t p_items, size_t fb_items) {
    if (c->tc_A_n < c->n) {
        if (c->tc_A) cudaFree(c->tc_A);
        c->tc_A = nullptr;
        ck(cudaMalloc(&c->tc_A, hk::tc_apre_bytes(c->n, c->L)), "cudaMalloc tc A");
        c->tc_A_n = c->n;
    }
    if (!c->tc_fb_count) {
        ck(cudaMalloc(&c->tc_fb_count, 4 * sizeof(int)), "cudaMalloc fb count");
        ck(cudaMemset(c->tc_fb_count, 0, 4 * sizeof(int)), "memset fb count");
    }
    if (fb_items > c->tc_fb_cap) {
        if (c->tc_fb) cudaFree(c->tc_fb);
        c->tc_fb = nullptr;
        ck(cudaMalloc(&c->tc_fb, fb_items * sizeof(long long)), "cudaMalloc fb list");
        c->tc_fb_cap = fb_items;
    }
    const size_t need = std::max<size_t>(p_items, 1) * hk::tc_scratch_limbs(c->L);
    if (c->tc_P_words >= need) return;
    if (c->tc_P) cudaFree(c->tc_P);
    if (c->tc_gcarry) cudaFree(c->tc_gcarry);
    c->tc_P = nullptr;
    c->tc_gcarry = nullptr;
    ck(cudaMalloc(&c->tc_gcarry, std::max<size_t>(p_items, 1) * (hk::kTcMaxGroups - 1) * sizeof(uint64_t)),
       "cudaMalloc tc carries");
    ck(cudaMalloc(&c->tc_P, need * sizeof(uint32_t)), "cudaMalloc tc scratch");
    c->tc_P_words = need;
}

// m == 0: the LDLT's needs; m > 0: the L^-1 steps' (N m products per step)
void ensure_tc_scratch(hk_ctx* c, int m = 0) {
    if (!use_tc(c)) return;
    const size_t tri = (size_t)c->n * (c->n + 1) / 2, nm = (size_t)c->n * m;
    const size_t p_items = m > 0 ? nm : (use_fuse(c) ? 0 : tri);
    ensure_tc_items(c, p_items, std::max(tri, nm + c->n));
}

// Buffers of the tensor-core L^-1 steps when they ride in the LDLT graph: the
// LDLT's A operand, redo list and counters are in use at the same time
void ensure_inv_overlap(hk_ctx* c, int m) {
    const size_t nm = (size_t)c->n * m;
    ensure_tc_items(c, nm, std::max((size_t)c->n * (c->n + 1) / 2, nm + c->n)); // product scratch + group carries (L^-1 only)
    if (c->inv_A_n < c->n) {
        if (c->inv_A) cudaFree(c->inv_A);
        c->inv_A = nullptr;
        c->inv_A_n = 0;
        ck(cudaMalloc(&c->inv_A, hk::tc_apre_bytes(c->n, c->L)), "cudaMalloc inv A");
        c->inv_A_n = c->n;
    }
    if (!c->inv_fb_count) {
        ck(cudaMalloc(&c->inv_fb_count, 2 * sizeof(int)), "cudaMalloc inv fb count");
        ck(cudaMemset(c->inv_fb_count, 0, 2 * sizeof(int)), "memset inv fb count");
    }
    if (nm + c->n > c->inv_fb_cap) {
        if (c->inv_fb) cudaFree(c->inv_fb);
        c->inv_fb = nullptr;
        c->inv_fb_cap = 0;
        ck(cudaMalloc(&c->inv_fb, (nm + c->n) * sizeof(long long)), "cudaMalloc inv fb list");
        c->inv_fb_cap = nm + c->n;
    }
}

// One L^-1 step of the N-step schedule (small p): few items a CTA per FMA, many a warp per FMA
void enqueue_inv_step(hk_ctx* c, int i, int m, cudaStream_t st, const int* err = nullptr) {
    const int N = c->n, L = c->L;
    const int b = i < m ? i : m;
    const long long items = (long long)(N - i - 1) * b + (i < m ? N - i - 1 : 0);
    if (items <= 4LL * c->sm_count) {
        hk::CItemInvStep f{c->S.view(), c->X.view(), N, L, m, i};
        f.err = err;
        launch_cta(c, f, items, ws_cta_words(L), st);
    } else {
        hk::ItemInvStep f{c->S.view(), c->X.view(), N, L, m, i};
        f.err = err;
        launch(c, f, items, ws_op_words(L), st);
    }
}

// inv_m > 0 (hk_ldlt_invert): the L^-1 row-elimination step i (inversion.cpp:93-102)
// rides in the same graph on a low-priority stream, right after column i of L
// is in place (StoreL(i)) and step i-1 — the steps need nothing else from the
// factorisation, so for latency-bound sizes the first m columns of L^-1 are
// ready a step after the LDLT ends instead of a whole pass later.
void enqueue_ldlt_steps(hk_ctx* c, int inv_m = 0) {
    const int N = c->n, L = c->L;
    const int wo = ws_op_words(L), wr = ws_recip_words(L);
    cudaStream_t la = c->st2, bulk = c->st;
    std::vector<cudaEvent_t>& evP = c->evP;
    std::vector<cudaEvent_t>& evR = c->evR;
    std::vector<cudaEvent_t>& evU = c->evU;
    std::vector<cudaEvent_t>& evD = c->evD;
    std::vector<cudaEvent_t>& evO = c->evO;
    std::vector<cudaEvent_t>& evC = c->evC;
    std::vector<cudaEvent_t>& evB1 = c->evB1;
    cudaStream_t la2 = c->st3, side = c->st4;
    static const char* pe = getenv("HK_PDL"); // programmatic dependent launch on the chain (default on)
    const bool pdl = !pe || pe[0] != '0';
    if (c->tc_fb_count) ck(cudaMemsetAsync(c->tc_fb_count, 0, 2 * sizeof(int), bulk), "memset fb counters");
    ck(cudaEventRecord(c->evFork, bulk), "fork");
    ck(cudaStreamWaitEvent(la, c->evFork, 0), "fork wait");
    ck(cudaStreamWaitEvent(side, c->evFork, 0), "fork wait side");
    cudaStream_t inv = c->st5;
    const bool inv_tc = inv_m > 0 && use_tc_inv(c);
    InvTarget itg;
    if (inv_m > 0) {
        ck(cudaStreamWaitEvent(inv, c->evFork, 0), "fork wait inv");
        hk::ItemInvInit ii{c->S.view(), c->X.view(), N, L, inv_m};
        ii.zero = 1; // column c of X is set at step c, before any use
        launch(c, ii, (long long)N * inv_m, 64, inv);
        if (inv_tc) {
            ck(cudaMemsetAsync(c->inv_fb_count, 0, 2 * sizeof(int), inv), "memset inv fb counters");
            itg.Lsrc = c->S.view();
            itg.X = c->X.view();
            itg.A = c->inv_A;
            itg.fb_count = c->inv_fb_count;
            itg.fb = c->inv_fb;
            itg.err = c->d_err;
        }
    }
    const int wc = ws_cta_words(L), wcr = ws_cta_recip_words(L);
    (void)wr;
    launch_recip(c, 0, la);
    launch_cta(c, hk::CItemMulB{c->S.view(), c->R.view(), b_buf(c, 0), N, L, 0, c->d_err}, N - 1, wc, la);
    ck(cudaEventRecord(evP[0], la), "evP");
    // bulk: U(i) -> evU(i) -> StoreL(i-1) -> evR(i-1);  LA: [evU(i-1)] P(i+1) with
    // MulB(i+1) (overwrites buffer (i+1) % 3 = that of B_{i-2}) after [evR(i-2)].
    c->kev_steps = 0;
    if (c->kprof) grow_events(c->kev, size_t(3 * N), cudaEventDefault);
    for (int i = 0; i < N; ++i) {
        ck(cudaStreamWaitEvent(bulk, evP[i], 0), "wait P");
        const bool timed = c->kprof && N - i - 2 > 0;
        enqueue_bulk(c, i, i + 2, bulk, pdl, timed ? c->kev_steps : -1);
        if (timed) ++c->kev_steps;
        ck(cudaEventRecord(evU[i], bulk), "evU");
        if (i >= 1) {
            // StoreL(i-1) on the side stream: column i-1 was last read by U(i-1)
            // (x operands) and P(i) (the look-ahead update of column i)
            ck(cudaStreamWaitEvent(side, evU[i - 1], 0), "wait U side");
            ck(cudaStreamWaitEvent(side, evP[i], 0), "wait P side");
            if (!dev_skip("storel"))
                launch(c, hk::ItemStoreL{c->S.view(), b_buf(c, i - 1), N, L, i - 1}, N - i, 64, side);
            ck(cudaEventRecord(evR[i - 1], side), "evR");
            if (inv_m > 0 && i - 1 < N - 1) { // L^-1 step i-1: column i-1 of L is in place
                ck(cudaStreamWaitEvent(inv, evR[i - 1], 0), "wait R inv");
                if (inv_tc)
                    enqueue_inv_tc(c, i - 1, inv, pdl, &itg);
                else
                    enqueue_inv_step(c, i - 1, inv_m, inv, c->d_err);
            }
        }
        if (i + 1 < N) {
            // P(i+1): the diagonal entry -> reciprocal on `la`, the rest of the
            // column concurrently on `la2`; B_{i+1} needs both.
            if (i > 0) ck(cudaStreamWaitEvent(la, evU[i - 1], 0), "wait U");
            ck(cudaEventRecord(evD[i + 1], la), "evD");
            ck(cudaStreamWaitEvent(la2, evD[i + 1], 0), "wait D");
            if (!dev_skip("coloff"))
                launch_cta(c, hk::CItemColUpd{c->S.view(), b_buf(c, i), N, L, i, c->d_err, 1}, N - i - 2, wc, la2,
                           pdl);
            ck(cudaEventRecord(evO[i + 1], la2), "evO");
            if (!dev_skip("coldiag"))
                launch_cta(c, hk::CItemColUpd{c->S.view(), b_buf(c, i), N, L, i, c->d_err, 0}, 1, wc, la, pdl);
            if (!dev_skip("recip"))
                launch_recip(c, i + 1, la, pdl);
            ck(cudaEventRecord(evC[i + 1], la), "evC");
            // B_{i+1}: the first entry (all the next diagonal update needs) on `la`,
            // the rest on `la2`; B buffer (i+1) % 3 was last read by StoreL(i-2)
            if (i >= 2) ck(cudaStreamWaitEvent(la, evR[i - 2], 0), "wait R");
            ck(cudaStreamWaitEvent(la, evO[i + 1], 0), "wait O");
            if (!dev_skip("mulb") && N - i - 2 > 0)
                launch_cta(c, hk::CItemMulB{c->S.view(), c->R.view(), b_buf(c, i + 1), N, L, i + 1, c->d_err, 1}, 1,
                           wc, la, pdl);
            ck(cudaEventRecord(evB1[i + 1], la), "evB1");
            ck(cudaStreamWaitEvent(la2, evC[i + 1], 0), "wait C");
            if (i >= 2) ck(cudaStreamWaitEvent(la2, evR[i - 2], 0), "wait R2");
            if (!dev_skip("mulb") && N - i - 3 > 0)
                launch_cta(c, hk::CItemMulB{c->S.view(), c->R.view(), b_buf(c, i + 1), N, L, i + 1, c->d_err, 2},
                           N - i - 3, wc, la2, pdl);
            ck(cudaStreamWaitEvent(la2, evB1[i + 1], 0), "wait B1");
            ck(cudaEventRecord(evP[i + 1], la2), "evP");
        }
    }
    // StoreL(N-1) has no rows; join the streams (the last ColUpd read S(N-1, N-2))
    ck(cudaEventRecord(c->evJoin, la), "join");
    ck(cudaStreamWaitEvent(bulk, c->evJoin, 0), "join wait");
    if (N >= 2) { // la2 joined the capture at step 0
        ck(cudaEventRecord(c->evJoin2, la2), "join2");
        ck(cudaStreamWaitEvent(bulk, c->evJoin2, 0), "join2 wait");
    }
    ck(cudaEventRecord(c->evJoin3, side), "join3");
    ck(cudaStreamWaitEvent(bulk, c->evJoin3, 0), "join3 wait");
    if (inv_m > 0) {
        graph_event(c->evMid, bulk); // the LDLT proper ends here (ldlt_s / invL_s split)
        ck(cudaEventRecord(c->evJoin4, inv), "join4");
        ck(cudaStreamWaitEvent(bulk, c->evJoin4, 0), "join4 wait");
    }
}

void ensure_step_events(hk_ctx* c, int N) {
    auto grow = [](std::vector<cudaEvent_t>& v, int n) {
        while ((int)v.size() < n) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            v.push_back(e);
        }
    };
    grow(c->evP, N);
    grow(c->evR, N);
    grow(c->evU, N);
    grow(c->evD, N);
    grow(c->evO, N);
    grow(c->evC, N);
    grow(c->evB1, N);
}

int check_pivots(hk_ctx* c) {
    int e = -1;
    ck(cudaMemcpyAsync(&e, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->st), "D2H err");
    ck(cudaStreamSynchronize(c->st), "sync");
    if (e == -2) { // k_ldlt_flow's watchdog: a flag never arrived
        c->factored = false;
        return fail(c, HK_ERR_RUNTIME, "hk_ldlt: the dataflow kernel's watchdog fired (a dependency flag never arrived)");
    }
    if (e >= 0) {
        c->bad_col = e;
        c->factored = false;
        return fail(c, HK_ERR_PRECISION,
                    "LDLT pivot <= 0 at column " + std::to_string(e) + ": matrix not positive definite at p=" +
                        std::to_string(32 * c->L) + " bits, increase the precision");
    }
    return HK_OK;
}

int dist_ldlt(hk_ctx* c); // multi-GPU factorisation (below)
int dist_invert(hk_ctx* c, int m);
int dist_block(hk_ctx* c, int k);
// HK_DIST_INV=0: a sharded context runs L^-1 and the block on rank 0 alone (the r01 schedule)
bool sharded_inv_off() {
    const char* e = getenv("HK_DIST_INV");
    return e && e[0] == '0';
}
int share_root_result(hk_ctx* c, int* rc, int s, double* hi, double* lo, double* te); // (below)

void drop_graphs(hk_ctx* c) {
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : c->inv_graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
    c->inv_graphs.clear();
    c->graph_sig.clear();
    c->inv_sig.clear();
    if (c->dist_graph) cudaGraphExecDestroy(c->dist_graph);
    c->dist_graph = nullptr;
    c->dist_sig.clear();
}

} // namespace

extern "C" {

int hk_version(void) { return 100; }

int hk_create(int device, int limbs, hk_ctx** out) {
    if (!out || limbs < 1 || limbs > 8192) return HK_ERR_INVALID;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return HK_ERR_RUNTIME;
    if (device < 0 || device >= ndev) return HK_ERR_INVALID;
    hk_ctx* c = new hk_ctx();
    c->device = device;
    c->L = limbs;
    const int rc = guarded(c, [&] {
        cudaDeviceProp prop{};
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        c->sm_count = prop.multiProcessorCount;
        c->smem_optin = prop.sharedMemPerBlockOptin;
        ck(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "cudaStreamCreate");
        int lo = 0, hi = 0;
        ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
        ck(cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi), "cudaStreamCreate la");
        ck(cudaStreamCreateWithPriority(&c->st3, cudaStreamNonBlocking, hi), "cudaStreamCreate la2");
        ck(cudaEventCreateWithFlags(&c->evFork, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->evJoin, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->evJoin2, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&c->evJoin3, cudaEventDisableTiming), "event");
        ck(cudaStreamCreateWithFlags(&c->st4, cudaStreamNonBlocking), "cudaStreamCreate side");
        ck(cudaStreamCreateWithPriority(&c->st5, cudaStreamNonBlocking, lo), "cudaStreamCreate inv");
        ck(cudaEventCreateWithFlags(&c->evJoin4, cudaEventDisableTiming), "event");
        ck(cudaEventCreate(&c->evMid), "event");
        ck(cudaMalloc(&c->d_err, 2 * sizeof(int)), "cudaMalloc err"); // [0] failing column, [1] inexact-moment flag
        ck(cudaEventCreate(&c->ev[0]), "event");
        ck(cudaEventCreate(&c->ev[1]), "event");
        ck(cudaMalloc(&c->fix_total, sizeof(unsigned long long)), "malloc fix counter");
        ck(cudaMemset(c->fix_total, 0, sizeof(unsigned long long)), "memset fix counter");
        if (const char* dv = getenv("HK_DEV_TCB"); dv && (atoi(dv) & 64)) {
            ck(cudaMalloc(&c->dev_cnt, 16 * sizeof(unsigned long long)), "malloc dev counters");
            ck(cudaMemset(c->dev_cnt, 0, 16 * sizeof(unsigned long long)), "memset dev counters");
        }
        return HK_OK;
    });
    if (rc != HK_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return HK_OK;
}

void hk_destroy(hk_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    drop_graphs(c);
    for (DevArr* a : {&c->mu, &c->S, &c->R, &c->B, &c->X, &c->Y, &c->T, &c->T2, &c->M, &c->Dg, &c->Vf}) a->release();
    for (auto& s : c->shards) {
        for (DevArr* a : {&s.S, &s.panel, &s.R, &s.B, &s.X, &s.Y, &s.T, &s.T2}) a->release();
        if (s.d_otiles) cudaFree(s.d_otiles);
        if (s.d_erow) cudaFree(s.d_erow);
        if (s.d_ecol) cudaFree(s.d_ecol);
        if (s.d_err) cudaFree(s.d_err);
        if (s.d_owned) cudaFree(s.d_owned);
        if (s.d_off) cudaFree(s.d_off);
        if (s.d_fb) cudaFree(s.d_fb);
    }
    if (c->nccl_comm) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        auto destroy = h ? (int (*)(void*))dlsym(h, "ncclCommDestroy") : nullptr;
        if (destroy) destroy(c->nccl_comm);
    }
    if (c->d_err) cudaFree(c->d_err);
    if (c->bcast_buf) cudaFree(c->bcast_buf);
    if (c->fix_total) cudaFree(c->fix_total);
    if (c->dev_cnt) {
        unsigned long long h[16] = {};
        cudaMemcpy(h, c->dev_cnt, sizeof h, cudaMemcpyDeviceToHost);
        const double tot = h[4] ? double(h[4]) : 1.0;
        fprintf(stderr, "k_tc_bulk issuer cycles: total %.3e over %llu CTAs; waiting empty %.1f%% full %.1f%% "
                        "efull %.1f%% accE %.1f%% peer %.1f%%\n", double(h[4]), h[5], 100 * h[0] / tot, 100 * h[1] / tot,
                100 * h[2] / tot, 100 * h[3] / tot, 100 * h[6] / tot);
        const double et = h[11] ? double(h[11]) : 1.0;
        fprintf(stderr, "fused epilogue (thread 128) cycles: total %.3e; waiting accF %.1f%% drain %.1f%% processing %.1f%%\n",
                double(h[11]), 100 * h[8] / et, 100 * h[9] / et, 100 * h[10] / et);
        cudaFree(c->dev_cnt);
    }
    if (c->tc_P) cudaFree(c->tc_P);
    if (c->tc_fb) cudaFree(c->tc_fb);
    if (c->tc_fb_count) cudaFree(c->tc_fb_count);
    if (c->tc_A) cudaFree(c->tc_A);
    if (c->tc_gcarry) cudaFree(c->tc_gcarry);
    if (c->flow_ready) cudaFree(c->flow_ready);
    if (c->lflow) cudaFree(c->lflow);
    if (c->inv_A) cudaFree(c->inv_A);
    if (c->inv_fb) cudaFree(c->inv_fb);
    if (c->inv_fb_count) cudaFree(c->inv_fb_count);
    for (auto e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto e : c->evP) cudaEventDestroy(e);
    for (auto e : c->evR) cudaEventDestroy(e);
    for (auto e : c->evU) cudaEventDestroy(e);
    for (auto e : c->evD) cudaEventDestroy(e);
    for (auto e : c->evO) cudaEventDestroy(e);
    for (auto e : c->evC) cudaEventDestroy(e);
    for (auto e : c->evB1) cudaEventDestroy(e);
    for (auto e : c->kev) cudaEventDestroy(e);
    for (auto e : c->cev) cudaEventDestroy(e);
    if (c->evJoin2) cudaEventDestroy(c->evJoin2);
    if (c->evJoin3) cudaEventDestroy(c->evJoin3);
    if (c->st4) cudaStreamDestroy(c->st4);
    if (c->st5) cudaStreamDestroy(c->st5);
    if (c->evJoin4) cudaEventDestroy(c->evJoin4);
    if (c->evMid) cudaEventDestroy(c->evMid);
    if (c->evFork) cudaEventDestroy(c->evFork);
    if (c->evJoin) cudaEventDestroy(c->evJoin);
    if (c->st2) cudaStreamDestroy(c->st2);
    if (c->st3) cudaStreamDestroy(c->st3);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

const char* hk_last_error(const hk_ctx* c) { return c ? c->err.c_str() : "null context"; }
int hk_bad_column(const hk_ctx* c) { return c ? c->bad_col : -1; }
int hk_limbs(const hk_ctx* c) { return c ? c->L : 0; }
long long hk_launch_count(const hk_ctx* c) { return c ? c->launches : 0; }

int hk_moments(unsigned beta_num, unsigned beta_den, int count, int limbs, uint32_t* out_limbs, int32_t* out_exps,
               int32_t* out_signs, int* exact) {
    const char* why = "";
    int ex = 0;
    const int rc = hk_moments_impl(beta_num, beta_den, count, limbs, out_limbs, out_exps, out_signs, &ex, &why);
    if (exact) *exact = ex;
    return rc;
}

int hk_load_moments(hk_ctx* c, int n, const uint32_t* limbs, const int32_t* exps, const int32_t* signs) {
    return guarded(c, [&] {
        if (n < 1) return fail(c, HK_ERR_INVALID, "matrix order must be >= 1");
        const double t0 = now_s();
        h2d_soa(c, c->mu, 2LL * n - 1, limbs, exps, signs);
        c->t[5] = now_s() - t0;
        c->n = n;
        c->factored = c->inverted = c->assembled = false;
        return HK_OK;
    });
}

// The 2n-1 moments generated on the device (csrc/moments_dev.cuh) straight
// into the context's moment array; even q = 2/beta only (the factorial branch).
int hk_generate_moments(hk_ctx* c, unsigned beta_num, unsigned beta_den, int n, int* exact) {
    return guarded(c, [&] {
        if (n < 1) return fail(c, HK_ERR_INVALID, "matrix order must be >= 1");
        if (beta_num == 0 || beta_den == 0 || (2ul * beta_den) % beta_num != 0)
            return fail(c, HK_ERR_INVALID, "unsupported beta: 2/beta must be a positive integer");
        const unsigned long q = 2ul * beta_den / beta_num;
        if (q % 2 != 0)
            return fail(c, HK_ERR_INVALID,
                        "hk_generate_moments: odd 2/beta (half-integer Gamma) is host-only: hk_moments + hk_load_moments");
        const double t0 = now_s();
        const int count = 2 * n - 1, L = c->L;
        // limbs of the largest value (q/2) (count q/2 - 1)!, with slack
        const double amax = double(count) * double(q / 2);
        const double bits = std::lgamma(amax + 1.0) / std::log(2.0) + std::log2(double(q / 2)) + 96.0;
        const long long need = (long long)(bits / 32.0) + 4;
        int threads = int(std::min<long long>(hk::kMomMaxThreads, (need + 31) / 32 * 32));
        int per = int((need + threads - 1) / threads);
        per |= 1; // odd stride between the threads' segments: no bank conflicts
        const size_t smem = ((q / 2 == 1 ? 1 : 2) * size_t(per) * threads + threads + 32) * sizeof(uint32_t);
        if (smem > c->smem_optin || q / 2 > 0xfffffffful)
            return fail(c, HK_ERR_INVALID, "hk_generate_moments: moments too large for the on-device generator");
        c->mu.ensure(count, L);
        int* d_inexact = c->d_err + 1; // second word of the error block
        ck(cudaMemsetAsync(d_inexact, 0, sizeof(int), c->st), "memset");
        func_smem((const void*)&hk::k_moments_fact, smem);
        hk::MomentsArgs a{c->mu.d, c->mu.m, count, L, unsigned(q), per, d_inexact};
        hk::k_moments_fact<<<1, threads, smem, c->st>>>(a);
        ck(cudaGetLastError(), "k_moments_fact");
        ++c->launches;
        int inexact = 0;
        ck(cudaMemcpyAsync(&inexact, d_inexact, sizeof(int), cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaStreamSynchronize(c->st), "sync");
        if (exact) *exact = inexact ? 0 : 1;
        c->t[5] = now_s() - t0;
        c->n = n;
        c->factored = c->inverted = c->assembled = false;
        return HK_OK;
    });
}

int hk_get_moments(hk_ctx* c, uint32_t* limbs, int32_t* exps, int32_t* signs) {
    return guarded(c, [&] {
        if (c->n < 1 || !c->mu.d) return fail(c, HK_ERR_INVALID, "hk_get_moments: no moments on the device");
        d2h_range(c, c->mu, 0, 2LL * c->n - 1, limbs, exps, signs);
        return HK_OK;
    });
}

} // extern "C"

namespace {
constexpr bool kInvOverlapTc = true; // default of HK_INV_OVERLAP_TC (C3 496 -> 448 ms, C4 4.65 -> 4.23 s)

// The L^-1 steps can ride in the LDLT graph (hk_ldlt_invert) when both run the
// N-step schedules on one GPU and L^-1 is latency-bound (small p, IMAD steps).
// HK_INV_OVERLAP=0 keeps the two passes apart.
bool can_overlap_inverse(const hk_ctx* c) {
    if (c->world > 1 || c->virt || c->nccl_comm) return false;
    if (use_ldlt_flow(c)) return false;
    const char* e = getenv("HK_INV_OVERLAP");
    if (e && e[0] == '0') return false;
    if (use_tc_inv(c)) { // tensor-core steps: they need the product scratch the unfused LDLT uses
        const char* t = getenv("HK_INV_OVERLAP_TC");
        return use_fuse(c) && (t ? t[0] == '1' : kInvOverlapTc);
    }
    return true;
}

// hk_ldlt (inv_m == 0) / the overlapped part of hk_ldlt_invert (inv_m > 0)
int ldlt_impl(hk_ctx* c, int inv_m) {
    return guarded(c, [&] {
        if (c->n < 1) return fail(c, HK_ERR_INVALID, "hk_ldlt: no moments loaded");
        if (c->world > 1 || c->virt || c->nccl_comm) return dist_ldlt(c);
        const int N = c->n, L = c->L;
        if (inv_m > 0) {
            c->X.ensure((long long)N * inv_m, L);
            c->m = inv_m; // (the tensor-core step enqueue reads it)
        }
        const long long ntri = (long long)N * (N + 1) / 2;
        c->S.ensure(ntri, L);
        c->R.ensure(N, L);
        c->bad_col = -1;
        if (use_ldlt_flow(c)) {
            // small p: the whole factorisation as one dataflow kernel (k_ldlt_flow)
            ensure_ldlt_flow(c, ntri);
            ck(cudaMemsetAsync(c->d_err, 0xff, sizeof(int), c->st), "memset err");
            ck(cudaEventRecord(c->ev[0], c->st), "event");
            enqueue_ldlt_flow(c, c->st);
            c->kev_steps = 0;
            ck(cudaEventRecord(c->ev[1], c->st), "event");
            ck(cudaEventSynchronize(c->ev[1]), "sync");
            float fms = 0;
            ck(cudaEventElapsedTime(&fms, c->ev[0], c->ev[1]), "elapsed");
            c->t[1] = fms * 1e-3;
            const int frc = check_pivots(c);
            if (frc != HK_OK) return frc;
            c->factored = true;
            c->inverted = c->assembled = false;
            return HK_OK;
        }
        c->B.ensure(3LL * N, L);
        ensure_tc_scratch(c);
        if (inv_m > 0 && use_tc_inv(c)) ensure_inv_overlap(c, inv_m);
        ensure_step_events(c, N);
        ck(cudaMemsetAsync(c->d_err, 0xff, sizeof(int), c->st), "memset err");
        ck(cudaEventRecord(c->ev[0], c->st), "event");
        launch(c, hk::ItemInitS{c->S.view(), c->mu.view(), N, L}, ntri, 64);
        // the cached step graphs are valid for the buffers and modes they were captured on
        // (the fused LDLT does not use the product scratch: L^-1 may re-size it freely)
        const std::vector<const void*> sig{c->S.d, c->S.m, c->R.d, c->B.d, c->mu.d,
                                           use_fuse(c) ? nullptr : (const void*)c->tc_P, c->tc_A, c->tc_fb,
                                           c->tc_fb_count, (const void*)(long long)use_tc(c),
                                           (const void*)(long long)use_fuse(c), (const void*)(long long)c->kprof,
                                           c->X.d, c->X.m, c->inv_A, c->inv_fb, c->inv_fb_count, c->tc_P, c->tc_gcarry};
        if (sig != c->graph_sig) {
            for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
            c->graphs.clear();
            c->graph_sig = sig;
        }
        const int key = N + (inv_m << 20); // graphs with the L^-1 steps interleaved are cached per (n, m)
        auto it = c->graphs.find(key);
        if (it == c->graphs.end()) {
            const long long before = c->launches;
            Capture cap(c->st);
            enqueue_ldlt_steps(c, inv_m);
            const cudaGraphExec_t ge = instantiate(cap.end(), cudaGraphInstantiateFlagUseNodePriority);
            it = c->graphs.emplace(key, ge).first;
            c->graph_launches[key] = c->launches - before;
            c->kev_steps_by_n[key] = c->kev_steps;
            c->launches = before;
        }
        ck(cudaGraphLaunch(it->second, c->st), "graph launch");
        c->launches += c->graph_launches[key];
        c->kev_steps = c->kev_steps_by_n[key];
        ck(cudaEventRecord(c->ev[1], c->st), "event");
        ck(cudaEventSynchronize(c->ev[1]), "sync");
        float ms = 0;
        if (inv_m > 0) { // the LDLT proper ends at evMid; what is left of L^-1 after it is invL_s
            ck(cudaEventElapsedTime(&ms, c->ev[0], c->evMid), "elapsed");
            c->t[1] = ms * 1e-3;
            ck(cudaEventElapsedTime(&ms, c->evMid, c->ev[1]), "elapsed");
            c->t[2] = ms * 1e-3;
        } else {
            ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
            c->t[1] = ms * 1e-3;
        }
        const int rc = check_pivots(c);
        if (rc != HK_OK) return rc;
        c->factored = true;
        c->inverted = c->assembled = false;
        if (inv_m > 0) {
            c->m = inv_m;
            c->inverted = true;
        }
        return HK_OK;
    });
}
} // namespace

extern "C" {

int hk_ldlt(hk_ctx* c) { return ldlt_impl(c, 0); }

// decompose + invert_L_partial(m) as one call (what compute() runs): the L^-1
// steps interleaved with the factorisation where that pays (can_overlap_inverse),
// otherwise the two passes one after the other.  Same results either way.
int hk_ldlt_invert(hk_ctx* c, int m) {
    if (!c) return HK_ERR_INVALID;
    if (c->n >= 1 && (m < 1 || m > c->n)) return fail(c, HK_ERR_INVALID, "invert_L_partial: need 1 <= m <= n");
    if (c->n >= 1 && can_overlap_inverse(c)) return ldlt_impl(c, m);
    const int rc = hk_ldlt(c);
    if (rc != HK_OK) return rc;
    if (c->rank != 0 && !((c->world > 1 || c->virt || c->nccl_comm) && !sharded_inv_off())) return HK_OK;
    return hk_invert_L_partial(c, m);
}

int hk_get_D(hk_ctx* c, uint32_t* limbs, int32_t* exps, int32_t* signs) {
    return guarded(c, [&] {
        if (!c->factored) return fail(c, HK_ERR_INVALID, "hk_get_D: not factored");
        c->Dg.ensure(c->n, c->L);
        k_gather_diag<<<unsigned(c->n), 128, 0, c->st>>>(c->S.view(), c->Dg.view(), c->n, c->L);
        ck(cudaGetLastError(), "gather launch");
        d2h_range(c, c->Dg, 0, c->n, limbs, exps, signs);
        return HK_OK;
    });
}

int hk_get_L_column(hk_ctx* c, int col, uint32_t* limbs, int32_t* exps, int32_t* signs) {
    return guarded(c, [&] {
        if (!c->factored) return fail(c, HK_ERR_INVALID, "hk_get_L_column: not factored");
        if (col < 0 || col >= c->n) return fail(c, HK_ERR_INVALID, "hk_get_L_column: column out of range");
        const long long cnt = c->n - col - 1;
        if (cnt > 0) d2h_range(c, c->S, hk::tri_idx(col + 1, col, c->n), cnt, limbs, exps, signs);
        return HK_OK;
    });
}

int hk_invert_L_partial(hk_ctx* c, int m) {
    return guarded(c, [&] {
        const bool sharded = c->world > 1 || c->virt || c->nccl_comm;
        if (!c->factored && !(sharded && c->dist_factored))
            return fail(c, HK_ERR_INVALID, "invert_L_partial: not factored");
        const int N = c->n, L = c->L;
        if (m < 1 || m > N) return fail(c, HK_ERR_INVALID, "invert_L_partial: need 1 <= m <= n");
        if (sharded && !sharded_inv_off()) return dist_invert(c, m);
        c->m = m;
        c->X.ensure((long long)N * m, L);
        const bool tc = use_tc_inv(c);
        // small p: the dataflow kernel (HK_INV_FLOW=0 forces the N-step schedule)
        const char* fe = getenv("HK_INV_FLOW");
        const bool flow = !tc && (fe ? fe[0] != '0' : true);
        if (flow) ensure_inv_flow(c, (long long)N * m);
        ensure_tc_scratch(c, m);
        // all N steps in one cached graph (invalidated when a buffer or mode changes)
        const std::vector<const void*> sig{c->S.d, c->S.m, c->X.d, c->tc_P, c->tc_A, c->tc_fb, c->tc_fb_count,
                                           c->tc_gcarry, c->flow_ready, (const void*)(long long)flow,
                                           (const void*)(long long)tc};
        if (sig != c->inv_sig) {
            for (auto& kv : c->inv_graphs) cudaGraphExecDestroy(kv.second);
            c->inv_graphs.clear();
            c->inv_sig = sig;
        }
        const long long key = ((long long)N << 20) | m;
        auto it = c->inv_graphs.find(key);
        if (it == c->inv_graphs.end()) {
            const long long before = c->launches;
            Capture cap(c->st);
            if (c->tc_fb_count) ck(cudaMemsetAsync(c->tc_fb_count, 0, 2 * sizeof(int), c->st), "memset fb counters");
            launch(c, hk::ItemInvInit{c->S.view(), c->X.view(), N, L, m}, (long long)N * m, 64);
            if (flow) enqueue_inv_flow(c, c->st);
            for (int i = 0; i < N && !flow; ++i) {
                const int b = i < m ? i : m;
                const long long items = (long long)(N - i - 1) * b + (i < m ? N - i - 1 : 0);
                if (tc) {
                    static const char* pe = getenv("HK_PDL");
                    enqueue_inv_tc(c, i, c->st, !pe || pe[0] != '0');
                    continue;
                }
                // few items: a CTA per FMA (latency); many: a warp per FMA (one wave)
                if (items <= 4LL * c->sm_count)
                    launch_cta(c, hk::CItemInvStep{c->S.view(), c->X.view(), N, L, m, i}, items, ws_cta_words(L));
                else
                    launch(c, hk::ItemInvStep{c->S.view(), c->X.view(), N, L, m, i}, items, ws_op_words(L));
            }
            const cudaGraphExec_t ge = instantiate(cap.end(), 0);
            it = c->inv_graphs.emplace(key, ge).first;
            c->inv_graph_launches[key] = c->launches - before;
            c->launches = before;
        }
        ck(cudaEventRecord(c->ev[0], c->st), "event");
        ck(cudaGraphLaunch(it->second, c->st), "graph launch");
        c->launches += c->inv_graph_launches[key];
        ck(cudaEventRecord(c->ev[1], c->st), "event");
        ck(cudaEventSynchronize(c->ev[1]), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
        c->t[2] = ms * 1e-3;
        c->inverted = true;
        c->assembled = false;
        return HK_OK;
    });
}

int hk_get_Linv(hk_ctx* c, uint32_t* limbs, int32_t* exps, int32_t* signs) {
    return guarded(c, [&] {
        if (!c->inverted) return fail(c, HK_ERR_INVALID, "hk_get_Linv: not inverted");
        d2h_range(c, c->X, 0, (long long)c->n * c->m, limbs, exps, signs);
        return HK_OK;
    });
}

int hk_assemble_block(hk_ctx* c, int k) {
    return guarded(c, [&] {
        if (!c->inverted) return fail(c, HK_ERR_INVALID, "assemble_truncated_inverse: not inverted");
        if (k < 1 || k > c->m) return fail(c, HK_ERR_INVALID, "assemble_truncated_inverse: need 1 <= k <= m");
        if ((c->world > 1 || c->virt || c->nccl_comm) && !sharded_inv_off()) return dist_block(c, k);
        const int N = c->n, L = c->L, m = c->m;
        int size = 1;
        while (size < N) size *= 2;
        const int npair = k * (k + 1) / 2;
        c->Y.ensure((long long)N * m, L);
        c->T.ensure((long long)npair * size, L);
        c->T2.ensure((long long)npair * (size / 2 > 0 ? size / 2 : 1), L);
        c->M.ensure((long long)k * k, L);
        const int wo = ws_op_words(L);
        ck(cudaEventRecord(c->ev[0], c->st), "event");
        launch(c, hk::ItemBlockY{c->X.view(), c->R.view(), c->Y.view(), N, L, m}, (long long)N * m, wo);
        launch(c, hk::ItemBlockTerms{c->X.view(), c->Y.view(), c->T.view(), N, L, m, k, size}, (long long)npair * size,
               wo);
        DevArr* cur = &c->T;
        DevArr* nxt = &c->T2;
        for (int half = size / 2; half >= 1; half /= 2) {
            launch(c, hk::ItemTreeLevel{cur->view(), nxt->view(), L, half}, (long long)npair * half, wo);
            std::swap(cur, nxt);
        }
        launch(c, hk::ItemBlockOut{cur->view(), c->M.view(), L, k}, npair, 64);
        ck(cudaEventRecord(c->ev[1], c->st), "event");
        ck(cudaEventSynchronize(c->ev[1]), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
        c->t[3] = ms * 1e-3;
        c->k = k;
        c->assembled = true;
        return HK_OK;
    });
}

int hk_get_block(hk_ctx* c, uint32_t* limbs, int32_t* exps, int32_t* signs) {
    return guarded(c, [&] {
        if (!c->assembled) return fail(c, HK_ERR_INVALID, "hk_get_block: not assembled");
        d2h_range(c, c->M, 0, (long long)c->k * c->k, limbs, exps, signs);
        return HK_OK;
    });
}

int hk_smallest_eigs(hk_ctx* c, int s, double* lambda_hi, double* lambda_lo, double* trunc_err) {
    return guarded(c, [&] {
        if (!c->assembled) return fail(c, HK_ERR_INVALID, "smallest_eigs_of_H: no block");
        const int k = c->k, L = c->L;
        const double t0 = now_s();
        c->h_limbs.resize(size_t(k) * k * L);
        c->h_e.resize(size_t(k) * k);
        c->h_s.resize(size_t(k) * k);
        d2h_range(c, c->M, 0, (long long)k * k, c->h_limbs.data(), c->h_e.data(), c->h_s.data());
        const double t1 = now_s();
        const char* why = "";
        const int rc = hk_block_eigs_impl(k, L, c->h_limbs.data(), c->h_e.data(), c->h_s.data(), s, lambda_hi,
                                          lambda_lo, trunc_err, &why);
        c->t[6] = t1 - t0;
        c->t[4] = now_s() - t1;
        if (rc != HK_OK) return fail(c, rc, why);
        return HK_OK;
    });
}

namespace {
// the path after the moments are on the device (pipeline.cpp:41-66)
int compute_tail(hk_ctx* c, int n, int rc, int k, double* lambda_hi, double* lambda_lo, double* trunc_err,
                 int* s_out, double t0) {
    const int kk = k < n ? k : n;    // pipeline.cpp:36
    const int s = kk < 3 ? kk : 3;   // pipeline.cpp:64
    // L^-1 and the block are sharded too (every rank takes part); rank 0 then
    // holds the block and runs the eigensolve.  HK_DIST_INV=0: rank 0 alone
    // from the gathered columns.
    const bool root = c->rank == 0;
    const bool all = (c->world > 1 || c->virt || c->nccl_comm) && !sharded_inv_off();
    if (rc == HK_OK) rc = hk_ldlt_invert(c, kk); // (ranks that take no part in L^-1 stop after the LDLT)
    if (rc == HK_OK && (root || all)) rc = hk_assemble_block(c, kk);
    if (rc == HK_OK && root) rc = hk_smallest_eigs(c, s, lambda_hi, lambda_lo, trunc_err);
    // every rank returns rank 0's record (status, lambdas), so a caller's
    // auto_precision / scan loop takes the same branch on every rank
    if (c->nccl_comm && c->world > 1 && c->n == n) {
        const int rb = share_root_result(c, &rc, s, lambda_hi, lambda_lo, trunc_err);
        if (rb != HK_OK) rc = rb;
    }
    if (s_out) *s_out = rc == HK_OK ? s : 0;
    c->t[0] = now_s() - t0;
    return rc;
}
} // namespace

int hk_compute(hk_ctx* c, int n, const uint32_t* limbs, const int32_t* exps, const int32_t* signs, int k,
               double* lambda_hi, double* lambda_lo, double* trunc_err, int* s_out) {
    if (!c) return HK_ERR_INVALID;
    if (n < 1) return fail(c, HK_ERR_INVALID, "compute: need N >= 1");
    if (k < 1) return fail(c, HK_ERR_INVALID, "compute: need k >= 1");
    const double t0 = now_s();
    const int rc = hk_load_moments(c, n, limbs, exps, signs);
    return compute_tail(c, n, rc, k, lambda_hi, lambda_lo, trunc_err, s_out, t0);
}

int hk_compute_generated(hk_ctx* c, unsigned beta_num, unsigned beta_den, int n, int k, double* lambda_hi,
                         double* lambda_lo, double* trunc_err, int* s_out, int* moments_exact) {
    if (!c) return HK_ERR_INVALID;
    if (n < 1) return fail(c, HK_ERR_INVALID, "compute: need N >= 1");
    if (k < 1) return fail(c, HK_ERR_INVALID, "compute: need k >= 1");
    const double t0 = now_s();
    const int rc = hk_generate_moments(c, beta_num, beta_den, n, moments_exact);
    return compute_tail(c, n, rc, k, lambda_hi, lambda_lo, trunc_err, s_out, t0);
}

int hk_set_limbs(hk_ctx* c, int limbs) {
    if (!c || limbs < 1 || limbs > 8192) return HK_ERR_INVALID;
    return guarded(c, [&] {
        if (limbs == c->L) return HK_OK;
        ck(cudaStreamSynchronize(c->st), "sync");
        drop_graphs(c);
        for (DevArr* a : {&c->mu, &c->S, &c->R, &c->B, &c->X, &c->Y, &c->T, &c->T2, &c->M, &c->Dg, &c->Vf}) a->release();
        for (auto& sh : c->shards) {
            for (DevArr* a : {&sh.S, &sh.panel, &sh.R, &sh.B, &sh.X, &sh.Y, &sh.T, &sh.T2}) a->release();
            sh.setup_n = -1;
            sh.rows_n = -1;
        }
        for (void* p : {(void*)c->tc_P, (void*)c->tc_A, (void*)c->tc_fb, (void*)c->tc_gcarry})
            if (p) cudaFree(p);
        if (c->inv_A) cudaFree(c->inv_A);
        c->inv_A = nullptr;
        c->inv_A_n = 0;
        c->tc_P = nullptr;
        c->tc_A = nullptr;
        c->tc_fb = nullptr;
        c->tc_gcarry = nullptr;
        c->tc_P_words = 0;
        c->tc_fb_cap = 0;
        c->tc_A_n = 0;
        c->L = limbs;
        c->n = c->m = c->k = 0;
        c->factored = c->inverted = c->assembled = false;
        return HK_OK;
    });
}

int hk_timings(const hk_ctx* c, double* out7) {
    if (!c || !out7) return HK_ERR_INVALID;
    for (int i = 0; i < 7; ++i) out7[i] = c->t[i];
    return HK_OK;
}

int hk_mp_batch(hk_ctx* c, int op, long long count, const uint32_t* a_l, const int32_t* a_e, const int32_t* a_s,
                const uint32_t* b_l, const int32_t* b_e, const int32_t* b_s, const uint32_t* c_l, const int32_t* c_e,
                const int32_t* c_s, uint32_t* o_l, int32_t* o_e, int32_t* o_s) {
    return guarded(c, [&] {
        const bool cta = (op & HK_OP_CTA) != 0;
        op &= ~HK_OP_CTA;
        if (op < 0 || op > 3 || count < 1 || (cta && op == HK_OP_ADD))
            return fail(c, HK_ERR_INVALID, "hk_mp_batch: bad op/count");
        if ((op != HK_OP_RECIP && (!b_l || !b_e || !b_s)) || (op == HK_OP_FMS && (!c_l || !c_e || !c_s)))
            return fail(c, HK_ERR_INVALID, "hk_mp_batch: missing operand");
        const int L = c->L;
        DevArr A, B, C, O;
        h2d_soa(c, A, count, a_l, a_e, a_s);
        if (op != HK_OP_RECIP) h2d_soa(c, B, count, b_l, b_e, b_s);
        if (op == HK_OP_FMS) h2d_soa(c, C, count, c_l, c_e, c_s);
        O.ensure(count, L);
        const int ws = op == HK_OP_RECIP ? ws_recip_words(L) : ws_op_words(L);
        if (cta)
            launch_cta(c, hk::CItemBatch{A.view(), B.view(), C.view(), O.view(), L, op == HK_OP_RECIP ? 2 : op}, count,
                       op == HK_OP_RECIP ? ws_cta_recip_words(L) : ws_cta_words(L));
        else
            launch(c, hk::ItemBatch{A.view(), B.view(), C.view(), O.view(), L, op}, count, ws);
        ck(cudaStreamSynchronize(c->st), "sync");
        d2h_range(c, O, 0, count, o_l, o_e, o_s);
        A.release();
        B.release();
        C.release();
        O.release();
        return HK_OK;
    });
}

} // extern "C"

// ------------------------------------------------------------------ measurement hooks

namespace {

// Register-only IMAD.WIDE carry-chain microkernel: 8 independent 96-bit
// accumulators per thread, the exact instruction mix of the column-sum loop.
__global__ void __launch_bounds__(256) k_peak_imad(int iters, uint32_t seed, uint32_t* sink) {
    uint32_t a0[8], a1[8], a2[8], x[8];
    const uint32_t y = seed ^ (threadIdx.x * 2654435761u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a0[j] = a1[j] = a2[j] = 0;
        x[j] = seed * (j + 1) + threadIdx.x;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
                         "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
                         "addc.u32 %2, %2, 0;"
                         : "+r"(a0[j]), "+r"(a1[j]), "+r"(a2[j])
                         : "r"(x[j]), "r"(y));
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s ^= a0[j] ^ a1[j] ^ a2[j];
    if (s == 0x12345678u) sink[threadIdx.x] = s;
}

// int8 tensor-core peak: one CTA per SM, thread 0 issues back-to-back
// tcgen05.mma kind::i8 M=128 N=256 K=32 (the product kernel's shape) from
// shared memory into two alternating TMEM accumulators.
__global__ void __launch_bounds__(128, 1) k_peak_i8(int iters, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t psm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr;
    const int tid = threadIdx.x;
    for (int q = tid; q < (4096 + 8192) / 4; q += blockDim.x) reinterpret_cast<uint32_t*>(psm)[q] = q * 2654435761u;
    hk::tc::fence_async_smem();
    if (tid < 32) hk::tc::tmem_alloc(&taddr, 512);
    if (tid == 0) hk::tc::mbar_init(&bar, 1);
    hk::tc::fence_before();
    __syncthreads();
    hk::tc::fence_after();
    const uint32_t tm = taddr;
    if (tid == 0) {
        const uint32_t idesc = hk::tc::idesc_u8(128, 256, false, true);
        const uint64_t ad = hk::tc::sdesc(psm, 128, 256), bd = hk::tc::sdesc(psm + 4096, 128, 512);
        for (int it = 0; it < iters; ++it) hk::tc::mma_i8(tm + uint32_t((it & 1) * 256), ad, bd, idesc, it > 1);
        hk::tc::commit(&bar);
        hk::tc::mbar_wait(&bar, 0);
    }
    __syncthreads();
    hk::tc::fence_after();
    uint32_t v[8];
    hk::tc::tmem_ld8(tm + ((uint32_t)((tid >> 5) * 32) << 16), v);
    hk::tc::tmem_ld_wait();
    if (v[0] == 0x12345678u && v[1] == 7u) sink[tid] = v[2];
    hk::tc::fence_before();
    __syncthreads();
    if (tid < 32) hk::tc::tmem_dealloc(tm, 512);
}

} // namespace

extern "C" {

void* hk_stream(const hk_ctx* c) { return c ? (void*)c->st : nullptr; }

int hk_profile_ldlt(hk_ctx* c, double* ms7, long long* n_trailing) {
    return guarded(c, [&] {
        if (c->n < 1) return fail(c, HK_ERR_INVALID, "hk_profile_ldlt: no moments loaded");
        const int N = c->n, L = c->L;
        const long long ntri = (long long)N * (N + 1) / 2;
        c->S.ensure(ntri, L);
        c->R.ensure(N, L);
        c->B.ensure(3LL * N, L);
        ensure_tc_scratch(c);
        ck(cudaMemsetAsync(c->d_err, 0xff, sizeof(int), c->st), "memset err");
        struct Rec {
            int kind;
            cudaEvent_t a, b, mid;
        };
        std::vector<Rec> recs;
        const bool tc = use_tc(c);
        auto timed = [&](int kind, auto&& fn) {
            Rec r{kind, nullptr, nullptr, nullptr};
            ck(cudaEventCreate(&r.a), "event");
            ck(cudaEventCreate(&r.b), "event");
            if (kind == 0 && tc) ck(cudaEventCreate(&r.mid), "event");
            c->prof_mid = r.mid;
            ck(cudaEventRecord(r.a, c->st), "event");
            fn();
            ck(cudaEventRecord(r.b, c->st), "event");
            c->prof_mid = nullptr;
            recs.push_back(r);
        };
        const int wo = ws_op_words(L), wr = ws_recip_words(L);
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        ck(cudaEventRecord(e0, c->st), "event");
        launch(c, hk::ItemInitS{c->S.view(), c->mu.view(), N, L}, ntri, 64);
        if (c->tc_fb_count) ck(cudaMemsetAsync(c->tc_fb_count, 0, 2 * sizeof(int), c->st), "memset fb counters");
        long long nt = 0;
        for (int i = 0; i < N; ++i) {
            timed(1, [&] {
                launch_recip(c, i, c->st);
            });
            const int nb = N - i - 1;
            if (nb == 0) continue;
            timed(2, [&] {
                launch_cta(c, hk::CItemMulB{c->S.view(), c->R.view(), b_buf(c, i), N, L, i, c->d_err}, nb,
                           ws_cta_words(L));
            });
            timed(0, [&] {
                enqueue_bulk(c, i, i + 1, c->st);
            });
            ++nt;
            timed(3, [&] { launch(c, hk::ItemStoreL{c->S.view(), b_buf(c, i), N, L, i}, nb, 64); });
        }
        ck(cudaEventRecord(e1, c->st), "event");
        ck(cudaEventSynchronize(e1), "sync");
        for (int q = 0; q < 7; ++q) ms7[q] = 0;
        for (auto& r : recs) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, r.a, r.b), "elapsed");
            ms7[r.kind] += ms;
            if (r.mid) {
                float m1 = 0, m2 = 0;
                ck(cudaEventElapsedTime(&m1, r.a, r.mid), "elapsed");
                ck(cudaEventElapsedTime(&m2, r.mid, r.b), "elapsed");
                ms7[5] += m1;
                ms7[6] += m2;
                cudaEventDestroy(r.mid);
            }
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        float tot = 0;
        ck(cudaEventElapsedTime(&tot, e0, e1), "elapsed");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ms7[4] = tot;
        *n_trailing = nt;
        const int rc = check_pivots(c);
        if (rc == HK_OK) c->factored = true;
        return rc;
    });
}

int hk_peak_imad(int device, double* out) {
    if (!out) return HK_ERR_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return HK_ERR_RUNTIME;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return HK_ERR_RUNTIME;
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 1024 * sizeof(uint32_t)) != cudaSuccess) return HK_ERR_RUNTIME;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    k_peak_imad<<<blocks, threads>>>(64, 1u, sink); // warm-up
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_peak_imad<<<blocks, threads>>>(iters, 12345u + rep, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double macs = double(blocks) * threads * iters * 8.0;
        if (ms > 0 && macs / (ms * 1e-3) > best) best = macs / (ms * 1e-3);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return HK_ERR_RUNTIME;
    *out = best;
    return HK_OK;
}

int hk_peak_i8mma(int device, double* out) {
    if (!out) return HK_ERR_INVALID;
    if (cudaSetDevice(device) != cudaSuccess) return HK_ERR_RUNTIME;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return HK_ERR_RUNTIME;
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 1024 * sizeof(uint32_t)) != cudaSuccess) return HK_ERR_RUNTIME;
    const int smem = 120 * 1024; // one CTA per SM (512 TMEM columns each)
    cudaFuncSetAttribute(k_peak_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = prop.multiProcessorCount, iters = 20000;
    k_peak_i8<<<blocks, 128, smem>>>(64, sink); // warm-up
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_peak_i8<<<blocks, 128, smem>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double macs = double(blocks) * iters * 128.0 * 256.0 * 32.0;
        if (ms > 0 && macs / (ms * 1e-3) > best) best = macs / (ms * 1e-3);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return HK_ERR_RUNTIME;
    *out = best;
    return HK_OK;
}

} // extern "C"

// ====================================================================== multi-GPU
//
// Column-sharded LDLT: rank r owns columns {c : owner[c] == r} of
// the boustrophedon map (ldlt.cpp:22-35), stored concatenated (rows j..N-1 of
// each owned column j).  Every rank holds the pivot column i in a panel slot
// (rows i..N-1) and B_i, both triple-buffered by i % 3.  The step loop is the
// reference's depth-1 look-ahead (ldlt.cpp:271-331), recorded into one CUDA
// graph on two streams of every rank:
//   BULK (ctx stream)  [P(i)] U(i): step-i update of the owned columns >= i+2,
//                      then StoreL(i) on the owner of i (D_i, L(:,i) in place)
//   LA (high priority) P(i+1): the owner of column i+1 updates it with step i
//                      straight into panel slot i+1 [after its U(i-1)];
//                      ncclBroadcast(panel, root = owner(i+1)) (ldlt.cpp:294-298
//                      publish / 248 wait_complete); every rank derives
//                      R_{i+1} = recip(panel[0]) and B_{i+1} = panel * R_{i+1}
//                      with the same deterministic kernels (B never travels, so
//                      the reference's BroadcastPolicy chunking is moot).
// The broadcast and the reciprocal chain of step i+1 thus overlap the bulk
// update of step i on every GPU.  Slot (i+1) % 3 is rewritten only after
// StoreL(i-2), its last reader.  After the loop all columns are gathered to
// rank 0 (ncclSend/Recv), which runs L^{-1}, the block and the eigensolve as on
// one GPU.  Every op is correctly rounded, so results are bit-identical for any
// world size.  Virtual mode runs all ranks' shards in one process on one GPU
// with the broadcast / gather as device-to-device copies (tests the sharded
// kernels, index maps and the schedule on a single B200).

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

// libnccl.so.2 is dlopen'ed: inside a torch process this resolves to the NCCL
// torch already loaded (same SONAME), standalone to the system one.
NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false, ok = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            ok = (api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId")) &&
                 (api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank")) &&
                 (api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy")) &&
                 (api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast")) &&
                 (api.Send = (decltype(api.Send))dlsym(h, "ncclSend")) &&
                 (api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv")) &&
                 (api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart")) &&
                 (api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd")) &&
                 (api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString"));
        }
    }
    return ok ? &api : nullptr;
}

void nk(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw HkError{HK_ERR_RUNTIME, std::string(what) + ": " + (nccl_api() ? nccl_api()->GetErrorString(r) : "?")};
}

using Shard = hk_ctx::Shard;

MpArr slot3(const DevArr& a, int N, int L, int i) {
    const long long off = (long long)(i % 3) * N;
    return MpArr{a.d + off * L, a.m + off};
}

void shard_setup(hk_ctx* c, Shard& s, int N) {
    if (s.setup_n == N) return; // the maps depend on (N, world, owner map) only (setup_n reset on a change)
    s.owned.clear();
    s.loc.assign(size_t(N), -1);
    s.off.assign(1, 0);
    std::vector<int> erow, ecol;
    for (int j = 0; j < N; ++j) {
        if (c->owner[size_t(j)] != s.rank) continue;
        s.loc[size_t(j)] = int(s.owned.size());
        s.owned.push_back(j);
        for (int k = j; k < N; ++k) {
            erow.push_back(k);
            ecol.push_back(j);
        }
        s.off.push_back((long long)erow.size());
    }
    const long long tot = (long long)erow.size();
    s.S.ensure(tot > 0 ? tot : 1, c->L);
    s.panel.ensure(3LL * N, c->L);
    s.R.ensure(N, c->L);
    s.B.ensure(3LL * N, c->L);
    if (s.d_erow) cudaFree(s.d_erow);
    if (s.d_ecol) cudaFree(s.d_ecol);
    ck(cudaMalloc(&s.d_erow, size_t(tot > 0 ? tot : 1) * sizeof(int)), "malloc erow");
    ck(cudaMalloc(&s.d_ecol, size_t(tot > 0 ? tot : 1) * sizeof(int)), "malloc ecol");
    if (tot > 0) {
        ck(cudaMemcpyAsync(s.d_erow, erow.data(), size_t(tot) * sizeof(int), cudaMemcpyHostToDevice, c->st), "H2D erow");
        ck(cudaMemcpyAsync(s.d_ecol, ecol.data(), size_t(tot) * sizeof(int), cudaMemcpyHostToDevice, c->st), "H2D ecol");
    }
    if (!s.d_err) ck(cudaMalloc(&s.d_err, sizeof(int)), "malloc err");
    if (!s.d_fb) ck(cudaMalloc(&s.d_fb, 2 * sizeof(int)), "malloc fb");
    if (s.d_owned) cudaFree(s.d_owned);
    if (s.d_off) cudaFree(s.d_off);
    ck(cudaMalloc(&s.d_owned, (s.owned.size() + 1) * sizeof(int)), "malloc owned");
    ck(cudaMalloc(&s.d_off, s.off.size() * sizeof(long long)), "malloc off");
    if (!s.owned.empty())
        ck(cudaMemcpyAsync(s.d_owned, s.owned.data(), s.owned.size() * sizeof(int), cudaMemcpyHostToDevice, c->st),
           "H2D owned");
    ck(cudaMemcpyAsync(s.d_off, s.off.data(), s.off.size() * sizeof(long long), cudaMemcpyHostToDevice, c->st),
       "H2D off");
    ck(cudaStreamSynchronize(c->st), "sync");
    s.setup_n = N;
}

// index of the first owned column >= j0 (owned columns of >= j0 form a suffix
// of the local storage, starting at entry off[q])
size_t first_owned(const Shard& s, int j0) {
    return size_t(std::lower_bound(s.owned.begin(), s.owned.end(), j0) - s.owned.begin());
}

// U(i) on one shard: step-i update of its owned columns >= i+2 (the look-ahead
// column i+1 is done by P(i+1)); IMAD warp FMAs or the tensor-core products
// (mode 2 of the product kernel) + the certified rounding pass — the same ops
// as ItemDTrailing, bit-identical.
bool dist_bulk(hk_ctx* c, Shard& s, int i, bool tc, cudaStream_t st, int kslot = -1) {
    const int N = c->n, L = c->L;
    const size_t q = first_owned(s, i + 2);
    const int ncols = int(s.owned.size() - q);
    if (ncols <= 0) return false;
    const long long e0 = s.off[q], n = s.off.back() - e0;
    const MpArr panel = slot3(s.panel, N, L, i), B = slot3(s.B, N, L, i);
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot)], st);
    if (!tc) {
        launch(c, hk::ItemDTrailing{s.S.view(), panel, B, s.d_erow, s.d_ecol, L, i, e0, s.d_err}, n, ws_op_words(L),
               st);
        if (kslot >= 0) {
            graph_event(c->kev[size_t(3 * kslot + 1)], st);
            graph_event(c->kev[size_t(3 * kslot + 2)], st);
        }
        return true;
    }
    // fallback counters alternate by step: the fix-up of step i clears the one step i+1 uses
    int* cnt = s.d_fb + (i & 1);
    int* nxt = s.d_fb + ((i + 1) & 1);
    hk::TcBulkArgs a{s.S.view(), panel, c->tc_A, c->tc_P, N, L, i, s.owned[q], 2, 0, 0, s.d_err};
    a.owned = s.d_owned;
    a.off = s.d_off;
    a.e0 = e0;
    a.first_loc = int(q);
    const bool fuse = use_fuse(c);
    if (fuse) {
        a.fuse = fuse_mode();
        a.Y = B;
        a.fb_count = cnt;
        a.fb = c->tc_fb;
        a.force_fb = force_fix();
        a.viol = c->tc_fb_count + 3;
    }
    tc_products(c, a, B, unsigned(ncols), st);
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot + 1)], st);
    if (!fuse) {
        hk::ItemTcRoundD rd{s.S.view(), panel, B, s.d_erow, s.d_ecol, c->tc_P, L, i, e0, s.d_err, cnt, c->tc_fb};
        rd.force_fb = force_fix();
        launch(c, rd, n, hk::tcround_words(L), st);
    }
    launch_fix(c, hk::FixD{s.S.view(), panel, B, s.d_erow, s.d_ecol, L, i, e0}, st, cnt, nxt);
    if (kslot >= 0) graph_event(c->kev[size_t(3 * kslot + 2)], st);
    return true;
}

// make every shard's panel slot `col` hold column col (rows col..N-1): the
// owner wrote it; broadcast from there (ldlt.cpp:294-298 publish / 248 wait)
void dist_publish(hk_ctx* c, int col, cudaStream_t st) {
    const int N = c->n, L = c->L, root = c->owner[size_t(col)];
    const long long cnt = N - col;
    if (c->virt) {
        const MpArr src = slot3(c->shards[size_t(root)].panel, N, L, col);
        for (auto& s : c->shards) {
            if (s.rank == root) continue;
            const MpArr dst = slot3(s.panel, N, L, col);
            ck(cudaMemcpyAsync(dst.d, src.d, size_t(cnt) * L * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st),
               "panel copy");
            ck(cudaMemcpyAsync(dst.m, src.m, size_t(cnt) * sizeof(Meta), cudaMemcpyDeviceToDevice, st),
               "panel meta copy");
        }
        return;
    }
    const MpArr p = slot3(c->shards[0].panel, N, L, col);
    NcclApi* A = nccl_api();
    ncclComm_t comm = (ncclComm_t)c->nccl_comm;
    nk(A->GroupStart(), "group start");
    nk(A->Broadcast(p.d, p.d, size_t(cnt) * L, ncclUint32, root, comm, st), "bcast limbs");
    nk(A->Broadcast(p.m, p.m, size_t(cnt) * 2, ncclInt32, root, comm, st), "bcast meta");
    nk(A->GroupEnd(), "group end");
}

// R_i = RNE(1/panel_i[0]) (pivot test) and B_i = panel_i * R_i, on every rank
void dist_derive(hk_ctx* c, Shard& s, int i, cudaStream_t st) {
    const int N = c->n, L = c->L;
    const MpArr p = slot3(s.panel, N, L, i);
    if (size_t(ws_cta_recip_words(L)) * 4 <= c->smem_optin)
        launch_cta(c, hk::CItemDRecip{p, s.R.view(), L, i, s.d_err}, 1, ws_cta_recip_words(L), st);
    else
        launch(c, hk::ItemDRecip{p, s.R.view(), L, i, s.d_err}, 1, ws_recip_words(L), st);
    if (N - i - 1 > 0)
        launch_cta(c, hk::CItemDMulB{p, s.R.view(), slot3(s.B, N, L, i), L, i, s.d_err}, N - i - 1, ws_cta_words(L),
                   st);
}

// rank 0's (status, lambdas) to every rank: one ncclBroadcast of 11 doubles
int share_root_result(hk_ctx* c, int* rc, int s, double* hi, double* lo, double* te) {
    return guarded(c, [&] {
        double h[11] = {double(*rc), double(s), 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (c->rank == 0 && *rc == HK_OK)
            for (int q = 0; q < s && q < 3; ++q) {
                h[2 + q] = hi[q];
                h[5 + q] = lo[q];
                h[8 + q] = te[q];
            }
        if (!c->bcast_buf) ck(cudaMalloc(&c->bcast_buf, sizeof(h)), "cudaMalloc bcast");
        ck(cudaMemcpyAsync(c->bcast_buf, h, sizeof(h), cudaMemcpyHostToDevice, c->st), "H2D result");
        nk(nccl_api()->Broadcast(c->bcast_buf, c->bcast_buf, sizeof(h), ncclUint8, 0, (ncclComm_t)c->nccl_comm, c->st),
           "bcast result");
        ck(cudaMemcpyAsync(h, c->bcast_buf, sizeof(h), cudaMemcpyDeviceToHost, c->st), "D2H result");
        ck(cudaStreamSynchronize(c->st), "sync");
        const int root_rc = int(h[0]);
        if (c->rank != 0) {
            if (root_rc != HK_OK && *rc == HK_OK) c->err = "rank 0 failed with status " + std::to_string(root_rc);
            if (*rc == HK_OK) *rc = root_rc;
            if (root_rc == HK_OK)
                for (int q = 0; q < s && q < 3; ++q) {
                    hi[q] = h[2 + q];
                    lo[q] = h[5 + q];
                    te[q] = h[8 + q];
                }
        }
        return HK_OK;
    });
}

void enqueue_dist_steps(hk_ctx* c, bool tc) {
    const int N = c->n, L = c->L;
    cudaStream_t bulk = c->st, la = c->st2;
    ck(cudaEventRecord(c->evFork, bulk), "fork");
    ck(cudaStreamWaitEvent(la, c->evFork, 0), "fork wait");
    // P(0): column 0 (owned by rank 0) is final as loaded
    for (auto& s : c->shards)
        if (c->owner[0] == s.rank)
            launch(c, hk::ItemCopy{slot3(s.panel, N, L, 0), s.S.view(), 0, s.off[size_t(s.loc[0])], L}, N, 64, la);
    grow_events(c->cev, size_t(2 * N), cudaEventDefault);
    c->cev_steps = 0;
    c->kev_steps = 0;
    if (c->kprof) grow_events(c->kev, size_t(3 * N), cudaEventDefault);
    auto publish = [&](int col) { // timed: the broadcast including the wait for its root (ldlt.cpp:248)
        graph_event(c->cev[size_t(2 * c->cev_steps)], la);
        dist_publish(c, col, la);
        graph_event(c->cev[size_t(2 * c->cev_steps + 1)], la);
        ++c->cev_steps;
    };
    publish(0);
    for (auto& s : c->shards) dist_derive(c, s, 0, la);
    ck(cudaEventRecord(c->evP[0], la), "evP");
    for (int i = 0; i < N; ++i) {
        ck(cudaStreamWaitEvent(bulk, c->evP[size_t(i)], 0), "wait P");
        // one real rank per process: its bulk kernels are timed when kprof is on
        const bool timed = c->kprof && c->shards.size() == 1;
        for (auto& s : c->shards)
            if (dist_bulk(c, s, i, tc, bulk, timed ? c->kev_steps : -1) && timed) ++c->kev_steps;
        ck(cudaEventRecord(c->evU[size_t(i)], bulk), "evU");
        for (auto& s : c->shards)
            if (c->owner[size_t(i)] == s.rank)
                launch(c,
                       hk::ItemDStoreL{s.S.view(), slot3(s.panel, N, L, i), slot3(s.B, N, L, i),
                                       s.off[size_t(s.loc[size_t(i)])], L, i},
                       N - i, 64, bulk);
        ck(cudaEventRecord(c->evR[size_t(i)], bulk), "evR");
        if (i + 1 >= N) continue;
        // P(i+1): slot (i+1) % 3 was last read by U(i-2) / StoreL(i-2)
        if (i >= 2) ck(cudaStreamWaitEvent(la, c->evR[size_t(i - 2)], 0), "wait R");
        for (auto& s : c->shards) {
            if (c->owner[size_t(i + 1)] != s.rank) continue;
            if (i >= 1) ck(cudaStreamWaitEvent(la, c->evU[size_t(i - 1)], 0), "wait U"); // column i+1 after step i-1
            launch_cta(c,
                       hk::CItemDColUpd{s.S.view(), slot3(s.panel, N, L, i), slot3(s.B, N, L, i),
                                        slot3(s.panel, N, L, i + 1), s.off[size_t(s.loc[size_t(i + 1)])], L, i,
                                        s.d_err},
                       N - i - 1, ws_cta_words(L), la);
        }
        publish(i + 1);
        for (auto& s : c->shards) dist_derive(c, s, i + 1, la);
        ck(cudaEventRecord(c->evP[size_t(i + 1)], la), "evP");
    }
    ck(cudaEventRecord(c->evJoin, la), "join");
    ck(cudaStreamWaitEvent(bulk, c->evJoin, 0), "join wait");
}

// gather all columns into the standard jagged S on rank 0 (+ R)
void gather_to_root(hk_ctx* c) {
    const int N = c->n, L = c->L;
    const long long ntri = (long long)N * (N + 1) / 2;
    if (c->rank == 0) {
        c->S.ensure(ntri, L);
        c->R.ensure(N, L);
    }
    if (c->virt) {
        for (int j = 0; j < N; ++j) {
            Shard& o = c->shards[size_t(c->owner[size_t(j)])];
            const long long src = o.off[size_t(o.loc[size_t(j)])], dst = hk::tri_idx(j, j, N), cnt = N - j;
            ck(cudaMemcpyAsync(c->S.d + dst * L, o.S.d + src * L, size_t(cnt) * L * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, c->st), "gather");
            ck(cudaMemcpyAsync(c->S.m + dst, o.S.m + src, size_t(cnt) * sizeof(Meta), cudaMemcpyDeviceToDevice, c->st),
               "gather meta");
        }
        Shard& s0 = c->shards[0];
        ck(cudaMemcpyAsync(c->R.d, s0.R.d, size_t(N) * L * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->st), "R");
        ck(cudaMemcpyAsync(c->R.m, s0.R.m, size_t(N) * sizeof(Meta), cudaMemcpyDeviceToDevice, c->st), "R meta");
        return;
    }
    Shard& s = c->shards[0];
    NcclApi* A = nccl_api();
    ncclComm_t comm = (ncclComm_t)c->nccl_comm;
    const int batch = 128;
    for (int j0 = 0; j0 < N; j0 += batch) {
        nk(A->GroupStart(), "group start");
        for (int j = j0; j < N && j < j0 + batch; ++j) {
            const int o = c->owner[size_t(j)];
            const long long cnt = N - j;
            if (c->rank == 0) {
                const long long dst = hk::tri_idx(j, j, N);
                if (o == 0) {
                    const long long src = s.off[size_t(s.loc[size_t(j)])];
                    ck(cudaMemcpyAsync(c->S.d + dst * L, s.S.d + src * L, size_t(cnt) * L * sizeof(uint32_t),
                                       cudaMemcpyDeviceToDevice, c->st), "gather");
                    ck(cudaMemcpyAsync(c->S.m + dst, s.S.m + src, size_t(cnt) * sizeof(Meta), cudaMemcpyDeviceToDevice,
                                       c->st), "gather meta");
                } else {
                    nk(A->Recv(c->S.d + dst * L, size_t(cnt) * L, ncclUint32, o, comm, c->st), "recv");
                    nk(A->Recv(c->S.m + dst, size_t(cnt) * 2, ncclInt32, o, comm, c->st), "recv meta");
                }
            } else if (o == c->rank) {
                const long long src = s.off[size_t(s.loc[size_t(j)])];
                nk(A->Send(s.S.d + src * L, size_t(cnt) * L, ncclUint32, 0, comm, c->st), "send");
                nk(A->Send(s.S.m + src, size_t(cnt) * 2, ncclInt32, 0, comm, c->st), "send meta");
            }
        }
        nk(A->GroupEnd(), "group end");
    }
    if (c->rank == 0) {
        ck(cudaMemcpyAsync(c->R.d, s.R.d, size_t(N) * L * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->st), "R");
        ck(cudaMemcpyAsync(c->R.m, s.R.m, size_t(N) * sizeof(Meta), cudaMemcpyDeviceToDevice, c->st), "R meta");
    }
}

// ---- sharded L^{-1} and H^{-1} block ------------------
// Rows are owned in 128-row blocks, block b by rank b % world (the row tiles of
// the tensor-core product kernel).  Step i of the reference's row elimination
// (inversion.cpp:93-102; parallel form 106-230 with a per-row publish, 145-195):
//   * the column owner broadcasts column i of L (its panel slot; the LDLT's
//     pivot-column broadcast again) and the owner of row i broadcasts X(i, :)
//     (final after step i - 1);
//   * every rank updates its own rows j > i: X(j,c) = RNE(X(j,c) - L(j,i) X(i,c)),
//     X(j,i) = -L(j,i) (i < m) — each entry's chain in the reference's order, so
//     bit-identical to one GPU for any world size.
// Every row is broadcast at its step, so after the last one each rank holds all
// of X.  The block M(j,c) = sum_l X(l,j) X(l,c) / D_l: each rank forms the terms
// of its rows (the others' are exact zeros) and reduces them up to 128-row
// subtrees of the fixed pairwise tree; rank 0 takes each subtree from its owner
// and finishes the same tree — the single-GPU sum, bit for bit.

void shard_rows_setup(hk_ctx* c, Shard& s) {
    const int N = c->n;
    if (s.rows_n == N) return;
    s.otiles.clear();
    for (int t = 0; t * hk::kRowBlock < N; ++t)
        if (t % c->world == s.rank) s.otiles.push_back(t);
    if (s.d_otiles) cudaFree(s.d_otiles);
    s.d_otiles = nullptr;
    ck(cudaMalloc(&s.d_otiles, (s.otiles.size() + 1) * sizeof(int)), "malloc otiles");
    if (!s.otiles.empty())
        ck(cudaMemcpy(s.d_otiles, s.otiles.data(), s.otiles.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D otiles");
    s.rows_n = N;
}

int row_owner(const hk_ctx* c, int j) { return (j / hk::kRowBlock) % c->world; }

// X(i, 0 .. cnt) of the row owner -> every rank
void dist_publish_xrow(hk_ctx* c, int i, int cnt, cudaStream_t st) {
    if (cnt <= 0) return;
    const int L = c->L, m = c->m, root = row_owner(c, i);
    const long long off = (long long)i * m;
    if (c->virt) {
        const Shard& src = c->shards[size_t(root)];
        for (auto& s : c->shards) {
            if (s.rank == root) continue;
            ck(cudaMemcpyAsync(s.X.d + off * L, src.X.d + off * L, size_t(cnt) * L * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, st), "xrow copy");
            ck(cudaMemcpyAsync(s.X.m + off, src.X.m + off, size_t(cnt) * sizeof(Meta), cudaMemcpyDeviceToDevice, st),
               "xrow meta copy");
        }
        return;
    }
    Shard& s = c->shards[0];
    NcclApi* A = nccl_api();
    ncclComm_t comm = (ncclComm_t)c->nccl_comm;
    nk(A->GroupStart(), "group start");
    nk(A->Broadcast(s.X.d + off * L, s.X.d + off * L, size_t(cnt) * L, ncclUint32, root, comm, st), "bcast xrow");
    nk(A->Broadcast(s.X.m + off, s.X.m + off, size_t(cnt) * 2, ncclInt32, root, comm, st), "bcast xrow meta");
    nk(A->GroupEnd(), "group end");
}

// column i of L -> every rank's panel slot i % 3 (the owner copies it out of its columns first)
void dist_publish_lcol(hk_ctx* c, int i, cudaStream_t st) {
    const int N = c->n, L = c->L;
    for (auto& s : c->shards)
        if (c->owner[size_t(i)] == s.rank)
            launch(c, hk::ItemCopy{slot3(s.panel, N, L, i), s.S.view(), 0, s.off[size_t(s.loc[size_t(i)])], L}, N - i,
                   64, st);
    dist_publish(c, i, st);
}

void enqueue_dist_inv(hk_ctx* c, bool tc, cudaStream_t st) {
    const int N = c->n, L = c->L, m = c->m;
    for (auto& s : c->shards) {
        hk::ItemInvInit ini{hk::MpArr{}, s.X.view(), N, L, m};
        ini.zero = 1;
        launch(c, ini, (long long)N * m, 64, st);
    }
    if (c->tc_fb_count) ck(cudaMemsetAsync(c->tc_fb_count, 0, 2 * sizeof(int), st), "memset fb counters");
    for (int i = 0; i + 1 < N; ++i) {
        dist_publish_lcol(c, i, st);
        dist_publish_xrow(c, i, std::min(i, m), st);
        const int b = i < m ? i : m;
        for (auto& s : c->shards) {
            InvTarget tg;
            tg.Lsrc = slot3(s.panel, N, L, i);
            tg.panel = 1;
            tg.X = s.X.view();
            tg.rw = c->world;
            tg.rr = s.rank;
            if (tc) {
                // this rank's row tiles holding rows > i
                size_t q = 0;
                while (q < s.otiles.size() && (s.otiles[q] + 1) * hk::kRowBlock <= i + 1) ++q;
                tg.otiles = s.d_otiles + q;
                tg.ntiles = int(s.otiles.size() - q);
                enqueue_inv_tc(c, i, st, false, &tg);
            } else {
                hk::ItemInvStep f{tg.Lsrc, tg.X, N, L, m, i};
                f.panel = 1;
                f.rw = c->world;
                f.rr = s.rank;
                launch(c, f, (long long)(N - i - 1) * b + (i < m ? N - i - 1 : 0), ws_op_words(L), st);
            }
        }
    }
    if (N >= 2) dist_publish_xrow(c, N - 1, std::min(N - 1, m), st); // the last row: now every rank holds all of X
}

int dist_invert(hk_ctx* c, int m) {
    const int N = c->n, L = c->L;
    c->m = m;
    for (auto& s : c->shards) {
        s.X.ensure((long long)N * m, L);
        shard_rows_setup(c, s);
    }
    const bool tc = use_tc_inv(c);
    if (tc) ensure_tc_items(c, (size_t)N * m, (size_t)N * m + N);
    ck(cudaEventRecord(c->ev[0], c->st), "event");
    enqueue_dist_inv(c, tc, c->st);
    if (c->rank == 0) { // rank 0's copy of X is the result (hk_get_Linv, the block)
        c->X.ensure((long long)N * m, L);
        const Shard& s0 = c->shards[0];
        ck(cudaMemcpyAsync(c->X.d, s0.X.d, size_t(N) * m * L * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->st), "X");
        ck(cudaMemcpyAsync(c->X.m, s0.X.m, size_t(N) * m * sizeof(Meta), cudaMemcpyDeviceToDevice, c->st), "X meta");
    }
    ck(cudaEventRecord(c->ev[1], c->st), "event");
    ck(cudaEventSynchronize(c->ev[1]), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
    c->t[2] = ms * 1e-3;
    c->inverted = true;
    c->assembled = false;
    return HK_OK;
}

int dist_block(hk_ctx* c, int k) {
    const int N = c->n, L = c->L, m = c->m;
    int size = 1;
    while (size < N) size *= 2;
    const int npair = k * (k + 1) / 2;
    const int B = std::min(hk::kRowBlock, size), nb = size / B; // subtrees of B leaves, block t on rank t % world
    const int wo = ws_op_words(L);
    ck(cudaEventRecord(c->ev[0], c->st), "event");
    for (auto& s : c->shards) {
        s.Y.ensure((long long)N * m, L);
        s.T.ensure((long long)npair * size, L);
        s.T2.ensure((long long)npair * std::max(size / 2, 1), L);
        launch(c, hk::ItemBlockY{s.X.view(), s.R.view(), s.Y.view(), N, L, m}, (long long)N * m, wo);
        hk::ItemBlockTerms tf{s.X.view(), s.Y.view(), s.T.view(), N, L, m, k, size};
        tf.rw = c->world;
        tf.rr = s.rank;
        launch(c, tf, (long long)npair * size, wo);
        DevArr* cur = &s.T;
        DevArr* nxt = &s.T2;
        for (int half = size / 2; half >= nb; half /= 2) {
            launch(c, hk::ItemTreeLevel{cur->view(), nxt->view(), L, half}, (long long)npair * half, wo);
            std::swap(cur, nxt);
        }
        if (cur != &s.T) std::swap(s.T, s.T2); // the subtree sums: s.T[q * nb + t]
    }
    // rank 0: subtree t from rank t % world, into its own T (then the remaining levels)
    const long long cnt = (long long)npair * nb;
    if (c->virt) {
        Shard& s0 = c->shards[0];
        for (int t = 0; t < nb; ++t) {
            const Shard& o = c->shards[size_t(t % c->world)];
            if (o.rank == 0) continue;
            for (int q = 0; q < npair; ++q) {
                const long long e = (long long)q * nb + t;
                ck(cudaMemcpyAsync(s0.T.d + e * L, o.T.d + e * L, size_t(L) * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                                   c->st), "subtree");
                ck(cudaMemcpyAsync(s0.T.m + e, o.T.m + e, sizeof(Meta), cudaMemcpyDeviceToDevice, c->st), "subtree m");
            }
        }
    } else if (c->world > 1) {
        // every rank sends its subtree array; rank 0 receives them into T2 [world][npair * nb] and picks
        Shard& s = c->shards[0];
        if (c->rank == 0) s.T2.ensure((long long)c->world * cnt, L);
        NcclApi* A = nccl_api();
        ncclComm_t comm = (ncclComm_t)c->nccl_comm;
        nk(A->GroupStart(), "group start");
        if (c->rank == 0) {
            for (int r = 1; r < c->world; ++r) {
                nk(A->Recv(s.T2.d + r * cnt * L, size_t(cnt) * L, ncclUint32, r, comm, c->st), "recv subtrees");
                nk(A->Recv(s.T2.m + r * cnt, size_t(cnt) * 2, ncclInt32, r, comm, c->st), "recv subtrees m");
            }
        } else {
            nk(A->Send(s.T.d, size_t(cnt) * L, ncclUint32, 0, comm, c->st), "send subtrees");
            nk(A->Send(s.T.m, size_t(cnt) * 2, ncclInt32, 0, comm, c->st), "send subtrees m");
        }
        nk(A->GroupEnd(), "group end");
        if (c->rank == 0)
            for (int t = 0; t < nb; ++t) {
                const int r = t % c->world;
                if (r == 0) continue;
                for (int q = 0; q < npair; ++q) {
                    const long long e = (long long)q * nb + t;
                    ck(cudaMemcpyAsync(s.T.d + e * L, s.T2.d + (r * cnt + e) * L, size_t(L) * sizeof(uint32_t),
                                       cudaMemcpyDeviceToDevice, c->st), "pick");
                    ck(cudaMemcpyAsync(s.T.m + e, s.T2.m + r * cnt + e, sizeof(Meta), cudaMemcpyDeviceToDevice, c->st),
                       "pick m");
                }
            }
    }
    if (c->rank == 0) {
        Shard& s0 = c->shards[0];
        DevArr* cur = &s0.T;
        DevArr* nxt = &s0.T2;
        nxt->ensure((long long)npair * std::max(nb / 2, 1), L);
        for (int half = nb / 2; half >= 1; half /= 2) {
            launch(c, hk::ItemTreeLevel{cur->view(), nxt->view(), L, half}, (long long)npair * half, wo);
            std::swap(cur, nxt);
        }
        c->M.ensure((long long)k * k, L);
        launch(c, hk::ItemBlockOut{cur->view(), c->M.view(), L, k}, npair, 64);
    }
    ck(cudaEventRecord(c->ev[1], c->st), "event");
    ck(cudaEventSynchronize(c->ev[1]), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
    c->t[3] = ms * 1e-3;
    c->k = k;
    c->assembled = c->rank == 0;
    return HK_OK;
}

int dist_ldlt(hk_ctx* c) {
    const int N = c->n, L = c->L;
    if ((int)c->owner.size() != N) {
        if (c->owner_custom)
            throw HkError{HK_ERR_INVALID, "decompose_parallel: the column assignment was set for another order"};
        c->owner.assign(size_t(N), 0);
        hk_assign_columns(N, c->world, c->owner.data());
        for (auto& s : c->shards) s.setup_n = -1;
        ++c->owner_version;
    }
    for (auto& s : c->shards) shard_setup(c, s, N);
    const bool tc = use_tc(c);
    if (tc) {
        long long most = 1;
        for (auto& s : c->shards) most = std::max(most, s.off.back());
        ensure_tc_items(c, use_fuse(c) ? 0 : size_t(most), size_t(most));
    }
    ensure_step_events(c, N);
    c->bad_col = -1;
    ck(cudaEventRecord(c->ev[0], c->st), "event");
    for (auto& s : c->shards) {
        ck(cudaMemsetAsync(s.d_err, 0xff, sizeof(int), c->st), "memset err");
        ck(cudaMemsetAsync(s.d_fb, 0, 2 * sizeof(int), c->st), "memset fb");
        launch(c, hk::ItemDInit{s.S.view(), c->mu.view(), s.d_erow, s.d_ecol, L}, s.off.back(), 64);
    }
    // the step graph is valid for the buffers it was captured on
    std::vector<const void*> sig{(const void*)(long long)N, (const void*)(long long)tc, c->tc_A, c->tc_P, c->tc_fb,
                                 (const void*)(long long)c->kprof, c->mu.d, (const void*)c->owner_version};
    for (auto& s : c->shards)
        for (const void* p : {(const void*)s.S.d, (const void*)s.panel.d, (const void*)s.B.d, (const void*)s.R.d,
                              (const void*)s.d_err, (const void*)s.d_fb, (const void*)s.d_erow, (const void*)s.d_owned})
            sig.push_back(p);
    if (!c->dist_graph || sig != c->dist_sig) {
        if (c->dist_graph) cudaGraphExecDestroy(c->dist_graph);
        c->dist_graph = nullptr;
        const long long before = c->launches;
        Capture cap(c->st);
        enqueue_dist_steps(c, tc);
        c->dist_graph = instantiate(cap.end(), cudaGraphInstantiateFlagUseNodePriority);
        c->dist_graph_launches = c->launches - before;
        c->launches = before;
        c->dist_sig = sig;
    }
    ck(cudaGraphLaunch(c->dist_graph, c->st), "graph launch");
    c->launches += c->dist_graph_launches;
    // pivot errors: every rank computed the same reciprocals, so the flags agree
    int bad = -1;
    for (auto& s : c->shards) {
        int e = -1;
        ck(cudaMemcpyAsync(&e, s.d_err, sizeof(int), cudaMemcpyDeviceToHost, c->st), "D2H err");
        ck(cudaStreamSynchronize(c->st), "sync");
        if (e >= 0 && (bad < 0 || e < bad)) bad = e;
    }
    if (bad >= 0) {
        c->bad_col = bad;
        c->factored = false;
        return fail(c, HK_ERR_PRECISION,
                    "LDLT pivot <= 0 at column " + std::to_string(bad) + ": matrix not positive definite at p=" +
                        std::to_string(32 * L) + " bits, increase the precision");
    }
    gather_to_root(c);
    ck(cudaEventRecord(c->ev[1], c->st), "event");
    ck(cudaEventSynchronize(c->ev[1]), "sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]), "elapsed");
    c->t[1] = ms * 1e-3;
    c->factored = c->rank == 0;
    c->dist_factored = true;
    c->inverted = c->assembled = false;
    return HK_OK;
}

} // namespace

extern "C" {

int hk_nccl_unique_id(void* out128) {
    NcclApi* A = nccl_api();
    if (!A || !out128) return HK_ERR_RUNTIME;
    ncclUniqueId id;
    if (A->GetUniqueId(&id) != ncclSuccess) return HK_ERR_RUNTIME;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, 128);
    return HK_OK;
}

int hk_create_sharded(int device, int limbs, int rank, int world, const void* nccl_id128, hk_ctx** out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return HK_ERR_INVALID;
    const int rc = hk_create(device, limbs, out);
    if (rc != HK_OK) return rc;
    hk_ctx* c = *out;
    c->world = world;
    c->rank = rank;
    c->virt = nccl_id128 == nullptr;
    const int r2 = guarded(c, [&] {
        if (c->virt) {
            if (rank != 0) return fail(c, HK_ERR_INVALID, "virtual mode emulates all ranks: rank must be 0");
            c->shards.resize(size_t(world));
            for (int r = 0; r < world; ++r) c->shards[size_t(r)].rank = r;
        } else {
            NcclApi* A = nccl_api();
            if (!A) return fail(c, HK_ERR_RUNTIME, "libnccl.so.2 not loadable");
            ncclUniqueId id;
            memcpy(&id, nccl_id128, 128);
            ncclComm_t comm;
            nk(A->CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
            c->nccl_comm = comm;
            c->shards.resize(1);
            c->shards[0].rank = rank;
        }
        return HK_OK;
    });
    if (r2 != HK_OK) {
        hk_destroy(c);
        *out = nullptr;
    }
    return r2;
}

int hk_fused_violations(hk_ctx* c, long long* out) {
    return guarded(c, [&] {
        if (!out) return fail(c, HK_ERR_INVALID, "hk_fused_violations: null output");
        int v = 0;
        if (c->tc_fb_count) {
            ck(cudaMemcpy(&v, c->tc_fb_count + 3, sizeof(int), cudaMemcpyDeviceToHost), "D2H violations");
        }
        *out = v;
        return HK_OK;
    });
}

int hk_fix_count(hk_ctx* c, long long* out) {
    return guarded(c, [&] {
        if (!out) return fail(c, HK_ERR_INVALID, "hk_fix_count: null output");
        unsigned long long v = 0;
        ck(cudaMemcpy(&v, c->fix_total, sizeof v, cudaMemcpyDeviceToHost), "D2H fix count");
        *out = (long long)v;
        return HK_OK;
    });
}

int hk_set_kernel_timing(hk_ctx* c, int on) {
    if (!c) return HK_ERR_INVALID;
    c->kprof = on != 0; // the LDLT graph signature includes it: recaptured on change
    return HK_OK;
}

int hk_kernel_times(hk_ctx* c, double* out6) {
    return guarded(c, [&] {
        if (!out6) return fail(c, HK_ERR_INVALID, "hk_kernel_times: null output");
        for (int q = 0; q < 6; ++q) out6[q] = 0.0;
        const bool dist = c->world > 1 || c->virt || c->nccl_comm;
        if (c->kprof && (dist ? c->dist_graph != nullptr : !c->graphs.empty())) {
            for (int s = 0; s < c->kev_steps; ++s) {
                out6[0] += event_ms(c->kev[size_t(3 * s)], c->kev[size_t(3 * s + 1)]);
                out6[1] += event_ms(c->kev[size_t(3 * s + 1)], c->kev[size_t(3 * s + 2)]);
            }
            out6[2] = c->kev_steps;
        }
        if (dist && c->dist_graph) {
            for (int s = 0; s < c->cev_steps; ++s) out6[3] += event_ms(c->cev[size_t(2 * s)], c->cev[size_t(2 * s + 1)]);
            out6[4] = c->cev_steps;
        }
        out6[5] = c->t[1] * 1e3;
        return HK_OK;
    });
}

int hk_set_owner_map(hk_ctx* c, int n, const int32_t* owner) {
    return guarded(c, [&] {
        if (!(c->world > 1 || c->virt || c->nccl_comm))
            return fail(c, HK_ERR_INVALID, "hk_set_owner_map: not a sharded context");
        if (n < 1 || !owner) return fail(c, HK_ERR_INVALID, "hk_set_owner_map: need n >= 1 and a map");
        for (int j = 0; j < n; ++j)
            if (owner[j] < 0 || owner[j] >= c->world)
                return fail(c, HK_ERR_INVALID, "hk_set_owner_map: owner out of range at column " + std::to_string(j));
        c->owner.assign(owner, owner + n);
        c->owner_custom = true;
        ++c->owner_version;
        for (auto& sh : c->shards) sh.setup_n = -1;
        return HK_OK;
    });
}

int hk_kernel_step_times(hk_ctx* c, double* out, int cap, int* count) {
    return guarded(c, [&] {
        if (!count) return fail(c, HK_ERR_INVALID, "hk_kernel_step_times: null count");
        *count = 0;
        if (!c->kprof) return HK_OK;
        for (int s = 0; s < c->kev_steps && s < cap; ++s) {
            out[2 * s] = event_ms(c->kev[size_t(3 * s)], c->kev[size_t(3 * s + 1)]);
            out[2 * s + 1] = event_ms(c->kev[size_t(3 * s + 1)], c->kev[size_t(3 * s + 2)]);
            *count = s + 1;
        }
        return HK_OK;
    });
}

int hk_world(const hk_ctx* c, int* rank, int* world) {
    if (!c) return HK_ERR_INVALID;
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    return HK_OK;
}

} // extern "C"
