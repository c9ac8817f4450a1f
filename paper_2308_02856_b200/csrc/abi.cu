// abi.cu — the C-ABI (include/ssbh_cuda.h): argument validation with the reference's error
// semantics, device buffer management (ssbh_plan), and the launch sequence of the fused
// sample -> seed -> hash -> concatenate path. All compute goes to the GPU; there is no
// CPU fallback (without a device every compute entry point returns SSBH_NO_DEVICE).
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ssbh_cuda.h"
#include "common.cuh"
#include "internal.h"

using namespace ssbh_impl;

namespace {

thread_local std::string g_err;

ssbh_status fail(ssbh_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

ssbh_status ok() {
    g_err.clear();
    return SSBH_OK;
}

#define CU(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(SSBH_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                                \
    } while (0)

ssbh_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SSBH_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return SSBH_OK;
}

int usable_devices() {
    static int cached = -1;
    static std::once_flag once;
    std::call_once(once, [] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        int good = 0;
        for (int d = 0; d < n; ++d) {
            cudaDeviceProp p;
            if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
        }
        cached = good;
    });
    return cached;
}

ssbh_status need_device() {
    if (usable_devices() <= 0)
        return fail(SSBH_NO_DEVICE,
                    "no sm_100 CUDA device available: the B200 path has no CPU fallback");
    return SSBH_OK;
}

#define NEED_DEVICE()                              \
    do {                                           \
        ssbh_status s_ = need_device();            \
        if (s_ != SSBH_OK) return s_;              \
    } while (0)

// RAII device buffer
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    cudaError_t alloc(size_t b) {
        release();
        bytes = b ? b : 16;
        return cudaMalloc(&p, bytes);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }
uint64_t words64(uint64_t bits) { return (bits + 63) / 64; }

// ---- per-thread call context of the reference-facing entry points ----------------------
// toeplitz_hash, KeyedStream::bits, assign_subblocks, sift_partition ... are called once per
// block by the reference's own callers (pipeline.cpp:129-136), so their fixed cost matters.
// Each thread keeps, per device, a non-blocking stream and a device arena that survives the
// call: buffers of one call are carved from it (256-B aligned), nothing is cudaMalloc'ed or
// freed in steady state, and every copy/launch of the call is ordered on the thread's stream
// (no legacy-stream device-wide syncs, so threads calling concurrently overlap). An arena
// that runs out mid-call chains one more block; at the end of the call the blocks are merged
// into one of the combined size for the next call.
struct CallArena {
    struct Blk {
        char* p;
        size_t cap, used;
    };
    int device = -1;
    cudaStream_t st = nullptr;
    std::vector<Blk> blks;
    size_t want = 0;  // capacity of the merged block to allocate at the next call
    int depth = 0;

    cudaError_t take(size_t bytes, void** out) {
        bytes = round_up(bytes ? bytes : 16, 256);
        if (blks.empty() || blks.back().used + bytes > blks.back().cap) {
            size_t cap = std::max(bytes, want);
            want = 0;
            if (!blks.empty()) cap = std::max(bytes, blks.back().cap);
            Blk b{nullptr, cap, 0};
            if (cudaError_t e = cudaMalloc(&b.p, cap)) return e;
            blks.push_back(b);
        }
        *out = blks.back().p + blks.back().used;
        blks.back().used += bytes;
        return cudaSuccess;
    }
    void end_call() {  // the call's work is complete (every entry point synchronises)
        for (auto& b : blks) b.used = 0;
        if (blks.size() > 1) {
            size_t tot = 0;
            for (auto& b : blks) {
                tot += b.cap;
                cudaFree(b.p);
            }
            blks.clear();
            want = tot;
        }
    }
    void release() {
        for (auto& b : blks) cudaFree(b.p);
        blks.clear();
        want = 0;
        if (st) cudaStreamDestroy(st);
        st = nullptr;
    }
    ~CallArena() { release(); }  // thread exit (errors during process teardown are ignored)
};

struct CallCtx {
    std::vector<std::unique_ptr<CallArena>> per_dev;
    CallArena* cur = nullptr;
};
thread_local CallCtx g_call;

// Opens the calling thread's context on the current device for one entry-point call.
struct CallScope {
    CallArena* a = nullptr;
    cudaError_t err = cudaSuccess;
    CallScope() {
        int dev = 0;
        if ((err = cudaGetDevice(&dev))) return;
        if ((size_t)dev >= g_call.per_dev.size()) g_call.per_dev.resize(dev + 1);
        auto& slot = g_call.per_dev[dev];
        if (!slot) {
            slot.reset(new CallArena());
            slot->device = dev;
            if ((err = cudaStreamCreateWithFlags(&slot->st, cudaStreamNonBlocking))) return;
        }
        a = slot.get();
        ++a->depth;
    }
    ~CallScope() {
        if (a && --a->depth == 0) {
            cudaStreamSynchronize(a->st);
            a->end_call();
        }
    }
    cudaStream_t stream() const { return a->st; }
};

// Arena-backed buffer with DBuf's interface (valid until the enclosing CallScope ends).
struct SBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t alloc(size_t b) {
        bytes = b ? b : 16;
        int dev = 0;
        if (cudaError_t e = cudaGetDevice(&dev)) return e;
        CallArena* a = (size_t)dev < g_call.per_dev.size() ? g_call.per_dev[dev].get() : nullptr;
        if (!a || !a->depth) return cudaErrorInvalidValue;  // only inside a CallScope
        return a->take(bytes, &p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace

#define CALL_SCOPE(name)                                                                   \
    CallScope name;                                                                        \
    if (name.err)                                                                          \
        return fail(SSBH_CUDA, "call context: %s", cudaGetErrorString(name.err));

// ======================================================================== runtime
extern "C" int ssbh_abi_version(void) { return SSBH_ABI_VERSION; }
extern "C" const char* ssbh_last_error(void) { return g_err.c_str(); }
extern "C" int ssbh_device_count(void) { return usable_devices(); }
extern "C" ssbh_status ssbh_set_device(int device) {
    NEED_DEVICE();
    if (device < 0 || device >= usable_devices())
        return fail(SSBH_INVALID_ARGUMENT, "set_device: device %d out of range", device);
    CU(cudaSetDevice(device));
    return ok();
}

// ======================================================================== PRF
extern "C" ssbh_status ssbh_prf_block(const uint64_t key[4], const uint64_t ctr[4],
                                      uint64_t out[4]) {
    uint64_t ks[5];
    ssbh_dev::threefry_ks(key, ks);
    const ssbh_dev::U64x4 r = ssbh_dev::threefry(ks, ctr[0], ctr[1], ctr[2], ctr[3]);
    for (int i = 0; i < 4; ++i) out[i] = r.v[i];
    return ok();
}

extern "C" uint64_t ssbh_prf_tag(const char* purpose, size_t len) {
    return ssbh_dev::fnv1a(purpose, len);
}

extern "C" ssbh_status ssbh_stream_bits(const uint64_t key[4], uint64_t tag, uint64_t sub,
                                        uint64_t nbits, uint64_t* out_words) {
    if (nbits == 0) return ok();
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    const uint64_t w64 = words64(nbits);
    SBuf d;
    CU(d.alloc(w64 * 8));
    CU(cudaMemsetAsync(d.p, 0, w64 * 8, st));
    launch_stream_bits(key, tag, sub, nbits, d.as<uint32_t>(), st);
    if (auto s = check_launch("stream_bits")) return s;
    CU(cudaMemcpyAsync(out_words, d.p, w64 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_stream_words(const uint64_t key[4], uint64_t tag, uint64_t sub,
                                         uint64_t first, uint64_t count, uint64_t* out) {
    if (count == 0) return ok();
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    SBuf d;
    CU(d.alloc(count * 8));
    launch_stream_words(key, tag, sub, first, count, d.as<uint64_t>(), st);
    if (auto s = check_launch("stream_words")) return s;
    CU(cudaMemcpyAsync(out, d.p, count * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_stream_uniform_below(const uint64_t key[4], uint64_t tag,
                                                 uint64_t sub, uint64_t bound, uint64_t first,
                                                 uint64_t count, uint64_t* out) {
    if (bound == 0) return fail(SSBH_INVALID_ARGUMENT, "uniform_below: bound must be positive");
    if (count == 0) return ok();
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    SBuf d;
    CU(d.alloc(count * 8));
    launch_stream_uniform(key, tag, sub, bound, first, count, d.as<uint64_t>(), st);
    if (auto s = check_launch("stream_uniform")) return s;
    CU(cudaMemcpyAsync(out, d.p, count * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_stream_bernoulli(const uint64_t key[4], uint64_t tag, uint64_t sub,
                                             double p, uint64_t first, uint64_t count,
                                             uint64_t* out_words) {
    if (p < 0.0 || p > 1.0) return fail(SSBH_INVALID_ARGUMENT, "bernoulli: p outside [0,1]");
    if (count == 0) return ok();
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    const uint64_t w64 = words64(count);
    SBuf d;
    CU(d.alloc(w64 * 8));
    CU(cudaMemsetAsync(d.p, 0, w64 * 8, st));
    launch_stream_bernoulli(key, tag, sub, p, first, count, d.as<uint32_t>(), st);
    if (auto s = check_launch("stream_bernoulli")) return s;
    CU(cudaMemcpyAsync(out_words, d.p, w64 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_make_input_device(const uint64_t key[4], double p, uint64_t nbits,
                                              uint32_t* d_out, void* stream) {
    if (p < 0.0 || p > 1.0) return fail(SSBH_INVALID_ARGUMENT, "bernoulli: p outside [0,1]");
    NEED_DEVICE();
    launch_make_input(key, p, nbits, d_out, static_cast<cudaStream_t>(stream));
    return check_launch("make_input");
}

// ======================================================================== host scalars
// sampling.cpp:41-96 restated (host numerics, not data-parallel).
static ssbh_status rel_entropy(double x, double p, double* out) {
    if (!(p > 0.0 && p < 1.0))
        return fail(SSBH_INVALID_ARGUMENT, "relative_entropy: p must lie in (0,1)");
    if (!(x >= 0.0 && x <= 1.0))
        return fail(SSBH_INVALID_ARGUMENT, "relative_entropy: x must lie in [0,1]");
    if (x == 0.0)
        *out = std::log(1.0 / (1.0 - p));
    else if (x == 1.0)
        *out = std::log(1.0 / p);
    else
        *out = x * std::log(x / p) + (1.0 - x) * std::log((1.0 - x) / (1.0 - p));
    return ok();
}

extern "C" ssbh_status ssbh_relative_entropy(double x, double p, double* out) {
    return rel_entropy(x, p, out);
}

extern "C" ssbh_status ssbh_binomial_tail_bound(uint64_t n, uint64_t limit, double p,
                                                double* out) {
    const double x = (double)limit / (double)n;
    double h = 0;
    if (auto s = rel_entropy(x, p, &h)) return s;
    const double arg = std::sqrt(2.0 * (double)n * h);
    *out = 0.5 * std::erfc(arg / std::sqrt(2.0));
    return ok();
}

extern "C" ssbh_status ssbh_block_limit(uint64_t n, double p, double eps, uint64_t m_blocks,
                                        uint64_t* limit) {
    if (n == 0) return fail(SSBH_INVALID_ARGUMENT, "block_limit: n_rounds must be positive");
    if (!(p > 0.0 && p < 1.0))
        return fail(SSBH_INVALID_ARGUMENT, "block_limit: p_sift must lie in (0,1)");
    if (!(eps > 0.0 && eps < 1.0))
        return fail(SSBH_INVALID_ARGUMENT, "block_limit: eps_abort must lie in (0,1)");
    if (m_blocks == 0)
        return fail(SSBH_INVALID_ARGUMENT, "block_limit: m_blocks must be positive");
    const double threshold = eps / (double)m_blocks;
    if (threshold < 1e-300)
        return fail(SSBH_INFEASIBLE, "block_limit: per-block budget below erfc resolution");
    auto tail = [&](uint64_t L) {
        double v = 0;
        ssbh_binomial_tail_bound(n, L, p, &v);
        return v;
    };
    const uint64_t lo0 = (uint64_t)std::ceil((double)n * p);
    if (tail(n) > threshold)
        return fail(SSBH_INFEASIBLE, "block_limit: bound not met even at L = n_rounds");
    if (tail(lo0) <= threshold) {
        *limit = lo0;
        return ok();
    }
    uint64_t lo = lo0, hi = n;
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (tail(mid) <= threshold)
            hi = mid;
        else
            lo = mid;
    }
    *limit = hi;
    return ok();
}

extern "C" int ssbh_abort_check(const uint64_t* lengths, uint64_t count, uint64_t limit) {
    for (uint64_t i = 0; i < count; ++i)
        if (lengths[i] > limit) return 0;
    return 1;
}

extern "C" uint64_t ssbh_fnv1a64(const uint64_t* words, uint64_t count) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t w = words[i];
        for (int b = 0; b < 8; ++b, w >>= 8) h = (h ^ (w & 0xff)) * 0x100000001b3ull;
    }
    return h;
}

extern "C" ssbh_status ssbh_cycle_estimate(uint64_t input_len, uint64_t output_len,
                                           uint64_t m_prime, uint64_t* out) {
    if (m_prime == 0)
        return fail(SSBH_INVALID_ARGUMENT, "cycle_estimate: m_prime must be positive");
    const uint64_t passes = (output_len + m_prime - 1) / m_prime;
    const unsigned __int128 total = (unsigned __int128)input_len + output_len +
                                    (unsigned __int128)(input_len + m_prime) * passes;
    if (total > (unsigned __int128)~0ull)
        return fail(SSBH_OVERFLOW, "cycle_estimate: result exceeds 64 bits");
    *out = (uint64_t)total;
    return ok();
}

// ======================================================================== device layout
namespace {

template <class Buf>
struct LayoutBufsT {
    Buf nj, yoff, ypad, ktl, items, soff, stats;
    cudaError_t alloc(uint32_t nown) {
        cudaError_t e;
        if ((e = nj.alloc((size_t)nown * 8 + 8))) return e;
        if ((e = yoff.alloc((size_t)(nown + 1) * 8))) return e;
        if ((e = ypad.alloc((size_t)nown * 4 + 4))) return e;
        if ((e = ktl.alloc((size_t)nown * 4 + 4))) return e;
        if ((e = items.alloc((size_t)(nown + 1) * 8))) return e;
        if ((e = soff.alloc((size_t)(nown + 1) * 8))) return e;
        if ((e = stats.alloc(sizeof(DevStats)))) return e;
        return cudaSuccess;
    }
    Layout view() const {
        Layout l;
        l.nj = nj.template as<unsigned long long>();
        l.yoff = yoff.template as<unsigned long long>();
        l.ypad = ypad.template as<uint32_t>();
        l.ktl = ktl.template as<uint32_t>();
        l.items = items.template as<unsigned long long>();
        l.soff = soff.template as<unsigned long long>();
        l.stats = stats.template as<DevStats>();
        return l;
    }
};
using LayoutBufs = LayoutBufsT<DBuf>;   // plans: owned for the plan's lifetime
using LayoutScratch = LayoutBufsT<SBuf>;  // one call (CallScope arena)

// Choose the k-tile so that the persistent grid gets enough items (>= ~16 per CTA)
// while keeping tiles long enough to amortise per-item overhead.
uint32_t choose_kt(uint64_t mean_nj, uint32_t nown, uint32_t rowtiles, int grid) {
    const uint64_t yw = std::max<uint64_t>(1, (mean_nj + 31) / 32);
    uint64_t kt = kHashKTMax;
    const uint64_t per_cta = 8;  // round 1: 8 items per CTA, config 2 hash 0.870 -> 0.888
    const uint64_t want_items = (uint64_t)grid * per_cta;
    while (kt > 64) {
        const uint64_t items = (uint64_t)rowtiles * nown * ((yw + kt - 1) / kt);
        if (items >= want_items) break;
        kt /= 2;
    }
    return (uint32_t)std::max<uint64_t>(kHashR, kt / kHashR * kHashR);
}

}  // namespace

// Engine of a new plan: the tensor cores (toeplitz_mma.cu: shared seeds as one GEMM over all
// blocks, per-block seeds as tiled matrix-vector products) unless SSBH_HASH_ENGINE=lop3 keeps
// the plan on the integer ALUs (toeplitz.cu).
// Plan-construction overrides (ssbh_set_plan_overrides): explicit testing / A-B hooks, never
// read from the environment — a plan's kernels depend only on its parameters unless a caller
// sets these. Process-wide; copied when a plan is created.
static std::mutex g_over_mu;
static ssbh_plan_overrides g_over{SSBH_ENGINE_AUTO, -1, 0, -1, -1, 0, 0};

static ssbh_plan_overrides overrides() {
    std::lock_guard<std::mutex> lk(g_over_mu);
    return g_over;
}

static int default_engine(uint32_t per_block_seed) {
    (void)per_block_seed;
    return overrides().engine == SSBH_ENGINE_LOP3 ? kEngineLop3 : kEngineMma;
}

// ======================================================================== plan
struct ssbh_plan {
    ssbh_extract_params p{};
    int device = 0;
    uint32_t nown = 0;
    SamplerGeom geom{};
    uint32_t kw = 0, rowtiles = 0, kt = 0;
    bool direct_out = true;
    int grid = 0;
    uint64_t ybuf_words = 0, sbuf_words = 0, key_words32 = 0;
    DBuf payload, counts, gsum, ybuf, sbuf, scratch;
    LayoutBufs lay;
    DevStats* h_stats = nullptr;
    bool timing = false;
    cudaEvent_t ev[6]{};
    cudaStream_t last_stream = nullptr;
    uint32_t launches_per_run = 0;
    // CUDA graph(s) of one run (captured per stream / buffers / seeds; replayed afterwards):
    // one graph untimed, one per segment when timing
    cudaGraphExec_t exec[4] = {nullptr, nullptr, nullptr, nullptr};
    struct GraphKey {
        cudaStream_t st;
        const void *in, *keep, *key, *len;
        uint64_t sk[4], hk[4];
        bool timing;
        bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof *this) == 0; }
    } gkey{};
    // two-level split (large key spaces, see internal.h BucketGeom)
    bool bucketed = false;
    BucketGeom bg{};
    DBuf counts_a, gsum_a, tot_a, staging, counts_b, gsum_b, nj_b;
    // streaming plans (no payload buffer; input fed chunk by chunk)
    bool streaming = false;
    uint64_t chunk_bits = 0;
    uint64_t stream_samp[4]{}, stream_hash[4]{};
    uint32_t stream_launches = 0;
    // forward streaming (two-level streaming plans): no count pass over the whole input; block
    // j's rounds fill [j * fwd_cap, ...) of yfwd in round order, run_rank = its length so far
    bool fwd_stream = false;
    uint64_t fwd_cap = 0;  // bits per block region (a multiple of 256)
    uint64_t next_chunk = 0;  // forward streaming takes the input chunks in order
    DBuf yfwd, run_rank;
    // hash engine (shared-seed plans may run on the tensor cores, toeplitz_mma.cu)
    int engine = kEngineLop3;
    MmaGeom mma{};
    PbGeom pb{};
    bool shared_pb = false;  // shared seed hashed by the tiled matrix-vector kernel (long blocks)
    // 3-for-4 split of the long shared-seed squares (toeplitz_split.cu)
    bool split = false;
    SplitGeom sg{};
    PbGeom pbv{};
    DBuf vs, vy, vout, vrem;
    DBuf vu;         // GEMM leaves: Hankel unit tables of the leaf seeds
    LayoutBufs vlay, rlay;
    DBuf mt_words;
    DBuf vmt;        // split leaves on the GEMM kernel: max ypad per virtual M tile
    MmaGeom mmv{};   // split leaves on the GEMM kernel
    MmaGeom mmr{};   // split remainder on the GEMM kernel (shared seed)
    // host-path staging; late input: during a host run the input is copied on copy_stream while
    // the count pass (which needs only the round indices) runs, and the passes that read the
    // data bits wait for late_ev
    DBuf d_input, d_key, d_len, d_keep;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t late_ev = nullptr, prev_ev = nullptr;
    const uint32_t* late_input = nullptr;
    // host runs of single-batch GEMM-split plans: the combine runs in block slices and each
    // slice of the key leaves for the host (copy_stream) while the next one is combined
    uint64_t* host_key = nullptr;
    bool host_key_sent = false;
    static constexpr int kKeySlices = 8;
    cudaEvent_t slice_ev[kKeySlices] = {};
    cudaStream_t own_stream = nullptr;
    uint64_t bytes = 0;
};

static ssbh_status phase_sample(ssbh_plan* pl, const uint32_t* d_input, const uint32_t* d_keep,
                                const uint64_t* sk, cudaStream_t st, uint32_t& launches);
static ssbh_status phase_finish(ssbh_plan* pl, uint32_t* d_key, uint64_t* d_lengths,
                                const uint64_t* hk, cudaStream_t st, uint32_t& launches);
static ssbh_status bucket_passes(ssbh_plan* pl, const SamplerGeom& ga, const uint64_t* sk,
                                 uint64_t base, const uint32_t* d_input, const uint32_t* d_keep,
                                 const void* d_payload_src, cudaStream_t st, uint32_t& launches);

static ssbh_status validate_params(const ssbh_extract_params* p, uint32_t* nown) {
    if (!p) return fail(SSBH_INVALID_ARGUMENT, "extract: null params");
    if (p->n_subblocks == 0)
        return fail(SSBH_INVALID_ARGUMENT, "assign_subblocks: n_subblocks must be positive");
    if (p->out_bits == 0)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    if (p->n_subblocks > (1u << 30))
        return fail(SSBH_INVALID_ARGUMENT, "extract: n_subblocks above 2^30 unsupported");
    const uint32_t cnt = p->block_count ? p->block_count : p->n_subblocks;
    if ((uint64_t)p->block_first + cnt > p->n_subblocks)
        return fail(SSBH_INVALID_ARGUMENT, "extract: owned block range exceeds n_subblocks");
    if (p->n_rounds == 0)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    *nown = cnt;
    return SSBH_OK;
}

// external_payload: the plan consumes a payload it does not own (shard owners), whose element
// size is external_payload_bytes.
// Parent mode of the leaf GEMM: leaves of <= 4096 positions (the parent's input, 2 leaves, fits
// the 8192-position leaf buffer) and L >= 2.
static bool leaf_parent_mode(const SplitGeom& g) { return g.gemm && g.L >= 2 && g.sL <= 4096; }

static ssbh_status plan_create_impl(const ssbh_extract_params* params, uint64_t chunk_bits,
                                    ssbh_plan** out, bool external_payload = false,
                                    int external_payload_bytes = 0) {
    uint32_t nown = 0;
    if (auto s = validate_params(params, &nown)) return s;
    NEED_DEVICE();
    int max_cs = 40;
    if (chunk_bits) {
        if (chunk_bits % 1024 != 0)
            return fail(SSBH_INVALID_ARGUMENT, "streaming: chunk_bits must be a multiple of 1024");
        max_cs = __builtin_ctzll(chunk_bits);
    }
    auto* pl = new ssbh_plan();
    pl->p = *params;
    pl->nown = nown;
    pl->streaming = chunk_bits != 0;
    pl->chunk_bits = chunk_bits;
    CU(cudaGetDevice(&pl->device));
    const uint64_t n = params->n_rounds, k = params->out_bits;
    pl->geom = make_sampler_geom(n, params->n_subblocks, params->block_first, nown, false, max_cs);
    if (external_payload && external_payload_bytes) pl->geom.payload_bytes = external_payload_bytes;
    // in-memory single-level plans: ranks found in pass 1, order-free pass 3 (make_ranked)
    if (!external_payload && !chunk_bits && nown < kBucketMinBlocks && overrides().buckets != 1)
        pl->geom = make_ranked(pl->geom);
    pl->geom.scatter_window = overrides().scatter_window;
    pl->kw = (uint32_t)((k + 31) / 32);
    pl->rowtiles = (pl->kw + kHashRowWords - 1) / kHashRowWords;
    pl->direct_out = (k % 32) == 0;
    pl->grid = hash_grid_size(pl->device);
    // expected block length: shard owners see only their received rounds (n = the receive
    // capacity, spread over the owned blocks); other plans the whole input over all s blocks
    const uint64_t mean_nj = external_payload ? n / std::max<uint32_t>(nown, 1)
                                              : n / params->n_subblocks;
    pl->kt = choose_kt(mean_nj, nown, pl->rowtiles, pl->grid);
    // buffer bounds (n_j unknown on the host until the device has sampled):
    // sum_j round_up(ceil(n_j/32), R) <= n/32 + nown*R
    const uint64_t ybound = (n + 31) / 32 + (uint64_t)nown * kHashR + 8;
    pl->ybuf_words = round_up(ybound, 8);
    const uint64_t seed_fixed = (uint64_t)pl->rowtiles * kHashRowWords + 8;
    if (params->per_block_seed)
        pl->sbuf_words = round_up((uint64_t)nown * (seed_fixed + 8) + ybound + 64, 8);
    else
        pl->sbuf_words = round_up(seed_fixed + round_up((n + 31) / 32, kHashR) + 64, 8);
    pl->key_words32 = ((uint64_t)nown * k + 31) / 32;
    pl->engine = default_engine(params->per_block_seed);
    pl->mma = make_mma_geom(nown, pl->kw, mean_nj, pl->device);
    pl->pb = make_pb_geom(nown, pl->kw, pl->device, mean_nj);
    // Long shared-seed blocks: the tiled matrix-vector kernel keeps each block's y chunks in
    // shared memory for 256 D steps instead of re-expanding them for every 256-row tile (config
    // 3: hash 155 -> 145 ms); its window ramp (255 D steps per item) costs < 5 % once the mean
    // block has > 620 K bits.
    const ssbh_plan_overrides ov = overrides();
    {
        pl->shared_pb = !params->per_block_seed &&
                        (ov.shared_tiled >= 0 ? ov.shared_tiled == 1 : mean_nj >= (uint64_t)620000);
        // 3-for-4 split (toeplitz_split.cu) of long blocks: levels by split_levels (or
        // forced by the overrides). Shared-seed leaves run on the all-blocks GEMM, or on the
        // tiled kernel (override split_tiled_leaves).
        bool gemm = !params->per_block_seed && !ov.split_tiled_leaves;
        const bool forced = ov.split_levels >= 0;
        uint32_t L = forced ? (uint32_t)ov.split_levels : split_levels(k, gemm);
        pl->split = (gemm || pl->shared_pb || params->per_block_seed) &&
                    pl->engine == kEngineMma && split_applicable(k, mean_nj, L);
        if (pl->split) {
            // leaf buffer budget, default 8 GB
            const uint64_t budget = (uint64_t)(ov.split_budget_mb ? ov.split_budget_mb : 8192u) << 20;
            const bool pb_ok = pl->shared_pb || params->per_block_seed;
            pl->sg = make_split_geom(nown, k, mean_nj, L, params->per_block_seed != 0, gemm,
                                     budget);
            // a batch the budget cannot hold (few, very long blocks: GEMM groups are padded to
            // 128 blocks; 3^L leaves of one square grow as 1.5^L): tiled leaves, then fewer
            // levels, then the direct kernel
            if (pl->sg.bytes > budget && gemm && pb_ok) {
                gemm = false;
                pl->sg = make_split_geom(nown, k, mean_nj, L, params->per_block_seed != 0, false,
                                         budget);
            }
            while (pl->sg.bytes > budget && L > 1 && !forced) {
                --L;
                pl->sg = make_split_geom(nown, k, mean_nj, L, params->per_block_seed != 0, gemm,
                                         budget);
            }
            if (pl->sg.bytes > budget && !forced)
                pl->split = false;
        }
        if (pl->split) {
            const uint32_t lw = (uint32_t)(pl->sg.sL / 32);
            if (pl->sg.gemm) {
                pl->mmv = make_leaf_geom((uint32_t)pl->sg.nvirt, lw, pl->device,
                                         leaf_parent_mode(pl->sg));
                const uint64_t tk = (uint64_t)pl->sg.T * k;  // remainder: one GEMM as well
                pl->mmr = make_mma_geom(nown, pl->kw, mean_nj > tk ? mean_nj - tk : 1, pl->device);
            }
            else
                pl->pbv = make_pb_geom((uint32_t)pl->sg.nvirt, lw, pl->device, pl->sg.sL);
        }
    }

    // two-level split for large key spaces (override buckets = 0 / 1 disables / forces it)
    pl->bucketed = ov.buckets >= 0 ? ov.buckets == 1 : nown >= kBucketMinBlocks;
    if (pl->bucketed) {
        const uint64_t n_src = pl->streaming ? chunk_bits : n;
        const double mean = (double)n / (double)(external_payload ? nown : params->n_subblocks);
        pl->bg = make_bucket_geom(n_src, params->n_subblocks, params->block_first, nown,
                                  pl->streaming ? (double)chunk_bits / params->n_subblocks : mean,
                                  false, max_cs);
        // pass-A payload: the received payload's type for shard owners; u16 whenever V fits
        // 15 bits and no keep marker can occur (streaming runs take no keep mask)
        pl->bg.a.payload_bytes = external_payload ? pl->geom.payload_bytes
                                 : (params->n_subblocks < 32768 ||
                                    (pl->streaming && params->n_subblocks == 32768)) ? 2 : 4;
    }
    const BucketGeom& bg = pl->bg;

    auto alloc = [&](DBuf& b, size_t bytes) -> cudaError_t {
        pl->bytes += bytes;
        return b.alloc(bytes);
    };
    cudaError_t e = cudaSuccess;
    if (!pl->bucketed) {
        if (!e && !pl->streaming && !external_payload)
            e = alloc(pl->payload, (size_t)n * pl->geom.payload_bytes);
    } else {
        if (!e && !external_payload)
            e = alloc(pl->payload, (size_t)bg.a.n * bg.a.payload_bytes + 16);
        if (!e) e = alloc(pl->counts_a, (size_t)bg.a.nchunks * bg.nbuckets * 4);
        if (!e) e = alloc(pl->gsum_a, (size_t)bg.a.ngroups * bg.nbuckets * 8);
        if (!e) e = alloc(pl->tot_a, (size_t)bg.nbuckets * 8);
        if (!e) e = alloc(pl->staging, (size_t)bg.b.n * 2);
        if (!e) e = alloc(pl->counts_b, (size_t)bg.b.nchunks * bg.b.nown * 4);
        if (!e) e = alloc(pl->gsum_b, (size_t)bg.b.ngroups * bg.b.nown * 8);
        if (!e) e = alloc(pl->nj_b, (size_t)bg.nbuckets * bg.b.nown * 8);
    }
    // single-level count table (two-level streaming plans do without: forward streaming)
    pl->fwd_stream = pl->bucketed && pl->streaming;
    // + the ranked count pass's chunk counter (zeroed with the table)
    if (!e && !pl->bucketed) e = alloc(pl->counts, (size_t)pl->geom.nchunks * nown * 4 + 4);
    if (!e && !pl->bucketed) e = alloc(pl->gsum, (size_t)pl->geom.ngroups * nown * 8);
    if (!e && pl->fwd_stream) {
        // region per block: mean + 16 sigma of Binomial(n, 1/s) (a longer block raises the
        // overflow flag -> SSBH_CUDA, never silently)
        const double mean = (double)n / (double)params->n_subblocks;
        const uint64_t cap = (uint64_t)(mean + 16.0 * std::sqrt(mean) + 64.0);
        pl->fwd_cap = round_up(cap, 256);
        e = alloc(pl->yfwd, (size_t)nown * (pl->fwd_cap / 8) + 64);
        if (!e) e = alloc(pl->run_rank, (size_t)nown * 4 + 16);
    }
    if (!e) e = alloc(pl->ybuf, pl->ybuf_words * 4);
    if (!e) e = alloc(pl->sbuf, pl->sbuf_words * 4);
    if (!e && !pl->direct_out) e = alloc(pl->scratch, (size_t)nown * pl->kw * 4);
    if (!e && !params->per_block_seed) e = alloc(pl->mt_words, (size_t)pl->mma.mtiles * 4);
    if (!e && pl->split) {
        const SplitGeom& g = pl->sg;
        e = alloc(pl->vs,
                  ((g.per_block ? g.nvirt : (size_t)g.T * g.leaves) * g.seed_words + 256) * 4);
        if (!e && g.gemm) e = alloc(pl->vu, (size_t)g.T * g.leaves * g.unit_stride * 16 + 16);
        // leaf inputs: materialised only for tiled leaves (the leaf GEMM builds its own)
        if (!e && !g.gemm) e = alloc(pl->vy, (size_t)g.nvirt * g.vlw * 4 + 16);
        // leaf outputs (parent mode: level L - 1 nodes, 2/3 of the leaves' bytes)
        if (!e)
            e = alloc(pl->vout, (size_t)g.nvirt * (g.sL / 8) / (leaf_parent_mode(g) ? 3 : 1) *
                                        (leaf_parent_mode(g) ? 2 : 1) + 16);
        if (!e) e = alloc(pl->vrem, (size_t)nown * pl->kw * 4 + 16);
        if (!e) e = pl->vlay.alloc((uint32_t)g.nvirt);
        if (!e && g.gemm) e = alloc(pl->vmt, (size_t)pl->mmv.mtiles * 4);
        if (!e) e = pl->rlay.alloc(nown);
    }
    if (!e) e = pl->lay.alloc(nown);
    if (!e) e = cudaMallocHost(&pl->h_stats, sizeof(DevStats));
    for (int i = 0; i < 6 && !e; ++i) e = cudaEventCreate(&pl->ev[i]);
    if (e) {
        ssbh_plan_destroy(pl);
        return fail(SSBH_CUDA, "plan_create: device allocation failed: %s", cudaGetErrorString(e));
    }
    *out = pl;
    return ok();
}

extern "C" ssbh_status ssbh_set_plan_overrides(const ssbh_plan_overrides* o) {
    std::lock_guard<std::mutex> lk(g_over_mu);
    g_over = o ? *o : ssbh_plan_overrides{SSBH_ENGINE_AUTO, -1, 0, -1, -1, 0, 0};
    return ok();
}

extern "C" ssbh_status ssbh_get_plan_overrides(ssbh_plan_overrides* o) {
    if (!o) return fail(SSBH_INVALID_ARGUMENT, "null overrides");
    std::lock_guard<std::mutex> lk(g_over_mu);
    *o = g_over;
    return ok();
}

extern "C" ssbh_status ssbh_plan_create(const ssbh_extract_params* params, ssbh_plan** out) {
    return plan_create_impl(params, 0, out);
}

extern "C" ssbh_status ssbh_plan_create_streaming(const ssbh_extract_params* params,
                                                  uint64_t chunk_bits, ssbh_plan** out) {
    if (chunk_bits == 0) return fail(SSBH_INVALID_ARGUMENT, "streaming: chunk_bits must be positive");
    return plan_create_impl(params, chunk_bits, out);
}

extern "C" ssbh_status ssbh_plan_stream_begin(ssbh_plan* pl, const uint64_t* samp_key,
                                              const uint64_t* hash_key, void* stream) {
    if (!pl || !pl->streaming) return fail(SSBH_INVALID_ARGUMENT, "stream_begin: not a streaming plan");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl->last_stream = st;
    std::memcpy(pl->stream_samp, samp_key ? samp_key : pl->p.samp_key, 32);
    std::memcpy(pl->stream_hash, hash_key ? hash_key : pl->p.hash_key, 32);
    pl->stream_launches = 0;
    pl->next_chunk = 0;
    if (auto s = phase_sample(pl, nullptr, nullptr, pl->stream_samp, st, pl->stream_launches))
        return s;
    return check_launch("stream_begin");
}

extern "C" ssbh_status ssbh_plan_stream_chunk(ssbh_plan* pl, uint64_t chunk_index,
                                              const uint32_t* d_chunk, void* stream) {
    if (!pl || !pl->streaming || !d_chunk)
        return fail(SSBH_INVALID_ARGUMENT, "stream_chunk: not a streaming plan / null chunk");
    const uint64_t first = chunk_index * pl->chunk_bits;
    if (first >= pl->p.n_rounds)
        return fail(SSBH_INVALID_ARGUMENT, "stream_chunk: chunk index past the input");
    const uint64_t count = std::min<uint64_t>(pl->chunk_bits, pl->p.n_rounds - first);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl->last_stream = st;
    const Layout lay = pl->lay.view();
    if (pl->bucketed) {
        // two-level split of this chunk. The blocks' ranks continue from chunk to chunk in a
        // running array (no count pass over the whole input), so the chunks come in order.
        if (chunk_index != pl->next_chunk)
            return fail(SSBH_INVALID_ARGUMENT,
                        "stream_chunk: a two-level streaming plan takes its chunks in order "
                        "(expected chunk %llu)", (unsigned long long)pl->next_chunk);
        ++pl->next_chunk;
        const SamplerGeom ga = geom_with_n(pl->bg.a, count);
        if (auto s = bucket_passes(pl, ga, pl->stream_samp, first, d_chunk, nullptr, nullptr, st,
                                   pl->stream_launches))
            return s;
        // forward streaming: ranks continue from the blocks' lengths so far; the bits go to the
        // blocks' fixed regions in round order
        launch_bucket_scatter(pl->bg, pl->staging.as<uint16_t>(), pl->counts_b.as<uint32_t>(),
                              lay.nj, lay.yoff, pl->yfwd.as<uint32_t>(),
                              pl->run_rank.as<uint32_t>(), st, pl->fwd_cap);
        launch_add_ranks(pl->run_rank.as<uint32_t>(), pl->nj_b.as<unsigned long long>(), pl->nown,
                         pl->fwd_cap, &lay.stats->pad, st);
        pl->stream_launches += 2;
        return check_launch("stream_chunk");
    }
    launch_scatter_stream(pl->geom, pl->stream_samp, d_chunk, first, count,
                          pl->counts.as<uint32_t>(), lay.nj, lay.yoff, pl->ybuf.as<uint32_t>(), st);
    pl->stream_launches += 1;
    return check_launch("stream_chunk");
}

extern "C" ssbh_status ssbh_plan_stream_finish(ssbh_plan* pl, uint32_t* d_key, uint64_t* d_lengths,
                                               void* stream) {
    if (!pl || !pl->streaming || !d_key)
        return fail(SSBH_INVALID_ARGUMENT, "stream_finish: not a streaming plan / null key");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl->last_stream = st;
    if (auto s = phase_finish(pl, d_key, d_lengths, pl->stream_hash, st, pl->stream_launches))
        return s;
    pl->launches_per_run = pl->stream_launches;
    return check_launch("stream_finish");
}

extern "C" ssbh_status ssbh_plan_destroy(ssbh_plan* pl) {
    if (!pl) return ok();
    for (auto& e : pl->ev)
        if (e) cudaEventDestroy(e);
    if (pl->h_stats) cudaFreeHost(pl->h_stats);
    if (pl->own_stream) cudaStreamDestroy(pl->own_stream);
    if (pl->copy_stream) cudaStreamDestroy(pl->copy_stream);
    if (pl->late_ev) cudaEventDestroy(pl->late_ev);
    if (pl->prev_ev) cudaEventDestroy(pl->prev_ev);
    for (auto& e : pl->slice_ev)
        if (e) cudaEventDestroy(e);
    for (auto x : pl->exec)
        if (x) cudaGraphExecDestroy(x);
    delete pl;
    return ok();
}

extern "C" uint64_t ssbh_plan_device_bytes(const ssbh_plan* pl) { return pl ? pl->bytes : 0; }

extern "C" ssbh_status ssbh_plan_set_engine(ssbh_plan* pl, int engine) {
    if (!pl) return fail(SSBH_INVALID_ARGUMENT, "null plan");
    if (engine < SSBH_ENGINE_AUTO || engine > SSBH_ENGINE_TENSOR)
        return fail(SSBH_INVALID_ARGUMENT, "set_engine: unknown engine %d", engine);
    int e = engine == SSBH_ENGINE_AUTO ? default_engine(pl->p.per_block_seed) : engine;
    if (e != pl->engine) {
        pl->engine = e;
        for (auto& x : pl->exec)  // captured graphs hold the other engine's launches
            if (x) {
                cudaGraphExecDestroy(x);
                x = nullptr;
            }
    }
    return ok();
}

extern "C" int ssbh_plan_engine(const ssbh_plan* pl) { return pl ? pl->engine : -1; }

extern "C" const char* ssbh_plan_hash_kernel(const ssbh_plan* pl) {
    if (!pl) return "";
    if (pl->engine != kEngineMma) return "k_toeplitz_hash";
    if (pl->split)  // engine checked above
        return pl->sg.gemm ? "k_leaf_gemm+split" : "k_toeplitz_mma_pb+split";
    if (pl->p.per_block_seed || pl->shared_pb)
        return "k_toeplitz_mma_pb";
    return "k_toeplitz_f4";
}

extern "C" ssbh_status ssbh_plan_split_geometry(const ssbh_plan* pl, uint32_t* levels,
                                                uint32_t* squares, uint32_t* batch_blocks) {
    if (!pl) return fail(SSBH_INVALID_ARGUMENT, "null plan");
    const bool on = pl->split && pl->engine == kEngineMma;
    if (levels) *levels = on ? pl->sg.L : 0u;
    if (squares) *squares = on ? pl->sg.T : 0u;
    if (batch_blocks) *batch_blocks = on ? pl->sg.batch : 0u;
    return ok();
}

extern "C" ssbh_status ssbh_plan_set_timing(ssbh_plan* pl, int enable) {
    if (!pl) return fail(SSBH_INVALID_ARGUMENT, "null plan");
    pl->timing = enable != 0;
    return ok();
}

// ---- the run as four stream segments ---------------------------------------------------
//  S0 sample: pass 1-2 (Threefry V per round + payload, counts, scan, device-side layout)
//  S1 scatter: pass 3 (stable partition into reversed packed blocks)
//  S2 seeds:   Toeplitz seed material
//  S3 hash:    GF(2) hash, concatenation, lengths / stats copies
// Timing events go BETWEEN segments: directly launched, or each segment replayed as its own
// CUDA graph (events inside a captured graph cannot be timed).
static void rec(ssbh_plan* pl, int i, cudaStream_t st) {
    if (pl->timing) cudaEventRecord(pl->ev[i], st);
}

// Two-level passes from a pass-A payload (or Threefry when d_input is given): bucket counts,
// scan, split into the staging regions, pass-B counts and per-region scan (-> nj_b).
static ssbh_status bucket_passes(ssbh_plan* pl, const SamplerGeom& ga, const uint64_t* sk,
                                 uint64_t base, const uint32_t* d_input, const uint32_t* d_keep,
                                 const void* d_payload_src, cudaStream_t st, uint32_t& launches) {
    const BucketGeom& bg = pl->bg;
    const Layout lay = pl->lay.view();
    uint32_t* flags = &lay.stats->pad;
    CU(cudaMemsetAsync(pl->counts_a.p, 0, pl->counts_a.bytes, st));
    if (d_payload_src) {
        launch_count_payload(ga, d_payload_src, pl->counts_a.as<uint32_t>(), st, bg.shift);
    } else {
        launch_sample_buckets(bg, ga, sk, base, d_input, d_keep, pl->payload.p,
                              pl->counts_a.as<uint32_t>(), st);
        d_payload_src = pl->payload.p;
    }
    launch_scan(with_keys(ga, bg.nbuckets), pl->counts_a.as<uint32_t>(),
                pl->gsum_a.as<unsigned long long>(), pl->tot_a.as<unsigned long long>(), st);
    CU(cudaMemsetAsync(pl->staging.p, 0xff, pl->staging.bytes, st));
    if (pl->late_input) CU(cudaStreamWaitEvent(st, pl->late_ev, 0));
    launch_bucket_split(bg, ga, d_payload_src, pl->counts_a.as<uint32_t>(),
                        pl->tot_a.as<unsigned long long>(), pl->staging.as<uint16_t>(), flags, st,
                        pl->late_input);
    CU(cudaMemsetAsync(pl->counts_b.p, 0, pl->counts_b.bytes, st));
    launch_bucket_count(bg, pl->staging.as<uint16_t>(), pl->counts_b.as<uint32_t>(), st);
    launch_scan(bg.b, pl->counts_b.as<uint32_t>(), pl->gsum_b.as<unsigned long long>(),
                pl->nj_b.as<unsigned long long>(), st, bg.gps);
    launches += 10;
    return SSBH_OK;
}

static ssbh_status seg_sample(ssbh_plan* pl, const uint32_t* d_input, const uint32_t* d_keep,
                              const uint64_t* sk, cudaStream_t st, uint32_t& launches) {
    const Layout lay = pl->lay.view();
    if (pl->bucketed || pl->streaming)
        CU(cudaMemsetAsync(&lay.stats->pad, 0, 4, st));  // kFlagBucketOverflow of this run
    if (pl->late_input) d_input = nullptr;  // the data bits join in the split / scatter
    if (pl->fwd_stream) {  // stream_begin: nothing is counted ahead of the chunks
        CU(cudaMemsetAsync(pl->run_rank.p, 0, pl->run_rank.bytes, st));
        CU(cudaMemsetAsync(pl->yfwd.p, 0, pl->yfwd.bytes, st));
        return SSBH_OK;
    }
    if (pl->bucketed && !pl->streaming) {
        if (auto s = bucket_passes(pl, pl->bg.a, sk, 0, d_input, d_keep, nullptr, st, launches))
            return s;
        // block lengths: the per-region totals of the first nown local keys
        CU(cudaMemcpyAsync(lay.nj, pl->nj_b.p, (size_t)pl->nown * 8, cudaMemcpyDeviceToDevice,
                           st));
        launch_layout(lay, pl->nown, pl->p.out_bits, pl->rowtiles, pl->kt, pl->p.per_block_seed,
                      pl->p.block_limit, st);
        launches += 1;
        CU(cudaMemsetAsync(pl->ybuf.p, 0, pl->ybuf.bytes, st));
        return SSBH_OK;
    }
    // the ranked count pass writes every row of the table with plain stores: only its chunk
    // counter (the word after the table) starts at zero
    if (pl->geom.ranked && !pl->streaming)
        CU(cudaMemsetAsync(pl->counts.as<uint8_t>() + pl->counts.bytes - 4, 0, 4, st));
    else
        CU(cudaMemsetAsync(pl->counts.p, 0, pl->counts.bytes, st));
    // streaming: count only (a bucketed streaming plan's payload buffer holds one chunk)
    launch_sample_count(pl->geom, sk, d_input, d_keep, pl->streaming ? nullptr : pl->payload.p,
                        pl->counts.as<uint32_t>(), nullptr, st);
    launch_scan(pl->geom, pl->counts.as<uint32_t>(), pl->gsum.as<unsigned long long>(), lay.nj,
                st);
    launch_layout(lay, pl->nown, pl->p.out_bits, pl->rowtiles, pl->kt, pl->p.per_block_seed,
                  pl->p.block_limit, st);
    launches += 5;
    CU(cudaMemsetAsync(pl->ybuf.p, 0, pl->ybuf.bytes, st));
    return SSBH_OK;
}

static ssbh_status seg_scatter(ssbh_plan* pl, cudaStream_t st, uint32_t& launches) {
    const Layout lay = pl->lay.view();
    if (pl->bucketed) {
        launch_bucket_scatter(pl->bg, pl->staging.as<uint16_t>(), pl->counts_b.as<uint32_t>(),
                              lay.nj, lay.yoff, pl->ybuf.as<uint32_t>(), nullptr, st);
        launches += 1;
        return SSBH_OK;
    }
    if (pl->late_input) CU(cudaStreamWaitEvent(st, pl->late_ev, 0));
    launch_scatter(pl->geom, pl->payload.p, pl->counts.as<uint32_t>(), lay.nj, lay.yoff,
                   pl->ybuf.as<uint32_t>(), nullptr, nullptr, st, pl->late_input);
    launches += 1;
    return SSBH_OK;
}

static ssbh_status seg_seeds(ssbh_plan* pl, const uint64_t* hk, cudaStream_t st,
                             uint32_t& launches) {
    launch_seeds(hk, pl->lay.view(), pl->nown, pl->p.block_first, pl->p.per_block_seed,
                 pl->sbuf_words, pl->sbuf.as<uint32_t>(), st);
    launches += 1;
    return SSBH_OK;
}

static ssbh_status seg_hash(ssbh_plan* pl, uint32_t* d_key, uint64_t* d_lengths,
                            cudaStream_t st, uint32_t& launches) {
    const Layout lay = pl->lay.view();
    uint32_t* out = pl->direct_out ? d_key : pl->scratch.as<uint32_t>();
    CU(cudaMemsetAsync(out, 0, pl->direct_out ? pl->key_words32 * 4 : pl->scratch.bytes, st));
    if (pl->split && pl->engine == kEngineMma) {
        // leaves of the 3-for-4 split + the remainder past T k, then the XOR combine
        const SplitGeom& g = pl->sg;
        const Layout vlay = pl->vlay.view(), rlay = pl->rlay.view();
        launch_split_setup(pl->sbuf.as<uint32_t>(), pl->sbuf_words, g, pl->vs.as<uint32_t>(), lay,
                           pl->nown, vlay, rlay, st);
        if (g.gemm) {  // the leaf GEMM's B operand: unit tables of the leaf seeds
            launch_hankel_units(pl->vs.as<uint32_t>(), g.seed_words, (uint64_t)g.T * g.leaves,
                                g.unit_stride, pl->vu.as<uint32_t>(), st);
            launches += 1;
        }
        CU(cudaMemsetAsync(pl->vrem.p, 0, pl->vrem.bytes, st));
        if (g.gemm) {  // shared seed: the remainders are one short GEMM (seed offset T k)
            MmaHashArgs r{};
            r.ybuf = pl->ybuf.as<uint32_t>();
            r.sbuf = pl->sbuf.as<uint32_t>();
            r.out = pl->vrem.as<uint32_t>();
            r.out_stride = pl->kw;
            r.lay = rlay;
            r.nown = pl->nown;
            r.kw = pl->kw;
            r.ntiles = pl->mmr.ntiles;
            r.ksplit = pl->mmr.ksplit;
            r.items = pl->mmr.items;
            r.mt_words = pl->mt_words.as<uint32_t>();
            launch_hash_mma(r, pl->mmr, st);
            launches += 5;
        } else {
            PbHashArgs r{};
            r.ybuf = pl->ybuf.as<uint32_t>();
            r.sbuf = pl->sbuf.as<uint32_t>();
            r.out = pl->vrem.as<uint32_t>();
            r.out_stride = pl->kw;
            r.lay = rlay;
            r.nown = pl->nown;
            r.kw = pl->kw;
            r.ntiles = pl->pb.ntiles;
            r.nwin = pl->pb.nwin;
            r.items = pl->pb.items;
            launch_hash_mma_pb(r, pl->pb, st);
            launches += 4;
        }
        for (uint32_t jj0 = 0; jj0 < pl->nown; jj0 += g.batch) {  // leaf batches
            const uint32_t cnt = std::min<uint32_t>(g.batch, pl->nown - jj0);
            if (!g.gemm) {  // tiled leaves: materialised leaf inputs (+ per-block leaf seeds)
                launch_split_batch(pl->ybuf.as<uint32_t>(), pl->sbuf.as<uint32_t>(),
                                   pl->sbuf_words, lay, pl->nown, g, jj0, pl->vy.as<uint32_t>(),
                                   pl->vs.as<uint32_t>(), st);
                launches += g.per_block ? 2 : 1;
            }
            if (g.gemm) {
                // leaf mode: the GEMM builds each M tile's leaf inputs in shared memory from the
                // original reversed blocks (no k_split_inputs, no leaf-input buffer)
                MmaHashArgs v{};
                v.ybuf = pl->vy.as<uint32_t>();
                // one CTA per M tile (round 2 A/B: a CTA-pair variant, cta_group::2 with M = 256
                // and half the Hankel table per SM, measured 32.3 vs 29.3 ms at config 3)
                v.leaf = leaf_parent_mode(g) ? 2 : 1;
                v.src.ybuf = pl->ybuf.as<uint32_t>();
                v.src.lay = lay;
                v.src.k = g.k;
                v.src.L = g.L;
                v.src.leaves = g.leaves;
                v.src.gpad = g.gpad;
                v.src.batch = g.batch;
                v.src.jj0 = jj0;
                v.src.nown = pl->nown;
                v.src.seed_words = g.seed_words;
                v.units = pl->vu.as<uint32_t>();
                v.unit_stride = g.unit_stride;
                v.src.kpw = leaf_parent_mode(g) ? (uint32_t)(2 * g.sL / 32)
                                                : (uint32_t)(g.sL / 32 / pl->mmv.ksplit);
                v.sbuf = pl->vs.as<uint32_t>();
                v.out = pl->vout.as<uint32_t>();
                // parent mode writes level L - 1 nodes (2 leaves wide, a third as many rows)
                v.out_stride = (leaf_parent_mode(g) ? 2 : 1) * (g.sL / 32);
                v.lay = vlay;  // soff per 128-block M tile = the group's leaf seed
                v.nown = (uint32_t)g.nvirt;
                v.kw = (uint32_t)(g.sL / 32);
                v.ntiles = pl->mmv.ntiles;
                v.ksplit = pl->mmv.ksplit;
                v.items = pl->mmv.items;
                v.mt_words = pl->vmt.as<uint32_t>();
                if (pl->mmv.ksplit > 1) CU(cudaMemsetAsync(pl->vout.p, 0, pl->vout.bytes, st));
                launch_hash_mma(v, pl->mmv, st);
                launches += 1;  // + k_mma_tiles
            } else {
                PbHashArgs v{};
                v.ybuf = pl->vy.as<uint32_t>();
                v.sbuf = pl->vs.as<uint32_t>();
                v.out = pl->vout.as<uint32_t>();
                v.out_stride = g.sL / 32;
                v.lay = vlay;
                v.nown = (uint32_t)g.nvirt;
                v.kw = (uint32_t)(g.sL / 32);
                v.ntiles = pl->pbv.ntiles;
                v.nwin = pl->pbv.nwin;
                v.items = pl->pbv.items;
                launch_hash_mma_pb(v, pl->pbv, st);
            }
            // the parent-mode leaf GEMM has done the deepest level: combine from level L - 1
            SplitGeom gc = g;
            if (leaf_parent_mode(g)) {
                gc.L = g.L - 1;
                gc.leaves = g.leaves / 3;
                gc.sL = 2 * g.sL;
            }
            const uint64_t ostride = pl->direct_out ? pl->p.out_bits / 32 : pl->kw;
            if (pl->host_key && pl->copy_stream && pl->direct_out && out == d_key &&
                cnt == pl->nown && pl->p.out_bits % 64 == 0 &&
                cnt >= 4u * ssbh_plan::kKeySlices) {
                for (int sl = 0; sl < ssbh_plan::kKeySlices; ++sl) {
                    const uint32_t a = (uint32_t)((uint64_t)cnt * sl / ssbh_plan::kKeySlices);
                    const uint32_t b = (uint32_t)((uint64_t)cnt * (sl + 1) / ssbh_plan::kKeySlices);
                    launches += launch_split_combine(pl->vout.as<uint32_t>(),
                                                     pl->vy.as<uint32_t>(), pl->vrem.as<uint32_t>(),
                                                     rlay.ktl, jj0, cnt, pl->kw, gc, out, ostride,
                                                     st, a, b);
                    if (!pl->slice_ev[sl])
                        CU(cudaEventCreateWithFlags(&pl->slice_ev[sl], cudaEventDisableTiming));
                    CU(cudaEventRecord(pl->slice_ev[sl], st));
                    CU(cudaStreamWaitEvent(pl->copy_stream, pl->slice_ev[sl], 0));
                    CU(cudaMemcpyAsync(pl->host_key + (uint64_t)a * (pl->p.out_bits / 64),
                                       d_key + (uint64_t)a * ostride,
                                       (uint64_t)(b - a) * (pl->p.out_bits / 8),
                                       cudaMemcpyDeviceToHost, pl->copy_stream));
                }
                launches += 2;
                pl->host_key_sent = true;
            } else {
                launches += 2 + launch_split_combine(pl->vout.as<uint32_t>(),
                                                     pl->vy.as<uint32_t>(), pl->vrem.as<uint32_t>(),
                                                     rlay.ktl, jj0, cnt, pl->kw, gc, out, ostride,
                                                     st);
            }
        }
    } else if (pl->engine == kEngineMma && (pl->p.per_block_seed || pl->shared_pb)) {
        PbHashArgs m{};
        m.ybuf = pl->ybuf.as<uint32_t>();
        m.sbuf = pl->sbuf.as<uint32_t>();
        m.out = out;
        m.out_stride = pl->direct_out ? pl->p.out_bits / 32 : pl->kw;
        m.lay = lay;
        m.nown = pl->nown;
        m.kw = pl->kw;
        m.ntiles = pl->pb.ntiles;
        m.nwin = pl->pb.nwin;
        m.items = pl->pb.items;
        launch_hash_mma_pb(m, pl->pb, st);
        launches += 1;
    } else if (pl->engine == kEngineMma) {
        MmaHashArgs m{};
        m.ybuf = pl->ybuf.as<uint32_t>();
        m.sbuf = pl->sbuf.as<uint32_t>();
        m.out = out;
        m.out_stride = pl->direct_out ? pl->p.out_bits / 32 : pl->kw;
        m.lay = lay;
        m.nown = pl->nown;
        m.kw = pl->kw;
        m.ntiles = pl->mma.ntiles;
        m.ksplit = pl->mma.ksplit;
        m.items = pl->mma.items;
        m.mt_words = pl->mt_words.as<uint32_t>();
        launch_hash_mma(m, pl->mma, st);
        launches += 2;
    } else {
    HashArgs a{};
    a.ybuf = pl->ybuf.as<uint32_t>();
    a.sbuf = pl->sbuf.as<uint32_t>();
    a.out = out;
    a.out_stride = pl->direct_out ? pl->p.out_bits / 32 : pl->kw;
    a.lay = lay;
    a.nown = pl->nown;
    a.kw = pl->kw;
    a.rowtiles = pl->rowtiles;
    a.per_block_seed = pl->p.per_block_seed;
    launch_hash(a, pl->grid, st);
    launches += 1;
    }
    if (!pl->direct_out) {
        launch_concat(pl->scratch.as<uint32_t>(), pl->kw, pl->nown, pl->p.out_bits, d_key, st);
        launches += 1;
    }
    if (d_lengths)
        CU(cudaMemcpyAsync(d_lengths, lay.nj, (size_t)pl->nown * 8, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(pl->h_stats, lay.stats, sizeof(DevStats), cudaMemcpyDeviceToHost, st));
    return SSBH_OK;
}

// Phase A (direct launches): S0 with its events. Streaming plans call it without input.
static ssbh_status phase_sample(ssbh_plan* pl, const uint32_t* d_input, const uint32_t* d_keep,
                                const uint64_t* sk, cudaStream_t st, uint32_t& launches) {
    rec(pl, 0, st);
    if (auto s = seg_sample(pl, d_input, d_keep, sk, st, launches)) return s;
    rec(pl, 1, st);
    return SSBH_OK;
}

// Phase C (direct launches): S2 + S3 with their events.
static ssbh_status phase_finish(ssbh_plan* pl, uint32_t* d_key, uint64_t* d_lengths,
                                const uint64_t* hk, cudaStream_t st, uint32_t& launches) {
    if (pl->fwd_stream) {
        // block lengths = the running ranks; layout; the forward regions reversed into the
        // compact padded blocks the hash kernels read
        const Layout lay = pl->lay.view();
        launch_ranks_to_nj(pl->run_rank.as<uint32_t>(), pl->nown, lay.nj, st);
        launch_layout(lay, pl->nown, pl->p.out_bits, pl->rowtiles, pl->kt, pl->p.per_block_seed,
                      pl->p.block_limit, st);
        CU(cudaMemsetAsync(pl->ybuf.p, 0, pl->ybuf.bytes, st));
        launch_reverse_blocks(pl->yfwd.as<uint32_t>(), pl->fwd_cap / 32, lay, pl->nown,
                              pl->p.n_rounds / pl->p.n_subblocks / 32 + 1,
                              pl->ybuf.as<uint32_t>(), st);
        launches += 3;
    }
    rec(pl, 2, st);
    if (auto s = seg_seeds(pl, hk, st, launches)) return s;
    rec(pl, 3, st);
    if (auto s = seg_hash(pl, d_key, d_lengths, st, launches)) return s;
    rec(pl, 4, st);
    rec(pl, 5, st);
    return SSBH_OK;
}

struct RunArgs {
    const uint32_t* d_input;
    const uint32_t* d_keep;
    uint32_t* d_key;
    uint64_t* d_lengths;
    const uint64_t* sk;
    const uint64_t* hk;
};

// Segments [s0, s1) of an in-memory run, without events.
static ssbh_status enqueue_segments(ssbh_plan* pl, const RunArgs& r, int s0, int s1,
                                    cudaStream_t st, uint32_t& launches) {
    for (int sgi = s0; sgi < s1; ++sgi) {
        ssbh_status s = SSBH_OK;
        switch (sgi) {
            case 0: s = seg_sample(pl, r.d_input, r.d_keep, r.sk, st, launches); break;
            case 1: s = seg_scatter(pl, st, launches); break;
            case 2: s = seg_seeds(pl, r.hk, st, launches); break;
            default: s = seg_hash(pl, r.d_key, r.d_lengths, st, launches); break;
        }
        if (s) return s;
    }
    return SSBH_OK;
}

// One in-memory fused run launched directly on `st`, events between segments.
static ssbh_status plan_enqueue(ssbh_plan* pl, const RunArgs& r, cudaStream_t st) {
    uint32_t launches = 0;
    for (int sgi = 0; sgi < 4; ++sgi) {
        rec(pl, sgi, st);
        if (auto s = enqueue_segments(pl, r, sgi, sgi + 1, st, launches)) return s;
    }
    rec(pl, 4, st);
    rec(pl, 5, st);
    pl->launches_per_run = launches;
    return check_launch("plan_run");
}

static bool graphs_enabled() { return true; }

static ssbh_status capture(ssbh_plan* pl, const RunArgs& r, int s0, int s1, cudaStream_t st,
                           cudaGraphExec_t* exec, uint32_t& launches) {
    CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const ssbh_status s = enqueue_segments(pl, r, s0, s1, st, launches);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(st, &g);
    if (s != SSBH_OK) {
        if (g) cudaGraphDestroy(g);
        return s;
    }
    if (e != cudaSuccess) return fail(SSBH_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
    const cudaError_t ie = cudaGraphInstantiate(exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
        *exec = nullptr;
        return fail(SSBH_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ie));
    }
    return SSBH_OK;
}

extern "C" ssbh_status ssbh_plan_run_device(ssbh_plan* pl, const uint32_t* d_input,
                                            uint32_t* d_key, uint64_t* d_lengths,
                                            const uint64_t* samp_key, const uint64_t* hash_key,
                                            void* stream) {
    return ssbh_plan_run_device_sifted(pl, d_input, nullptr, d_key, d_lengths, samp_key, hash_key,
                                       stream);
}

extern "C" ssbh_status ssbh_plan_run_device_sifted(ssbh_plan* pl, const uint32_t* d_input,
                                                   const uint32_t* d_keep, uint32_t* d_key,
                                                   uint64_t* d_lengths, const uint64_t* samp_key,
                                                   const uint64_t* hash_key, void* stream) {
    if (!pl || !d_input || !d_key) return fail(SSBH_INVALID_ARGUMENT, "plan_run: null argument");
    if (pl->streaming)
        return fail(SSBH_INVALID_ARGUMENT, "plan_run: streaming plans take stream_begin/chunk/finish");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl->last_stream = st;
    const RunArgs r{d_input, d_keep, d_key, d_lengths, samp_key ? samp_key : pl->p.samp_key,
                    hash_key ? hash_key : pl->p.hash_key};
    // the legacy default stream cannot be captured: launch directly there
    if (st == nullptr || !graphs_enabled()) return plan_enqueue(pl, r, st);
    ssbh_plan::GraphKey key{};
    key.st = st;
    key.in = d_input;
    key.key = d_key;
    key.len = d_lengths;
    key.keep = d_keep;
    std::memcpy(key.sk, r.sk, 32);
    std::memcpy(key.hk, r.hk, 32);
    key.timing = pl->timing;
    // untimed: one graph for the whole run; timed: one graph per segment, events between
    const int nseg = pl->timing ? 4 : 1;
    if (!(pl->exec[0] && key == pl->gkey)) {
        for (auto& x : pl->exec)
            if (x) {
                cudaGraphExecDestroy(x);
                x = nullptr;
            }
        uint32_t launches = 0;
        for (int sgi = 0; sgi < nseg; ++sgi) {
            const int s0 = nseg == 1 ? 0 : sgi, s1 = nseg == 1 ? 4 : sgi + 1;
            if (auto s = capture(pl, r, s0, s1, st, &pl->exec[sgi], launches)) return s;
        }
        pl->launches_per_run = launches;
        pl->gkey = key;
    }
    for (int sgi = 0; sgi < nseg; ++sgi) {
        if (nseg > 1) rec(pl, sgi, st);
        CU(cudaGraphLaunch(pl->exec[sgi], st));
    }
    if (nseg > 1) {
        rec(pl, 4, st);
        rec(pl, 5, st);
    }
    return ok();
}

extern "C" ssbh_status ssbh_plan_check(ssbh_plan* pl, ssbh_extract_stats* stats) {
    if (!pl) return fail(SSBH_INVALID_ARGUMENT, "null plan");
    CU(cudaStreamSynchronize(pl->last_stream));
    const DevStats& d = *pl->h_stats;
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->hash_word_ops = d.hash_word_ops;
        stats->max_len = d.max_nj;
        stats->min_len = d.min_nj;
        stats->hash_launches = 1;
        stats->launches = pl->launches_per_run;
        if (pl->timing) {
            float ms[5] = {0, 0, 0, 0, 0};
            for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&ms[i], pl->ev[i], pl->ev[i + 1]);
            cudaEventElapsedTime(&ms[4], pl->ev[0], pl->ev[5]);
            stats->ms_sample = ms[0];
            stats->ms_scatter = ms[1];
            stats->ms_seed = ms[2];
            stats->ms_hash = ms[3];
            stats->ms_total = ms[4];
        }
    }
    if (d.pad & kFlagBucketOverflow)
        return fail(SSBH_CUDA, "extract: a two-level staging region overflowed (> mean + 16 "
                               "sigma rounds in one bucket)");
    if (d.flags & kFlagTooLong)
        return fail(SSBH_INVALID_ARGUMENT,
                    "extract: sub-block of >= 2^32 bits is beyond the device path");
    if (d.flags & kFlagOversize)
        return fail(SSBH_ABORT_OVERSIZE, "abort: oversize_block (some n_j > block_limit %llu)",
                    (unsigned long long)pl->p.block_limit);
    if (d.flags & kFlagEmpty)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    return ok();
}

extern "C" ssbh_status ssbh_plan_run_host(ssbh_plan* pl, const uint64_t* input, uint64_t* out_key,
                                          uint64_t* out_lengths, ssbh_extract_stats* stats) {
    return ssbh_plan_run_host_sifted(pl, input, nullptr, out_key, out_lengths, stats);
}

extern "C" ssbh_status ssbh_plan_run_host_sifted(ssbh_plan* pl, const uint64_t* input,
                                                 const uint64_t* keep, uint64_t* out_key,
                                                 uint64_t* out_lengths,
                                                 ssbh_extract_stats* stats) {
    if (!pl || !input || !out_key) return fail(SSBH_INVALID_ARGUMENT, "plan_run_host: null argument");
    if (pl->streaming)
        return fail(SSBH_INVALID_ARGUMENT, "plan_run_host: streaming plans take stream_begin/chunk/finish");
    CU(cudaSetDevice(pl->device));
    if (!pl->own_stream) CU(cudaStreamCreateWithFlags(&pl->own_stream, cudaStreamNonBlocking));
    const uint64_t in_w64 = words64(pl->p.n_rounds);
    const uint64_t key_w64 = words64((uint64_t)pl->nown * pl->p.out_bits);
    if (!pl->d_input.p) {
        CU(pl->d_input.alloc(in_w64 * 8 + 16));
        CU(pl->d_key.alloc(key_w64 * 8 + 16));
        CU(pl->d_len.alloc((size_t)pl->nown * 8 + 8));
    }
    if (keep && !pl->d_keep.p) CU(pl->d_keep.alloc(in_w64 * 8 + 16));
    cudaStream_t st = pl->own_stream;
    // large inputs without a keep mask: copy the input on a second stream while the count pass
    // runs (it needs only the round indices); the split / scatter wait for the copy
    const bool late = !keep && pl->p.n_rounds >= (1ull << 24);
    if (late) {
        if (!pl->copy_stream) {
            CU(cudaStreamCreateWithFlags(&pl->copy_stream, cudaStreamNonBlocking));
            CU(cudaEventCreateWithFlags(&pl->late_ev, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&pl->prev_ev, cudaEventDisableTiming));
        }
        CU(cudaEventRecord(pl->prev_ev, st));  // the previous run is done with d_input
        CU(cudaStreamWaitEvent(pl->copy_stream, pl->prev_ev, 0));
        CU(cudaMemcpyAsync(pl->d_input.p, input, in_w64 * 8, cudaMemcpyHostToDevice,
                           pl->copy_stream));
        CU(cudaEventRecord(pl->late_ev, pl->copy_stream));
    } else {
        CU(cudaMemcpyAsync(pl->d_input.p, input, in_w64 * 8, cudaMemcpyHostToDevice, st));
        if (keep) CU(cudaMemcpyAsync(pl->d_keep.p, keep, in_w64 * 8, cudaMemcpyHostToDevice, st));
    }
    // the key buffer's last u32 of an odd word count must read as zero in the u64 view
    if ((pl->key_words32 & 1) != 0) CU(cudaMemsetAsync(pl->d_key.p, 0, key_w64 * 8, st));
    if (late) {  // direct launches: the cross-stream wait is not part of a captured graph
        pl->late_input = pl->d_input.as<uint32_t>();
        pl->host_key = out_key;
        pl->host_key_sent = false;
        pl->last_stream = st;
        const RunArgs r{pl->d_input.as<uint32_t>(), nullptr, pl->d_key.as<uint32_t>(),
                        pl->d_len.as<uint64_t>(), pl->p.samp_key, pl->p.hash_key};
        const ssbh_status s = plan_enqueue(pl, r, st);
        pl->late_input = nullptr;
        pl->host_key = nullptr;
        if (s) {
            if (pl->host_key_sent) cudaStreamSynchronize(pl->copy_stream);
            pl->host_key_sent = false;
            return s;
        }
    } else if (auto s = ssbh_plan_run_device_sifted(pl, pl->d_input.as<uint32_t>(),
                                                    keep ? pl->d_keep.as<uint32_t>() : nullptr,
                                                    pl->d_key.as<uint32_t>(),
                                                    pl->d_len.as<uint64_t>(), nullptr, nullptr,
                                                    st))
        return s;
    const bool key_sent = pl->host_key_sent;  // the key left in slices behind the combine
    pl->host_key_sent = false;
    // the read-backs are queued behind the run, so the one synchronisation of plan_check also
    // covers them (a failed run leaves unspecified bytes in the caller's buffers)
    if (!key_sent)
        CU(cudaMemcpyAsync(out_key, pl->d_key.p, key_w64 * 8, cudaMemcpyDeviceToHost, st));
    if (out_lengths)
        CU(cudaMemcpyAsync(out_lengths, pl->d_len.p, (size_t)pl->nown * 8, cudaMemcpyDeviceToHost,
                           st));
    const ssbh_status s = ssbh_plan_check(pl, stats);  // synchronises st
    if (key_sent) {
        const std::string msg = g_err;
        cudaStreamSynchronize(pl->copy_stream);
        g_err = msg;
    }
    return s;
}

extern "C" ssbh_status ssbh_extract(const ssbh_extract_params* params, const uint64_t* input,
                                    uint64_t* out_key, uint64_t* out_lengths,
                                    ssbh_extract_stats* stats) {
    return ssbh_extract_sifted(params, input, nullptr, out_key, out_lengths, stats);
}

extern "C" ssbh_status ssbh_extract_sifted(const ssbh_extract_params* params,
                                           const uint64_t* input, const uint64_t* keep,
                                           uint64_t* out_key, uint64_t* out_lengths,
                                           ssbh_extract_stats* stats) {
    ssbh_plan* pl = nullptr;
    if (auto s = ssbh_plan_create(params, &pl)) return s;
    const ssbh_status s = ssbh_plan_run_host_sifted(pl, input, keep, out_key, out_lengths, stats);
    std::string msg = g_err;
    ssbh_plan_destroy(pl);
    g_err = msg;
    return s;
}

// ======================================================================== sampler API
extern "C" ssbh_status ssbh_assign_subblocks(uint64_t n, uint32_t s, const uint64_t key[4],
                                             uint32_t* assignment, uint64_t* raw_counts) {
    if (s == 0)
        return fail(SSBH_INVALID_ARGUMENT, "assign_subblocks: n_subblocks must be positive");
    if (n == 0) {
        std::memset(raw_counts, 0, (size_t)s * 8);
        return ok();
    }
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    const SamplerGeom g = make_sampler_geom(n, s, 0, s, false);
    SBuf assign, counts, gsum, nj;
    CU(assign.alloc((size_t)n * 4));
    CU(counts.alloc((size_t)g.nchunks * s * 4));
    CU(gsum.alloc((size_t)g.ngroups * s * 8));
    CU(nj.alloc((size_t)s * 8));
    CU(cudaMemsetAsync(counts.p, 0, counts.bytes, st));
    launch_sample_count(g, key, nullptr, nullptr, nullptr, counts.as<uint32_t>(),
                        assign.as<uint32_t>(), st);
    launch_scan(g, counts.as<uint32_t>(), gsum.as<unsigned long long>(),
                nj.as<unsigned long long>(), st);
    if (auto e_ = check_launch("assign_subblocks")) return e_;
    CU(cudaMemcpyAsync(assignment, assign.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(raw_counts, nj.p, (size_t)s * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

namespace ssbh_impl {
void launch_payload_from_assignment(const SamplerGeom& g, const uint32_t* d_assign,
                                    const uint8_t* d_keep, uint32_t* d_payload,
                                    uint32_t* d_counts, uint32_t* d_bad, cudaStream_t st);
void launch_csr_offsets(const unsigned long long* d_nj, uint32_t nown,
                        unsigned long long* d_off, cudaStream_t st);
}  // namespace ssbh_impl

extern "C" ssbh_status ssbh_sift_partition(const uint8_t* keep, uint64_t n,
                                           const uint32_t* assignment, uint32_t s,
                                           uint64_t* offsets, uint64_t* indices,
                                           uint64_t* max_len) {
    if (s == 0)
        return fail(SSBH_INVALID_ARGUMENT, "sift_partition: n_subblocks must be positive");
    if (n == 0) {
        std::memset(offsets, 0, ((size_t)s + 1) * 8);
        if (max_len) *max_len = 0;
        return ok();
    }
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    const SamplerGeom g = make_sampler_geom(n, s, 0, s, true);
    SBuf dassign, dkeep, payload, counts, gsum, nj, off, idx, bad;
    CU(dassign.alloc((size_t)n * 4));
    CU(cudaMemcpyAsync(dassign.p, assignment, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    if (keep) {
        CU(dkeep.alloc((size_t)n));
        CU(cudaMemcpyAsync(dkeep.p, keep, (size_t)n, cudaMemcpyHostToDevice, st));
    }
    CU(payload.alloc((size_t)n * 4));
    CU(counts.alloc((size_t)g.nchunks * s * 4));
    CU(gsum.alloc((size_t)g.ngroups * s * 8));
    CU(nj.alloc((size_t)s * 8));
    CU(off.alloc(((size_t)s + 1) * 8));
    CU(idx.alloc((size_t)n * 8));
    CU(bad.alloc(4));
    CU(cudaMemsetAsync(counts.p, 0, counts.bytes, st));
    CU(cudaMemsetAsync(bad.p, 0, 4, st));
    launch_payload_from_assignment(g, dassign.as<uint32_t>(), keep ? dkeep.as<uint8_t>() : nullptr,
                                   payload.as<uint32_t>(), counts.as<uint32_t>(),
                                   bad.as<uint32_t>(), st);
    uint32_t hbad = 0;
    CU(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (hbad)
        return fail(SSBH_INVALID_ARGUMENT,
                    "sift_partition: assignment value outside [1, n_subblocks]");
    launch_scan(g, counts.as<uint32_t>(), gsum.as<unsigned long long>(),
                nj.as<unsigned long long>(), st);
    launch_csr_offsets(nj.as<unsigned long long>(), s, off.as<unsigned long long>(), st);
    launch_scatter(g, payload.p, counts.as<uint32_t>(), nj.as<unsigned long long>(), nullptr,
                   nullptr, idx.as<unsigned long long>(), off.as<unsigned long long>(), st);
    if (auto e_ = check_launch("sift_partition")) return e_;
    CU(cudaMemcpyAsync(offsets, off.p, ((size_t)s + 1) * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const uint64_t kept = offsets[s];
    if (kept) CU(cudaMemcpyAsync(indices, idx.p, kept * 8, cudaMemcpyDeviceToHost, st));
    if (max_len) {
        uint64_t m = 0;
        for (uint32_t j = 0; j < s; ++j) m = std::max<uint64_t>(m, offsets[j + 1] - offsets[j]);
        *max_len = m;
    }
    CU(cudaStreamSynchronize(st));
    return ok();
}

// ======================================================================== toeplitz API
namespace ssbh_impl {
void launch_pack_blocks(const uint64_t* d_seeds, const unsigned long long* d_seed_off,
                        const uint64_t* d_inputs, const unsigned long long* d_in_off,
                        const Layout& lay, uint32_t count, uint64_t m, uint32_t* d_sbuf,
                        uint32_t* d_ybuf, cudaStream_t st, uint64_t max_words);
}

// One batched hash through the calling thread's CallScope: block b's input words come from
// in_ptr[b] (or inputs + in_off[b]), its seed words from seed_ptr[b] (or seeds + seed_off[b]).
static ssbh_status hash_batch_impl(uint64_t count, uint64_t m, const uint64_t* n,
                                   const uint64_t* inputs, const uint64_t* in_off,
                                   const uint64_t* const* in_ptr, const uint64_t* seeds,
                                   const uint64_t* seed_off, const uint64_t* const* seed_ptr,
                                   uint64_t* out) {
    if (m == 0) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    for (uint64_t b = 0; b < count; ++b)
        if (n[b] == 0) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    if (count == 0) return ok();
    if (count > (1u << 30)) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: batch too large");
    NEED_DEVICE();
    CALL_SCOPE(scope);
    const cudaStream_t st = scope.stream();
    int dev = 0;
    CU(cudaGetDevice(&dev));
    const uint32_t nown = (uint32_t)count;
    const uint32_t kw = (uint32_t)((m + 31) / 32);
    const uint32_t rowtiles = (kw + kHashRowWords - 1) / kHashRowWords;
    // device-side offsets: the contiguous form keeps the caller's, the pointer form packs
    std::vector<uint64_t> meta(3 * count);  // n | in_off | seed_off
    uint64_t in_words = 0, seed_words = 0, sum_n = 0, ybound = 8, sbound = 8, maxw = 0;
    for (uint64_t b = 0; b < count; ++b) {
        const uint64_t iw = words64(n[b]), sw = words64(m + n[b] - 1);
        meta[b] = n[b];
        meta[count + b] = in_ptr ? in_words : in_off[b];
        meta[2 * count + b] = seed_ptr ? seed_words : seed_off[b];
        in_words = in_ptr ? in_words + iw : std::max<uint64_t>(in_words, in_off[b] + iw);
        seed_words = seed_ptr ? seed_words + sw : std::max<uint64_t>(seed_words, seed_off[b] + sw);
        sum_n += n[b];
        const uint64_t yp = round_up((n[b] + 31) / 32, kHashR);
        ybound += yp;
        sbound += round_up((uint64_t)rowtiles * kHashRowWords + 8 + yp, 8);
        maxw = std::max<uint64_t>(maxw, 2 * sw);
    }
    LayoutScratch lb;
    SBuf din, dseeds, dmeta, ybuf, sbuf, scratch, key;
    CU(lb.alloc(nown));
    CU(din.alloc(in_words * 8));
    CU(dseeds.alloc(seed_words * 8));
    CU(dmeta.alloc(count * 24));
    CU(ybuf.alloc(ybound * 4));
    CU(sbuf.alloc((sbound + 64) * 4));  // + the tensor kernels' read-ahead of unused units
    CU(scratch.alloc((size_t)nown * kw * 4));
    const uint64_t key_w64 = words64(count * m);
    CU(key.alloc(key_w64 * 8));
    if (in_ptr) {
        for (uint64_t b = 0; b < count; ++b)
            CU(cudaMemcpyAsync(din.as<uint64_t>() + meta[count + b], in_ptr[b],
                               words64(n[b]) * 8, cudaMemcpyHostToDevice, st));
    } else {
        CU(cudaMemcpyAsync(din.p, inputs, in_words * 8, cudaMemcpyHostToDevice, st));
    }
    if (seed_ptr) {
        for (uint64_t b = 0; b < count; ++b)
            CU(cudaMemcpyAsync(dseeds.as<uint64_t>() + meta[2 * count + b], seed_ptr[b],
                               words64(m + n[b] - 1) * 8, cudaMemcpyHostToDevice, st));
    } else {
        CU(cudaMemcpyAsync(dseeds.p, seeds, seed_words * 8, cudaMemcpyHostToDevice, st));
    }
    CU(cudaMemcpyAsync(dmeta.p, meta.data(), count * 24, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(lb.nj.p, meta.data(), count * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(ybuf.p, 0, ybuf.bytes, st));
    CU(cudaMemsetAsync(sbuf.p, 0, sbuf.bytes, st));
    CU(cudaMemsetAsync(key.p, 0, key.bytes, st));
    const Layout lay = lb.view();
    const int grid = hash_grid_size(dev);
    const uint32_t kt = choose_kt(sum_n / count, nown, rowtiles, grid);
    launch_layout(lay, nown, m, rowtiles, kt, 1, 0, st);
    launch_pack_blocks(dseeds.as<uint64_t>(), dmeta.as<unsigned long long>() + 2 * count,
                       din.as<uint64_t>(), dmeta.as<unsigned long long>() + count, lay, nown, m,
                       sbuf.as<uint32_t>(), ybuf.as<uint32_t>(), st, maxw);
    if (default_engine(1) == kEngineMma) {  // every block its own matrix: tiled matvec MMAs
        const PbGeom pg = make_pb_geom(nown, kw, dev, sum_n / count);
        PbHashArgs a{};
        a.ybuf = ybuf.as<uint32_t>();
        a.sbuf = sbuf.as<uint32_t>();
        a.out = scratch.as<uint32_t>();
        a.out_stride = kw;
        a.lay = lay;
        a.nown = nown;
        a.kw = kw;
        a.ntiles = pg.ntiles;
        a.nwin = pg.nwin;
        launch_hash_mma_pb(a, pg, st);
    } else {
        CU(cudaMemsetAsync(scratch.p, 0, scratch.bytes, st));
        HashArgs a{};
        a.ybuf = ybuf.as<uint32_t>();
        a.sbuf = sbuf.as<uint32_t>();
        a.out = scratch.as<uint32_t>();
        a.out_stride = kw;
        a.lay = lay;
        a.nown = nown;
        a.kw = kw;
        a.rowtiles = rowtiles;
        a.per_block_seed = 1;
        launch_hash(a, grid, st);
    }
    launch_concat(scratch.as<uint32_t>(), kw, nown, m, key.as<uint32_t>(), st);
    if (auto e = check_launch("toeplitz_hash")) return e;
    CU(cudaMemcpyAsync(out, key.p, key_w64 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_toeplitz_hash_batch(uint64_t count, uint64_t m, const uint64_t* n,
                                                const uint64_t* inputs, const uint64_t* in_off,
                                                const uint64_t* seeds, const uint64_t* seed_off,
                                                uint64_t* out) {
    return hash_batch_impl(count, m, n, inputs, in_off, nullptr, seeds, seed_off, nullptr, out);
}

extern "C" ssbh_status ssbh_toeplitz_hash_batch_ptrs(uint64_t count, uint64_t m,
                                                     const uint64_t* n,
                                                     const uint64_t* const* inputs,
                                                     const uint64_t* const* seeds,
                                                     uint64_t* out) {
    return hash_batch_impl(count, m, n, nullptr, nullptr, inputs, nullptr, nullptr, seeds, out);
}

// Prepared batch (device-resident inputs and seeds; see include/ssbh_cuda.h).
struct ssbh_hash_batch {
    uint32_t nown = 0, kw = 0, rowtiles = 0, kt = 0;
    uint64_t m = 0, mean_n = 0, key_w64 = 0;
    int device = 0, grid = 0;
    LayoutBufs lb;
    DBuf ybuf, sbuf, scratch, key;
    cudaStream_t st = nullptr;
};

extern "C" ssbh_status ssbh_hash_batch_create(uint64_t count, uint64_t m, const uint64_t* n,
                                              const uint64_t* const* inputs,
                                              const uint64_t* const* seeds,
                                              ssbh_hash_batch** out) {
    if (!out || !n || !inputs || !seeds)
        return fail(SSBH_INVALID_ARGUMENT, "hash_batch_create: null argument");
    if (m == 0 || count == 0)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    for (uint64_t b = 0; b < count; ++b)
        if (n[b] == 0) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    if (count > (1u << 30)) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: batch too large");
    NEED_DEVICE();
    std::unique_ptr<ssbh_hash_batch> hb(new ssbh_hash_batch());
    CU(cudaGetDevice(&hb->device));
    hb->nown = (uint32_t)count;
    hb->m = m;
    hb->kw = (uint32_t)((m + 31) / 32);
    hb->rowtiles = (hb->kw + kHashRowWords - 1) / kHashRowWords;
    std::vector<uint64_t> meta(3 * count);  // n | in_off | seed_off (u64 words)
    uint64_t in_words = 0, seed_words = 0, sum_n = 0, ybound = 8, sbound = 8, maxw = 0;
    for (uint64_t b = 0; b < count; ++b) {
        const uint64_t iw = words64(n[b]), sw = words64(m + n[b] - 1);
        meta[b] = n[b];
        meta[count + b] = in_words;
        meta[2 * count + b] = seed_words;
        in_words += iw;
        seed_words += sw;
        sum_n += n[b];
        const uint64_t yp = round_up((n[b] + 31) / 32, kHashR);
        ybound += yp;
        sbound += round_up((uint64_t)hb->rowtiles * kHashRowWords + 8 + yp, 8);
        maxw = std::max<uint64_t>(maxw, 2 * sw);
    }
    hb->mean_n = sum_n / count;
    hb->key_w64 = words64(count * m);
    DBuf din, dseeds, dmeta;  // only needed until the blocks are packed
    CU(hb->lb.alloc(hb->nown));
    CU(din.alloc(in_words * 8));
    CU(dseeds.alloc(seed_words * 8));
    CU(dmeta.alloc(count * 24));
    CU(hb->ybuf.alloc(ybound * 4));
    CU(hb->sbuf.alloc((sbound + 64) * 4));
    CU(hb->scratch.alloc((size_t)hb->nown * hb->kw * 4));
    CU(hb->key.alloc(hb->key_w64 * 8));
    CU(cudaStreamCreateWithFlags(&hb->st, cudaStreamNonBlocking));
    const cudaStream_t st = hb->st;
    for (uint64_t b = 0; b < count; ++b) {
        CU(cudaMemcpyAsync(din.as<uint64_t>() + meta[count + b], inputs[b], words64(n[b]) * 8,
                           cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(dseeds.as<uint64_t>() + meta[2 * count + b], seeds[b],
                           words64(m + n[b] - 1) * 8, cudaMemcpyHostToDevice, st));
    }
    CU(cudaMemcpyAsync(dmeta.p, meta.data(), count * 24, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(hb->lb.nj.p, meta.data(), count * 8, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(hb->ybuf.p, 0, hb->ybuf.bytes, st));
    CU(cudaMemsetAsync(hb->sbuf.p, 0, hb->sbuf.bytes, st));
    const Layout lay = hb->lb.view();
    hb->grid = hash_grid_size(hb->device);
    hb->kt = choose_kt(hb->mean_n, hb->nown, hb->rowtiles, hb->grid);
    launch_layout(lay, hb->nown, m, hb->rowtiles, hb->kt, 1, 0, st);
    launch_pack_blocks(dseeds.as<uint64_t>(), dmeta.as<unsigned long long>() + 2 * count,
                       din.as<uint64_t>(), dmeta.as<unsigned long long>() + count, lay, hb->nown,
                       m, hb->sbuf.as<uint32_t>(), hb->ybuf.as<uint32_t>(), st, maxw);
    if (auto e = check_launch("hash_batch_create")) return e;
    CU(cudaStreamSynchronize(st));
    *out = hb.release();
    return ok();
}

extern "C" ssbh_status ssbh_hash_batch_run(ssbh_hash_batch* hb, uint64_t* out) {
    if (!hb || !out) return fail(SSBH_INVALID_ARGUMENT, "hash_batch_run: null argument");
    CU(cudaSetDevice(hb->device));
    const cudaStream_t st = hb->st;
    const Layout lay = hb->lb.view();
    CU(cudaMemsetAsync(hb->key.p, 0, hb->key.bytes, st));
    if (default_engine(1) == kEngineMma) {  // every block its own matrix: tiled matvec MMAs
        const PbGeom pg = make_pb_geom(hb->nown, hb->kw, hb->device, hb->mean_n);
        PbHashArgs a{};
        a.ybuf = hb->ybuf.as<uint32_t>();
        a.sbuf = hb->sbuf.as<uint32_t>();
        a.out = hb->scratch.as<uint32_t>();
        a.out_stride = hb->kw;
        a.lay = lay;
        a.nown = hb->nown;
        a.kw = hb->kw;
        a.ntiles = pg.ntiles;
        a.nwin = pg.nwin;
        launch_hash_mma_pb(a, pg, st);
    } else {
        CU(cudaMemsetAsync(hb->scratch.p, 0, hb->scratch.bytes, st));
        HashArgs a{};
        a.ybuf = hb->ybuf.as<uint32_t>();
        a.sbuf = hb->sbuf.as<uint32_t>();
        a.out = hb->scratch.as<uint32_t>();
        a.out_stride = hb->kw;
        a.lay = lay;
        a.nown = hb->nown;
        a.kw = hb->kw;
        a.rowtiles = hb->rowtiles;
        a.per_block_seed = 1;
        launch_hash(a, hb->grid, st);
    }
    launch_concat(hb->scratch.as<uint32_t>(), hb->kw, hb->nown, hb->m, hb->key.as<uint32_t>(), st);
    if (auto e = check_launch("hash_batch_run")) return e;
    CU(cudaMemcpyAsync(out, hb->key.p, hb->key_w64 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return ok();
}

extern "C" ssbh_status ssbh_hash_batch_destroy(ssbh_hash_batch* hb) {
    if (!hb) return ok();
    if (hb->st) cudaStreamDestroy(hb->st);
    delete hb;
    return ok();
}

extern "C" ssbh_status ssbh_release_thread_cache(void) {
    for (auto& a : g_call.per_dev)
        if (a && !a->depth) a.reset();
    return ok();
}

extern "C" ssbh_status ssbh_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                                          const uint64_t* input, uint64_t input_bits,
                                          uint64_t* out) {
    // ToeplitzSeed ctor (toeplitz.cpp:9-15) then check_input (toeplitz.cpp:19-22)
    if (m == 0 || n == 0) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    if (input_bits != n)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: input length does not match seed.n");
    const uint64_t zero = 0;
    return ssbh_toeplitz_hash_batch(1, m, &n, input, &zero, seed, &zero, out);
}

extern "C" ssbh_status ssbh_blocked_toeplitz_hash(const uint64_t* seed, uint64_t m, uint64_t n,
                                                  const uint64_t* input, uint64_t input_bits,
                                                  uint64_t m_prime, uint64_t n_prime,
                                                  uint64_t* out) {
    if (m == 0 || n == 0) return fail(SSBH_INVALID_ARGUMENT, "toeplitz: m and n must be positive");
    if (input_bits != n)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: input length does not match seed.n");
    if (m_prime == 0 || n_prime == 0)
        return fail(SSBH_INVALID_ARGUMENT, "toeplitz: blocking dimensions must be positive");
    // toeplitz.hpp:29-32: bit-for-bit identical to toeplitz_hash for every blocking; the
    // GPU tiling is our own (row tiles x k tiles), so the blocking is validated only.
    return ssbh_toeplitz_hash(seed, m, n, input, input_bits, out);
}

// ======================================================================== multi-GPU shards
// One process per GPU. Rank r samples only its slice of rounds, stores every round's payload
// straight into the owning rank's receive buffer through NVLink peer memory (CUDA IPC
// mappings; the dispatch of an all-to-all fused into the stable owner split), and then each
// owner partitions / hashes only its received rounds. Host barriers separate the phases;
// no kernel ever waits on another rank.
struct ssbh_shard {
    ssbh_extract_params p{};  // block_first/count = this rank's owned blocks
    uint32_t rank = 0, world = 1;
    int device = 0;
    uint64_t slice_lo = 0, slice_n = 0;
    SamplerGeom gs{};  // slice geometry, keys = owning ranks
    DBuf slice_payload, slice_counts, slice_gsum, slice_tot;
    uint64_t recv_cap = 0, n_recv = 0;
    DBuf recv, d_dst, d_dst_base;
    std::vector<void*> peer;   // receive buffers of all ranks (own = recv.p)
    std::vector<bool> opened;  // IPC-opened (to close)
    ssbh_plan* plan = nullptr;  // owner pipeline over the received payload
    uint64_t* h_tot = nullptr;  // pinned, world entries
    uint32_t launches = 0;
};

static uint64_t slice_bound(uint64_t n, uint32_t world, uint32_t r) {
    if (r >= world) return n;
    return (n * r / world) / 1024 * 1024;
}

extern "C" ssbh_status ssbh_shard_create(const ssbh_extract_params* params, uint32_t rank,
                                         uint32_t world, ssbh_shard** out) {
    if (!params || !out) return fail(SSBH_INVALID_ARGUMENT, "shard_create: null argument");
    if (world == 0 || rank >= world || world > params->n_subblocks)
        return fail(SSBH_INVALID_ARGUMENT, "shard_create: need 0 <= rank < world <= n_subblocks");
    NEED_DEVICE();
    auto* sh = new ssbh_shard();
    sh->p = *params;
    sh->rank = rank;
    sh->world = world;
    CU(cudaGetDevice(&sh->device));
    const uint64_t n = params->n_rounds, s = params->n_subblocks;
    sh->p.block_first = (uint32_t)(s * rank / world);
    sh->p.block_count = (uint32_t)(s * (rank + 1) / world) - sh->p.block_first;
    sh->slice_lo = slice_bound(n, world, rank);
    sh->slice_n = slice_bound(n, world, rank + 1) - sh->slice_lo;
    sh->gs = make_sampler_geom(sh->slice_n ? sh->slice_n : 1, s, 0, world, false);
    sh->gs.n = sh->slice_n;
    // shards take no keep mask, so no u16 sift marker: V up to 0x7fff fits (s <= 2^15)
    sh->gs.payload_bytes = s <= 32768 ? 2 : 4;
    // receive capacity: the largest owner's expected share + 16 sigma + slack
    uint64_t maxc = 0;
    for (uint32_t o = 0; o < world; ++o)
        maxc = std::max<uint64_t>(maxc, s * (o + 1) / world - s * o / world);
    const double mean = (double)n * (double)maxc / (double)s;
    sh->recv_cap = (uint64_t)(mean + 16.0 * std::sqrt(mean) + 65536.0);
    sh->recv_cap = std::min<uint64_t>(sh->recv_cap, n);
    const int pb = sh->gs.payload_bytes;
    cudaError_t e = cudaSuccess;
    if (!e) e = sh->slice_payload.alloc(sh->slice_n * pb + 16);
    if (!e) e = sh->slice_counts.alloc((size_t)sh->gs.nchunks * world * 4);
    if (!e) e = sh->slice_gsum.alloc((size_t)sh->gs.ngroups * world * 8);
    if (!e) e = sh->slice_tot.alloc((size_t)world * 8);
    if (!e) e = sh->recv.alloc(sh->recv_cap * pb + 16);
    if (!e) e = sh->d_dst.alloc((size_t)world * sizeof(void*));
    if (!e) e = sh->d_dst_base.alloc((size_t)world * 8);
    if (!e) e = cudaMallocHost(&sh->h_tot, (size_t)world * 8);
    if (e) {
        ssbh_shard_destroy(sh);
        return fail(SSBH_CUDA, "shard_create: allocation failed: %s", cudaGetErrorString(e));
    }
    sh->peer.assign(world, nullptr);
    sh->opened.assign(world, false);
    sh->peer[rank] = sh->recv.p;
    ssbh_extract_params op = sh->p;
    op.n_rounds = sh->recv_cap;
    if (auto st = plan_create_impl(&op, 0, &sh->plan, /*external_payload=*/true, pb)) {
        const std::string msg = g_err;
        ssbh_shard_destroy(sh);
        g_err = msg;
        return st;
    }
    *out = sh;
    return ok();
}

extern "C" const char* ssbh_shard_hash_kernel(const ssbh_shard* sh) {
    return sh ? ssbh_plan_hash_kernel(sh->plan) : "";
}

extern "C" ssbh_status ssbh_shard_split_geometry(const ssbh_shard* sh, uint32_t* levels,
                                                 uint32_t* squares, uint32_t* batch_blocks) {
    if (!sh) return fail(SSBH_INVALID_ARGUMENT, "null shard");
    return ssbh_plan_split_geometry(sh->plan, levels, squares, batch_blocks);
}

extern "C" ssbh_status ssbh_shard_destroy(ssbh_shard* sh) {
    if (!sh) return ok();
    for (uint32_t r = 0; r < sh->peer.size(); ++r)
        if (sh->opened[r]) cudaIpcCloseMemHandle(sh->peer[r]);
    if (sh->plan) ssbh_plan_destroy(sh->plan);
    if (sh->h_tot) cudaFreeHost(sh->h_tot);
    delete sh;
    return ok();
}

extern "C" ssbh_status ssbh_shard_info(const ssbh_shard* sh, uint64_t* slice_first,
                                       uint64_t* slice_rounds, uint32_t* block_first,
                                       uint32_t* block_count) {
    if (!sh) return fail(SSBH_INVALID_ARGUMENT, "null shard");
    if (slice_first) *slice_first = sh->slice_lo;
    if (slice_rounds) *slice_rounds = sh->slice_n;
    if (block_first) *block_first = sh->p.block_first;
    if (block_count) *block_count = sh->p.block_count;
    return ok();
}

extern "C" ssbh_status ssbh_shard_ipc_handle(ssbh_shard* sh, void* handle_out) {
    if (!sh || !handle_out) return fail(SSBH_INVALID_ARGUMENT, "null argument");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, sh->recv.p));
    static_assert(sizeof(h) == SSBH_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof h);
    return ok();
}

extern "C" ssbh_status ssbh_shard_open_peers(ssbh_shard* sh, const void* handles) {
    if (!sh || !handles) return fail(SSBH_INVALID_ARGUMENT, "null argument");
    for (uint32_t r = 0; r < sh->world; ++r) {
        if (r == sh->rank || sh->opened[r]) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof h, sizeof h);
        void* ptr = nullptr;
        CU(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        sh->peer[r] = ptr;
        sh->opened[r] = true;
    }
    CU(cudaMemcpy(sh->d_dst.p, sh->peer.data(), (size_t)sh->world * sizeof(void*),
                  cudaMemcpyHostToDevice));
    return ok();
}

extern "C" ssbh_status ssbh_shard_sample(ssbh_shard* sh, const uint32_t* d_slice_input,
                                         const uint64_t* samp_key, uint64_t* owner_counts,
                                         void* stream) {
    if (!sh || !owner_counts || (sh->slice_n && !d_slice_input))
        return fail(SSBH_INVALID_ARGUMENT, "shard_sample: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t* sk = samp_key ? samp_key : sh->p.samp_key;
    sh->launches = 0;
    CU(cudaMemsetAsync(sh->slice_counts.p, 0, sh->slice_counts.bytes, st));
    CU(cudaMemsetAsync(sh->slice_tot.p, 0, sh->slice_tot.bytes, st));
    if (sh->slice_n) {
        launch_sample_slice(sh->gs, sk, sh->slice_lo, d_slice_input, sh->slice_payload.p,
                            sh->world, sh->slice_counts.as<uint32_t>(), st);
        launch_scan(sh->gs, sh->slice_counts.as<uint32_t>(),
                    sh->slice_gsum.as<unsigned long long>(),
                    sh->slice_tot.as<unsigned long long>(), st);
        sh->launches += 4;
    }
    CU(cudaMemcpyAsync(sh->h_tot, sh->slice_tot.p, (size_t)sh->world * 8, cudaMemcpyDeviceToHost,
                       st));
    CU(cudaStreamSynchronize(st));
    std::memcpy(owner_counts, sh->h_tot, (size_t)sh->world * 8);
    return check_launch("shard_sample");
}

extern "C" ssbh_status ssbh_shard_exchange(ssbh_shard* sh, const uint64_t* counts, void* stream) {
    if (!sh || !counts) return fail(SSBH_INVALID_ARGUMENT, "shard_exchange: null argument");
    const uint32_t W = sh->world;
    std::vector<uint64_t> base(W, 0);
    for (uint32_t o = 0; o < W; ++o) {
        uint64_t tot = 0;
        for (uint32_t r = 0; r < W; ++r) {
            if (r == sh->rank) base[o] = tot;
            tot += counts[(size_t)r * W + o];
        }
        if (tot > sh->recv_cap)
            return fail(SSBH_INVALID_ARGUMENT, "shard_exchange: owner %u receives %llu rounds > "
                        "capacity %llu", o, (unsigned long long)tot,
                        (unsigned long long)sh->recv_cap);
        if (o == sh->rank) sh->n_recv = tot;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CU(cudaMemcpyAsync(sh->d_dst_base.p, base.data(), (size_t)W * 8, cudaMemcpyHostToDevice, st));
    launch_owner_split(sh->gs, sh->slice_payload.p, W, sh->slice_counts.as<uint32_t>(),
                       sh->d_dst.as<void* const>(), sh->d_dst_base.as<unsigned long long>(), st);
    sh->launches += 1;
    CU(cudaStreamSynchronize(st));  // this rank's stores are complete before its barrier
    return check_launch("shard_exchange");
}

extern "C" ssbh_status ssbh_shard_finish(ssbh_shard* sh, uint32_t* d_key, uint64_t* d_lengths,
                                         const uint64_t* hash_key, void* stream) {
    if (!sh || !d_key) return fail(SSBH_INVALID_ARGUMENT, "shard_finish: null argument");
    ssbh_plan* pl = sh->plan;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    pl->last_stream = st;
    const uint64_t* hk = hash_key ? hash_key : sh->p.hash_key;
    const SamplerGeom g = geom_with_n(pl->geom, sh->n_recv);
    const Layout lay = pl->lay.view();
    uint32_t launches = sh->launches;
    if (pl->timing) CU(cudaEventRecord(pl->ev[0], st));
    if (pl->bucketed) {
        // many owned blocks: two-level split of the received rounds (see BucketGeom)
        CU(cudaMemsetAsync(&lay.stats->pad, 0, 4, st));
        if (auto s = bucket_passes(pl, geom_with_n(pl->bg.a, sh->n_recv), nullptr, 0, nullptr,
                                   nullptr, sh->recv.p, st, launches))
            return s;
        CU(cudaMemcpyAsync(lay.nj, pl->nj_b.p, (size_t)pl->nown * 8, cudaMemcpyDeviceToDevice,
                           st));
    } else {
        CU(cudaMemsetAsync(pl->counts.p, 0, pl->counts.bytes, st));
        launch_count_payload(g, sh->recv.p, pl->counts.as<uint32_t>(), st);
        launch_scan(g, pl->counts.as<uint32_t>(), pl->gsum.as<unsigned long long>(), lay.nj, st);
        launches += 4;
    }
    launch_layout(lay, pl->nown, pl->p.out_bits, pl->rowtiles, pl->kt, pl->p.per_block_seed,
                  pl->p.block_limit, st);
    launches += 1;
    if (pl->timing) CU(cudaEventRecord(pl->ev[1], st));
    CU(cudaMemsetAsync(pl->ybuf.p, 0, pl->ybuf.bytes, st));
    if (pl->bucketed)
        launch_bucket_scatter(pl->bg, pl->staging.as<uint16_t>(), pl->counts_b.as<uint32_t>(),
                              lay.nj, lay.yoff, pl->ybuf.as<uint32_t>(), nullptr, st);
    else
        launch_scatter(g, sh->recv.p, pl->counts.as<uint32_t>(), lay.nj, lay.yoff,
                       pl->ybuf.as<uint32_t>(), nullptr, nullptr, st);
    launches += 1;
    if (auto s = phase_finish(pl, d_key, d_lengths, hk, st, launches)) return s;
    pl->launches_per_run = launches;
    return check_launch("shard_finish");
}

extern "C" ssbh_status ssbh_shard_check(ssbh_shard* sh, ssbh_extract_stats* stats) {
    if (!sh) return fail(SSBH_INVALID_ARGUMENT, "null shard");
    return ssbh_plan_check(sh->plan, stats);
}

extern "C" ssbh_status ssbh_shard_set_timing(ssbh_shard* sh, int enable) {
    if (!sh) return fail(SSBH_INVALID_ARGUMENT, "null shard");
    return ssbh_plan_set_timing(sh->plan, enable);
}

// ======================================================================== protocol rounds
static ssbh_status check_round_params(const ssbh_round_params* p) {
    if (!p) return fail(SSBH_INVALID_ARGUMENT, "simulate_rounds: null params");
    const double ps[4] = {p->p_x, p->e_ph, p->e_bit, p->p_det};
    for (double v : ps)
        if (!(v >= 0.0 && v <= 1.0)) return fail(SSBH_INVALID_ARGUMENT, "bernoulli: p outside [0,1]");
    return SSBH_OK;
}

extern "C" ssbh_status ssbh_simulate_rounds_device(const ssbh_round_params* params,
                                                   const uint64_t seed[4], uint8_t* d_rounds,
                                                   void* stream) {
    if (auto s = check_round_params(params)) return s;
    if (params->n_rounds == 0) return ok();
    if (!seed || !d_rounds) return fail(SSBH_INVALID_ARGUMENT, "simulate_rounds: null argument");
    NEED_DEVICE();
    launch_simulate_rounds(seed, params->n_rounds, params->p_x, params->e_ph, params->e_bit,
                           params->p_det, d_rounds, static_cast<cudaStream_t>(stream));
    return check_launch("simulate_rounds");
}

extern "C" ssbh_status ssbh_simulate_rounds(const ssbh_round_params* params,
                                            const uint64_t seed[4], uint8_t* rounds) {
    if (auto s = check_round_params(params)) return s;
    if (params->n_rounds == 0) return ok();
    if (!seed || !rounds) return fail(SSBH_INVALID_ARGUMENT, "simulate_rounds: null argument");
    NEED_DEVICE();
    DBuf d;
    CU(d.alloc(params->n_rounds));
    if (auto s = ssbh_simulate_rounds_device(params, seed, d.as<uint8_t>(), nullptr)) return s;
    CU(cudaMemcpy(rounds, d.p, params->n_rounds, cudaMemcpyDeviceToHost));
    return ok();
}

// pipeline.cpp:84-136 from device-resident RoundRecord bytes. The two host decisions of the
// reference (statistics abort, then oversize abort / bits_per_block) need the counters and
// the block lengths, so the call synchronises twice.
extern "C" ssbh_status ssbh_run_extraction_device(const uint8_t* d_rounds, uint64_t n,
                                                  const ssbh_extraction_params* p,
                                                  uint64_t* out_key, uint64_t* out_lengths,
                                                  ssbh_extraction_result* res) {
    if (!p || !res) return fail(SSBH_INVALID_ARGUMENT, "run_extraction: null argument");
    if (p->n_subblocks == 0)
        return fail(SSBH_INVALID_ARGUMENT, "run_extraction: plan.n_subblocks must be positive");
    if (p->block_limit == 0)
        return fail(SSBH_INVALID_ARGUMENT, "run_extraction: plan.block_limit must be set");
    if (n == 0 || !d_rounds)
        return fail(SSBH_INVALID_ARGUMENT, "run_extraction: round count does not match params");
    NEED_DEVICE();
    std::memset(res, 0, sizeof *res);
    const uint32_t ns = p->n_subblocks;
    // pipeline.cpp:86-88, same operation order
    res->total_epsilon = static_cast<double>(ns) * (p->eps_sec - p->eps_abort) /
                             static_cast<double>(ns) +
                         p->eps_abort;

    const uint64_t w32 = (n + 31) / 32;
    DBuf bits, keep, cnt;
    CU(bits.alloc(round_up(w32, 2) * 4));
    CU(keep.alloc(round_up(w32, 2) * 4));
    CU(cnt.alloc(4 * 8));
    CU(cudaMemset(cnt.p, 0, 4 * 8));
    launch_rounds_split(d_rounds, n, bits.as<uint32_t>(), keep.as<uint32_t>(),
                        cnt.as<unsigned long long>(), nullptr);
    if (auto s = check_launch("rounds_split")) return s;
    uint64_t c[4];
    CU(cudaMemcpy(c, cnt.p, sizeof c, cudaMemcpyDeviceToHost));
    res->test_rounds = c[0];
    res->phase_errors = c[1];
    res->no_detections = c[2];
    res->key_rounds = c[3];

    // statistics check (pipeline.cpp:90-104)
    const double nd = static_cast<double>(n);
    const double px2 = p->p_x * p->p_x;
    if (static_cast<double>(c[1]) / nd > px2 * p->eta_tol * p->q_tol ||
        static_cast<double>(c[2]) / nd > px2 * (1.0 - p->eta_tol)) {
        res->abort = 2;
        return ok();
    }

    // sift + sample + abort_check + per-block seeds + hash (pipeline.cpp:107-136)
    const uint64_t bpb = p->key_length / ns;
    res->bits_per_block = bpb;
    ssbh_extract_params ep{};
    ep.n_rounds = n;
    ep.n_subblocks = ns;
    ep.per_block_seed = 1;
    ep.out_bits = bpb ? bpb : 32;  // bpb == 0: lengths only, the hash output is discarded
    std::memcpy(ep.samp_key, p->seed, 32);
    std::memcpy(ep.hash_key, p->seed, 32);
    ep.block_limit = p->block_limit;
    ssbh_plan* pl = nullptr;
    if (auto s = ssbh_plan_create(&ep, &pl)) return s;
    std::unique_ptr<ssbh_plan, ssbh_status (*)(ssbh_plan*)> guard(pl, ssbh_plan_destroy);
    ssbh_plan_set_timing(pl, 1);
    DBuf key, len;
    const uint64_t key_w64 = words64((uint64_t)ns * ep.out_bits);
    CU(key.alloc(key_w64 * 8 + 16));
    CU(len.alloc((size_t)ns * 8));
    CU(cudaMemset(key.p, 0, key_w64 * 8 + 16));
    if (auto s = ssbh_plan_run_device_sifted(pl, bits.as<uint32_t>(), keep.as<uint32_t>(),
                                             key.as<uint32_t>(), len.as<uint64_t>(), nullptr,
                                             nullptr, nullptr))
        return s;
    ssbh_extract_stats st{};
    ssbh_status s = ssbh_plan_check(pl, &st);
    if (s == SSBH_ABORT_OVERSIZE) {
        res->abort = 1;
        res->bits_per_block = 0;  // the reference returns before sizing the key
        s = SSBH_OK;
    } else if (s == SSBH_INVALID_ARGUMENT && bpb == 0 && st.min_len == 0) {
        s = SSBH_OK;  // no hashing when nothing is extractable: empty blocks are fine
    }
    if (s != SSBH_OK) return s;
    if (out_lengths) CU(cudaMemcpy(out_lengths, len.p, (size_t)ns * 8, cudaMemcpyDeviceToHost));
    res->lengths_valid = out_lengths != nullptr;
    if (res->abort || bpb == 0) return ok();
    res->key_bits = (uint64_t)ns * bpb;
    res->hash_seconds = (st.ms_seed + st.ms_hash) * 1e-3;
    if (out_key) CU(cudaMemcpy(out_key, key.p, words64(res->key_bits) * 8, cudaMemcpyDeviceToHost));
    return ok();
}

extern "C" ssbh_status ssbh_run_extraction(const uint8_t* rounds, uint64_t n,
                                           const ssbh_extraction_params* p, uint64_t* out_key,
                                           uint64_t* out_lengths, ssbh_extraction_result* res) {
    if (!p || !res) return fail(SSBH_INVALID_ARGUMENT, "run_extraction: null argument");
    if (n == 0 || !rounds)
        return fail(SSBH_INVALID_ARGUMENT, "run_extraction: round count does not match params");
    NEED_DEVICE();
    DBuf d;
    CU(d.alloc(n));
    CU(cudaMemcpy(d.p, rounds, n, cudaMemcpyHostToDevice));
    return ssbh_run_extraction_device(d.as<uint8_t>(), n, p, out_key, out_lengths, res);
}

// ======================================================================== in-process multi-GPU
namespace {

// dst bits [off, off + nbits) |= src bits [0, nbits) (dst pre-zeroed; host words)
void or_bits(uint64_t* dst, uint64_t off, const uint64_t* src, uint64_t nbits) {
    const uint64_t nw = words64(nbits);
    const unsigned sh = (unsigned)(off & 63);
    uint64_t* d = dst + (off >> 6);
    for (uint64_t w = 0; w < nw; ++w) {
        uint64_t v = src[w];
        if (w + 1 == nw && (nbits & 63)) v &= (1ull << (nbits & 63)) - 1;
        d[w] |= v << sh;
        if (sh && (w + 1 < nw || ((nbits & 63) == 0 ? 64 : (nbits & 63)) + sh > 64))
            d[w + 1] |= v >> (64 - sh);
    }
}

struct RankRun {
    ssbh_shard* sh = nullptr;
    int device = 0;
    cudaStream_t st = nullptr;
    DBuf slice, key, len;
    std::vector<uint64_t> counts, key_host, len_host;
    ssbh_status status = SSBH_OK;
    std::string msg;
};

// Runs fn(rank) on one host thread per rank (each bound to its device); the first failure's
// status and message become the caller's.
template <class Fn>
ssbh_status on_ranks(std::vector<RankRun>& rr, Fn fn) {
    std::vector<std::thread> th;
    for (size_t r = 0; r < rr.size(); ++r)
        th.emplace_back([&, r] {
            if (cudaSetDevice(rr[r].device) != cudaSuccess) {
                rr[r].status = SSBH_CUDA;
                rr[r].msg = "set_device failed";
                return;
            }
            rr[r].status = fn(r);
            if (rr[r].status != SSBH_OK) rr[r].msg = g_err;
        });
    for (auto& t : th) t.join();
    for (auto& x : rr)
        if (x.status != SSBH_OK) return fail(x.status, "%s", x.msg.c_str());
    return SSBH_OK;
}

}  // namespace

// One process driving several GPUs: the sharded protocol of ssbh_shard_* with the receive
// buffers exchanged as plain device pointers (peer access enabled between distinct devices)
// and the three phases separated by thread joins instead of torch.distributed.
extern "C" ssbh_status ssbh_extract_multi(const ssbh_extract_params* params, const uint64_t* input,
                                          const int* devices, uint32_t ndev, uint64_t* out_key,
                                          uint64_t* out_lengths, ssbh_extract_stats* stats) {
    if (!params || !input || !out_key || !devices || ndev == 0)
        return fail(SSBH_INVALID_ARGUMENT, "extract_multi: null argument / no devices");
    if (params->block_first != 0 || (params->block_count && params->block_count != params->n_subblocks))
        return fail(SSBH_INVALID_ARGUMENT, "extract_multi: produces the whole key (block range 0, all)");
    NEED_DEVICE();
    for (uint32_t r = 0; r < ndev; ++r)
        if (devices[r] < 0 || devices[r] >= usable_devices())
            return fail(SSBH_INVALID_ARGUMENT, "extract_multi: device %d out of range", devices[r]);
    int prev = 0;
    CU(cudaGetDevice(&prev));
    if (ndev == 1) {
        CU(cudaSetDevice(devices[0]));
        const ssbh_status s = ssbh_extract(params, input, out_key, out_lengths, stats);
        cudaSetDevice(prev);
        return s;
    }
    const uint64_t n = params->n_rounds, k = params->out_bits, s = params->n_subblocks;
    std::vector<RankRun> rr(ndev);
    for (uint32_t r = 0; r < ndev; ++r) rr[r].device = devices[r];
    auto cleanup = [&] {
        for (auto& x : rr) {
            cudaSetDevice(x.device);
            if (x.sh) ssbh_shard_destroy(x.sh);
            if (x.st) cudaStreamDestroy(x.st);
            x.slice.release();
            x.key.release();
            x.len.release();
        }
        cudaSetDevice(prev);
    };
    ssbh_status st = on_ranks(rr, [&](size_t r) -> ssbh_status {
        if (auto e = ssbh_shard_create(params, (uint32_t)r, ndev, &rr[r].sh)) return e;
        CU(cudaStreamCreateWithFlags(&rr[r].st, cudaStreamNonBlocking));
        return SSBH_OK;
    });
    if (st == SSBH_OK) {
        // receive buffers as plain pointers; peer access between distinct devices
        for (uint32_t r = 0; r < ndev; ++r) {
            cudaSetDevice(rr[r].device);
            for (uint32_t q = 0; q < ndev; ++q) {
                rr[r].sh->peer[q] = rr[q].sh->recv.p;
                if (rr[q].device != rr[r].device) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(rr[q].device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else if (e != cudaSuccess) {
                        st = fail(SSBH_CUDA, "extract_multi: peer access %d -> %d: %s", rr[r].device,
                                  rr[q].device, cudaGetErrorString(e));
                        break;
                    }
                }
            }
            if (st != SSBH_OK) break;
            if (cudaMemcpy(rr[r].sh->d_dst.p, rr[r].sh->peer.data(), (size_t)ndev * sizeof(void*),
                           cudaMemcpyHostToDevice) != cudaSuccess) {
                st = fail(SSBH_CUDA, "extract_multi: peer table upload failed");
                break;
            }
        }
    }
    // phase 1: each rank samples its slice of rounds
    if (st == SSBH_OK)
        st = on_ranks(rr, [&](size_t r) -> ssbh_status {
            RankRun& x = rr[r];
            const uint64_t lo = x.sh->slice_lo, cnt = x.sh->slice_n;
            const uint64_t w0 = lo / 64, w1 = words64(lo + cnt);
            CU(x.slice.alloc((w1 - w0) * 8 + 16));
            if (cnt)
                CU(cudaMemcpyAsync(x.slice.p, input + w0, (w1 - w0) * 8, cudaMemcpyHostToDevice,
                                   x.st));
            x.counts.assign(ndev, 0);
            return ssbh_shard_sample(x.sh, x.slice.as<uint32_t>(), nullptr, x.counts.data(), x.st);
        });
    // phase 2: owner split through peer memory (every rank needs every rank's counts)
    std::vector<uint64_t> matrix((size_t)ndev * ndev);
    for (uint32_t r = 0; r < ndev && st == SSBH_OK; ++r)
        std::memcpy(matrix.data() + (size_t)r * ndev, rr[r].counts.data(), (size_t)ndev * 8);
    if (st == SSBH_OK)
        st = on_ranks(rr, [&](size_t r) -> ssbh_status {
            return ssbh_shard_exchange(rr[r].sh, matrix.data(), rr[r].st);
        });
    // phase 3 (after the join = barrier): owners hash their blocks
    if (st == SSBH_OK)
        st = on_ranks(rr, [&](size_t r) -> ssbh_status {
            RankRun& x = rr[r];
            const uint64_t cnt = x.sh->p.block_count;
            const uint64_t kw64 = words64(cnt * k);
            CU(x.key.alloc(kw64 * 8 + 16));
            CU(x.len.alloc(cnt * 8 + 8));
            CU(cudaMemsetAsync(x.key.p, 0, kw64 * 8 + 16, x.st));
            if (auto e = ssbh_shard_finish(x.sh, x.key.as<uint32_t>(), x.len.as<uint64_t>(), nullptr,
                                           x.st))
                return e;
            if (auto e = ssbh_shard_check(x.sh, nullptr)) return e;
            x.key_host.resize(kw64 + 1);
            x.len_host.resize(cnt + 1);
            CU(cudaMemcpy(x.key_host.data(), x.key.p, kw64 * 8, cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(x.len_host.data(), x.len.p, cnt * 8, cudaMemcpyDeviceToHost));
            return SSBH_OK;
        });
    if (st == SSBH_OK) {
        std::memset(out_key, 0, words64(s * k) * 8);
        ssbh_extract_stats agg{};
        agg.min_len = ~0ull;
        for (auto& x : rr) {
            const uint64_t first = x.sh->p.block_first, cnt = x.sh->p.block_count;
            or_bits(out_key, first * k, x.key_host.data(), cnt * k);
            if (out_lengths) std::memcpy(out_lengths + first, x.len_host.data(), cnt * 8);
            for (uint64_t i = 0; i < cnt; ++i) {
                agg.max_len = std::max<uint64_t>(agg.max_len, x.len_host[i]);
                agg.min_len = std::min<uint64_t>(agg.min_len, x.len_host[i]);
                agg.hash_word_ops += x.len_host[i] * k / 32;
            }
        }
        agg.hash_launches = ndev;
        if (stats) *stats = agg;
        (void)n;
    }
    cleanup();
    return st == SSBH_OK ? ok() : st;
}
