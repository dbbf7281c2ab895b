// spk_capi.cu — C-ABI (include/spike_b200.h) over the SPIKE device kernels.
//
// The host side is a compiler, not an interpreter: at factorization time the
// reference's stage structure (src/factorize.cpp:133-257, src/solve.cpp:81-380)
// is lowered into three static "programs" (factor, forward solve, transpose
// solve).  Each program is a short list of stages; each stage is ONE batched
// launch over all partitions / coupling blocks.  Job descriptors live in one
// device blob uploaded once, and address per-call buffers through a Bufs table,
// so a solve issues O(stages + reduced levels) launches independent of p.
#include "../../include/spike_b200.h"
#include "spk_launch.h"
#include "spk_piv_blocked.cuh"
#include "spk_sweep_fast.cuh"
#include "spk_sweep_dmma.cuh"

namespace spk {
struct PivLuArgs {  // spk_lu_fast.cu
    const int* units;
    const PartDev* parts;
    const double* band;
    int akl, aku;
    double* fac;
    int* piv;
    int* status;
};
}  // namespace spk

#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

using namespace spk;

// ---------------------------------------------------------------------------
// errors
namespace {
thread_local std::string g_err;
thread_local long long g_launches = 0;
// launches of the generic correctness-baseline kernels (k_sweep, k_band_lu)
// on SPIKE-partition stages whose shape no tuned kernel covers, or of every
// generic kernel when spk_set_generic_path(1) forces that path (tests).  The
// coupling units' generic pivoted LU is not counted: it is the designated
// path of pairs with |W| > 1 (guarded off on the device otherwise)
thread_local long long g_generic_launches = 0;
std::atomic<int> g_generic{0};
bool generic_path() { return g_generic.load(std::memory_order_relaxed) != 0; }

struct SpkError {
    spk_status st;
    std::string msg;
};

[[noreturn]] void fail(spk_status st, const std::string& m) { throw SpkError{st, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation) fail(SPK_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
        fail(SPK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <class F>
spk_status guarded(F&& f) {
    try {
        f();
        return SPK_OK;
    } catch (const SpkError& e) {
        g_err = e.msg;
        return e.st;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SPK_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPK_EINVAL;
    }
}
}  // namespace

namespace spk {
// every launcher calls this right after its launch: a launch that failed
// (configuration, resources) raises here instead of leaving its output unwritten
void count_launch(int n) {
    g_launches += n;
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(SPK_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    }
}

// The dynamic shared-memory limit of a kernel is a per-device attribute: keep
// the largest value set per (device, kernel) and only ever raise it, so
// concurrent launchers never lower it under each other.
void set_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    int& cur = done[{dev, fn}];
    if (bytes <= cur) return;
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "cudaFuncSetAttribute");
    cur = bytes;
}

unsigned long long* g_sk_trace = nullptr;

int device_sms() {
    static std::mutex mu;
    static std::map<int, int> sms;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    auto it = sms.find(dev);
    if (it != sms.end()) return it->second;
    int v = 0;
    ck(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    sms[dev] = v;
    return v;
}
}  // namespace spk

#include <chrono>
namespace {
// SPK_TRACE=1: host-side phase timestamps of factorize / solve on stderr
struct Tracer {
    bool on;
    std::chrono::steady_clock::time_point t0;
    const char* what;
    explicit Tracer(const char* w) : on(getenv("SPK_TRACE") && atoi(getenv("SPK_TRACE"))), what(w) {
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char* phase) {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[spk %s] %-24s %9.3f ms\n", what, phase, ms);
    }
};
}  // namespace

// ---------------------------------------------------------------------------
// optional per-kernel-class CUDA-event profiling (bench.py roofline):
// events are recorded on the launching stream around each stage launch.
namespace {
struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double flops, bytes;
};
thread_local bool g_prof_on = false;
thread_local std::vector<ProfRec> g_prof;
thread_local std::vector<cudaEvent_t> g_evpool;
// one class per StageType (same order), then the factorization prologue
constexpr int kNumClasses = 14;
const char* kClassName[kNumClasses] = {"sweep",     "copy",       "gemm",         "band_lu",  "coupling",
                                       "memset",    "memcpy_fx",  "memcpy_fs",    "transpose", "wcheck",
                                       "schur_init", "dense_lu",  "fill_factors", "corners"};
enum { PC_FILL = 12, PC_CORNERS = 13 };
struct ProfAcc {
    double ms = 0, flops = 0, bytes = 0;
    long long launches = 0;
};
thread_local ProfAcc g_acc[kNumClasses];

cudaEvent_t prof_event() {
    if (!g_evpool.empty()) {
        cudaEvent_t e = g_evpool.back();
        g_evpool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    bool on;
    ProfRec r;
    cudaStream_t s;
    ProfScope(int cls, cudaStream_t st, double flops, double bytes) : on(g_prof_on), s(st) {
        if (!on) return;
        r.a = prof_event();
        r.b = prof_event();
        r.cls = cls;
        r.flops = flops;
        r.bytes = bytes;
        cudaEventRecord(r.a, s);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(r.b, s);
        g_prof.push_back(r);
    }
};

void prof_drain() {
    for (ProfRec& r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        g_acc[r.cls].ms += ms;
        g_acc[r.cls].flops += r.flops;
        g_acc[r.cls].bytes += r.bytes;
        g_acc[r.cls].launches += 1;
        g_evpool.push_back(r.a);
        g_evpool.push_back(r.b);
    }
    g_prof.clear();
}
}  // namespace

// ---------------------------------------------------------------------------
// programs
namespace {

enum StageType {
    ST_SWEEP, ST_COPY, ST_GEMM, ST_LU, ST_CPL, ST_MEMSET, ST_MEMCPY_FX, ST_MEMCPY_FS, ST_TRANSPOSE,
    ST_WCHECK, ST_SCHUR_INIT, ST_SCHUR_INV,
    ST_PHASE = 100  // exchange-point marker (no work, not profiled)
};

struct Stage {
    StageType t;
    int njobs = 0;
    size_t off = 0;  // byte offset of the job array in the device blob
    int max_nc = 0;  // sweep/gemm: max explicit columns; -1: call columns
    long long max_elems = 0;
    int max_r = 0;
    int max_kk = 0;  // gemm: longest inner dimension (split-K choice)
    int buf = 0;  // memset target
    int cols = -1;  // memset columns (-1: call columns)
    // algorithmic work per call column (explicit-column stages: per launch)
    double flops_per_col = 0.0, bytes_per_col = 0.0;
    // sweeps: register-window fast path (spk_sweep_fast.cuh) when every job is
    // a SPIKE partition it supports
    bool fast = false;
    int mode = 0, kwmax = 0, tr = 0, piv = 0;
    // sweeps on short units: shared-memory staged kernel (k_sweep_small)
    int small_ch = 0, small_rows = 0;
    bool partitions = false;  // ST_LU / ST_SWEEP over SPIKE partitions (LU: fill from the input band)
};

struct ProgramBuilder {
    std::vector<char> blob;
    template <class T>
    size_t push(const std::vector<T>& v) {
        size_t off = (blob.size() + 15) & ~size_t(15);
        blob.resize(off + v.size() * sizeof(T));
        if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
        return off;
    }
};

using Program = std::vector<Stage>;

View view(int buf, long long base, int rev = 0, int off = 0, int mrows = 0, long long ld = -1) {
    View v;
    v.base = base;
    v.ld = ld;
    v.buf = buf;
    v.rev = rev;
    v.off = off;
    v.mrows = mrows;
    return v;
}

struct Level {
    int units = 0;
    std::vector<int> uoff, uh;
    std::vector<long long> voff, woff;  // pool offsets, -1 when never formed
    std::vector<int> pair_part;         // PartDev index per pair: generic 2k coupling unit
    std::vector<int> spart;             // PartDev index per pair: k x k Schur-complement unit
    std::vector<int> gidx;              // flag index per pair (1 = Schur path, 0 = generic)
    std::vector<long long> sinv;        // pool offset of S^-1 (k x k, ld k) per pair, Schur path
};

}  // namespace

namespace {

// Device arena: factorizations and solves allocate gigabytes of factor and
// scratch storage per call.  Freed blocks go to a free list (exact size class,
// 2 MiB granularity) with an event recorded on the freeing stream; a reuse on
// another stream waits on that event, a reuse on the same stream is ordered by
// the stream itself.  Growth uses cudaMalloc once; nothing is re-mapped on the
// hot path (cudaMallocAsync re-mapped the pool on every factorization: ~22 ms
// per C3 factorization).
struct ArenaBlock {
    void* p;
    size_t bytes;
    cudaStream_t stream;
    cudaEvent_t ev;
};

struct Arena {
    std::mutex mu;
    std::vector<ArenaBlock> free_list;
    size_t cached = 0;

    static size_t round_up(size_t b) {
        const size_t g = b >= (2u << 20) ? (2u << 20) : 256;
        return (b + g - 1) / g * g;
    }

    static bool tracing() {
        static const bool t = getenv("SPK_TRACE") && atoi(getenv("SPK_TRACE")) > 1;
        return t;
    }

    // SPK_POISON=1 (debugging aid): every block handed out is filled with
    // 0xFF bytes (NaN doubles, -1 ints) on the requesting stream, so a read of
    // memory its kernel chain never wrote shows up as NaN in the results
    // instead of depending on what the block held before.
    static bool poisoning() {
        static const bool t = getenv("SPK_POISON") && atoi(getenv("SPK_POISON")) > 0;
        return t;
    }

    void* alloc(size_t bytes, cudaStream_t s) {
        void* p = alloc_block(bytes, s);
        if (poisoning()) cudaMemsetAsync(p, 0xFF, round_up(bytes == 0 ? 1 : bytes), s);
        return p;
    }

    void* alloc_block(size_t bytes, cudaStream_t s) {
        bytes = round_up(bytes == 0 ? 1 : bytes);
        {
            std::lock_guard<std::mutex> lk(mu);
            // best fit, preferring blocks already free for this stream (released
            // on it, or their last use finished): a block still in flight on
            // another stream would order this stream behind that work.  A
            // large in-flight block is left alone and a new one allocated.
            int best = -1;
            bool best_ready = false;
            for (int i = 0; i < (int)free_list.size(); ++i) {
                const ArenaBlock& b = free_list[i];
                if (b.bytes < bytes || b.bytes > bytes + bytes / 4) continue;
                const bool ready = b.stream == s || cudaEventQuery(b.ev) == cudaSuccess;
                if (best < 0 || (ready && !best_ready) || (ready == best_ready && b.bytes < free_list[best].bytes)) {
                    best = i;
                    best_ready = ready;
                }
            }
            (void)cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady
            if (best >= 0 && !best_ready && bytes >= (64u << 20)) best = -1;
            if (best >= 0) {
                ArenaBlock b = free_list[best];
                free_list.erase(free_list.begin() + best);
                cached -= b.bytes;
                if (b.stream != s) cudaStreamWaitEvent(s, b.ev, 0);
                cudaEventDestroy(b.ev);
                if (tracing() && bytes > (1u << 30))
                    fprintf(stderr, "[spk arena] reuse %.3f GB for %.3f GB\n", b.bytes / 1e9, bytes / 1e9);
                return b.p;
            }
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (tracing()) {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            fprintf(stderr, "[spk arena] cudaMalloc %.3f GB (%s), cached %.3f GB, free %.3f GB\n", bytes / 1e9,
                    e == cudaSuccess ? "ok" : "failed", cached / 1e9, fr / 1e9);
        }
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            trim();  // give cached blocks back and retry once
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
        }
        std::lock_guard<std::mutex> lk(mu);
        sizes[p] = bytes;
        return p;
    }

    void release(void* p, cudaStream_t s) {
        if (!p) return;
        std::lock_guard<std::mutex> lk(mu);
        auto it = sizes.find(p);
        if (it == sizes.end()) return;
        ArenaBlock b{p, it->second, s, nullptr};
        cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
        cudaEventRecord(b.ev, s);
        free_list.push_back(b);
        cached += b.bytes;
        if (tracing() && b.bytes > (1u << 30))
            fprintf(stderr, "[spk arena] release %.3f GB, cached %.3f GB\n", b.bytes / 1e9, cached / 1e9);
        // Bound the cache at 3/4 of HBM: drop the oldest blocks beyond it
        // (waits for their last use; only reached when shapes keep changing;
        // a failing cudaMalloc also trims).  C5 keeps ~104 GB cached.
        while (cached > cap() && free_list.size() > 1) {
            ArenaBlock o = free_list.front();
            free_list.erase(free_list.begin());
            cudaEventSynchronize(o.ev);
            cudaEventDestroy(o.ev);
            sizes.erase(o.p);
            cudaFree(o.p);
            cached -= o.bytes;
            if (tracing()) fprintf(stderr, "[spk arena] evict %.3f GB\n", o.bytes / 1e9);
        }
    }

    static size_t cap() {
        static size_t c = [] {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            return tot / 4 * 3;
        }();
        return c;
    }

    void trim() {
        std::lock_guard<std::mutex> lk(mu);
        for (ArenaBlock& b : free_list) {
            cudaEventSynchronize(b.ev);
            cudaEventDestroy(b.ev);
            sizes.erase(b.p);
            cudaFree(b.p);
        }
        free_list.clear();
        cached = 0;
    }

    std::unordered_map<void*, size_t> sizes;
};

Arena& arena() {
    static Arena* a = new Arena();  // leaked on purpose: no teardown-order issues at exit
    return *a;
}

template <class T>
T* dalloc(size_t count, cudaStream_t s) {
    return static_cast<T*>(arena().alloc(sizeof(T) * (count == 0 ? 1 : count), s));
}

inline void dfree(void* p, cudaStream_t s) { arena().release(p, s); }

}  // namespace

struct spk_fact {
    long long n = 0;
    int kl = 0, ku = 0, k = 0, p = 0, piv_on = 0;
    // Slab of a multi-GPU system: an open edge couples to the neighbouring
    // slab, so the edge partition carries that spike too and the local
    // hierarchy ends in one unit with V (open right) / W (open left) spikes.
    int open_l = 0, open_r = 0;
    double boost_eps = 0.0;
    bool reduced_only = false;
    std::vector<long long> bounds;
    std::vector<int> kinds;
    std::vector<PartDev> parts;  // [0,p) partitions, [p, p+ncpl) couplings
    std::vector<Level> levels;
    long long off_bhat = 0, off_chat = 0, pool_size = 0, fac_size = 0, piv_size = 0;
    long long aux_rows = 0, auxf_rows = 0;
    int tau_first = 0, tau_last = 0, z_first = 0, z_last = 0, tau_w = 0;  // AUX row offsets
    // device
    PartDev* d_parts = nullptr;
    double* d_fac = nullptr;
    int* d_piv = nullptr;
    double* d_pool = nullptr;
    long long* d_bounds = nullptr;
    unsigned long long* d_amax = nullptr;
    int* d_boost = nullptr;
    int* d_fell = nullptr;
    int* d_status = nullptr;
    char* d_blob = nullptr;   // factor program jobs
    char* d_sblob = nullptr;  // solve program jobs (built once the coupling paths are known)
    int* d_flags = nullptr;   // per-pair coupling path
    std::vector<int> flags;   // host copy after factorization
    int npairs = 0;
    double* d_tfac = nullptr;
    double* d_dinv = nullptr;
    long long tfac_size = 0;
    double* d_lblk = nullptr;  // pivoted: blocked L records (spk_piv_blocked.cuh)
    int lblk_trw = 0;
    bool lblk_ok = false;      // written by the blocked pivoted LU of this factorization
    Program prog_factor, prog_fwd, prog_tr, prog_rfwd, prog_rtr;  // r*: reduced system only
    // the general reduced-hierarchy stages (factorize.cpp:46-120); prog_factor
    // holds the partition stages before them
    Program prog_levels;
    // small-k engine (spk_smallk.cu): tables in the factor blob, a fallback
    // flag and grid-barrier words per factorization
    bool sk = false;
    bool sk_schur_all = false;  // finished, every pair on the Schur path: k_sk_solve applies
    size_t sk_units = 0, sk_pairs = 0, sk_items = 0, sk_levels = 0;  // blob offsets
    int sk_nlevels = 0, sk_mmax = 0, sk_rmax = 0;
    unsigned* d_skmisc = nullptr;  // small-k: [0] status, [2, 2+nparts) fell, then 4 barrier words
    bool tables_shared = false;    // d_parts / d_bounds / d_blob belong to the symbolic
    // the small-k engine writes the packed factor only; the row-major copy the
    // general programs' transposed sweeps read is made at their first use
    std::atomic<bool> tfac_ready{true};
    std::mutex tfac_mu;
    bool want_tfac = false;  // the symbolic has seen transposed solves (setup_fact)
    std::shared_ptr<struct Symbolic> sym;  // cached geometry + programs (shared by equal factorizations)
    std::vector<long long> factor_sweeps;
    int boost_count = 0, boost_warnings = 0;
    cudaStream_t stream = nullptr;
    // spk_factorize returns once the work is enqueued; the host-side finish
    // (status, boost counts, coupling paths -> solve programs) runs once, at
    // the first call that needs it (ensure_finished, under fin_mu).  Its
    // outcome is sticky: every later consumer re-raises a failure.
    std::mutex fin_mu;
    std::atomic<bool> pending{false};
    spk_status fin_status = SPK_OK;
    std::string fin_msg;
    cudaEvent_t upload_ev = nullptr;  // host band upload done (orders later host-solve uploads after it)
    // recorded on `stream` after the factor program and after every upload of
    // solve jobs: solves on other streams wait on it (wait_ready)
    cudaEvent_t ready_ev = nullptr;
    char* d_sblob_prev = nullptr;     // guarded solve jobs used while pending
    // last use of the factorization by each solve stream other than `stream`:
    // the destructor orders the release of the device memory after them
    std::mutex use_mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;

    // closed-edge predicates (reference kinds: the first partition has no W,
    // the last no V and is factored as UL)
    bool first(int i) const { return i == 0 && !open_l; }
    bool last(int i) const { return i == p - 1 && !open_r; }
    bool open() const { return open_l || open_r; }
    bool coupled() const { return k > 0 && (p > 1 || open()); }
    int top_level() const { return levels.empty() ? -1 : (int)levels.size() - 1; }

    ~spk_fact() {
        // stream-ordered release on the factorization's stream (which must
        // outlive it), after the last use by any other solve stream; no
        // device-wide synchronisation
        for (auto& u : uses) {
            cudaStreamWaitEvent(stream, u.second, 0);
            cudaEventDestroy(u.second);
        }
        if (tables_shared) {
            d_parts = nullptr;
            d_bounds = nullptr;
            d_blob = nullptr;
        }
        if (d_skmisc) {  // status / fell live inside it
            d_status = nullptr;
            d_fell = nullptr;
        }
        for (void* q : {(void*)d_parts, (void*)d_fac, (void*)d_piv, (void*)d_pool, (void*)d_bounds,
                        (void*)d_amax, (void*)d_boost, (void*)d_fell, (void*)d_status, (void*)d_blob,
                        (void*)d_tfac, (void*)d_dinv, (void*)d_sblob, (void*)d_flags, (void*)d_sblob_prev,
                        (void*)d_lblk, (void*)d_skmisc})
            if (q) dfree(q, stream);
        if (upload_ev) cudaEventDestroy(upload_ev);
        if (ready_ev) cudaEventDestroy(ready_ev);
    }
};

struct spk_reduced {
    std::unique_ptr<spk_fact> f;
};

namespace {

// ---------------------------------------------------------------------------
// geometry
PartDev make_part(long long r0, int m, int akl, int aku, int piv_on, int rev, int kcorner) {
    PartDev P{};
    P.r0 = r0;
    P.m = m;
    P.rev = rev;
    P.kl = std::min(rev ? aku : akl, m - 1);
    P.ku = std::min(rev ? akl : aku, m - 1);
    P.pivoting = piv_on;
    P.ubw = piv_on ? std::min(P.kl + P.ku, m - 1) : P.ku;
    P.d = P.ubw;
    P.rows = P.ubw + P.kl + 1;
    P.trunc = std::max(0, m - kcorner - (piv_on ? P.kl : 0));
    P.bofs = -1;
    P.tofs = -1;
    P.rowsT = 0;
    P.guard = -1;
    return P;
}

void build_levels(spk_fact& f, long long& pool_cursor) {
    const int p = f.p, k = f.k;
    f.levels.clear();
    if (!f.coupled()) return;
    int L = 0;
    for (int u = p; u > 1; u = (u + 1) / 2) ++L;
    f.levels.resize(L + 1);
    for (int l = 0; l <= L; ++l) {
        Level& lv = f.levels[l];
        lv.units = l == 0 ? p : (f.levels[l - 1].units + 1) / 2;
        lv.uoff.assign(lv.units, 0);
        lv.uh.assign(lv.units, 0);
        lv.voff.assign(lv.units, -1);
        lv.woff.assign(lv.units, -1);
        for (int a = 0; a < lv.units; ++a) {
            if (l == 0) {
                lv.uoff[a] = 2 * a * k;
                lv.uh[a] = 2 * k;
            } else {
                const Level& pv = f.levels[l - 1];
                lv.uoff[a] = pv.uoff[2 * a];
                lv.uh[a] = pv.uh[2 * a] + (2 * a + 1 < pv.units ? pv.uh[2 * a + 1] : 0);
            }
        }
    }
    // spike storage: level 0 holds [vt; vb] / [wt; wb].  A merged unit has a V
    // spike when its right-most sub-unit has one and a W spike when its
    // left-most has one (factorize.cpp:104-115 forms exactly those; carried
    // odd units keep theirs).  Closed slabs: the top unit has neither.
    for (int l = 0; l <= L; ++l) {
        Level& lv = f.levels[l];
        for (int a = 0; a < lv.units; ++a) {
            const long long sz = (long long)lv.uh[a] * k;
            bool hv = false, hw = false;
            if (l == 0) {
                hv = a < p - 1 || f.open_r;
                hw = a > 0 || f.open_l;
            } else {
                const Level& pv = f.levels[l - 1];
                const int right = 2 * a + 1 < pv.units ? 2 * a + 1 : 2 * a;
                hv = pv.voff[right] >= 0;
                hw = pv.woff[2 * a] >= 0;
            }
            if (hv) {
                lv.voff[a] = pool_cursor;
                pool_cursor += sz;
            }
            if (hw) {
                lv.woff[a] = pool_cursor;
                pool_cursor += sz;
            }
        }
    }
}

void add_couplings(spk_fact& f, long long& fac_cursor) {
    const int k = f.k;
    int idx = 0;
    for (size_t l = 0; l + 1 < f.levels.size(); ++l) {
        Level& lv = f.levels[l];
        lv.pair_part.clear();
        lv.spart.clear();
        lv.gidx.clear();
        for (int a = 0; a < lv.units / 2; ++a) {
            const int nn = 2 * k;
            // generic path: the full 2k coupling, pivoted with boosted fallback
            PartDev P = make_part(f.n + (long long)idx * nn, nn, nn - 1, nn - 1, 1, 0, 0);
            P.fallback = 1;
            P.fofs = fac_cursor;
            fac_cursor += (long long)P.m * P.rows;
            P.bofs = fac_cursor;
            fac_cursor += (long long)P.m * P.rows;
            P.guard = 2 * f.npairs + 0;
            lv.pair_part.push_back((int)f.parts.size());
            f.parts.push_back(P);
            // Schur path: S = I - W V as a pivoted dense k x k unit (full band)
            PartDev S = make_part(f.n + (long long)idx * nn + k, k, k - 1, k - 1, 1, 0, 0);
            S.fofs = fac_cursor;
            fac_cursor += (long long)S.m * S.rows;
            lv.spart.push_back((int)f.parts.size());
            f.parts.push_back(S);
            lv.gidx.push_back(f.npairs++);
            ++idx;
        }
    }
}

struct Builder {
    spk_fact& f;
    ProgramBuilder& pb;
    Program& prog;

    void sweep(const std::vector<SweepJob>& jobs) {
        if (jobs.empty()) return;
        Stage s{ST_SWEEP};
        s.njobs = (int)jobs.size();
        s.off = pb.push(jobs);
        int mx = 0;
        for (auto& j : jobs) {
            mx = j.nc < 0 ? -1 : (mx < 0 ? -1 : std::max(mx, j.nc));
            const PartDev& P = f.parts[j.part];
            const double rows = (j.mode == SW_BWD_U) ? (j.hi - j.lo + 1) : (P.m - j.lo);
            const double bw = (j.mode == SW_FWD_L || j.mode == SW_BWD_LT) ? P.kl : P.ubw;
            const double nc = j.nc < 0 ? 1.0 : j.nc;
            s.flops_per_col += 2.0 * rows * bw * nc;
            s.bytes_per_col += 8.0 * rows * (bw + 1) + 16.0 * rows * nc;
        }
        s.max_nc = mx;
        // fast-path eligibility
        bool fast = !generic_path() && !f.reduced_only;
        int kwneed = 1, kwmax = 1;
        for (auto& j : jobs) {
            const PartDev& P = f.parts[j.part];
            if (j.part >= f.p) fast = false;
            // pivoted transposed L sweeps need the blocked L records
            if (j.mode == SW_BWD_LT && P.pivoting && !piv_trw(f.kl, f.ku)) fast = false;
            if (j.mode != jobs[0].mode) fast = false;
            const int kw = (j.mode == SW_FWD_L || j.mode == SW_BWD_LT) ? P.kl : P.ubw;
            kwmax = std::max(kwmax, kw);
            kwneed = std::max(kwneed, (j.mode == SW_FWD_L && P.pivoting) ? P.kl + 1 : kw);
        }
        const int tr = (kwneed + 31) / 32;
        if (tr > 8) fast = false;
        // staged rows per job (the rows k_sweep touches) and factor entries per row
        int srows = 0, sbw = 0;
        for (auto& j : jobs) {
            const PartDev& P = f.parts[j.part];
            int a = j.lo, e = P.m, bw = P.kl;
            if (j.mode == SW_BWD_U || j.mode == SW_FWD_UT) {
                a = std::max(j.lo - P.ubw, j.v.off);
                bw = P.ubw;
            }
            if (j.mode == SW_BWD_U) e = j.hi + 1;
            srows = std::max(srows, e - a);
            sbw = std::max(sbw, bw);
        }
        if (srows <= 1024 && sbw <= 320) {
            s.small_rows = std::max(srows, 1);
            s.small_ch = std::max(1, (sbw + 31) / 32);
        }
        s.fast = fast;
        s.partitions = jobs[0].part < f.p && !f.reduced_only;
        s.mode = jobs[0].mode;
        s.kwmax = kwmax;
        s.tr = tr;
        s.piv = f.piv_on && (jobs[0].mode == SW_FWD_L || jobs[0].mode == SW_BWD_LT);
        prog.push_back(s);
    }
    void transpose_factors() { prog.push_back(Stage{ST_TRANSPOSE}); }
    void copy(const std::vector<CopyJob>& jobs) {
        if (jobs.empty()) return;
        Stage s{ST_COPY};
        s.njobs = (int)jobs.size();
        s.off = pb.push(jobs);
        long long mx = 0;
        int mnc = 0;
        for (auto& j : jobs) {
            mx = std::max(mx, (long long)(j.L1 - j.L0));
            mnc = j.nc < 0 ? -1 : (mnc < 0 ? -1 : std::max(mnc, j.nc));
        }
        s.max_elems = mx;
        s.max_nc = mnc;
        for (auto& j : jobs) s.bytes_per_col += 16.0 * (j.L1 - j.L0) * (j.nc < 0 ? 1.0 : j.nc);
        prog.push_back(s);
    }
    void gemm(const std::vector<GemmJob>& jobs) {
        if (jobs.empty()) return;
        Stage s{ST_GEMM};
        s.njobs = (int)jobs.size();
        s.off = pb.push(jobs);
        int mr = 0, mnc = 0;
        for (auto& j : jobs) {
            mr = std::max(mr, j.r);
            mnc = j.nc < 0 ? -1 : (mnc < 0 ? -1 : std::max(mnc, j.nc));
        }
        s.max_r = mr;
        s.max_nc = mnc;
        for (auto& j : jobs) s.max_kk = std::max(s.max_kk, j.kk);
        for (auto& j : jobs) {
            const double nc = j.nc < 0 ? 1.0 : j.nc;
            s.flops_per_col += 2.0 * j.r * j.kk * nc;
            s.bytes_per_col += 8.0 * (j.r * j.kk + (j.kk + 2.0 * j.r) * nc);
        }
        prog.push_back(s);
    }
    void lu(const std::vector<int>& units, bool partitions = false) {
        if (units.empty()) return;
        Stage s{ST_LU};
        s.partitions = partitions;
        s.njobs = (int)units.size();
        s.off = pb.push(units);
        for (int u : units) {
            const PartDev& P = f.parts[u];
            s.max_r = std::max(s.max_r, P.m);
            s.flops_per_col += 2.0 * P.m * P.kl * P.ubw;
            s.bytes_per_col += 16.0 * P.m * P.rows;
        }
        prog.push_back(s);
    }
    void cpl(const std::vector<CouplingJob>& jobs) {
        if (jobs.empty()) return;
        Stage s{ST_CPL};
        s.njobs = (int)jobs.size();
        s.off = pb.push(jobs);
        s.max_elems = (long long)(2 * f.k) * (4 * f.k - 1);
        prog.push_back(s);
    }
    void cjobs(StageType t, const std::vector<CouplingJob>& jobs) {
        if (jobs.empty()) return;
        Stage s{t};
        s.njobs = (int)jobs.size();
        s.off = pb.push(jobs);
        s.max_elems = (long long)f.k * (2 * f.k - 1);
        prog.push_back(s);
    }
    void memset_buf(int buf, int cols = -1) {
        Stage s{ST_MEMSET};
        s.buf = buf;
        s.cols = cols;
        prog.push_back(s);
    }
    void memcpy_fx() { prog.push_back(Stage{ST_MEMCPY_FX}); }
    void phase() { prog.push_back(Stage{ST_PHASE}); }
    void memcpy_fs() { prog.push_back(Stage{ST_MEMCPY_FS}); }
};

SweepJob sj(View v, int part, int mode, int lo, int hi, int c0 = 0, int nc = -1) {
    SweepJob j;
    j.v = v;
    j.part = part;
    j.mode = mode;
    j.lo = lo;
    j.hi = hi;
    j.c0 = c0;
    j.nc = nc;
    j.guard = -1;
    return j;
}

CopyJob cj(View src, View dst, int L0, int L1, int op = CP_COPY, int c0 = 0, int nc = -1) {
    CopyJob j;
    j.src = src;
    j.dst = dst;
    j.L0 = L0;
    j.L1 = L1;
    j.op = op;
    j.c0 = c0;
    j.nc = nc;
    j.guard = -1;
    return j;
}

GemmJob gj(View a, int transA, View b, int brow0, View c, int crow0, int r, int kk, int op,
           int nc = -1) {
    GemmJob j;
    j.a = a;
    j.b = b;
    j.c = c;
    j.transA = transA;
    j.brow0 = brow0;
    j.crow0 = crow0;
    j.r = r;
    j.kk = kk;
    j.nc = nc;
    j.op = op;
    j.guard = -1;
    return j;
}

// pair_solve (factorize.cpp:19-32) / pair_solve_transpose (:34-44) over a
// batch of z blocks (z = {buf, base row, ld}).  Two realisations per pair:
//  * generic: gather red = z[hL-k, hL+k) into its own region, solve with the
//    pivoted 2k coupling unit, two GEMM updates, scatter back;
//  * Schur (spk_coupling.cu): in place on z with the k x k unit S = I - W V:
//      forward   z2 -= W z1; z2 = S^-1 z2; z[0:hL] -= vl z2; z[hL+k:] -= wr[k:] z1
//      transpose z1 -= wr[k:]^T z[hL+k:]; z2 -= vl[0:hL-k]^T z[0:hL-k];
//                z2 -= V^T z1; z2 = S^-T z2; z1 -= W^T z2
// `path` bit 0 emits the generic jobs, bit 1 the Schur jobs; when both are
// emitted (factor time, before the path is known) the jobs carry guards.
struct PairZ {
    long long sinv;  // pool offset of S^-1 (Schur unit)
    int spart;  // Schur unit
    int gidx;   // flag index of the pair
    int pair_part;
    long long vl_off, wr_off;
    int hL, hR;
    int zbuf;
    long long zbase, zld;
    long long red_row;  // row offset of this job's 2k red region in redbuf
    int path;           // bit0 generic, bit1 Schur
};

template <class Jb>
Jb guarded_job(Jb j, const PairZ& z, int want) {
    j.guard = (z.path == 3) ? 2 * z.gidx + want : -1;
    return j;
}

void emit_pair_solves(Builder& b, const std::vector<PairZ>& zs, int redbuf, long long redld,
                      int ncols_explicit, bool transpose, int k) {
    if (zs.empty()) return;
    std::vector<CopyJob> gather, scatter, gsc;
    std::vector<SweepJob> s1, s2;
    std::vector<GemmJob> g, ga, gb, gd, ge, gs;
    const int nc = ncols_explicit;
    for (const PairZ& z : zs) {
        const View zv = view(z.zbuf, z.zbase, 0, 0, 0, z.zld);
        const int hL = z.hL, hR = z.hR;
        if (z.path & 1) {
            // red logical row L in [hL-k, hL+k) <-> red region row red_row + L - (hL-k)
            const View rv_z = view(redbuf, z.red_row, 0, hL - k, 0, redld);
            const View rv = view(redbuf, z.red_row, 0, 0, 2 * k, redld);
            gather.push_back(guarded_job(cj(zv, rv_z, hL - k, hL + k, CP_COPY, 0, nc), z, 0));
            scatter.push_back(guarded_job(cj(rv_z, zv, hL - k, hL + k, CP_COPY, 0, nc), z, 0));
            const View vl = view(B_POOL, z.vl_off, 0, 0, 0, hL);
            const View wr = view(B_POOL, z.wr_off + k, 0, 0, 0, hR);  // rows k.. of wr
            if (!transpose) {
                s1.push_back(guarded_job(sj(rv, z.pair_part, SW_FWD_L, 0, 0, 0, nc), z, 0));
                s2.push_back(guarded_job(sj(rv, z.pair_part, SW_BWD_U, 0, 2 * k - 1, 0, nc), z, 0));
                if (hL - k > 0) g.push_back(guarded_job(gj(vl, 0, rv, k, zv, 0, hL - k, k, GM_SUB, nc), z, 0));
                if (hR - k > 0) g.push_back(guarded_job(gj(wr, 0, rv, 0, zv, hL + k, hR - k, k, GM_SUB, nc), z, 0));
            } else {
                if (hR - k > 0) g.push_back(guarded_job(gj(wr, 1, zv, hL + k, rv, 0, k, hR - k, GM_SUB, nc), z, 0));
                if (hL - k > 0) g.push_back(guarded_job(gj(vl, 1, zv, 0, rv, k, k, hL - k, GM_SUB, nc), z, 0));
                s1.push_back(guarded_job(sj(rv, z.pair_part, SW_FWD_UT, 0, 0, 0, nc), z, 0));
                s2.push_back(guarded_job(sj(rv, z.pair_part, SW_BWD_LT, 0, 0, 0, nc), z, 0));
            }
        }
        if (z.path & 2) {
            const View z2 = view(z.zbuf, z.zbase + hL, 0, 0, k, z.zld);  // rows [hL, hL+k)
            const View W = view(B_POOL, z.wr_off, 0, 0, 0, hR);            // wr[0:k]
            const View Wk = view(B_POOL, z.wr_off + k, 0, 0, 0, hR);       // wr[k:hR]
            const View V = view(B_POOL, z.vl_off + hL - k, 0, 0, 0, hL);   // vl[hL-k:hL]
            const View Vt = view(B_POOL, z.vl_off, 0, 0, 0, hL);           // vl[0:hL-k]
            // z2 = S^-1 z2 (S^-T z2): GEMM into the pair's red region, copied back
            const View Si = view(B_POOL, z.sinv, 0, 0, 0, k);
            const View red = view(redbuf, z.red_row, 0, 0, 2 * k, redld);
            gs.push_back(guarded_job(gj(Si, transpose ? 1 : 0, zv, hL, red, 0, k, k, GM_SET, nc), z, 1));
            gsc.push_back(guarded_job(cj(red, z2, 0, k, CP_COPY, 0, nc), z, 1));
            if (!transpose) {
                ga.push_back(guarded_job(gj(W, 0, zv, hL - k, zv, hL, k, k, GM_SUB, nc), z, 1));
                gd.push_back(guarded_job(gj(V, 0, zv, hL, zv, hL - k, k, k, GM_SUB, nc), z, 1));
                if (hL - k > 0) ge.push_back(guarded_job(gj(Vt, 0, zv, hL, zv, 0, hL - k, k, GM_SUB, nc), z, 1));
                if (hR - k > 0) ge.push_back(guarded_job(gj(Wk, 0, zv, hL - k, zv, hL + k, hR - k, k, GM_SUB, nc), z, 1));
            } else {
                if (hR - k > 0) ga.push_back(guarded_job(gj(Wk, 1, zv, hL + k, zv, hL - k, k, hR - k, GM_SUB, nc), z, 1));
                if (hL - k > 0) ga.push_back(guarded_job(gj(Vt, 1, zv, 0, zv, hL, k, hL - k, GM_SUB, nc), z, 1));
                gb.push_back(guarded_job(gj(V, 1, zv, hL - k, zv, hL, k, k, GM_SUB, nc), z, 1));
                ge.push_back(guarded_job(gj(W, 1, zv, hL, zv, hL - k, k, k, GM_SUB, nc), z, 1));
            }
        }
    }
    // generic path
    b.copy(gather);
    if (!transpose) {
        b.sweep(s1);
        b.sweep(s2);
        b.gemm(g);
    } else {
        b.gemm(g);
        b.sweep(s1);
        b.sweep(s2);
    }
    b.copy(scatter);
    // Schur path
    if (!transpose) {
        b.gemm(ga);
        b.gemm(gs);
        b.copy(gsc);
        b.gemm(gd);
        b.gemm(ge);
    } else {
        b.gemm(ga);
        b.gemm(gb);
        b.gemm(gs);
        b.copy(gsc);
        b.gemm(ge);
    }
}

// ---------------------------------------------------------------------------
// factor program (factorize.cpp:133-257 + reduce_factorize :46-120)
void build_factor_program(spk_fact& f, ProgramBuilder& pb) {
    Builder b{f, pb, f.prog_factor};
    Builder bl{f, pb, f.prog_levels};
    const int p = f.p, k = f.k;
    const long long n = f.n, kk = (long long)k * k;
    if (!f.reduced_only) {
        std::vector<int> units(p);
        for (int i = 0; i < p; ++i) units[i] = i;
        b.lu(units, true);  // register-window LU from the band, or fill + generic LU
        b.transpose_factors();
    }
    if (!f.coupled()) return;
    if (!f.reduced_only) {
        // spike right-hand sides in FS (n x 2k): V = [0; bhat], W = [chat; 0]
        b.memset_buf(B_FS, 2 * k);
        std::vector<CopyJob> init;
        std::vector<SweepJob> fl, bu;
        std::vector<CopyJob> tips;
        for (int i = 0; i < p; ++i) {
            const PartDev& P = f.parts[i];
            const int m = P.m;
            const long long r0 = f.bounds[i];
            const bool first = f.first(i), last = f.last(i);  // open edges act as inner partitions
            const View fsv = view(B_FS, r0, 0, 0, m, n);
            const View fsr = view(B_FS, r0, P.rev, 0, m, n);
            const View fsw = view(B_FS, r0 + (long long)k * n, 0, 0, m, n);  // W columns
            if (!last) {
                const View bh = view(B_POOL, f.off_bhat + i * kk, 0, m - k, k, k);
                init.push_back(cj(bh, fsv, m - k, m, CP_COPY, 0, k));
            }
            if (!first && !last) {
                const View ch = view(B_POOL, f.off_chat + i * kk, 0, 0, k, k);
                init.push_back(cj(ch, fsw, 0, k, CP_COPY, 0, k));
            }
            if (last) {
                // [0; rev chat] in reversed space == chat in physical rows [0, k)
                const View ch = view(B_POOL, f.off_chat + i * kk, 0, 0, k, k);
                init.push_back(cj(ch, fsv, 0, k, CP_COPY, 0, k));
            }
            const View vv = last ? fsr : fsv;
            fl.push_back(sj(vv, i, SW_FWD_L, P.trunc, 0, 0, k));
            if (!first && !last) {
                fl.push_back(sj(fsv, i, SW_FWD_L, 0, 0, k, k));
                bu.push_back(sj(fsv, i, SW_BWD_U, 0, m - 1, 0, 2 * k));
            } else {
                bu.push_back(sj(vv, i, SW_BWD_U, m - k, m - 1, 0, k));
            }
            // tips into level-0 spike columns (2k x k, ld 2k)
            const Level& l0 = f.levels[0];
            if (!last) {
                const View vdst_b = view(B_POOL, l0.voff[i] + k, 0, m - k, k, 2 * k);
                tips.push_back(cj(fsv, vdst_b, m - k, m, CP_COPY, 0, k));
                if (!first) {
                    const View vdst_t = view(B_POOL, l0.voff[i], 0, 0, k, 2 * k);
                    tips.push_back(cj(fsv, vdst_t, 0, k, CP_COPY, 0, k));
                }
            }
            if (!first) {
                const View wdst_t = view(B_POOL, l0.woff[i], 0, 0, k, 2 * k);
                if (last) {
                    tips.push_back(cj(fsv, wdst_t, 0, k, CP_COPY, 0, k));
                } else {
                    tips.push_back(cj(fsw, wdst_t, 0, k, CP_COPY, 0, k));
                    const View wdst_b = view(B_POOL, l0.woff[i] + k, 0, m - k, k, 2 * k);
                    tips.push_back(cj(fsw, wdst_b, m - k, m, CP_COPY, 0, k));
                }
            }
        }
        b.copy(init);
        b.sweep(fl);
        b.sweep(bu);
        b.copy(tips);
    }
    // reduced hierarchy: per level, both coupling paths guarded by the
    // device-side per-pair flag (Schur when max|W| <= 1 and S is nonsingular)
    const int L = (int)f.levels.size() - 1;
    const bool schur_ok = k <= 160;
    const int both = schur_ok ? 3 : 1;
    long long red_cursor = 0;
    for (int l = 0; l < L; ++l) {
        const Level& lv = f.levels[l];
        const int np = lv.units / 2;
        std::vector<CouplingJob> cplS, cplG;
        std::vector<GemmJob> sgemm;
        std::vector<int> lus;
        for (int a = 0; a < np; ++a) {
            CouplingJob c;
            c.vl_off = lv.voff[2 * a];
            c.wr_off = lv.woff[2 * a + 1];
            c.hL = lv.uh[2 * a];
            c.hR = lv.uh[2 * a + 1];
            c.k = k;
            c.guard = lv.gidx[a];
            c.pad = 0;
            c.aux = -1;
            c.part = lv.pair_part[a];
            cplG.push_back(c);
            lus.push_back(lv.pair_part[a]);
            if (schur_ok) {
                c.part = lv.spart[a];
                cplS.push_back(c);
                const PartDev& S = f.parts[lv.spart[a]];
                const View Sv = view(B_FAC, S.fofs + (k - 1), 0, 0, 0, S.rows - 1);  // dense k x k
                const View W = view(B_POOL, c.wr_off, 0, 0, 0, c.hR);
                const View V = view(B_POOL, c.vl_off, 0, 0, 0, c.hL);
                GemmJob gjb = gj(W, 0, V, c.hL - k, Sv, 0, k, k, GM_SUB, k);
                gjb.guard = 2 * lv.gidx[a] + 1;
                sgemm.push_back(gjb);
            }
        }
        if (schur_ok) {
            bl.cjobs(ST_WCHECK, cplS);
            bl.cjobs(ST_SCHUR_INIT, cplS);
            bl.gemm(sgemm);
            for (int a = 0; a < np; ++a) cplS[a].aux = lv.sinv[a];
            bl.cjobs(ST_SCHUR_INV, cplS);  // S^-1 into the pool (S stays in the factor pool)
        }
        bl.cpl(cplG);
        bl.lu(lus);
        const Level& nx = f.levels[l + 1];
        std::vector<CopyJob> init;
        std::vector<PairZ> zs;
        for (int a = 0; a < np; ++a) {
            const int hL = lv.uh[2 * a], hR = lv.uh[2 * a + 1], H = hL + hR;
            if (nx.voff[a] >= 0) {
                const View src = view(B_POOL, lv.voff[2 * a + 1], 0, hL, hR, hR);
                const View dst = view(B_POOL, nx.voff[a], 0, 0, H, H);
                init.push_back(cj(src, dst, hL, H, CP_COPY, 0, k));
                zs.push_back(PairZ{lv.sinv[a], lv.spart[a], lv.gidx[a], lv.pair_part[a], lv.voff[2 * a],
                                   lv.woff[2 * a + 1], hL, hR, B_POOL, nx.voff[a], H, red_cursor, both});
                red_cursor += 2 * k;
            }
            if (nx.woff[a] >= 0) {
                const View src = view(B_POOL, lv.woff[2 * a], 0, 0, hL, hL);
                const View dst = view(B_POOL, nx.woff[a], 0, 0, H, H);
                init.push_back(cj(src, dst, 0, hL, CP_COPY, 0, k));
                zs.push_back(PairZ{lv.sinv[a], lv.spart[a], lv.gidx[a], lv.pair_part[a], lv.voff[2 * a],
                                   lv.woff[2 * a + 1], hL, hR, B_POOL, nx.woff[a], H, red_cursor, both});
                red_cursor += 2 * k;
            }
        }
        if (lv.units % 2 == 1) {
            // carried unit: its spikes move up unchanged
            const int h = lv.uh[lv.units - 1];
            if (lv.woff[lv.units - 1] >= 0) {
                const View src = view(B_POOL, lv.woff[lv.units - 1], 0, 0, h, h);
                const View dst = view(B_POOL, nx.woff[np], 0, 0, h, h);
                init.push_back(cj(src, dst, 0, h, CP_COPY, 0, k));
            }
            if (lv.voff[lv.units - 1] >= 0) {
                const View src = view(B_POOL, lv.voff[lv.units - 1], 0, 0, h, h);
                const View dst = view(B_POOL, nx.voff[np], 0, 0, h, h);
                init.push_back(cj(src, dst, 0, h, CP_COPY, 0, k));
            }
        }
        bl.copy(init);
        emit_pair_solves(bl, zs, B_AUX, -1, k, false, k);
    }
    f.auxf_rows = std::max<long long>(red_cursor, 1);
}

// ---------------------------------------------------------------------------
// forward solve program (solve.cpp:81-223)
void build_reduced_solve(spk_fact& f, Builder& b, bool transpose, long long aux_base) {
    const int L = (int)f.levels.size() - 1;
    const int k = f.k;
    long long cur = aux_base;
    std::vector<long long> level_base(L);
    for (int l = 0; l < L; ++l) {
        level_base[l] = cur;
        cur += (long long)(f.levels[l].units / 2) * 2 * k;
    }
    for (int s = 0; s < L; ++s) {
        const int l = transpose ? L - 1 - s : s;
        const Level& lv = f.levels[l];
        std::vector<PairZ> zs;
        for (int a = 0; a < lv.units / 2; ++a)
            zs.push_back(PairZ{lv.sinv[a], lv.spart[a], lv.gidx[a], lv.pair_part[a], lv.voff[2 * a],
                               lv.woff[2 * a + 1], lv.uh[2 * a], lv.uh[2 * a + 1], B_T, (long long)lv.uoff[2 * a], -1,
                               level_base[l] + 2LL * k * a,
                               // paths unknown (factorization still running): both, device-guarded
                               f.flags.empty() ? (k <= 160 ? 3 : 1) : (f.flags[lv.gidx[a]] ? 2 : 1)});
        emit_pair_solves(b, zs, B_AUX, -1, -1, transpose, k);
    }
}

// Slab exchange (open edges): T rows [0, k) / [H-k, H) are the slab's top and
// bottom tips, H = 2pk; T has k halo rows on each side, [-k, 0) holding the
// left neighbour's bottom tip and [H, H+k) the right neighbour's top tip.
// Export / import blocks are column-major with ld = their row count.
void emit_unit_correction(spk_fact& f, Builder& b) {
    // y -= V_unit xi + W_unit eta over the slab's reduced rows (two stages:
    // both update every row of T)
    const Level& top = f.levels[f.top_level()];
    const int H = top.uh[0], k = f.k;
    const View tview = view(B_T, 0);
    if (top.voff[0] >= 0) b.gemm({gj(view(B_POOL, top.voff[0], 0, 0, 0, H), 0, tview, H, tview, 0, H, k, GM_SUB)});
    if (top.woff[0] >= 0) b.gemm({gj(view(B_POOL, top.woff[0], 0, 0, 0, H), 0, tview, -k, tview, 0, H, k, GM_SUB)});
}

void build_forward_program(spk_fact& f, ProgramBuilder& pb) {
    Builder b{f, pb, f.prog_fwd};
    const int p = f.p, k = f.k;
    const long long kk = (long long)k * k;
    b.memcpy_fx();
    std::vector<SweepJob> s_fl, s_bu;
    if (!f.coupled()) {
        for (int i = 0; i < p; ++i) {
            const PartDev& P = f.parts[i];
            const View xv = view(B_X, f.bounds[i], P.rev, 0, P.m);
            s_fl.push_back(sj(xv, i, SW_FWD_L, 0, 0));
            s_bu.push_back(sj(xv, i, SW_BWD_U, 0, P.m - 1));
        }
        b.sweep(s_fl);
        b.sweep(s_bu);
        return;
    }
    std::vector<CopyJob> c_edge, c_inner;
    for (int i = 0; i < p; ++i) {
        const PartDev& P = f.parts[i];
        const int m = P.m;
        const long long r0 = f.bounds[i];
        const View xv = view(B_X, r0, P.rev, 0, m);
        s_fl.push_back(sj(xv, i, SW_FWD_L, 0, 0));
        if (f.first(i)) {
            const View tv = view(B_T, k, 0, m - k, k);
            c_edge.push_back(cj(xv, tv, m - k, m));
            s_bu.push_back(sj(tv, i, SW_BWD_U, m - k, m - 1));
        } else if (f.last(i)) {
            const View tv = view(B_T, 2LL * i * k, 1, m - k, k);
            c_edge.push_back(cj(xv, tv, m - k, m));
            s_bu.push_back(sj(tv, i, SW_BWD_U, m - k, m - 1));
        } else {
            s_bu.push_back(sj(xv, i, SW_BWD_U, 0, m - 1));
            c_inner.push_back(cj(xv, view(B_T, 2LL * i * k, 0, 0, k), 0, k));
            c_inner.push_back(cj(xv, view(B_T, (2LL * i + 1) * k, 0, m - k, k), m - k, m));
        }
    }
    b.sweep(s_fl);
    b.copy(c_edge);
    b.sweep(s_bu);
    b.copy(c_inner);
    build_reduced_solve(f, b, false, 0);
    if (f.open()) {
        // export [y_top; y_bot]; import [xi; eta] = [right neighbour's x_top;
        // left neighbour's x_bot] from the slab-level reduced solve
        const int H = 2 * p * k;
        b.copy({cj(view(B_T, 0), view(B_XCH, 0), 0, k), cj(view(B_T, 0), view(B_XCH, 2 * k - H), H - k, H)});
        b.phase();
        std::vector<CopyJob> imp;
        if (f.open_r) imp.push_back(cj(view(B_XIN, -H), view(B_T, 0), H, H + k));
        if (f.open_l) imp.push_back(cj(view(B_XIN, 2 * k), view(B_T, 0), -k, 0));
        b.copy(imp);
        emit_unit_correction(f, b);
    }
    // retrieval (solve.cpp:180-223): x_i = A_i^-1 (f_i - C_i eta - B_i xi), solved
    // again from F with corrected tip rows (X = F, X[tips] -= corner products,
    // then the full L and U sweeps): no correction buffer, no memset, no
    // X -= S pass; the D-stage result Y was only needed for its tips
    b.memcpy_fx();
    std::vector<GemmJob> g;
    std::vector<SweepJob> r_fl, r_bu;
    const View tview = view(B_T, 0);
    for (int i = 0; i < p; ++i) {
        const PartDev& P = f.parts[i];
        const int m = P.m;
        const long long r0 = f.bounds[i];
        const View xp = view(B_X, r0, 0, 0, m);      // physical rows
        const View xv = view(B_X, r0, P.rev, 0, m);  // LU space (reversed for the UL partition)
        const View bh = view(B_POOL, f.off_bhat + i * kk, 0, 0, 0, k);
        const View ch = view(B_POOL, f.off_chat + i * kk, 0, 0, 0, k);
        if (!f.last(i)) g.push_back(gj(bh, 0, tview, 2 * (i + 1) * k, xp, m - k, k, k, GM_SUB));
        if (!f.first(i)) g.push_back(gj(ch, 0, tview, (2 * i - 1) * k, xp, 0, k, k, GM_SUB));
        r_fl.push_back(sj(xv, i, SW_FWD_L, 0, 0));
        r_bu.push_back(sj(xv, i, SW_BWD_U, 0, m - 1));
    }
    b.gemm(g);
    b.sweep(r_fl);
    b.sweep(r_bu);
}

// transpose solve program (solve.cpp:225-380)
void build_transpose_program(spk_fact& f, ProgramBuilder& pb) {
    Builder b{f, pb, f.prog_tr};
    const int p = f.p, k = f.k;
    const long long kk = (long long)k * k;
    b.memcpy_fx();
    if (!f.coupled()) {
        std::vector<SweepJob> a, c;
        for (int i = 0; i < p; ++i) {
            const PartDev& P = f.parts[i];
            const View xv = view(B_X, f.bounds[i], P.rev, 0, P.m);
            a.push_back(sj(xv, i, SW_FWD_UT, 0, 0));
            c.push_back(sj(xv, i, SW_BWD_LT, 0, 0));
        }
        b.sweep(a);
        b.sweep(c);
        return;
    }
    b.memcpy_fs();
    const long long red_rows = (long long)(p - 1) * 2 * k;
    std::vector<CopyJob> zero, tau_copy, gcopy, d_copy, d_add;
    std::vector<SweepJob> s_fut, s_blt, tau_blt, d_fut, d_blt;
    std::vector<GemmJob> g;
    for (int i = 0; i < p; ++i) {
        const PartDev& P = f.parts[i];
        const int m = P.m;
        const long long r0 = f.bounds[i];
        const View sv = view(B_S, r0, 0, 0, m);
        const View xv = view(B_X, r0, P.rev, 0, m);
        if (f.first(i) || f.last(i)) {
            const bool last = f.last(i);
            zero.push_back(cj(xv, xv, m - k, m, CP_ZERO));
            s_fut.push_back(sj(xv, i, SW_FWD_UT, 0, 0));
            const int w = std::min(m, k + (f.piv_on ? P.kl : 0));
            const long long taoff = red_rows + (last ? f.tau_w : 0);
            const View av = view(B_AUX, taoff, 0, m - w, w);
            tau_copy.push_back(cj(xv, av, m - w, m));
            tau_blt.push_back(sj(av, i, SW_BWD_LT, m - w, 0));
            // D^T stage: z = U_tail^-T tip, X_tail += z, full P^T L^-T
            const long long zoff = red_rows + 2LL * f.tau_w + (last ? k : 0);
            const View zv = view(B_AUX, zoff, 0, m - k, k);
            const View tip = last ? view(B_T, 2LL * i * k, 1, m - k, k) : view(B_T, k, 0, m - k, k);
            d_copy.push_back(cj(tip, zv, m - k, m));
            d_fut.push_back(sj(zv, i, SW_FWD_UT, m - k, 0));
            d_add.push_back(cj(zv, xv, m - k, m, CP_ADD));
            d_blt.push_back(sj(xv, i, SW_BWD_LT, 0, 0));
        } else {
            zero.push_back(cj(sv, sv, 0, k, CP_ZERO));
            zero.push_back(cj(sv, sv, m - k, m, CP_ZERO));
            s_fut.push_back(sj(sv, i, SW_FWD_UT, 0, 0));
            s_blt.push_back(sj(sv, i, SW_BWD_LT, 0, 0));
            d_copy.push_back(cj(view(B_T, 2LL * i * k, 0, 0, k), xv, 0, k));
            d_copy.push_back(cj(view(B_T, (2LL * i + 1) * k, 0, m - k, k), xv, m - k, m));
            d_fut.push_back(sj(xv, i, SW_FWD_UT, 0, 0));
            d_blt.push_back(sj(xv, i, SW_BWD_LT, 0, 0));
        }
    }
    // G tips (solve.cpp:313-325): boundary rows of F minus corner^T * tau
    const View fg = view(B_F, 0);
    for (int i = 0; i < p; ++i) {
        const long long b0 = f.bounds[i], b1 = f.bounds[i + 1];
        gcopy.push_back(cj(fg, view(B_T, 2LL * i * k, 0, (int)b0, k), (int)b0, (int)b0 + k));
        gcopy.push_back(cj(fg, view(B_T, (2LL * i + 1) * k, 0, (int)(b1 - k), k), (int)(b1 - k), (int)b1));
    }
    const View tview = view(B_T, 0);
    // where tau lives: the whole partition in S (inner), the tip rows in AUX
    // (closed first: bottom, closed last: top, in reversed space)
    auto tau_b = [&](int i) {  // view whose rows [m-k, m) are tau_b(i)
        const PartDev& Q = f.parts[i];
        if (f.first(i)) {
            const int w = std::min(Q.m, k + (f.piv_on ? Q.kl : 0));
            return view(B_AUX, red_rows, 0, Q.m - w, w);
        }
        return view(B_S, f.bounds[i], 0, 0, Q.m);
    };
    auto tau_t = [&](int i) {  // view whose rows [0, k) are tau_t(i)
        const PartDev& Q = f.parts[i];
        if (f.last(i)) {
            const int w = std::min(Q.m, k + (f.piv_on ? Q.kl : 0));
            return view(B_AUX, red_rows + f.tau_w, 1, 0, w);
        }
        return view(B_S, f.bounds[i], 0, 0, Q.m);
    };
    for (int i = 1; i < p; ++i) {
        // tip_t(i) -= bhat_{i-1}^T tau_b(i-1)
        const View bh = view(B_POOL, f.off_bhat + (i - 1) * kk, 0, 0, 0, k);
        g.push_back(gj(bh, 1, tau_b(i - 1), f.parts[i - 1].m - k, tview, 2 * i * k, k, k, GM_SUB));
    }
    for (int i = 0; i + 1 < p; ++i) {
        // tip_b(i) -= chat_{i+1}^T tau_t(i+1)
        const View ch = view(B_POOL, f.off_chat + (i + 1) * kk, 0, 0, 0, k);
        g.push_back(gj(ch, 1, tau_t(i + 1), 0, tview, (2 * i + 1) * k, k, k, GM_SUB));
    }
    b.copy(zero);
    b.sweep(s_fut);
    b.copy(tau_copy);
    for (const SweepJob& j : tau_blt) s_blt.push_back(j);  // one launch with the inner sweeps
    b.sweep(s_blt);
    b.copy(gcopy);
    b.gemm(g);
    if (f.open()) {
        // exchange 1: the neighbours' G-tip terms across the slab edges.
        // export [chat_0^T tau_t(0); bhat_{p-1}^T tau_b(p-1)], import
        // [left neighbour's bhat^T tau_b; right neighbour's chat^T tau_t]
        const int H = 2 * p * k;
        b.memset_buf(B_XCH);
        std::vector<GemmJob> ex;
        if (f.open_l)
            ex.push_back(gj(view(B_POOL, f.off_chat, 0, 0, 0, k), 1, tau_t(0), 0, view(B_XCH, 0), 0, k, k, GM_SET));
        if (f.open_r)
            ex.push_back(gj(view(B_POOL, f.off_bhat + (p - 1) * kk, 0, 0, 0, k), 1, tau_b(p - 1), f.parts[p - 1].m - k,
                            view(B_XCH, 0), k, k, k, GM_SET));
        b.gemm(ex);
        b.phase();
        std::vector<CopyJob> imp;
        if (f.open_l) imp.push_back(cj(view(B_XIN, 0), tview, 0, k, CP_SUB));
        if (f.open_r) imp.push_back(cj(view(B_XIN, 2 * k - H), tview, H - k, H, CP_SUB));
        b.copy(imp);
        // exchange 2: slab-level transposed reduced system.  export [t_top;
        // t_bot; V_int^T t_int; W_int^T t_int], import [z_top; z_bot]
        b.memset_buf(B_XCH);
        b.copy({cj(tview, view(B_XCH, 0), 0, k), cj(tview, view(B_XCH, 2 * k - H), H - k, H)});
        const Level& top = f.levels[f.top_level()];
        std::vector<GemmJob> proj;
        if (H > 2 * k) {
            if (top.voff[0] >= 0)
                proj.push_back(gj(view(B_POOL, top.voff[0] + k, 0, 0, 0, H), 1, tview, k, view(B_XCH, 0), 2 * k, k,
                                  H - 2 * k, GM_SET));
            if (top.woff[0] >= 0)
                proj.push_back(gj(view(B_POOL, top.woff[0] + k, 0, 0, 0, H), 1, tview, k, view(B_XCH, 0), 3 * k, k,
                                  H - 2 * k, GM_SET));
        }
        b.gemm(proj);
        b.phase();
        b.copy({cj(view(B_XIN, 0), tview, 0, k), cj(view(B_XIN, 2 * k - H), tview, H - k, H)});
    }
    build_reduced_solve(f, b, true, 0);
    b.copy(d_copy);
    b.sweep(d_fut);
    b.copy(d_add);
    b.sweep(d_blt);
}

// ---------------------------------------------------------------------------
// execution
struct Exec {
    spk_fact& f;
    cudaStream_t s;
    Bufs B;
    int ncols;
    // memcpy sources
    const double* F = nullptr;
    long long ldf = 0, n = 0;
    const double* band = nullptr;  // factorization input (device)
    long long band_cols = 0, band_col0 = 0;  // its readable columns: [-band_col0, band_cols - band_col0)
    bool lu_fast_done = false;

    bool run_fast_sweep(const Stage& st, const SweepJob* jobs, int nc) {
        if (nc <= 0) return true;
        if (st.piv && f.lblk_ok) {
            // pivoted forward / transposed L sweeps, 8 rows per step on the
            // tensor cores from the LU's blocked records: <= 16 warps x 8
            // columns per CTA
            const int groups = (nc + 127) / 128;
            const int cols = ((nc + groups - 1) / groups + 7) / 8 * 8;
            const dim3 grid(st.njobs, (nc + cols - 1) / cols);
            PivSweepArgs A{jobs, f.d_parts, f.d_lblk, B, ncols, f.d_fac, f.d_piv};
            if (st.mode == SW_FWD_L ? launch_sweep_piv_dmma(f.lblk_trw, cols / 8, grid, A, s)
                                    : launch_sweep_piv_dmma_t(f.lblk_trw, cols / 8, grid, A, s))
                return true;
        }
        // pivoted transposed sweeps have no register-window kernel
        if (st.piv && st.mode == SW_BWD_LT) return false;
        // narrow solves (<= 8 right-hand sides): the producer/consumer sweep
        // with the window split over a pair of warps (k_sweep_dmma2<..., PAIR>).
        // Measured: narrow solves gain at every bandwidth; wider ones were
        // slower paired (C2's 64/128-column factor sweeps, C5's 32-column
        // solves, C3)
        constexpr int pair_maxnc = 8;
        if (!st.piv && nc <= pair_maxnc && st.kwmax >= 8 && st.kwmax <= 192) {
            static const int ntws[] = {3, 5, 9, 13, 17, 21, 25};
            int ntw = 0;
            for (int t : ntws)
                if (8 * (t - 1) >= st.kwmax) {
                    ntw = t;
                    break;
                }
            FastSweepArgs A{jobs, f.d_parts, f.d_fac, f.d_tfac, f.d_dinv, f.d_piv, B, ncols};
            const int groups = (nc + 55) / 56;  // <= 7 pairs per CTA (16 warps with the producers: launch bound 512)
            const int cols = ((nc + groups - 1) / groups + 7) / 8 * 8;
            const int ncw = 2 * (cols / 8);  // one warp pair per 8 columns
            const dim3 grid(st.njobs, (nc + cols - 1) / cols);
            bool ok = false;
            switch (st.mode) {
                case SW_FWD_L: ok = launch_sweep_dmma2_fl(ntw, ncw, grid, A, s, true); break;
                case SW_BWD_U: ok = launch_sweep_dmma2_bu(ntw, ncw, grid, A, s, true); break;
                case SW_FWD_UT: ok = launch_sweep_dmma2_fut(ntw, ncw, grid, A, s, true); break;
                default: ok = launch_sweep_dmma2_blt(ntw, ncw, grid, A, s, true); break;
            }
            if (ok) return true;
        }
        // producer/consumer DMMA sweep (spk_sweep_dmma2.cuh): <= 14 compute warps
        // (8 columns each) + 2 producer warps per CTA.  Taken when it needs no
        // more column groups than the 16-warp kernel below (each group re-reads
        // the factor) and keeps >= 6 compute warps busy (with fewer, one warp's
        // dependency chain sets the pace and the synchronous kernel wins).
        const int groups2 = (nc + 111) / 112, groups1 = (nc + 127) / 128;
        const int cols2 = ((nc + groups2 - 1) / groups2 + 7) / 8 * 8;
        if (!st.piv && nc >= 8 && st.kwmax <= 192 && groups2 == groups1 && cols2 >= 48) {
            static const int ntws[] = {3, 5, 9, 13, 17, 21, 25};
            int ntw = 0;
            for (int t : ntws)
                if (8 * (t - 1) >= st.kwmax) {
                    ntw = t;
                    break;
                }
            const int cols = cols2;
            const dim3 grid(st.njobs, (nc + cols - 1) / cols);
            FastSweepArgs A{jobs, f.d_parts, f.d_fac, f.d_tfac, f.d_dinv, f.d_piv, B, ncols};
            bool ok = false;
            switch (st.mode) {
                case SW_FWD_L: ok = launch_sweep_dmma2_fl(ntw, cols / 8, grid, A, s); break;
                case SW_BWD_U: ok = launch_sweep_dmma2_bu(ntw, cols / 8, grid, A, s); break;
                case SW_FWD_UT: ok = launch_sweep_dmma2_fut(ntw, cols / 8, grid, A, s); break;
                default: ok = launch_sweep_dmma2_blt(ntw, cols / 8, grid, A, s); break;
            }
            if (ok) return true;
        }
        if (!st.piv && st.kwmax <= 192) {
            // blocked tensor-core sweep: 8 columns per warp, <= 16 warps per CTA,
            // column groups balanced across CTAs.  Narrow solves (nc < 8) run
            // padded to one warp: the chain per 8-row block (~4 DMMA latencies)
            // beats the per-row chain of the DFMA kernel ~10x, and the tensor
            // pipe has room for the padding
            static const int ntws[] = {3, 5, 9, 13, 17, 21, 25};
            int ntw = 0;
            for (int t : ntws)
                if (8 * (t - 1) >= st.kwmax) {
                    ntw = t;
                    break;
                }
            // 9..32 columns: warp pairs per 8 columns (the window split; a warp
            // issues at most one DMMA per ~32 cycles)
            const bool pair = ntw >= 9 && nc > 8 && nc <= 32;
            const int groups = pair ? (nc + 63) / 64 : (nc + 127) / 128;  // <= 16 warps per CTA
            const int cols = ((nc + groups - 1) / groups + 7) / 8 * 8;
            const int nwd = (pair ? 2 : 1) * (cols / 8);
            const dim3 grid(st.njobs, (nc + cols - 1) / cols);
            const size_t smem = dmma_sweep_smem(ntw, nwd, pair);
            FastSweepArgs A{jobs, f.d_parts, f.d_fac, f.d_tfac, f.d_dinv, f.d_piv, B, ncols};
            if (smem <= 227 * 1024) {
                bool ok = false;
                switch (st.mode) {
                    case SW_FWD_L: ok = launch_sweep_dmma_fl(ntw, nwd, grid, smem, A, s, pair); break;
                    case SW_BWD_U: ok = launch_sweep_dmma_bu(ntw, nwd, grid, smem, A, s, pair); break;
                    case SW_FWD_UT: ok = launch_sweep_dmma_fut(ntw, nwd, grid, smem, A, s, pair); break;
                    default: ok = launch_sweep_dmma_blt(ntw, nwd, grid, smem, A, s, pair); break;
                }
                if (ok) return true;
            }
        }
        int NC, nw;
        if (nc >= 64) {
            NC = 4;
            nw = std::min(20, (nc + 3) / 4);
        } else if (nc >= 8) {
            NC = 2;
            nw = std::min(16, (nc + 1) / 2);
        } else {
            NC = 1;
            nw = nc;
        }
        const dim3 grid(st.njobs, (nc + nw * NC - 1) / (nw * NC));
        const size_t smem = fast_sweep_smem(st.tr, nw, NC);
        if (smem > 227 * 1024) return false;
        FastSweepArgs A{jobs, f.d_parts, f.d_fac, f.d_tfac, f.d_dinv, f.d_piv, B, ncols};
        switch (st.mode) {
            case SW_FWD_L: return launch_sweep_fast_fl(st.tr, NC, st.piv, nw, grid, smem, A, s);
            case SW_BWD_U: return launch_sweep_fast_bu(st.tr, NC, false, nw, grid, smem, A, s);
            case SW_FWD_UT: return launch_sweep_fast_fut(st.tr, NC, false, nw, grid, smem, A, s);
            default: return launch_sweep_fast_blt(st.tr, NC, false, nw, grid, smem, A, s);
        }
    }

    // phase < 0: every stage; else only the stages between the phase-th and
    // (phase+1)-th ST_PHASE markers (the exchange points of a slab solve)
    void run(const Program& prog, const char* blob, int phase = -1) {
        int cur = 0;
        for (const Stage& st : prog) {
            if (st.t == ST_PHASE) {
                ++cur;
                continue;
            }
            if (phase >= 0 && cur != phase) continue;
            const char* jobs = blob + st.off;
            const double mult = st.max_nc < 0 ? ncols : 1.0;
            ProfScope ps((int)st.t, s, st.flops_per_col * mult, st.bytes_per_col * mult);
            switch (st.t) {
                case ST_SWEEP: {
                    const int nc = st.max_nc < 0 ? ncols : st.max_nc;
                    if (st.fast && run_fast_sweep(st, (const SweepJob*)jobs, nc)) break;
                    if (st.small_ch > 0 && !generic_path() &&
                        launch_sweep_small((const SweepJob*)jobs, st.njobs, nc, st.small_ch, st.small_rows, f.d_parts,
                                           f.d_fac, f.d_piv, B, ncols, s))
                        break;
                    if (st.partitions) ++g_generic_launches;
                    launch_sweep((const SweepJob*)jobs, st.njobs, nc, f.d_parts, f.d_fac, f.d_piv, B,
                                 ncols, s);
                    break;
                }
                case ST_TRANSPOSE: {
                    if (lu_fast_done) break;
                    long long mx = 0;
                    for (int i = 0; i < f.p; ++i) mx = std::max(mx, (long long)f.parts[i].m * f.parts[i].rowsT);
                    launch_transpose_factors(f.d_parts, f.p, mx, f.d_fac, f.d_tfac, f.d_dinv, s);
                    break;
                }
                case ST_COPY: {
                    const int nc = st.max_nc < 0 ? ncols : st.max_nc;
                    launch_copy((const CopyJob*)jobs, st.njobs, st.max_elems * nc, B, ncols, s);
                    break;
                }
                case ST_GEMM: {
                    const int nc = st.max_nc < 0 ? ncols : st.max_nc;
                    if (generic_path()) {
                        ++g_generic_launches;
                        launch_gemm((const GemmJob*)jobs, st.njobs, st.max_r, nc, B, ncols, s);
                    } else {
                        const int ns = gemm_splitk_factor(st.njobs, st.max_r, nc, st.max_kk);
                        if (ns > 1) {
                            double* ws = dalloc<double>(gemm_splitk_workspace(st.njobs, st.max_r, nc, ns), s);
                            launch_gemm_dmma((const GemmJob*)jobs, st.njobs, st.max_r, nc, B, ncols, s, ws, ns);
                            dfree(ws, s);
                        } else {
                            launch_gemm_dmma((const GemmJob*)jobs, st.njobs, st.max_r, nc, B, ncols, s);
                        }
                    }
                    break;
                }
                case ST_LU: {
                    if (st.partitions) {
                        const bool generic_only = generic_path();
                        const int kmax = std::max(f.kl, f.ku);
                        if (!f.piv_on && !generic_only && kmax <= 160) {
                            // the DMMA LU (k <= 160) writes the packed factor only; the
                            // row-major copy is made when a transposed solve needs it
                            // the DMMA LU (k <= 160) writes the row-major copy only
                            // where transposed solves have been seen for this shape;
                            // otherwise it is made on demand (ensure_tfac)
                            const bool wt = kmax <= 16 || f.want_tfac;
                            FastLuArgs A{(const int*)jobs, f.d_parts, band, f.kl, f.ku, f.d_fac,
                                         wt ? f.d_tfac : nullptr, f.d_dinv, f.d_piv, f.boost_eps, f.d_boost,
                                         band_cols, band_col0};
                            if (launch_band_lu_fast((const int*)jobs, st.njobs, kmax, A, s)) {
                                lu_fast_done = true;
                                if (!wt) f.tfac_ready.store(false);
                                break;
                            }
                        }
                        if (f.piv_on && !generic_only) {
                            // pivoted: blocked DMMA kernel (factor, pivots, row-major copy, 1/u_jj)
                            PivDmmaArgs A{(const int*)jobs, f.d_parts, band, f.kl, f.ku, f.d_fac,
                                          f.d_tfac, f.d_dinv, f.d_piv, f.d_status, f.d_lblk};
                            if (launch_band_lu_piv_dmma(st.njobs, f.kl, f.ku, A, s)) {
                                lu_fast_done = true;  // it writes the row-major copy and 1/u_jj too
                                f.lblk_ok = f.d_lblk != nullptr;
                                break;
                            }
                        }
                        if (f.piv_on && !generic_only) {
                            // pivoted: shared-memory window kernel (factor + pivots; the
                            // transpose stage then builds the row-major copy and 1/u_jj)
                            PivLuArgs A{(const int*)jobs, f.d_parts, band, f.kl, f.ku, f.d_fac, f.d_piv, f.d_status};
                            if (launch_band_lu_piv((const int*)jobs, st.njobs, f.kl, f.ku, A, s)) break;
                        }
                        long long max_elems = 0;
                        for (int i = 0; i < f.p; ++i)
                            max_elems = std::max(max_elems, (long long)f.parts[i].m * f.parts[i].rows);
                        launch_fill_factors(band, n, f.kl, f.ku, f.d_parts, f.p, max_elems, f.d_fac, f.d_piv,
                                            f.d_amax, s);
                    }
                    {
                        const bool generic_only = generic_path();
                        if (!st.partitions && !generic_only) {
                            // the pivoted 2k coupling units: blocked DMMA LU in place, then
                            // the shared-memory kernel redoes any unit with an exactly zero
                            // column (boosted non-pivoting fallback, kernels.cpp:67-77)
                            PivDmmaArgs A{(const int*)jobs, f.d_parts, nullptr, 0, 0, f.d_fac, nullptr, nullptr,
                                          f.d_piv, f.d_status, nullptr, f.d_flags, f.d_fell};
                            if (launch_dense_lu_piv_dmma(st.njobs, st.max_r, A, s) &&
                                launch_band_lu_small((const int*)jobs, st.njobs, st.max_r, f.d_parts, f.d_fac,
                                                     f.d_piv, f.d_amax, f.boost_eps, f.d_boost, f.d_fell,
                                                     f.d_status, f.d_flags, s, true))
                                break;
                        }
                        if (!generic_only && launch_band_lu_small((const int*)jobs, st.njobs, st.max_r, f.d_parts,
                                                              f.d_fac, f.d_piv, f.d_amax, f.boost_eps, f.d_boost,
                                                              f.d_fell, f.d_status, f.d_flags, s))
                            break;
                    }
                    if (st.partitions) ++g_generic_launches;
                    launch_band_lu((const int*)jobs, st.njobs, f.d_parts, f.d_fac, f.d_piv, f.d_amax,
                                   f.boost_eps, f.d_boost, f.d_fell, f.d_status, f.d_flags, s);
                    break;
                }
                case ST_CPL:
                    launch_build_coupling((const CouplingJob*)jobs, st.njobs, st.max_elems, f.d_parts,
                                          f.d_pool, f.d_fac, f.d_piv, f.d_amax, f.d_flags, s);
                    break;
                case ST_WCHECK:
                    launch_wcheck((const CouplingJob*)jobs, st.njobs, f.k, f.d_pool, f.d_flags, s);
                    break;
                case ST_SCHUR_INIT:
                    launch_schur_init((const CouplingJob*)jobs, st.njobs, st.max_elems, f.d_parts, f.d_fac,
                                      f.d_piv, f.d_flags, s);
                    break;
                case ST_SCHUR_INV:
                    if (!launch_schur_inverse((const CouplingJob*)jobs, st.njobs, f.k, f.d_parts, f.d_fac, f.d_pool,
                                              f.d_flags, s))
                        fail(SPK_EINVAL, "schur inverse: k > 160");
                    break;
                case ST_MEMSET: {
                    const int nc = st.cols < 0 ? ncols : st.cols;
                    if (B.p[st.buf] && nc > 0)
                        ck(cudaMemsetAsync(B.p[st.buf], 0, sizeof(double) * B.ld[st.buf] * nc, s), "memset");
                    break;
                }
                case ST_MEMCPY_FX:
                case ST_MEMCPY_FS: {
                    double* dst = st.t == ST_MEMCPY_FX ? B.p[B_X] : B.p[B_S];
                    const long long ldd = st.t == ST_MEMCPY_FX ? B.ld[B_X] : B.ld[B_S];
                    if (ncols > 0 && dst != B.p[B_F]) launch_copy_cols(B.p[B_F], B.ld[B_F], dst, ldd, n, ncols, s);
                    break;
                }
            }
        }
    }
};


void validate_plan(long long n, const spk_plan* plan) {
    if (!plan || plan->p < 1 || !plan->bounds) fail(SPK_EINVAL, "factorize: invalid plan");
    if (plan->bounds[0] != 0 || plan->bounds[plan->p] != n)
        fail(SPK_EINVAL, "factorize: plan does not match matrix");
    for (int i = 0; i < plan->p; ++i)
        if (plan->bounds[i + 1] - plan->bounds[i] < 1) fail(SPK_EINVAL, "factorize: empty partition");
}

}  // namespace

// Symbolic state of a factorization: everything that depends only on the
// shape, the plan and the options (geometry, pool layout, compiled programs),
// shared by repeated factorizations of the same structure.  Solve programs are
// cached per vector of coupling-path flags.  (Host program construction is
// ~8 ms at p = 1184: most of C1's factorization before this cache.)
struct SolveProgs {
    Program fwd, tr, rfwd, rtr;
    std::vector<char> blob;
};
struct Symbolic {
    std::vector<PartDev> parts;
    std::vector<Level> levels;
    long long off_bhat = 0, off_chat = 0, pool_size = 0, fac_size = 0, piv_size = 0, tfac_size = 0;
    long long aux_rows = 0, auxf_rows = 0;
    int tau_w = 0, npairs = 0;
    Program prog_factor, prog_levels;
    bool sk = false;
    size_t sk_units = 0, sk_pairs = 0, sk_items = 0, sk_levels = 0;
    int sk_nlevels = 0, sk_mmax = 0, sk_rmax = 0;
    std::vector<char> blob;
    std::map<std::vector<int>, SolveProgs> solves;
    // device copies of parts / bounds / blob for the small-k engine (one
    // upload per shape and device instead of one per factorization); kept
    // for the process lifetime of the cache entry
    struct DevTables {
        PartDev* parts = nullptr;
        long long* bounds = nullptr;
        char* blob = nullptr;
    };
    std::mutex dev_mu;
    std::map<int, DevTables> dev;
    // a transposed solve has run on a factorization of this shape: later
    // ones write the row-major copy inside their LU (instead of on demand)
    std::atomic<bool> want_tfac{false};
};

namespace {

struct SymCache {
    std::mutex mu;
    std::map<std::string, std::shared_ptr<Symbolic>> map;
};
SymCache& sym_cache() {
    static SymCache* c = new SymCache();
    return *c;
}
std::string sym_key(const spk_fact& f) {
    std::string key;
    auto put = [&](long long v) { key.append(reinterpret_cast<const char*>(&v), sizeof(v)); };
    for (long long v : {f.n, (long long)f.kl, (long long)f.ku, (long long)f.k, (long long)f.p, (long long)f.piv_on,
                        (long long)f.open_l, (long long)f.open_r, (long long)f.reduced_only,
                        (long long)generic_path()})
        put(v);
    for (long long b : f.bounds) put(b);
    return key;
}

void alloc_fact(spk_fact& f, cudaStream_t s, const std::vector<char>& blob);

// The small-k engine takes non-pivoting closed systems with kl, ku <= 16, at
// least two partitions, every partition at least 2k rows and short enough
// for its shared-memory staging (spk_smallk.cu).
constexpr int kSkMaxRows = 384;
bool sk_eligible(const spk_fact& f) {
    if (f.piv_on || f.open() || f.reduced_only || generic_path()) return false;
    if (f.kl > 16 || f.ku > 16 || f.k < 1 || f.p < 2) return false;
    for (int i = 0; i < f.p; ++i) {
        const long long m = f.bounds[i + 1] - f.bounds[i];
        if (m < 2LL * f.k || m > kSkMaxRows) return false;
    }
    return true;
}

// Level tables of the small-k engine (SkUnit / SkPair / SkItem / SkLevel, in
// the factor blob): units of every level with their pool offsets, pairs with
// their S^-1 slot, and per level the work items (pair, 32-row chunk of the
// merged unit; carried odd units).
void build_sk_tables(spk_fact& f, ProgramBuilder& pb) {
    std::vector<SkUnit> units;
    std::vector<SkPair> pairs;
    std::vector<SkItem> items;
    std::vector<SkLevel> lvls;
    std::vector<int> ubase;
    for (const Level& lv : f.levels) {
        ubase.push_back((int)units.size());
        for (int u = 0; u < lv.units; ++u) units.push_back(SkUnit{lv.voff[u], lv.woff[u], lv.uh[u], lv.uoff[u]});
    }
    const int L = (int)f.levels.size() - 1;
    for (int l = 0; l < L; ++l) {
        const Level& lv = f.levels[l];
        const int np = lv.units / 2, pbase = (int)pairs.size();
        SkLevel d{(int)items.size(), 0, pbase, np, -1, -1};
        if (lv.units % 2 == 1) {
            d.carry = ubase[l] + lv.units - 1;
            d.carry_next = ubase[l + 1] + np;
        }
        for (int a = 0; a < np; ++a) {
            const Level& nx = f.levels[l + 1];
            pairs.push_back(SkPair{lv.sinv[a], lv.voff[2 * a], lv.woff[2 * a], lv.voff[2 * a + 1], lv.woff[2 * a + 1],
                                   nx.voff[a], nx.woff[a], lv.uh[2 * a], lv.uh[2 * a + 1], lv.uoff[2 * a], lv.gidx[a],
                                   ubase[l] + 2 * a, ubase[l + 1] + a});
            const int H = lv.uh[2 * a] + lv.uh[2 * a + 1];
            for (int r = 0; r < H; r += kSkChunk) items.push_back(SkItem{pbase + a, r, -1, 0});
        }
        if (lv.units % 2 == 1) {
            const int u = lv.units - 1;
            for (int r = 0; r < lv.uh[u]; r += kSkChunk)
                items.push_back(SkItem{-(ubase[l] + u) - 1, r, ubase[l + 1] + np, 0});
        }
        d.nitems = (int)items.size() - d.item0;
        lvls.push_back(d);
    }
    f.sk_units = pb.push(units);
    f.sk_pairs = pb.push(pairs);
    f.sk_items = pb.push(items);
    f.sk_levels = pb.push(lvls);
    f.sk_nlevels = L;
    int mmax = 0, rmax = 0;
    for (int i = 0; i < f.p; ++i) {
        mmax = std::max(mmax, f.parts[i].m);
        rmax = std::max(rmax, f.parts[i].rows);
    }
    f.sk_mmax = mmax;
    f.sk_rmax = rmax;
}

// Symbolic part: geometry, pool layout, programs (cached), device allocations.
void setup_fact(spk_fact& f, cudaStream_t s) {
    Tracer tr("setup");
    const int p = f.p, k = f.k;
    const long long kk = (long long)k * k;
    const std::string key = sym_key(f);
    {
        SymCache& c = sym_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.map.find(key);
        if (it != c.map.end()) f.sym = it->second;
    }
    if (f.sym) {
        const Symbolic& y = *f.sym;
        f.parts = y.parts;
        f.levels = y.levels;
        f.off_bhat = y.off_bhat;
        f.off_chat = y.off_chat;
        f.pool_size = y.pool_size;
        f.fac_size = y.fac_size;
        f.piv_size = y.piv_size;
        f.tfac_size = y.tfac_size;
        f.aux_rows = y.aux_rows;
        f.auxf_rows = y.auxf_rows;
        f.tau_w = y.tau_w;
        f.npairs = y.npairs;
        f.prog_factor = y.prog_factor;
        f.prog_levels = y.prog_levels;
        f.sk = y.sk;
        f.sk_units = y.sk_units;
        f.sk_pairs = y.sk_pairs;
        f.sk_items = y.sk_items;
        f.sk_levels = y.sk_levels;
        f.sk_nlevels = y.sk_nlevels;
        f.sk_mmax = y.sk_mmax;
        f.sk_rmax = y.sk_rmax;
        f.want_tfac = y.want_tfac.load();
        tr.mark("symbolic (cached)");
        alloc_fact(f, s, y.blob);
        return;
    }
    f.parts.clear();
    long long fac_cursor = 0;
    if (!f.reduced_only) {
        for (int i = 0; i < p; ++i) {
            const int m = (int)(f.bounds[i + 1] - f.bounds[i]);
            const int rev = (f.coupled() && f.last(i)) ? 1 : 0;
            PartDev P = make_part(f.bounds[i], m, f.kl, f.ku, f.piv_on, rev, k);
            // partition factors start on 64-byte boundaries: the LU's 8-entry
            // runs (U columns, L rows) are then whole sectors for k = 0 mod 4
            P.fofs = fac_cursor;
            fac_cursor += ((long long)P.m * P.rows + 7) / 8 * 8;
            P.rowsT = P.kl + P.ubw + 1;
            P.tofs = f.tfac_size;
            f.tfac_size += ((long long)P.m * P.rowsT + 7) / 8 * 8;
            f.parts.push_back(P);
        }
        if (f.coupled())
            for (int i = 0; i < p; ++i)
                if (f.parts[i].m < k)
                    fail(SPK_EINVAL, "factorize: partition smaller than the half-bandwidth");
    } else {
        for (int i = 0; i < p; ++i) f.parts.push_back(PartDev{});
    }
    long long pool = 0;
    f.off_bhat = pool;
    pool += kk * p;
    f.off_chat = pool;
    pool += kk * p;
    build_levels(f, pool);
    add_couplings(f, fac_cursor);
    // explicit S^-1 per pair (Schur path): pair solves apply it as one GEMM
    for (size_t l = 0; l + 1 < f.levels.size(); ++l) {
        Level& lv = f.levels[l];
        lv.sinv.assign(lv.units / 2, -1);
        for (int a = 0; a < lv.units / 2; ++a) {
            lv.sinv[a] = pool;
            pool += kk;
        }
    }
    f.pool_size = pool;
    f.fac_size = fac_cursor;
    f.piv_size = f.n + (long long)(f.parts.size() - p) * 2 * k + 1;
    // AUX layout for solves: reduced red regions, then tau (first, last), z (first, last)
    int wmax = k;
    if (!f.reduced_only && p > 1)
        wmax = std::max(std::min(f.parts[0].m, k + (f.piv_on ? f.parts[0].kl : 0)),
                        std::min(f.parts[p - 1].m, k + (f.piv_on ? f.parts[p - 1].kl : 0)));
    f.tau_w = wmax;
    f.aux_rows = std::max<long long>((long long)std::max(p - 1, 0) * 2 * k + 2LL * wmax + 2LL * k, 1);
    tr.mark("geometry");
    ProgramBuilder pb;
    build_factor_program(f, pb);
    if (f.sk) build_sk_tables(f, pb);
    tr.mark("factor program");
    auto y = std::make_shared<Symbolic>();
    y->parts = f.parts;
    y->levels = f.levels;
    y->off_bhat = f.off_bhat;
    y->off_chat = f.off_chat;
    y->pool_size = f.pool_size;
    y->fac_size = f.fac_size;
    y->piv_size = f.piv_size;
    y->tfac_size = f.tfac_size;
    y->aux_rows = f.aux_rows;
    y->auxf_rows = f.auxf_rows;
    y->tau_w = f.tau_w;
    y->npairs = f.npairs;
    y->prog_factor = f.prog_factor;
    y->prog_levels = f.prog_levels;
    y->sk = f.sk;
    y->sk_units = f.sk_units;
    y->sk_pairs = f.sk_pairs;
    y->sk_items = f.sk_items;
    y->sk_levels = f.sk_levels;
    y->sk_nlevels = f.sk_nlevels;
    y->sk_mmax = f.sk_mmax;
    y->sk_rmax = f.sk_rmax;
    y->blob = std::move(pb.blob);
    {
        SymCache& c = sym_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.map.size() >= 32) c.map.clear();  // bounded: shapes rarely vary that much
        c.map[key] = y;
    }
    f.sym = y;
    alloc_fact(f, s, y->blob);
}

// device allocations (stream ordered) and uploads of the symbolic state
// The symbolic's device tables for the current device, uploaded once.
Symbolic::DevTables sym_device_tables(Symbolic& y, const spk_fact& f) {
    int dev = 0;
    ck(cudaGetDevice(&dev), "device");
    std::lock_guard<std::mutex> lk(y.dev_mu);
    auto it = y.dev.find(dev);
    if (it != y.dev.end()) return it->second;
    Symbolic::DevTables t;
    ck(cudaMalloc(&t.parts, sizeof(PartDev) * std::max<size_t>(y.parts.size(), 1)), "alloc");
    ck(cudaMalloc(&t.bounds, sizeof(long long) * (f.p + 1)), "alloc");
    ck(cudaMalloc(&t.blob, std::max<size_t>(y.blob.size(), 1)), "alloc");
    ck(cudaMemcpy(t.parts, y.parts.data(), sizeof(PartDev) * y.parts.size(), cudaMemcpyHostToDevice), "upload");
    ck(cudaMemcpy(t.bounds, f.bounds.data(), sizeof(long long) * (f.p + 1), cudaMemcpyHostToDevice), "upload");
    if (!y.blob.empty()) ck(cudaMemcpy(t.blob, y.blob.data(), y.blob.size(), cudaMemcpyHostToDevice), "upload");
    y.dev[dev] = t;
    return t;
}

void alloc_fact(spk_fact& f, cudaStream_t s, const std::vector<char>& blob) {
    Tracer tr("alloc");
    const int p = f.p;
    const int nparts = (int)f.parts.size();
    if (f.sk && f.sym) {
        // small-k engine: the symbolic's device tables, the factor, the pool
        // (every entry any consumer reads is written by the engine's kernels:
        // no memset) and one small zeroed block (status, fell, barrier words)
        const Symbolic::DevTables t = sym_device_tables(*f.sym, f);
        f.d_parts = t.parts;
        f.d_bounds = t.bounds;
        f.d_blob = t.blob;
        f.tables_shared = true;
        f.d_fac = dalloc<double>(f.fac_size, s);
        f.d_pool = dalloc<double>(f.pool_size, s);
        f.d_tfac = dalloc<double>(f.tfac_size, s);
        f.d_dinv = dalloc<double>(f.n, s);
        f.d_piv = dalloc<int>(1, s);
        f.d_amax = dalloc<unsigned long long>(1, s);
        f.d_boost = dalloc<int>(nparts, s);
        f.d_flags = dalloc<int>(std::max(f.npairs, 1), s);
        const size_t misc = 2 + nparts + 4;  // status, pad, fell[nparts], barrier words
        f.d_skmisc = dalloc<unsigned>(misc, s);
        ck(cudaMemsetAsync(f.d_skmisc, 0, sizeof(unsigned) * misc, s), "memset");
        f.d_status = reinterpret_cast<int*>(f.d_skmisc);
        f.d_fell = reinterpret_cast<int*>(f.d_skmisc) + 2;
        tr.mark("small-k allocations");
        return;
    }
    f.d_parts = dalloc<PartDev>(nparts, s);
    f.d_fac = dalloc<double>(f.fac_size, s);
    f.d_piv = dalloc<int>(f.piv_size, s);
    f.d_pool = dalloc<double>(f.pool_size, s);
    f.d_bounds = dalloc<long long>(p + 1, s);
    f.d_amax = dalloc<unsigned long long>(nparts, s);
    f.d_boost = dalloc<int>(nparts, s);
    f.d_fell = dalloc<int>(nparts, s);
    f.d_status = dalloc<int>(1, s);
    f.d_blob = dalloc<char>(std::max<size_t>(blob.size(), 1), s);
    f.d_tfac = dalloc<double>(f.tfac_size, s);
    f.d_dinv = dalloc<double>(f.n, s);
    f.lblk_trw = (!f.reduced_only && f.piv_on) ? piv_trw(f.kl, f.ku) : 0;
    if (f.lblk_trw)
        f.d_lblk = dalloc<double>((f.bounds[p] / 8 + nparts + 2) * piv_rec_size(f.lblk_trw), s);
    tr.mark("allocations");
    f.d_flags = dalloc<int>(std::max(f.npairs, 1), s);
    ck(cudaMemsetAsync(f.d_flags, 0, sizeof(int) * std::max(f.npairs, 1), s), "memset");
    if (f.sk) {
        f.d_skmisc = dalloc<unsigned>(4, s);
        ck(cudaMemsetAsync(f.d_skmisc, 0, sizeof(unsigned) * 4, s), "memset");
    }
    ck(cudaMemcpyAsync(f.d_parts, f.parts.data(), sizeof(PartDev) * nparts, cudaMemcpyHostToDevice, s), "upload");
    ck(cudaMemcpyAsync(f.d_bounds, f.bounds.data(), sizeof(long long) * (p + 1), cudaMemcpyHostToDevice, s),
       "upload");
    if (!blob.empty())
        ck(cudaMemcpyAsync(f.d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice, s), "upload");
    ck(cudaMemsetAsync(f.d_pool, 0, sizeof(double) * f.pool_size, s), "memset");
    ck(cudaMemsetAsync(f.d_amax, 0, sizeof(unsigned long long) * nparts, s), "memset");
    ck(cudaMemsetAsync(f.d_boost, 0, sizeof(int) * nparts, s), "memset");
    ck(cudaMemsetAsync(f.d_fell, 0, sizeof(int) * nparts, s), "memset");
    ck(cudaMemsetAsync(f.d_status, 0, sizeof(int), s), "memset");
    tr.mark("uploads");
}

void build_solve_programs(spk_fact& f, cudaStream_t s);
Bufs make_bufs(const spk_fact* f);

// The small-k engine's factorization: partitions (LU, factor layouts,
// corners, level-0 tips) and the whole reduced hierarchy, two launches.
// false when its kernels do not cover the shape (the caller runs the general
// programs).
bool run_sk_factor(spk_fact& f, const double* dband, cudaStream_t s) {
    const char* blob = f.d_blob;
    SkPartsArgs P{dband, f.n, f.kl, f.ku, f.k, f.p, f.d_parts, f.d_fac, f.d_dinv, f.d_boost, f.d_pool,
                  f.off_bhat, f.off_chat, reinterpret_cast<const SkUnit*>(blob + f.sk_units), f.boost_eps, f.sk_mmax};
    {
        ProfScope ps(ST_LU, s, 8.0 * f.n * f.k * f.k, 16.0 * f.n * (f.kl + f.ku + 1));
        if (!launch_sk_parts(P, s)) return false;
    }
    SkLevelsArgs L{f.d_pool, reinterpret_cast<const SkUnit*>(blob + f.sk_units),
                   reinterpret_cast<const SkPair*>(blob + f.sk_pairs), reinterpret_cast<const SkItem*>(blob + f.sk_items),
                   reinterpret_cast<const SkLevel*>(blob + f.sk_levels), f.sk_nlevels, f.k, f.d_flags,
                   f.boost_eps, f.d_skmisc + 2 + f.parts.size(), g_sk_trace};
    {
        ProfScope ps(ST_CPL, s, 0.0, 0.0);
        launch_sk_levels(L, s);
    }
    return true;
}

// the factorization's device state (factors, pool, flags, solve jobs) is
// complete on f.stream up to here
void mark_ready(spk_fact& f, cudaStream_t s) {
    if (!f.ready_ev) ck(cudaEventCreateWithFlags(&f.ready_ev, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(f.ready_ev, s), "event");
}

// forward solves with few right-hand sides of a small-k factorization run
// the engine's own cooperative kernel (k_sk_solve)
bool sk_kernel_solve(const spk_fact& f, int transpose, int nrhs) {
    return f.sk_schur_all && !transpose && nrhs >= 1 && nrhs <= kSkMaxRhs && !f.open() && f.coupled() &&
           sk_solve_smem(f.sk_mmax, f.sk_rmax, nrhs) <= 227u * 1024;
}

// the row-major factor copy of a small-k factorization, once, ordered on
// the factorization's stream (later solves on other streams wait on ready_ev)
void ensure_tfac(const spk_fact* fc) {
    spk_fact& f = const_cast<spk_fact&>(*fc);
    if (f.tfac_ready.load()) return;
    std::lock_guard<std::mutex> lk(f.tfac_mu);
    if (f.tfac_ready.load()) return;
    long long mx = 0;
    for (int i = 0; i < f.p; ++i) mx = std::max(mx, (long long)f.parts[i].m * f.parts[i].rowsT);
    launch_transpose_factors(f.d_parts, f.p, mx, f.d_fac, f.d_tfac, f.d_dinv, f.stream);
    mark_ready(f, f.stream);
    f.tfac_ready.store(true);
    if (f.sym && !f.sk) f.sym->want_tfac.store(true);
}

// order work on s after the factorization (a no-op on its own stream)
void wait_ready(const spk_fact& f, cudaStream_t s) {
    if (f.ready_ev && s != f.stream) ck(cudaStreamWaitEvent(s, f.ready_ev, 0), "wait");
}

// record the last use of f by stream s (see ~spk_fact)
void note_use(const spk_fact& fc, cudaStream_t s) {
    if (s == fc.stream) return;
    spk_fact& f = const_cast<spk_fact&>(fc);
    std::lock_guard<std::mutex> lk(f.use_mu);
    for (auto& u : f.uses)
        if (u.first == s) {
            ck(cudaEventRecord(u.second, s), "event");
            return;
        }
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventRecord(e, s), "event");
    f.uses.emplace_back(s, e);
}

void finish_factor(spk_fact& f, cudaStream_t s) {
    Tracer tr("finish");
    int status = 0;
    const int nparts = (int)f.parts.size();
    std::vector<int> boost(nparts), fell(nparts);
    ck(cudaMemcpyAsync(&status, f.d_status, sizeof(int), cudaMemcpyDeviceToHost, s), "download");
    ck(cudaMemcpyAsync(boost.data(), f.d_boost, sizeof(int) * nparts, cudaMemcpyDeviceToHost, s), "download");
    ck(cudaMemcpyAsync(fell.data(), f.d_fell, sizeof(int) * nparts, cudaMemcpyDeviceToHost, s), "download");
    // coupling paths, known once the factor program ran
    std::vector<int> flags(std::max(f.npairs, 1), 0);
    if (f.npairs > 0)
        ck(cudaMemcpyAsync(flags.data(), f.d_flags, sizeof(int) * f.npairs, cudaMemcpyDeviceToHost, s), "flags");
    ck(cudaStreamSynchronize(s), "factorize");
    tr.mark("stream synced");
    ck(cudaGetLastError(), "factorize kernels");
    if (status == 2) fail(SPK_ESINGULAR, "lu_factor: exactly singular column in pivoting mode");
    f.boost_count = 0;
    if (!f.reduced_only)
        for (int i = 0; i < f.p; ++i) f.boost_count += boost[i];
    f.boost_warnings = 0;
    for (int i = f.p; i < nparts; ++i) f.boost_warnings += fell[i];
    f.factor_sweeps.assign(f.p, 0);
    if (!f.reduced_only && f.coupled())
        for (int i = 0; i < f.p; ++i) f.factor_sweeps[i] = (!f.first(i) && !f.last(i)) ? 3 : 0;
    // coupling paths are known now: compile the solve programs without guards
    f.flags = std::move(flags);
    build_solve_programs(f, s);
    mark_ready(f, s);
}

// Solve programs for f.flags (the per-pair coupling paths), or -- flags empty,
// factorization still running -- with both paths emitted and device-guarded.
// Cached per flag pattern in the symbolic.
void build_solve_programs(spk_fact& f, cudaStream_t s) {
    if (f.d_sblob) {
        // solves already enqueued may still read the previous jobs: kept to the end
        if (f.d_sblob_prev) dfree(f.d_sblob_prev, f.stream);
        f.d_sblob_prev = f.d_sblob;
        f.d_sblob = nullptr;
    }
    if (f.sym) {
        SymCache& c = sym_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = f.sym->solves.find(f.flags);
        if (it != f.sym->solves.end()) {
            const SolveProgs& sp = it->second;
            f.prog_fwd = sp.fwd;
            f.prog_tr = sp.tr;
            f.prog_rfwd = sp.rfwd;
            f.prog_rtr = sp.rtr;
            f.d_sblob = dalloc<char>(std::max<size_t>(sp.blob.size(), 1), s);
            if (!sp.blob.empty())
                ck(cudaMemcpyAsync(f.d_sblob, sp.blob.data(), sp.blob.size(), cudaMemcpyHostToDevice, s), "upload");
            return;
        }
    }
    ProgramBuilder pb;
    f.prog_fwd.clear();
    f.prog_tr.clear();
    f.prog_rfwd.clear();
    f.prog_rtr.clear();
    if (!f.reduced_only) {
        build_forward_program(f, pb);
        build_transpose_program(f, pb);
        Builder bf{f, pb, f.prog_rfwd}, bt{f, pb, f.prog_rtr};
        if (f.p > 1 && f.k > 0) {
            build_reduced_solve(f, bf, false, 0);
            build_reduced_solve(f, bt, true, 0);
        }
    } else {
        Builder bf{f, pb, f.prog_fwd}, bt{f, pb, f.prog_tr};
        if (f.p > 1 && f.k > 0) {
            build_reduced_solve(f, bf, false, 0);
            build_reduced_solve(f, bt, true, 0);
        }
    }
    f.d_sblob = dalloc<char>(std::max<size_t>(pb.blob.size(), 1), s);
    if (!pb.blob.empty())
        ck(cudaMemcpyAsync(f.d_sblob, pb.blob.data(), pb.blob.size(), cudaMemcpyHostToDevice, s), "upload");
    if (f.sym) {
        SymCache& c = sym_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        if (f.sym->solves.size() >= 8) f.sym->solves.clear();
        SolveProgs& sp = f.sym->solves[f.flags];
        sp.fwd = f.prog_fwd;
        sp.tr = f.prog_tr;
        sp.rfwd = f.prog_rfwd;
        sp.rtr = f.prog_rtr;
        sp.blob = std::move(pb.blob);
    }
}

// the deferred host-side finish of a factorization (stream-ordered
// spk_factorize): synchronises its stream, reports an exactly singular pivot
void ensure_finished(const spk_fact* fc) {
    if (!fc) fail(SPK_EINVAL, "null factorization handle");
    spk_fact& f = const_cast<spk_fact&>(*fc);
    if (f.pending.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lk(f.fin_mu);
        if (f.pending.load(std::memory_order_relaxed)) {
            try {
                finish_factor(f, f.stream);
            } catch (const SpkError& e) {
                f.fin_status = e.st;
                f.fin_msg = e.msg;
            } catch (const std::bad_alloc&) {
                f.fin_status = SPK_ENOMEM;
                f.fin_msg = "host allocation failed";
            }
            f.pending.store(false, std::memory_order_release);
        }
    }
    if (f.fin_status != SPK_OK) fail(f.fin_status, f.fin_msg);
}

Bufs make_bufs(const spk_fact* f = nullptr) {
    Bufs B;
    for (int i = 0; i < kMaxBufs; ++i) {
        B.p[i] = nullptr;
        B.ld[i] = 1;
    }
    B.flags = f ? f->d_flags : nullptr;
    if (f) {
        B.p[B_FAC] = f->d_fac;
        B.p[B_POOL] = f->d_pool;
    }
    return B;
}

}  // namespace

// ===========================================================================
// C-ABI
extern "C" {

const char* spk_last_error(void) { return g_err.c_str(); }
const char* spk_version(void) { return "spike_b200 0.1 (sm_100a)"; }

void spk_profile_enable(int32_t on) { g_prof_on = on != 0; }

int32_t spk_profile_classes(void) { return kNumClasses; }

/* Drains pending events (synchronising on them) and returns the accumulated
 * per-class totals since the last reset. */
const char* spk_profile_read(int32_t cls, double* ms, double* flops, double* bytes, int64_t* launches) {
    prof_drain();
    if (cls < 0 || cls >= kNumClasses) return nullptr;
    if (ms) *ms = g_acc[cls].ms;
    if (flops) *flops = g_acc[cls].flops;
    if (bytes) *bytes = g_acc[cls].bytes;
    if (launches) *launches = g_acc[cls].launches;
    return kClassName[cls];
}

void spk_profile_reset(void) {
    prof_drain();
    for (auto& a : g_acc) a = ProfAcc{};
}

int64_t spk_arena_cached(void) { return (int64_t)arena().cached; }

void spk_arena_trim(void) { arena().trim(); }

int64_t spk_launch_count(int32_t reset) {
    const long long v = g_launches;
    if (reset) g_launches = 0;
    return v;
}

int64_t spk_generic_launch_count(int32_t reset) {
    const long long v = g_generic_launches;
    if (reset) g_generic_launches = 0;
    return v;
}

void spk_set_generic_path(int32_t on) { g_generic.store(on ? 1 : 0); }

void spk_compute_ratios(double K, int32_t nrhs, int32_t k, double* r12, double* r13) {
    // partition.cpp:47-54
    const double rho = static_cast<double>(nrhs) / k;
    const double t = 1.0 / (1.0 + K * rho) + (1.5 + 2.0 * rho) / (1.0 / K + rho);
    *r13 = t;
    *r12 = t / 2.0;
}

spk_status spk_distribute_threads(int32_t t, int32_t cap_p, int32_t* p, int32_t* kinds, int32_t kinds_cap,
                                  int32_t* threads_used, int32_t* idle) {
    // partition.cpp:24-45
    return guarded([&] {
        if (t < 1) fail(SPK_EINVAL, "distribute_threads: t must be >= 1");
        int pp = 1;
        while (2 * pp <= t) pp *= 2;
        if (cap_p > 0) pp = std::min(pp, cap_p);
        *p = pp;
        std::vector<int> kd(pp, SPK_INNER_SINGLE);
        int used = 1;
        if (pp == 1) {
            kd[0] = SPK_FIRSTLAST;
        } else {
            kd.front() = kd.back() = SPK_FIRSTLAST;
            const int extra = std::min(t - pp, pp - 2);
            for (int i = 0; i < extra; ++i) kd[1 + i] = SPK_INNER_DUAL;
            used = pp + extra;
        }
        if (kinds)
            for (int i = 0; i < pp && i < kinds_cap; ++i) kinds[i] = kd[i];
        if (threads_used) *threads_used = used;
        if (idle) *idle = t - used;
    });
}

spk_status spk_compute_sizes(int64_t n, int32_t p, const int32_t* kinds, double r12, double r13,
                             int64_t min_single, int64_t min_dual, int64_t* sizes) {
    // partition.cpp:56-87
    return guarded([&] {
        if (p == 1) {
            if (n < min_single) fail(SPK_EDOMAIN, "compute_sizes: matrix too small");
            sizes[0] = n;
            return;
        }
        int x = 0;
        for (int i = 0; i < p; ++i) x += kinds[i] == SPK_INNER_DUAL;
        const int y = (p - x) - 2;
        const double denom = 2.0 * r12 * r13 + x * r13 + y * r12;
        const double n1 = n * r12 * r13 / denom, n2 = n1 / r12, n3 = n1 / r13;
        long long rest = 0;
        for (int i = 1; i < p; ++i) {
            double want = n1;
            if (kinds[i] == SPK_INNER_DUAL) want = n2;
            else if (kinds[i] == SPK_INNER_SINGLE) want = n3;
            sizes[i] = std::llround(want);
            rest += sizes[i];
        }
        sizes[0] = n - rest;
        for (int i = 0; i < p; ++i) {
            const long long need = kinds[i] == SPK_INNER_DUAL ? min_dual : min_single;
            if (sizes[i] < need) fail(SPK_EDOMAIN, "compute_sizes: partition below its minimum size");
        }
    });
}

spk_status spk_make_plan(int64_t n, int32_t kl, int32_t ku, int32_t t, double r12, double r13, int32_t cap,
                         int32_t* p, int64_t* bounds, int32_t* kinds, int32_t* threads_used, int32_t* idle) {
    // partition.cpp:89-118
    return guarded([&] {
        if (t < 1) fail(SPK_EINVAL, "distribute_threads: t must be >= 1");
        const int khat = std::max(kl, ku);
        const long long min_single = 2LL * khat + 1;
        const long long min_dual = std::max(min_single, 2LL * (kl + ku + 1));
        int p0 = 0, tu = 0, id = 0;
        spk_distribute_threads(t, 0, &p0, nullptr, 0, &tu, &id);
        for (int pp = p0; pp >= 1; pp /= 2) {
            int pq = 0;
            std::vector<int32_t> kd(pp);
            spk_distribute_threads(t, pp, &pq, kd.data(), pp, &tu, &id);
            std::vector<int64_t> sizes(pq);
            if (spk_compute_sizes(n, pq, kd.data(), r12, r13, min_single, min_dual, sizes.data()) == SPK_OK) {
                if (pq > cap) fail(SPK_EINVAL, "make_plan: capacity too small");
                *p = pq;
                bounds[0] = 0;
                for (int i = 0; i < pq; ++i) {
                    bounds[i + 1] = bounds[i] + sizes[i];
                    kinds[i] = kd[i];
                }
                *threads_used = tu;
                *idle = id;
                return;
            }
            if (pp == 1) break;
        }
        *p = 1;
        bounds[0] = 0;
        bounds[1] = n;
        kinds[0] = SPK_FIRSTLAST;
        *threads_used = 1;
        *idle = t - 1;
    });
}

spk_status spk_gpu_plan(int64_t n, int32_t kl, int32_t ku, int32_t nrhs, int32_t pivoting, int32_t p_hint,
                        int32_t cap, int32_t* p, int64_t* bounds, int32_t* kinds) {
    return guarded([&] {
        const int k = std::max(kl, ku);
        const long long min_part = std::max<long long>(2LL * k + 1, 1);
        int pp = p_hint;
        if (pp <= 0) {
            // one partition per SM for wide bands (the sweep kernels then split
            // the right-hand sides across SMs); more for narrow bands, where a
            // partition's column chain is short per step.
            // Narrow solves (nrhs <= 64) on wide bands get two partitions per SM:
            // their sweeps are latency-bound at <= 8 warps per partition (C5:
            // 238 -> 216 ms per step); wide ones fill an SM per partition (C3:
            // p = 296 would cost 9 ms).
            // SMs of the current device (148 on B200; the planner is host-only
            // and may run without a GPU, where it plans for a B200)
            int ndev = 0, sms = 148;
            if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) sms = device_sms();
            (void)cudaGetLastError();
            if (k >= 96) pp = nrhs <= 64 ? 2 * sms : sms;
            else if (k >= 32) pp = 2 * sms;
            // narrow bands: up to 8 partitions per SM, but no shorter than
            // ~2k rows (more reduced-system levels cost more than the shorter
            // column chain saves: C1 n=1e5 p=1184 3.6 ms, p=148 2.0 ms)
            // narrow non-pivoting bands take the small-k engine (spk_smallk*.cu):
            // partitions of ~96 rows (a half-warp per partition, the block
            // staged in shared memory; the solve keeps a warp's partition
            // factor resident between its D-stage and retrieval)
            else if (!pivoting && kl <= 16 && ku <= 16) pp = (int)std::max<long long>(2, (n + 95) / 96);
            else pp = (int)std::min<long long>(8 * sms, std::max<long long>(sms, n / 2048));
        }
        pp = (int)std::max<long long>(1, std::min<long long>(pp, n / std::max<long long>(min_part, 1)));
        if (pp > cap) fail(SPK_EINVAL, "gpu_plan: capacity too small");
        // first/last partitions carry no spike sweeps (0 vs 3 in factor, 2 vs 4
        // in solve): give them the reference's R13 ratio with K = 1.
        // Equal sizes: on the GPU every stage is one launch over all
        // partitions, so a stage costs its largest partition; first/last
        // partitions do full sweeps in the D stage and the LU like everyone
        // else, so the CPU ratio model (partition.cpp:47-54) would make them
        // the critical path.
        const long long base = n / pp, extra = n % pp;
        bounds[0] = 0;
        for (int i = 0; i < pp; ++i) bounds[i + 1] = bounds[i] + base + (i < extra ? 1 : 0);
        for (int i = 0; i < pp; ++i) {
            if (bounds[i + 1] - bounds[i] < min_part && pp > 1) fail(SPK_EDOMAIN, "gpu_plan: partition too small");
            kinds[i] = (i == 0 || i == pp - 1) ? SPK_FIRSTLAST : SPK_INNER_SINGLE;
        }
        *p = pp;
    });
}

spk_status spk_gpu_plan_ratio(int64_t n, int32_t kl, int32_t ku, int32_t nrhs, int32_t pivoting, int32_t p_hint,
                              double r13, int32_t cap, int32_t* p, int64_t* bounds, int32_t* kinds) {
    return guarded([&] {
        if (!(r13 > 0.0)) fail(SPK_EDOMAIN, "gpu_plan_ratio: r13 must be positive");
        spk_status st = spk_gpu_plan(n, kl, ku, nrhs, pivoting, p_hint, cap, p, bounds, kinds);
        if (st != SPK_OK) fail(st, g_err.c_str());
        const int pp = *p;
        if (pp < 3) return;  // both partitions first/last: equal halves (as compute_sizes)
        // first/last = r13 * inner (compute_sizes, partition.cpp:47-76, without dual partitions)
        const int k = std::max(kl, ku);
        const long long min_part = std::max<long long>(2LL * k + 1, 1);
        const double inner = (double)n / (pp - 2 + 2.0 * r13);
        const long long fl = std::max<long long>(std::llround(r13 * inner), min_part);
        const long long rest = n - 2 * fl, ni = pp - 2;
        if (rest < ni * min_part) fail(SPK_EDOMAIN, "gpu_plan_ratio: partition too small");
        const long long base = rest / ni, extra = rest % ni;
        bounds[0] = 0;
        bounds[1] = fl;
        for (int i = 1; i < pp - 1; ++i) bounds[i + 1] = bounds[i] + base + (i - 1 < extra ? 1 : 0);
        bounds[pp] = n;
        for (int i = 0; i < pp; ++i)
            if (bounds[i + 1] - bounds[i] < min_part) fail(SPK_EDOMAIN, "gpu_plan_ratio: partition too small");
    });
}

spk_status spk_default_k_cache_path(char* buf, int32_t cap) {
    return guarded([&] {
        const char* env = getenv("SPIKE_K_CACHE");
        const std::string path = env ? env : "spike_k.cache";  // partition.cpp:149-152
        if ((int)path.size() + 1 > cap) fail(SPK_EINVAL, "k_cache_path: buffer too small");
        std::memcpy(buf, path.c_str(), path.size() + 1);
    });
}

spk_status spk_write_k_cache(const char* path, double k) {
    return guarded([&] {
        FILE* fp = fopen(path, "w");
        if (!fp) fail(SPK_EIO, std::string("cannot write calibration cache ") + path);
        fprintf(fp, "K %.17g\n", k);  // os.precision(17); os << "K " << k (partition.cpp:154-159)
        fclose(fp);
    });
}

spk_status spk_read_k_cache(const char* path, double* k, int32_t* found) {
    return guarded([&] {
        *found = 0;
        FILE* fp = fopen(path, "r");
        if (!fp) return;
        char key[256];
        double v = 0.0;
        while (fscanf(fp, "%255s %lf", key, &v) == 2)  // partition.cpp:161-169: first "K" wins
            if (std::strcmp(key, "K") == 0) {
                *k = v;
                *found = 1;
                break;
            }
        fclose(fp);
    });
}

spk_status spk_calibrate_k(int64_t n_sample, int32_t k_sample, int32_t reps, void* stream, spk_calibration* out) {
    return guarded([&] {
        if (k_sample < 1) fail(SPK_EINVAL, "calibrate_k: k_sample must be >= 1");
        if (n_sample <= 0) n_sample = 200LL * k_sample;
        if (k_sample >= n_sample) fail(SPK_EINVAL, "calibrate_k: k_sample must be < n_sample");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const long long n = n_sample, ld = 2LL * k_sample + 1;
        double* band = dalloc<double>((size_t)(ld * n), s);
        double* F = dalloc<double>((size_t)(n * k_sample), s);
        double* X = dalloc<double>((size_t)(n * k_sample), s);
        launch_generate_band(1234, n, k_sample, k_sample, 1.5, 0, n, band, s);
        launch_generate_rhs(5678, 0, n, k_sample, F, n, s);
        ck(cudaGetLastError(), "calibrate_k");
        // one partition: the serial LU and two-sweep solve of partition.cpp:131-135
        int64_t bnds[2] = {0, n};
        int32_t kind = SPK_FIRSTLAST;
        spk_plan plan{1, bnds, &kind};
        spk_factor_options opts{0, 0.0};
        cudaEvent_t e[3];
        for (auto& x : e) ck(cudaEventCreate(&x), "event");
        std::vector<double> ratios;
        double tf_total = 0.0, ts_total = 0.0;
        const int R = std::max(reps, 1);
        for (int rep = 0; rep < R + 1; ++rep) {  // rep 0 warms up (symbolic cache, arena)
            spk_fact* f = nullptr;
            ck(cudaEventRecord(e[0], s), "event");
            spk_status st = spk_factorize(band, SPK_MEM_DEVICE, n, k_sample, k_sample, &plan, &opts, s, &f);
            if (st != SPK_OK) fail(st, g_err.c_str());
            ck(cudaEventRecord(e[1], s), "event");
            st = spk_solve(f, 0, F, n, k_sample, X, n, SPK_MEM_DEVICE, s, nullptr);
            if (st != SPK_OK) {
                spk_fact_destroy(f);
                fail(st, g_err.c_str());
            }
            ck(cudaEventRecord(e[2], s), "event");
            ck(cudaEventSynchronize(e[2]), "calibrate_k");
            spk_fact_destroy(f);
            if (rep == 0) continue;
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, e[0], e[1]);
            cudaEventElapsedTime(&b, e[1], e[2]);
            const double tf = a * 1e-3, ts = b * 1e-3;
            tf_total += tf;
            ts_total += ts;
            ratios.push_back(ts / std::max(tf, 1e-12));
        }
        for (auto& x : e) cudaEventDestroy(x);
        for (double* q : {band, F, X}) dfree(q, s);
        std::sort(ratios.begin(), ratios.end());
        out->k = ratios[ratios.size() / 2];
        out->factor_seconds = tf_total / R;
        out->solve_seconds = ts_total / R;
        out->timer_warning = (tf_total + ts_total) < 0.010;
    });
}

static spk_status factorize_impl(const double* band, int32_t band_mem, int64_t n, int32_t kl, int32_t ku,
                                 const spk_plan* plan, const spk_factor_options* opts, int open_l, int open_r,
                                 void* stream, spk_fact** out) {
    return guarded([&] {
        if (!out) fail(SPK_EINVAL, "factorize: null output");
        *out = nullptr;
        if (n < 1 || kl < 0 || ku < 0 || kl >= n || ku >= n) fail(SPK_EINVAL, "BandedMatrix: bad shape");
        validate_plan(n, plan);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto f = std::make_unique<spk_fact>();
        f->open_l = open_l ? 1 : 0;
        f->open_r = open_r ? 1 : 0;
        f->n = n;
        f->kl = kl;
        f->ku = ku;
        f->k = std::max(kl, ku);
        f->p = plan->p;
        f->piv_on = opts ? opts->pivoting : 0;
        f->boost_eps = (opts && opts->boost_eps > 0) ? opts->boost_eps : std::sqrt(DBL_EPSILON);
        f->bounds.assign(plan->bounds, plan->bounds + plan->p + 1);
        f->kinds.assign(plan->p, SPK_INNER_SINGLE);
        if (plan->kinds) f->kinds.assign(plan->kinds, plan->kinds + plan->p);
        f->stream = s;
        f->sk = sk_eligible(*f);
        Tracer tr("factorize");
        setup_fact(*f, s);
        // until the factorization is finished (ensure_finished) solves run
        // device-guarded programs; built and uploaded here, ahead of the work
        f->flags.clear();
        if (!f->sk) build_solve_programs(*f, s);  // small-k: built at the finish, when a general program needs them
        tr.mark("setup (symbolic)");
        // band on device; a slab's band starts k halo columns early when its
        // left edge is open and carries k more when its right edge is
        const long long ld = kl + ku + 1;
        const long long hl = (long long)f->k * f->open_l, hr = (long long)f->k * f->open_r;
        const double* dband = band;
        double* tmp = nullptr;
        if (band_mem == SPK_MEM_HOST) {
            tmp = dalloc<double>(ld * (n + hl + hr), s);
            ck(cudaMemcpyAsync(tmp, band, sizeof(double) * ld * (n + hl + hr), cudaMemcpyHostToDevice, s),
               "band upload");
            ck(cudaEventCreateWithFlags(&f->upload_ev, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(f->upload_ev, s), "event");
            dband = tmp;
        }
        dband += ld * hl;  // column 0 of the slab
        const int p = f->p;
        if (f->sk) {
            if (!run_sk_factor(*f, dband, s)) fail(SPK_ECUDA, "factorize: small-k engine launch");
            f->tfac_ready.store(false);
            f->sk_schur_all = true;
            mark_ready(*f, s);
            tr.mark("enqueued (small-k engine)");
            if (tmp) dfree(tmp, s);
            f->pending.store(true);
            *out = f.release();
            return;
        }
        {
            ProfScope ps(PC_CORNERS, s, 0.0, 16.0 * p * f->k * f->k);
            launch_corners(dband, n, kl, ku, f->d_bounds, p, f->k, f->open_l, f->open_r, f->d_pool + f->off_bhat,
                           f->d_pool + f->off_chat, s);
        }
        double* fs = nullptr;
        double* auxf = nullptr;
        if (f->coupled()) {
            fs = dalloc<double>((size_t)n * 2 * f->k, s);
            auxf = dalloc<double>((size_t)f->auxf_rows * f->k, s);
        }
        Bufs B = make_bufs(f.get());
        B.p[B_POOL] = f->d_pool;
        B.ld[B_POOL] = 1;
        B.p[B_FS] = fs;
        B.ld[B_FS] = n;
        B.p[B_AUX] = auxf;
        B.ld[B_AUX] = f->auxf_rows;
        Exec ex{*f, s, B, f->k};
        ex.n = n;
        ex.band = dband;
        ex.band_cols = n + hl + hr;
        ex.band_col0 = hl;
        ex.run(f->prog_factor, f->d_blob);
        ex.run(f->prog_levels, f->d_blob);
        mark_ready(*f, s);
        tr.mark("enqueued");
        if (fs) dfree(fs, s);
        if (auxf) dfree(auxf, s);
        if (tmp) dfree(tmp, s);
        f->pending.store(true);  // finished lazily (ensure_finished)
        *out = f.release();
    });
}

spk_status spk_factorize(const double* band, int32_t band_mem, int64_t n, int32_t kl, int32_t ku,
                         const spk_plan* plan, const spk_factor_options* opts, void* stream,
                         spk_fact** out) {
    return factorize_impl(band, band_mem, n, kl, ku, plan, opts, 0, 0, stream, out);
}

spk_status spk_factorize_slab(const double* band, int32_t band_mem, int64_t n, int32_t kl, int32_t ku,
                              const spk_plan* plan, const spk_factor_options* opts, int32_t open_left,
                              int32_t open_right, void* stream, spk_fact** out) {
    return factorize_impl(band, band_mem, n, kl, ku, plan, opts, open_left, open_right, stream, out);
}

spk_status spk_fact_unit_tips(const spk_fact* f, double* d_tips, void* stream) {
    return guarded([&] {
        ensure_finished(f);
        const int k = f->k;
        const long long kk = (long long)k * k;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (k == 0) return;
        ck(cudaMemsetAsync(d_tips, 0, sizeof(double) * 4 * kk, s), "memset");
        if (!f->coupled()) return;
        const Level& top = f->levels[f->top_level()];
        const long long H = top.uh[0];
        const long long offs[2] = {top.voff[0], top.woff[0]};
        for (int w = 0; w < 2; ++w) {
            if (offs[w] < 0) continue;
            // top rows [0, k) and bottom rows [H-k, H) of the unit spike (ld H)
            ck(cudaMemcpy2DAsync(d_tips + (2 * w) * kk, sizeof(double) * k, f->d_pool + offs[w], sizeof(double) * H,
                                 sizeof(double) * k, k, cudaMemcpyDeviceToDevice, s),
               "unit tips");
            ck(cudaMemcpy2DAsync(d_tips + (2 * w + 1) * kk, sizeof(double) * k, f->d_pool + offs[w] + H - k,
                                 sizeof(double) * H, sizeof(double) * k, k, cudaMemcpyDeviceToDevice, s),
               "unit tips");
        }
    });
}

void spk_debug_set_trace(void* d_buf) { spk::g_sk_trace = static_cast<unsigned long long*>(d_buf); }

int32_t spk_fact_engine(const spk_fact* f) {
    if (!f) return -1;
    if (guarded([&] { ensure_finished(f); }) != SPK_OK) return -1;
    return f->sk ? (f->sk_schur_all ? 1 : 2) : 0;
}

int32_t spk_fact_open(const spk_fact* f) { return f ? (f->open_l | (f->open_r << 1)) : 0; }

void spk_fact_destroy(spk_fact* f) { delete f; }

spk_status spk_fact_sync(const spk_fact* f) {
    return guarded([&] { ensure_finished(f); });
}

spk_status spk_stream_sync(void* stream) {
    return guarded([&] { ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "stream sync"); });
}

spk_status spk_fact_info(const spk_fact* f, int64_t* n, int32_t* kl, int32_t* ku, int32_t* k, int32_t* p,
                         int32_t* levels, int32_t* boost_count, int32_t* boost_warnings) {
    return guarded([&] {
        ensure_finished(f);
        if (n) *n = f->n;
        if (kl) *kl = f->kl;
        if (ku) *ku = f->ku;
        if (k) *k = f->k;
        if (p) *p = f->p;
        if (levels) *levels = f->levels.empty() ? 0 : (int)f->levels.size() - 1;
        if (boost_count) *boost_count = f->boost_count;
        if (boost_warnings) *boost_warnings = f->boost_warnings;
    });
}

spk_status spk_fact_bounds(const spk_fact* f, int64_t* bounds) {
    return guarded([&] {
        if (!f || !bounds) fail(SPK_EINVAL, "fact_bounds: null argument");
        std::copy(f->bounds.begin(), f->bounds.end(), bounds); });
}

spk_status spk_fact_factor_sweeps(const spk_fact* f, int64_t* sweeps) {
    return guarded([&] {
        ensure_finished(f); std::copy(f->factor_sweeps.begin(), f->factor_sweeps.end(), sweeps); });
}

spk_status spk_fact_tip(const spk_fact* f, int32_t which, int32_t i, double* out) {
    return guarded([&] {
        ensure_finished(f);
        const int k = f->k, p = f->p;
        if (i < 0 || i >= p || which < 0 || which > 5) fail(SPK_ERANGE, "fact_tip: index out of range");
        const long long kk = (long long)k * k;
        std::fill(out, out + kk, 0.0);
        if (k == 0) return;
        if (which == SPK_BHAT || which == SPK_CHAT) {
            const long long off = (which == SPK_BHAT ? f->off_bhat : f->off_chat) + i * kk;
            ck(cudaMemcpy(out, f->d_pool + off, sizeof(double) * kk, cudaMemcpyDeviceToHost), "tip");
            return;
        }
        if (p < 2) return;
        const Level& l0 = f->levels[0];
        const long long base = (which == SPK_TIP_VT || which == SPK_TIP_VB) ? l0.voff[i] : l0.woff[i];
        if (base < 0) return;
        const long long roff = (which == SPK_TIP_VB || which == SPK_TIP_WB) ? k : 0;
        ck(cudaMemcpy2D(out, sizeof(double) * k, f->d_pool + base + roff, sizeof(double) * 2 * k,
                        sizeof(double) * k, k, cudaMemcpyDeviceToHost),
           "tip");
    });
}

int64_t spk_fact_dump(const spk_fact* f, int32_t which, double* out) {
    // debug/test hook: 0 packed LU pool, 1 row-major copies, 2 1/u_jj
    const long long sz = which == 0 ? f->fac_size : which == 1 ? f->tfac_size : f->n;
    const double* src = which == 0 ? f->d_fac : which == 1 ? f->d_tfac : f->d_dinv;
    try {
        ensure_finished(f);
        if (which == 1) {
            ensure_tfac(f);
            cudaStreamSynchronize(f->stream);
        }
    } catch (...) {
    }
    if (out) cudaMemcpy(out, src, sizeof(double) * sz, cudaMemcpyDeviceToHost);
    return sz;
}

int32_t spk_fact_units(const spk_fact* f, int32_t l) {
    if (!f || l < 0 || l >= (int)f->levels.size()) return 0;
    return f->levels[l].units;
}

spk_status spk_fact_level_spike(const spk_fact* f, int32_t l, int32_t which, int32_t u, int32_t* h,
                                double* out) {
    return guarded([&] {
        ensure_finished(f);
        if (l < 0 || l + 1 >= (int)f->levels.size()) fail(SPK_ERANGE, "level_spike: level out of range");
        const Level& lv = f->levels[l];
        if (u < 0 || u >= lv.units) fail(SPK_ERANGE, "level_spike: unit out of range");
        *h = lv.uh[u];
        if (!out) return;
        const long long sz = (long long)lv.uh[u] * f->k;
        const long long off = which == 0 ? lv.voff[u] : lv.woff[u];
        if (off < 0) {
            std::fill(out, out + sz, 0.0);
            return;
        }
        ck(cudaMemcpy(out, f->d_pool + off, sizeof(double) * sz, cudaMemcpyDeviceToHost), "level_spike");
    });
}

spk_status spk_fact_coupling(const spk_fact* f, int32_t l, int32_t a, double* lu, int32_t* piv,
                             int32_t* fell_back) {
    return guarded([&] {
        ensure_finished(f);
        if (l < 0 || l + 1 >= (int)f->levels.size()) fail(SPK_ERANGE, "coupling: level out of range");
        const Level& lv = f->levels[l];
        if (a < 0 || a >= (int)lv.pair_part.size()) fail(SPK_ERANGE, "coupling: pair out of range");
        const int k = f->k, nn = 2 * k;
        const bool schur = f->flags.size() > (size_t)lv.gidx[a] && f->flags[lv.gidx[a]] == 1;
        auto unpack = [&](const PartDev& P, std::vector<double>& dense, std::vector<int>& pv) {
            std::vector<double> band((size_t)P.m * P.rows);
            ck(cudaMemcpy(band.data(), f->d_fac + P.fofs, sizeof(double) * band.size(), cudaMemcpyDeviceToHost),
               "coupling");
            dense.assign((size_t)P.m * P.m, 0.0);
            for (int j = 0; j < P.m; ++j)
                for (int i = 0; i < P.m; ++i) {
                    const int q = P.d + i - j;
                    dense[(size_t)j * P.m + i] = (q >= 0 && q < P.rows) ? band[(size_t)j * P.rows + q] : 0.0;
                }
            pv.resize(P.m);
            ck(cudaMemcpy(pv.data(), f->d_piv + P.r0, sizeof(int) * P.m, cudaMemcpyDeviceToHost), "coupling");
        };
        std::vector<double> dense;
        std::vector<int> pv;
        if (!schur) {
            unpack(f->parts[lv.pair_part[a]], dense, pv);
            std::copy(dense.begin(), dense.end(), lu);
            if (piv) std::copy(pv.begin(), pv.end(), piv);
            if (fell_back) {
                int fb = 0;
                ck(cudaMemcpy(&fb, f->d_fell + lv.pair_part[a], sizeof(int), cudaMemcpyDeviceToHost), "coupling");
                *fell_back = fb;
            }
            return;
        }
        // Schur path: [[I, 0], [W, L_S]] [[I, V], [0, U_S]] with rows k.. permuted by P_S.
        // The factorization keeps S itself (the solves use S^-1): factor a
        // scratch copy with the gbtf2-convention dense LU on demand.
        {
            PartDev S = f->parts[lv.spart[a]];
            const size_t fsz = (size_t)S.m * S.rows;
            double* d_s = nullptr;
            int* d_i = nullptr;
            void* d_meta = nullptr;
            ck(cudaMalloc(&d_s, sizeof(double) * fsz), "coupling");
            ck(cudaMalloc(&d_i, sizeof(int) * (S.m + 1)), "coupling");
            ck(cudaMalloc(&d_meta, sizeof(PartDev) + sizeof(CouplingJob)), "coupling");
            if (f->sk_schur_all) {
                // the small-k engine keeps only S^-1: S = I - Wt Vb from the level's spikes
                const int hL = lv.uh[2 * a], hR = lv.uh[2 * a + 1];
                std::vector<double> vl((size_t)hL * k), wr((size_t)hR * k), band(fsz, 0.0);
                ck(cudaMemcpy(vl.data(), f->d_pool + lv.voff[2 * a], sizeof(double) * vl.size(),
                              cudaMemcpyDeviceToHost), "coupling");
                ck(cudaMemcpy(wr.data(), f->d_pool + lv.woff[2 * a + 1], sizeof(double) * wr.size(),
                              cudaMemcpyDeviceToHost), "coupling");
                for (int j = 0; j < k; ++j)
                    for (int i = 0; i < k; ++i) {
                        double v = i == j ? 1.0 : 0.0;
                        for (int t = 0; t < k; ++t) v -= wr[(size_t)t * hR + i] * vl[(size_t)j * hL + hL - k + t];
                        const int q = S.d + i - j;
                        if (q >= 0 && q < S.rows) band[(size_t)j * S.rows + q] = v;
                    }
                ck(cudaMemcpy(d_s, band.data(), sizeof(double) * fsz, cudaMemcpyHostToDevice), "coupling");
            } else {
                ck(cudaMemcpy(d_s, f->d_fac + S.fofs, sizeof(double) * fsz, cudaMemcpyDeviceToDevice), "coupling");
            }
            S.fofs = 0;
            S.r0 = 0;
            CouplingJob J{};
            J.part = 0;
            J.k = k;
            J.guard = S.m;  // flag slot after the pivots
            const int one = 1;
            ck(cudaMemcpy(d_i + S.m, &one, sizeof(int), cudaMemcpyHostToDevice), "coupling");
            ck(cudaMemcpy(d_meta, &S, sizeof(PartDev), cudaMemcpyHostToDevice), "coupling");
            ck(cudaMemcpy((char*)d_meta + sizeof(PartDev), &J, sizeof(CouplingJob), cudaMemcpyHostToDevice),
               "coupling");
            launch_dense_lu((const CouplingJob*)((char*)d_meta + sizeof(PartDev)), 1, S.m, (const PartDev*)d_meta, d_s,
                            d_i, d_i, 0);
            ck(cudaDeviceSynchronize(), "coupling");
            std::vector<double> band(fsz);
            ck(cudaMemcpy(band.data(), d_s, sizeof(double) * fsz, cudaMemcpyDeviceToHost), "coupling");
            pv.resize(S.m);
            ck(cudaMemcpy(pv.data(), d_i, sizeof(int) * S.m, cudaMemcpyDeviceToHost), "coupling");
            cudaFree(d_s);
            cudaFree(d_i);
            cudaFree(d_meta);
            dense.assign((size_t)S.m * S.m, 0.0);
            for (int j = 0; j < S.m; ++j)
                for (int i = 0; i < S.m; ++i) {
                    const int q = S.d + i - j;
                    dense[(size_t)j * S.m + i] = (q >= 0 && q < S.rows) ? band[(size_t)j * S.rows + q] : 0.0;
                }
        }
        const int hL = lv.uh[2 * a], hR = lv.uh[2 * a + 1];
        std::vector<double> vl((size_t)hL * k), wr((size_t)hR * k);
        ck(cudaMemcpy(vl.data(), f->d_pool + lv.voff[2 * a], sizeof(double) * vl.size(), cudaMemcpyDeviceToHost),
           "coupling");
        ck(cudaMemcpy(wr.data(), f->d_pool + lv.woff[2 * a + 1], sizeof(double) * wr.size(), cudaMemcpyDeviceToHost),
           "coupling");
        std::fill(lu, lu + (size_t)nn * nn, 0.0);
        for (int j = 0; j < nn; ++j)
            for (int i = 0; i < nn; ++i) {
                double v = 0.0;
                if (j < k) {
                    if (i == j) v = 1.0;
                    else if (i >= k) v = wr[(size_t)j * hR + (i - k)];
                } else if (i < k) {
                    v = vl[(size_t)(j - k) * hL + (hL - k + i)];
                } else {
                    v = dense[(size_t)(j - k) * k + (i - k)];
                }
                lu[(size_t)j * nn + i] = v;
            }
        if (piv)
            for (int i = 0; i < nn; ++i) piv[i] = i < k ? i : k + pv[i - k];
        if (fell_back) *fell_back = 0;
    });
}

}  // extern "C"

// One solve in flight: device buffers plus the program phase it stopped at.
// A closed factorization runs every phase in one call; a slab runs up to each
// exchange point and resumes when the neighbours' blocks are imported.
struct spk_xsolve {
    spk_fact* f = nullptr;
    int transpose = 0, nrhs = 0, phase = 0, nphases = 1;
    cudaStream_t s = nullptr;
    double *S = nullptr, *T = nullptr, *AUX = nullptr, *tF = nullptr, *tX = nullptr;
    double *XCH = nullptr, *XIN = nullptr;
    // small-k engine (k_sk_solve): grid-barrier words + tree counters, z blocks
    bool sk = false;
    unsigned* bar = nullptr;
    double* ZS = nullptr;
    Bufs B;

    ~spk_xsolve() {
        for (double* q : {S, T, AUX, tF, tX, XCH, XIN, ZS})
            if (q) dfree(q, s);
        if (bar) dfree(bar, s);
    }
    const Program& prog() const { return transpose ? f->prog_tr : f->prog_fwd; }
    // rows of the export block after phase q (column-major, ld = rows)
    int export_rows(int q) const { return (transpose && q == 1) ? 4 * f->k : 2 * f->k; }
    void run_phase() {
        if (sk) {
            const char* blob = f->d_blob;
            SkSolveArgs A{f->d_parts, f->p, f->k, nrhs, f->d_fac, f->fac_size, f->d_pool, f->off_bhat, f->off_chat,
                          reinterpret_cast<const SkUnit*>(blob + f->sk_units),
                          reinterpret_cast<const SkPair*>(blob + f->sk_pairs),
                          reinterpret_cast<const SkItem*>(blob + f->sk_items),
                          reinterpret_cast<const SkLevel*>(blob + f->sk_levels), f->sk_nlevels, B.p[B_F], B.ld[B_F],
                          B.p[B_X], B.ld[B_X], T, ZS, bar + 2, bar, f->sk_mmax, f->sk_rmax,
                          g_sk_trace ? g_sk_trace + 4096 * 16 : nullptr};
            ProfScope ps(ST_SWEEP, s, 8.0 * f->n * f->k * nrhs, 16.0 * f->n * (f->kl + f->ku + 1));
            launch_sk_solve(A, s);
            ++phase;
            return;
        }
        Exec ex{*f, s, B, nrhs};
        ex.n = f->n;
        if (phase + 1 < nphases) {
            B.ld[B_XCH] = export_rows(phase);
            ex.B.ld[B_XCH] = B.ld[B_XCH];
        }
        ex.run(prog(), f->d_sblob, f->open() ? phase : -1);
        ++phase;
    }
};

namespace {

// Validates the call and sets up buffers; F/X device (or host with staging).
std::unique_ptr<spk_xsolve> open_solve(const spk_fact* fc, int32_t transpose, const double* F, int64_t ldf,
                                       int32_t nrhs, double* X, int64_t ldx, int32_t mem, cudaStream_t s) {
    spk_fact& f = const_cast<spk_fact&>(*fc);
    const long long n = f.n;
    const bool sk_kernel = sk_kernel_solve(f, transpose, nrhs);
    if (transpose) ensure_tfac(fc);  // only the transposed sweeps read the row-major copy
    wait_ready(f, s);
    auto x = std::make_unique<spk_xsolve>();
    x->f = &f;
    x->transpose = transpose;
    x->nrhs = nrhs;
    x->s = s;
    x->nphases = f.open() ? (transpose ? 3 : 2) : 1;
    const double* dF = F;
    double* dX = X;
    long long lf = ldf, lx = ldx;
    if (mem == SPK_MEM_HOST) {
        x->tF = dalloc<double>((size_t)n * nrhs, s);
        x->tX = dalloc<double>((size_t)n * nrhs, s);
        ck(cudaMemcpy2DAsync(x->tF, sizeof(double) * n, F, sizeof(double) * ldf, sizeof(double) * n, nrhs,
                             cudaMemcpyHostToDevice, s),
           "F upload");
        dF = x->tF;
        dX = x->tX;
        lf = lx = n;
    } else if (transpose || f.coupled()) {
        // both programs re-read F after writing X (the transpose program's
        // G tips, the forward retrieval's re-solve): never alias
        const char* f0 = (const char*)F;
        const char* f1 = (const char*)(F + ldf * (nrhs - 1) + n);
        const char* x0 = (const char*)X;
        const char* x1 = (const char*)(X + ldx * (nrhs - 1) + n);
        if (!(f1 <= x0 || x1 <= f0)) {
            x->tF = dalloc<double>((size_t)n * nrhs, s);
            ck(cudaMemcpy2DAsync(x->tF, sizeof(double) * n, F, sizeof(double) * ldf, sizeof(double) * n, nrhs,
                                 cudaMemcpyDeviceToDevice, s),
               "F copy");
            dF = x->tF;
            lf = n;
        }
    }
    Bufs& B = x->B;
    B = make_bufs(&f);
    B.p[B_X] = dX;
    B.ld[B_X] = lx;
    B.p[B_F] = const_cast<double*>(dF);
    B.ld[B_F] = lf;
    if (f.coupled()) {
        const long long H = 2LL * f.p * f.k, halo = f.open() ? f.k : 0;
        if (transpose) x->S = dalloc<double>((size_t)n * nrhs, s);  // tau (the forward solve needs none)
        x->T = dalloc<double>((size_t)(H + 2 * halo) * nrhs, s);
        if (!sk_kernel) x->AUX = dalloc<double>((size_t)f.aux_rows * nrhs, s);
        if (f.open()) {
            // dead tips of closed edges are read (times zero) by transposed
            // pair solves: keep them finite
            ck(cudaMemsetAsync(x->T, 0, sizeof(double) * (H + 2 * halo) * nrhs, s), "memset");
            x->XCH = dalloc<double>((size_t)4 * f.k * nrhs, s);
            x->XIN = dalloc<double>((size_t)2 * f.k * nrhs, s);
        }
        B.p[B_S] = x->S;
        B.ld[B_S] = n;
        B.p[B_T] = x->T + halo;
        B.ld[B_T] = H + 2 * halo;
        B.p[B_AUX] = x->AUX;
        B.ld[B_AUX] = f.aux_rows;
        B.p[B_XCH] = x->XCH;
        B.ld[B_XCH] = 2 * f.k;
        B.p[B_XIN] = x->XIN;
        B.ld[B_XIN] = 2 * f.k;
    }
    B.p[B_POOL] = f.d_pool;
    B.ld[B_POOL] = 1;
    // forward solves with few right-hand sides of a small-k factorization
    // whose pairs all took the Schur path: one cooperative kernel
    if (sk_kernel) {
        x->sk = true;
        const long long H = 2LL * f.p * f.k;
        // grid-barrier words, then the reduced-solve tree's per-pair counters
        const size_t nw = 2 + (size_t)std::max(f.npairs, 1);
        x->bar = static_cast<unsigned*>(arena().alloc(nw * sizeof(unsigned), s));
        ck(cudaMemsetAsync(x->bar, 0, nw * sizeof(unsigned), s), "memset");
        x->ZS = dalloc<double>((size_t)std::max(f.npairs, 1) * 32 * 8, s);
        B.ld[B_T] = H;
        B.p[B_T] = x->T;
    }
    return x;
}

// Host-buffer solve, pipelined over right-hand-side column chunks: uploads
// run ahead on one copy stream, downloads follow on another, so PCIe in both
// directions overlaps the solve of the neighbouring chunks (columns are
// independent; each chunk runs the full program on its columns).
struct CopyStreams {
    cudaStream_t up = nullptr, down = nullptr;
    int dev = -1;
};
CopyStreams& copy_streams() {
    static thread_local CopyStreams cs;
    int dev = 0;
    cudaGetDevice(&dev);
    if (cs.dev != dev) {
        ck(cudaStreamCreateWithFlags(&cs.up, cudaStreamNonBlocking), "copy stream");
        ck(cudaStreamCreateWithFlags(&cs.down, cudaStreamNonBlocking), "copy stream");
        cs.dev = dev;
    }
    return cs;
}

void solve_host_pipelined(const spk_fact* fc, int32_t transpose, const double* F, int64_t ldf, int32_t nrhs,
                          double* X, int64_t ldx, cudaStream_t s) {
    const long long n = fc->n;
    // no host wait for a pending factorization: its guarded solve programs
    // are used, and fin_mu keeps a concurrent finish from swapping them while
    // this call enqueues
    spk_fact& fm = const_cast<spk_fact&>(*fc);
    if (fm.sk) ensure_finished(fc);  // (the small-k engine has no device-guarded programs)
    if (transpose) ensure_tfac(fc);
    std::lock_guard<std::mutex> lk(fm.fin_mu);
    if (!fm.pending.load() && fm.fin_status != SPK_OK) fail(fm.fin_status, fm.fin_msg);
    CopyStreams& cs = copy_streams();
    // three column chunks: enough to hide the solve behind PCIe in both
    // directions while each chunk still fills the sweep kernels
    constexpr int want = 3;
    const int chunk = std::max(16, ((nrhs + want - 1) / want + 7) / 8 * 8);
    const int nch = (nrhs + chunk - 1) / chunk;
    // F's staging buffer belongs to the upload stream, so the uploads start
    // at once -- under a still running factorization (stream-ordered
    // spk_factorize) or the previous call's downloads
    double* dF = dalloc<double>((size_t)n * nrhs, cs.up);
    if (fc->upload_ev) ck(cudaStreamWaitEvent(cs.up, fc->upload_ev, 0), "wait");  // PCIe: the band first
    std::vector<cudaEvent_t> ev(3 * nch);
    for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (int c = 0; c < nch; ++c) {
        const int c0 = c * chunk, nc = std::min(chunk, nrhs - c0);
        ck(cudaMemcpy2DAsync(dF + (size_t)c0 * n, sizeof(double) * n, F + (size_t)c0 * ldf, sizeof(double) * ldf,
                             sizeof(double) * n, nc, cudaMemcpyHostToDevice, cs.up),
           "F upload");
        ck(cudaEventRecord(ev[c], cs.up), "event");
    }
    // no host wait: while the factorization is pending its solve programs are
    // device-guarded on the coupling paths
    double* dX = dalloc<double>((size_t)n * nrhs, s);
    for (int c = 0; c < nch; ++c) {
        const int c0 = c * chunk, nc = std::min(chunk, nrhs - c0);
        ck(cudaStreamWaitEvent(s, ev[c], 0), "wait");
        {
            auto x = open_solve(fc, transpose, dF + (size_t)c0 * n, n, nc, dX + (size_t)c0 * n, n, SPK_MEM_DEVICE, s);
            x->run_phase();
        }
        ck(cudaEventRecord(ev[nch + c], s), "event");
        ck(cudaStreamWaitEvent(cs.down, ev[nch + c], 0), "wait");
        ck(cudaMemcpy2DAsync(X + (size_t)c0 * ldx, sizeof(double) * ldx, dX + (size_t)c0 * n, sizeof(double) * n,
                             sizeof(double) * n, nc, cudaMemcpyDeviceToHost, cs.down),
           "X download");
        ck(cudaEventRecord(ev[2 * nch + c], cs.down), "event");
    }
    dfree(dF, s);  // last read by the solve on s
    // stream-ordered completion: s (and whoever synchronises it) is ordered
    // after the downloads; the host is not blocked
    ck(cudaStreamWaitEvent(s, ev[3 * nch - 1], 0), "wait");
    note_use(*fc, s);
    dfree(dX, s);
    ck(cudaGetLastError(), "solve kernels");
    for (auto& e : ev) cudaEventDestroy(e);
}

void fill_stats(const spk_fact& f, spk_solve_stats* stats) {
    if (!stats) return;
    if (stats->partition_full_sweeps)
        for (int i = 0; i < f.p; ++i) {
            const bool edge = f.first(i) || f.last(i);
            stats->partition_full_sweeps[i] = !f.coupled() ? 2 : (edge ? 2 : 4);
        }
    stats->reduced_coupling_solves = f.coupled() ? f.p - 1 : 0;
}

}  // namespace

extern "C" {

spk_status spk_solve(const spk_fact* fc, int32_t transpose, const double* F, int64_t ldf, int32_t nrhs,
                     double* X, int64_t ldx, int32_t mem, void* stream, spk_solve_stats* stats) {
    return guarded([&] {
        if (!fc) fail(SPK_EINVAL, "solve: null factorization handle");
        if (nrhs > 0 && (!F || !X)) fail(SPK_EINVAL, "solve: null F or X");
        const spk_fact& f = *fc;
        const long long n = f.n;
        if (nrhs < 0) fail(SPK_EINVAL, "solve: negative nrhs");
        if (ldf < n || ldx < n) fail(SPK_EINVAL, transpose ? "transpose_solve: F.rows must equal n"
                                                           : "solve: F.rows must equal n");
        if (f.open()) fail(SPK_EINVAL, "solve: slab factorization (open edges) needs spk_xsolve_begin");
        fill_stats(f, stats);
        if (nrhs == 0) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (mem == SPK_MEM_HOST && nrhs >= 32) {
            solve_host_pipelined(fc, transpose, F, ldf, nrhs, X, ldx, s);
            return;
        }
        // the small-k engine's own solve kernel reads only device state: no
        // host finish (and no host wait) before it
        if (!sk_kernel_solve(f, transpose, nrhs)) ensure_finished(fc);
        auto x = open_solve(fc, transpose, F, ldf, nrhs, X, ldx, mem, s);
        x->run_phase();
        note_use(f, s);
        if (mem == SPK_MEM_HOST)
            ck(cudaMemcpy2DAsync(X, sizeof(double) * ldx, x->tX, sizeof(double) * n, sizeof(double) * n, nrhs,
                                 cudaMemcpyDeviceToHost, s),
               "X download");
        x.reset();
        ck(cudaGetLastError(), "solve kernels");
        if (mem == SPK_MEM_HOST) ck(cudaStreamSynchronize(s), "solve");
    });
}

int32_t spk_xsolve_exchanges(const spk_fact* f, int32_t transpose) {
    return f && f->open() && f->coupled() ? (transpose ? 2 : 1) : 0;
}

spk_status spk_xsolve_begin(const spk_fact* f, int32_t transpose, const double* d_F, int64_t ldf, int32_t nrhs,
                            double* d_X, int64_t ldx, void* stream, double* d_export, spk_xsolve** out) {
    return guarded([&] {
        if (!out) fail(SPK_EINVAL, "xsolve: null output");
        *out = nullptr;
        ensure_finished(f);
        if (nrhs < 1) fail(SPK_EINVAL, "xsolve: nrhs must be positive");
        if (ldf < f->n || ldx < f->n) fail(SPK_EINVAL, "xsolve: F.rows must equal n");
        if (!f->open() || !f->coupled()) fail(SPK_EINVAL, "xsolve: not a slab factorization");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        auto x = open_solve(f, transpose, d_F, ldf, nrhs, d_X, ldx, SPK_MEM_DEVICE, s);
        x->run_phase();
        const long long rows = x->export_rows(0);
        ck(cudaMemcpyAsync(d_export, x->XCH, sizeof(double) * rows * nrhs, cudaMemcpyDeviceToDevice, s), "export");
        ck(cudaGetLastError(), "xsolve");
        note_use(*f, s);
        *out = x.release();
    });
}

spk_status spk_xsolve_step(spk_xsolve* x, const double* d_import, double* d_export) {
    return guarded([&] {
        if (!x) fail(SPK_EINVAL, "xsolve: null handle");
        if (x->phase >= x->nphases) fail(SPK_EINVAL, "xsolve: solve already complete");
        const long long k = x->f->k;
        ck(cudaMemcpyAsync(x->XIN, d_import, sizeof(double) * 2 * k * x->nrhs, cudaMemcpyDeviceToDevice, x->s),
           "import");
        const int q = x->phase;
        x->run_phase();
        if (x->phase < x->nphases && d_export)
            ck(cudaMemcpyAsync(d_export, x->XCH, sizeof(double) * x->export_rows(q) * x->nrhs,
                               cudaMemcpyDeviceToDevice, x->s),
               "export");
        ck(cudaGetLastError(), "xsolve");
        note_use(*x->f, x->s);
    });
}

void spk_xsolve_end(spk_xsolve* x) { delete x; }

// The slab-level (or any) reduced system from its units' tips.  load(l0,
// pool) writes each unit's [vt; vb] / [wt; wb] (2k x k, column-major) at
// l0.voff / l0.woff; everything else runs on stream s.
}  // extern "C"
template <class Load>
static spk_status reduced_create_impl(int32_t p, int32_t k, double boost_eps, cudaStream_t s, spk_reduced** out,
                                      Load load) {
    return guarded([&] {
        if (!out) fail(SPK_EINVAL, "reduce_factorize: null output");
        *out = nullptr;
        if (p < 1 || k < 0) fail(SPK_EINVAL, "reduce_factorize: bad shape");
        auto r = std::make_unique<spk_reduced>();
        r->f = std::make_unique<spk_fact>();
        spk_fact& f = *r->f;
        f.reduced_only = true;
        f.n = 2LL * p * k;
        f.k = k;
        f.kl = f.ku = k;
        f.p = p;
        f.boost_eps = boost_eps > 0 ? boost_eps : std::sqrt(DBL_EPSILON);
        f.bounds.assign(p + 1, 0);
        f.stream = s;
        setup_fact(f, s);
        if (p > 1 && k > 0) {
            load(f.levels[0], f.d_pool);
            double* auxf = dalloc<double>((size_t)f.auxf_rows * k, s);
            Bufs B = make_bufs(&f);
            B.p[B_POOL] = f.d_pool;
            B.p[B_AUX] = auxf;
            B.ld[B_AUX] = f.auxf_rows;
            Exec ex{f, s, B, k};
            ex.run(f.prog_factor, f.d_blob);
            ex.run(f.prog_levels, f.d_blob);
            dfree(auxf, s);
        }
        finish_factor(f, s);
        *out = r.release();
    });
}
extern "C" {

spk_status spk_reduced_create(const double* vt, const double* vb, const double* wt, const double* wb, int32_t p,
                              int32_t k, double boost_eps, spk_reduced** out) {
    if (p > 1 && k > 0 && (!vt || !vb || !wt || !wb)) {
        if (out) *out = nullptr;
        return guarded([] { fail(SPK_EINVAL, "reduce_factorize: null tips"); });
    }
    const long long kk = (long long)k * k;
    return reduced_create_impl(p, k, boost_eps, nullptr, out, [&](const Level& l0, double* pool) {
        std::vector<double> col(2 * kk);
        auto put = [&](long long off, const double* top, const double* bot) {
            for (int c = 0; c < k; ++c)
                for (int q = 0; q < k; ++q) {
                    col[(size_t)c * 2 * k + q] = top[(size_t)c * k + q];
                    col[(size_t)c * 2 * k + k + q] = bot[(size_t)c * k + q];
                }
            ck(cudaMemcpy(pool + off, col.data(), sizeof(double) * 2 * kk, cudaMemcpyHostToDevice), "tips");
        };
        for (int i = 0; i < p; ++i) {
            if (l0.voff[i] >= 0) put(l0.voff[i], vt + i * kk, vb + i * kk);
            if (l0.woff[i] >= 0) put(l0.woff[i], wt + i * kk, wb + i * kk);
        }
    });
}

spk_status spk_reduced_create_device(const double* d_tips, int32_t p, int32_t k, double boost_eps, void* stream,
                                     spk_reduced** out) {
    if (p > 1 && k > 0 && !d_tips) {
        if (out) *out = nullptr;
        return guarded([] { fail(SPK_EINVAL, "reduce_factorize: null tips"); });
    }
    const long long kk = (long long)k * k;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return reduced_create_impl(p, k, boost_eps, s, out, [&](const Level& l0, double* pool) {
        // unit i's tips [vt; vb; wt; wb] at d_tips + 4 i k^2: columns of vt and vb
        // interleave into the 2k x k unit spike (two strided copies each)
        auto put = [&](long long off, const double* top, const double* bot) {
            ck(cudaMemcpy2DAsync(pool + off, sizeof(double) * 2 * k, top, sizeof(double) * k, sizeof(double) * k, k,
                                 cudaMemcpyDeviceToDevice, s),
               "tips");
            ck(cudaMemcpy2DAsync(pool + off + k, sizeof(double) * 2 * k, bot, sizeof(double) * k, sizeof(double) * k,
                                 k, cudaMemcpyDeviceToDevice, s),
               "tips");
        };
        for (int i = 0; i < p; ++i) {
            const double* t = d_tips + 4 * i * kk;
            if (l0.voff[i] >= 0) put(l0.voff[i], t, t + kk);
            if (l0.woff[i] >= 0) put(l0.woff[i], t + 2 * kk, t + 3 * kk);
        }
    });
}

static spk_status reduced_solve_on(spk_fact& f, bool own_programs, int32_t transpose, double* z, int32_t ncols,
                                   int64_t* couplings, bool device = false, cudaStream_t s = nullptr) {
    return guarded([&] {
        if (couplings) *couplings += (f.p > 1 && f.k > 0) ? f.p - 1 : 0;
        if (ncols == 0 || f.p < 2 || f.k == 0) return;
        wait_ready(f, s);
        const long long rows = 2LL * f.p * f.k;
        double* T = device ? z : dalloc<double>((size_t)rows * ncols, s);
        double* AUX = dalloc<double>((size_t)f.aux_rows * ncols, s);
        if (!device) ck(cudaMemcpyAsync(T, z, sizeof(double) * rows * ncols, cudaMemcpyHostToDevice, s), "z upload");
        Bufs B = make_bufs(&f);
        B.p[B_T] = T;
        B.ld[B_T] = rows;
        B.p[B_AUX] = AUX;
        B.ld[B_AUX] = f.aux_rows;
        B.p[B_POOL] = f.d_pool;
        Exec ex{f, s, B, ncols};
        ex.run(own_programs ? (transpose ? f.prog_tr : f.prog_fwd) : (transpose ? f.prog_rtr : f.prog_rfwd), f.d_sblob);
        dfree(AUX, s);
        note_use(f, s);
        if (device) {
            ck(cudaGetLastError(), "reduced_solve");
            return;
        }
        ck(cudaMemcpyAsync(z, T, sizeof(double) * rows * ncols, cudaMemcpyDeviceToHost, s), "z download");
        dfree(T, s);
        ck(cudaStreamSynchronize(s), "reduced_solve");
    });
}

spk_status spk_reduced_solve_device(const spk_reduced* r, int32_t transpose, double* d_z, int32_t ncols,
                                    void* stream) {
    return reduced_solve_on(*r->f, true, transpose, d_z, ncols, nullptr, true, static_cast<cudaStream_t>(stream));
}

spk_status spk_reduced_solve(const spk_reduced* r, int32_t transpose, double* z, int32_t ncols,
                             int64_t* couplings) {
    return reduced_solve_on(*r->f, true, transpose, z, ncols, couplings);
}

spk_status spk_fact_reduced_solve(const spk_fact* f, int32_t transpose, double* z, int32_t ncols,
                                  int64_t* couplings) {
    const spk_status st = guarded([&] { ensure_finished(f); });
    if (st != SPK_OK) return st;
    return reduced_solve_on(const_cast<spk_fact&>(*f), false, transpose, z, ncols, couplings);
}

int32_t spk_reduced_levels(const spk_reduced* r) {
    return r->f->levels.empty() ? 0 : (int)r->f->levels.size() - 1;
}
int32_t spk_reduced_boost_warnings(const spk_reduced* r) { return r->f->boost_warnings; }
const spk_fact* spk_reduced_fact(const spk_reduced* r) { return r ? r->f.get() : nullptr; }
void spk_reduced_destroy(spk_reduced* r) { delete r; }

spk_status spk_band_matmul(const double* band, int64_t n, int32_t kl, int32_t ku, const double* X, int64_t ldx,
                           int32_t ncols, int32_t transpose, double* Y, int64_t ldy, int32_t mem, void* stream) {
    return guarded([&] {
        if (ldx < n || ldy < n) fail(SPK_EINVAL, "band_matmul: X.rows must equal n");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (ncols == 0) return;
        if (mem == SPK_MEM_DEVICE) {
            launch_band_mm(band, n, kl, ku, X, ldx, ncols, transpose, nullptr, 0, Y, ldy, s);
            ck(cudaGetLastError(), "band_matmul");
            return;
        }
        const long long ld = kl + ku + 1;
        double* db = dalloc<double>((size_t)ld * n, s);
        double* dx = dalloc<double>((size_t)n * ncols, s);
        double* dy = dalloc<double>((size_t)n * ncols, s);
        ck(cudaMemcpyAsync(db, band, sizeof(double) * ld * n, cudaMemcpyHostToDevice, s), "upload");
        ck(cudaMemcpy2DAsync(dx, sizeof(double) * n, X, sizeof(double) * ldx, sizeof(double) * n, ncols,
                             cudaMemcpyHostToDevice, s),
           "upload");
        launch_band_mm(db, n, kl, ku, dx, n, ncols, transpose, nullptr, 0, dy, n, s);
        ck(cudaMemcpy2DAsync(Y, sizeof(double) * ldy, dy, sizeof(double) * n, sizeof(double) * n, ncols,
                             cudaMemcpyDeviceToHost, s),
           "download");
        for (double* q : {db, dx, dy}) dfree(q, s);
        ck(cudaStreamSynchronize(s), "band_matmul");
    });
}

// ---------------------------------------------------------------------------
// verification and refinement on the device
}  // extern "C"

namespace {

// per-column {sum|x|, sum x^2, max|x|} of an n x ncols device block, to the host
std::vector<double> col_stats_host(const double* X, long long ldx, long long n, int ncols, cudaStream_t s) {
    std::vector<double> h((size_t)3 * ncols);
    if (ncols <= 0) return h;
    const int nblk = col_stats_blocks(n);
    double* part = dalloc<double>((size_t)3 * nblk * ncols, s);
    double* out = dalloc<double>((size_t)3 * ncols, s);
    launch_col_stats(X, ldx, n, ncols, part, out, s);
    ck(cudaGetLastError(), "col_stats");
    ck(cudaMemcpyAsync(h.data(), out, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s), "col_stats");
    ck(cudaStreamSynchronize(s), "col_stats");
    dfree(part, s);
    dfree(out, s);
    return h;
}

void device_solve(const spk_fact* fc, int transpose, const double* F, long long ldf, int nrhs, double* X,
                  long long ldx, cudaStream_t s) {
    ensure_finished(fc);
    auto x = open_solve(fc, transpose, F, ldf, nrhs, X, ldx, SPK_MEM_DEVICE, s);
    x->run_phase();
    note_use(*fc, s);
}

}  // namespace

extern "C" {

spk_status spk_residual_device(const double* d_band, int64_t n, int32_t kl, int32_t ku, const double* d_X,
                               int64_t ldx, const double* d_F, int64_t ldf, int32_t ncols, int32_t transpose,
                               double* d_R, int64_t ldr, void* stream, double* out) {
    return guarded([&] {
        if (n < 1 || kl < 0 || ku < 0) fail(SPK_EINVAL, "residual: bad shape");
        if (ldx < n || ldf < n || (d_R && ldr < n)) fail(SPK_EINVAL, "residual: X.rows must equal n");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (ncols <= 0) return;
        double* R = d_R;
        long long lr = ldr;
        if (!R) {
            R = dalloc<double>((size_t)n * ncols, s);
            lr = n;
        }
        launch_band_mm(d_band, n, kl, ku, d_X, ldx, ncols, transpose, d_F, ldf, R, lr, s);
        ck(cudaGetLastError(), "residual");
        const std::vector<double> sr = col_stats_host(R, lr, n, ncols, s);
        const std::vector<double> sf = col_stats_host(d_F, ldf, n, ncols, s);
        const std::vector<double> sx = col_stats_host(d_X, ldx, n, ncols, s);
        if (!d_R) dfree(R, s);
        for (int c = 0; c < ncols; ++c) {
            out[4 * c + 0] = sr[3 * c + 1];
            out[4 * c + 1] = sf[3 * c + 1];
            out[4 * c + 2] = sr[3 * c + 2];
            out[4 * c + 3] = sx[3 * c + 2];
        }
    });
}

spk_status spk_band_norms_device(const double* d_band, int64_t n, int32_t kl, int32_t ku, void* stream,
                                 double* out) {
    return guarded([&] {
        if (n < 1 || kl < 0 || ku < 0) fail(SPK_EINVAL, "band_norms: bad shape");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        unsigned long long* d = dalloc<unsigned long long>(3, s);
        ck(cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), s), "band_norms");
        launch_band_norms(d_band, n, kl, ku, d, s);
        ck(cudaGetLastError(), "band_norms");
        unsigned long long h[3];
        ck(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s), "band_norms");
        ck(cudaStreamSynchronize(s), "band_norms");
        dfree(d, s);
        for (int i = 0; i < 3; ++i) out[i] = __builtin_bit_cast(double, h[i]);
    });
}

}  // extern "C"

namespace {
void refine_on_device(const spk_fact* fc, const double* d_band, const double* d_F, int64_t ldf, int32_t nrhs,
                      double* d_X, int64_t ldx, int32_t transpose, int32_t max_iters, double tol, cudaStream_t s,
                      spk_refine_result* res) {
        const spk_fact& f = *fc;
        const long long n = f.n;
        *res = spk_refine_result{0, 0, 0, 0.0};
        // ||F||_F (band_ops.cpp frobenius_norm), column sums of squares in order
        double fn2 = 0.0;
        {
            const std::vector<double> sf = col_stats_host(d_F, ldf, n, nrhs, s);
            for (int c = 0; c < nrhs; ++c) fn2 += sf[3 * c + 1];
        }
        const double fnorm = std::sqrt(fn2);
        double* R = dalloc<double>((size_t)n * std::max(nrhs, 1), s);
        double prev = INFINITY;
        for (int it = 0; it <= max_iters; ++it) {
            // r = f - op(A) x  (solve.cpp:412-413)
            if (nrhs > 0) launch_band_mm(d_band, n, f.kl, f.ku, d_X, ldx, nrhs, transpose, d_F, ldf, R, n, s);
            ck(cudaGetLastError(), "iterative_refine");
            double rn2 = 0.0;
            const std::vector<double> sr = col_stats_host(R, n, n, nrhs, s);
            for (int c = 0; c < nrhs; ++c) rn2 += sr[3 * c + 1];
            const double rn = std::sqrt(rn2);
            res->residual = fnorm == 0.0 ? (rn == 0.0 ? 0.0 : INFINITY) : rn / fnorm;
            res->iterations = it;
            if (res->residual <= tol) {
                res->converged = 1;
                break;
            }
            if (it > 0 && res->residual * 1.1 > prev) {
                res->stagnated = 1;
                break;
            }
            if (it == max_iters) break;
            prev = res->residual;
            // d = op(A)^-1 r in place; x += d  (solve.cpp:427-429)
            device_solve(fc, transpose, R, n, nrhs, R, n, s);
            launch_axpy(d_X, ldx, R, n, n, nrhs, s);
            ck(cudaGetLastError(), "iterative_refine");
        }
        dfree(R, s);
}

// a host band / block staged on the device (arena), or the caller's device pointer
struct Staged {
    double* p = nullptr;
    bool own = false;
    cudaStream_t s = nullptr;
    Staged(const double* src, long long rows, long long ld, int cols, int mem, cudaStream_t st) : s(st) {
        if (mem == SPK_MEM_DEVICE) {
            p = const_cast<double*>(src);
            return;
        }
        own = true;
        p = dalloc<double>((size_t)rows * std::max(cols, 1), s);
        if (cols > 0)
            ck(cudaMemcpy2DAsync(p, sizeof(double) * rows, src, sizeof(double) * ld, sizeof(double) * rows, cols,
                                 cudaMemcpyHostToDevice, s),
               "upload");
    }
    ~Staged() {
        if (own) dfree(p, s);
    }
};
}  // namespace

extern "C" {

spk_status spk_refine(const spk_fact* fc, const double* band, const double* F, int64_t ldf, int32_t nrhs, double* X,
                      int64_t ldx, int32_t transpose, int32_t max_iters, double tol, int32_t mem, void* stream,
                      spk_refine_result* res) {
    return guarded([&] {
        if (!fc) fail(SPK_EINVAL, "null factorization handle");
        const spk_fact& f = *fc;
        const long long n = f.n;
        if (ldf < n || ldx < n) fail(SPK_EINVAL, "iterative_refine: F.rows must equal n");
        if (f.open()) fail(SPK_EINVAL, "iterative_refine: slab factorization");
        if (nrhs < 0 || max_iters < 0) fail(SPK_EINVAL, "iterative_refine: negative nrhs or max_iters");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const long long ld = f.kl + f.ku + 1;
        Staged b(band, ld * n, ld * n, 1, mem, s), fs(F, n, ldf, nrhs, mem, s), xs(X, n, ldx, nrhs, mem, s);
        const long long lf = mem == SPK_MEM_DEVICE ? ldf : n, lx = mem == SPK_MEM_DEVICE ? ldx : n;
        refine_on_device(fc, b.p, fs.p, lf, nrhs, xs.p, lx, transpose, max_iters, tol, s, res);
        if (mem != SPK_MEM_DEVICE && nrhs > 0)
            ck(cudaMemcpy2DAsync(X, sizeof(double) * ldx, xs.p, sizeof(double) * n, sizeof(double) * n, nrhs,
                                 cudaMemcpyDeviceToHost, s),
               "download");
        ck(cudaStreamSynchronize(s), "iterative_refine");
    });
}

spk_status spk_condest_1norm(const spk_fact* fc, const double* band, int32_t mem, void* stream, double* cond) {
    return guarded([&] {
        if (!fc) fail(SPK_EINVAL, "null factorization handle");
        const spk_fact& f = *fc;
        const long long n = f.n;
        if (f.open()) fail(SPK_EINVAL, "condition_estimate: slab factorization");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const long long ld = f.kl + f.ku + 1;
        Staged b(band, ld * n, ld * n, 1, mem, s);
        const double* d_band = b.p;
        double norms[3];
        spk_status st = spk_band_norms_device(d_band, n, f.kl, f.ku, stream, norms);
        if (st != SPK_OK) fail(st, g_err.c_str());
        double* x = dalloc<double>((size_t)n, s);
        double* y = dalloc<double>((size_t)n, s);
        double* xi = dalloc<double>((size_t)n, s);
        const int nblk = dot_argmax_blocks(n);
        double* part = dalloc<double>((size_t)3 * nblk, s);
        std::vector<double> hp((size_t)3 * nblk);
        launch_fill(x, n, 1.0 / n, s);
        double est = 0.0;
        // Hager / Higham 1-norm estimator, oracle.cpp:132-166: at most 6 steps
        for (int it = 0; it < 6; ++it) {
            device_solve(fc, 0, x, n, 1, y, n, s);
            const std::vector<double> sy = col_stats_host(y, n, n, 1, s);
            est = std::max(est, sy[0]);
            launch_sign(y, xi, n, s);
            device_solve(fc, 1, xi, n, 1, xi, n, s);
            launch_dot_argmax(xi, x, n, part, s);
            ck(cudaGetLastError(), "condition_estimate");
            ck(cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, s),
               "condition_estimate");
            ck(cudaStreamSynchronize(s), "condition_estimate");
            double zdx = 0.0, zmax = -1.0;
            long long jmax = 0;
            for (int b = 0; b < nblk; ++b) {  // blocks in index order: first max wins
                zdx += hp[3 * b];
                if (hp[3 * b + 1] > zmax) {
                    zmax = hp[3 * b + 1];
                    jmax = (long long)hp[3 * b + 2];
                }
            }
            if (zmax <= zdx) break;
            launch_unit(x, n, jmax, s);
        }
        for (double* q : {x, y, xi, part}) dfree(q, s);
        ck(cudaStreamSynchronize(s), "condition_estimate");
        *cond = est * norms[0];
    });
}

// ---------------------------------------------------------------------------
// .spkb files (band_io.cpp:98-143)
}  // extern "C"

namespace {

constexpr long long kSpkbHeader = 4 + 3 * 8;

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

void full_pread(int fd, void* dst, size_t bytes, long long off, const char* what) {
    char* p = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t r = pread(fd, p, bytes, off);
        if (r <= 0) fail(SPK_EIO, what);
        p += r;
        bytes -= (size_t)r;
        off += r;
    }
}

void full_write(int fd, const void* src, size_t bytes, const std::string& path) {
    const char* p = static_cast<const char*>(src);
    while (bytes > 0) {
        const ssize_t r = write(fd, p, bytes);
        if (r <= 0) fail(SPK_EIO, "write to " + path + " failed");
        p += r;
        bytes -= (size_t)r;
    }
}

// header + size check; little-endian host (x86-64 / aarch64) assumed, like the
// reference's get_i64 / get_f64 byte order
void spkb_open(const char* path, Fd& f, long long& n, int& kl, int& ku) {
    static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "spkb: little-endian host");
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) fail(SPK_EIO, std::string("cannot open ") + path);
    char head[kSpkbHeader];
    struct stat st;
    if (fstat(f.fd, &st) != 0) fail(SPK_EIO, std::string("cannot open ") + path);
    if (st.st_size < 4 || pread(f.fd, head, 4, 0) != 4 || std::memcmp(head, "SPKB", 4) != 0)
        fail(SPK_EIO, "bad SPKB magic");
    if (st.st_size < kSpkbHeader) fail(SPK_EIO, "SPKB file truncated");
    full_pread(f.fd, head, kSpkbHeader, 0, "SPKB file truncated");
    int64_t v[3];
    std::memcpy(v, head + 4, sizeof(v));
    if (v[0] < 1 || v[1] < 0 || v[2] < 0 || v[1] >= v[0] || v[2] >= v[0]) fail(SPK_EIO, "bad SPKB dimensions");
    n = v[0];
    kl = (int)v[1];
    ku = (int)v[2];
    if ((long long)st.st_size < kSpkbHeader + 8LL * (kl + ku + 1) * n) fail(SPK_EIO, "SPKB file truncated");
}

// two pinned staging buffers, cached per thread (pinned allocation is slow)
struct Staging {
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    size_t bytes = 0;
};
Staging& staging(size_t want) {
    static thread_local Staging st;
    if (st.bytes < want) {
        for (int i = 0; i < 2; ++i) {
            if (st.buf[i]) cudaFreeHost(st.buf[i]);
            if (st.ev[i]) cudaEventDestroy(st.ev[i]);
            ck(cudaHostAlloc(&st.buf[i], want, cudaHostAllocDefault), "pinned staging");
            ck(cudaEventCreateWithFlags(&st.ev[i], cudaEventDisableTiming), "event");
        }
        st.bytes = want;
    }
    return st;
}

size_t spkb_chunk_bytes() { return (size_t)64 << 20; }

}  // namespace

extern "C" {

spk_status spk_spkb_header(const char* path, int64_t* n, int32_t* kl, int32_t* ku) {
    return guarded([&] {
        Fd f;
        long long nn;
        int a, b;
        spkb_open(path, f, nn, a, b);
        *n = nn;
        *kl = a;
        *ku = b;
    });
}

spk_status spk_spkb_load(const char* path, int64_t col0, int64_t ncols, double* dst, int32_t mem, void* stream) {
    return guarded([&] {
        Fd f;
        long long n;
        int kl, ku;
        spkb_open(path, f, n, kl, ku);
        if (col0 < 0 || ncols < 0 || col0 + ncols > n) fail(SPK_ERANGE, "spkb_load: column window out of range");
        const long long ld = kl + ku + 1;
        const long long off = kSpkbHeader + 8LL * ld * col0;
        const size_t total = (size_t)(8LL * ld * ncols);
        if (total == 0) return;
        if (mem != SPK_MEM_DEVICE) {
            full_pread(f.fd, dst, total, off, "SPKB file truncated");
            return;
        }
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t chunk = std::min(total, spkb_chunk_bytes());
        Staging& st = staging(chunk);
        size_t done = 0;
        for (int c = 0; done < total; ++c) {
            const int b = c & 1;
            const size_t len = std::min(chunk, total - done);
            if (c >= 2) ck(cudaEventSynchronize(st.ev[b]), "spkb_load");  // buffer b's previous upload
            full_pread(f.fd, st.buf[b], len, off + (long long)done, "SPKB file truncated");
            ck(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + done, st.buf[b], len, cudaMemcpyHostToDevice, s),
               "spkb upload");
            ck(cudaEventRecord(st.ev[b], s), "event");
            done += len;
        }
        ck(cudaStreamSynchronize(s), "spkb_load");
    });
}

spk_status spk_spkb_store(const char* path, const double* band, int64_t n, int32_t kl, int32_t ku, int32_t mem,
                          void* stream) {
    return guarded([&] {
        if (n < 1 || kl < 0 || ku < 0 || kl >= n || ku >= n) fail(SPK_EINVAL, "BandedMatrix: bad shape");
        Fd f;
        f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (f.fd < 0) fail(SPK_EIO, std::string("cannot open ") + path + " for writing");
        char head[kSpkbHeader];
        std::memcpy(head, "SPKB", 4);
        const int64_t v[3] = {n, kl, ku};
        std::memcpy(head + 4, v, sizeof(v));
        const std::string p(path);
        full_write(f.fd, head, kSpkbHeader, p);
        const size_t total = (size_t)(8LL * (kl + ku + 1) * n);
        if (mem != SPK_MEM_DEVICE) {
            full_write(f.fd, band, total, p);
            return;
        }
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t chunk = std::min(total, spkb_chunk_bytes());
        Staging& st = staging(chunk);
        // download chunk c+1 while chunk c is written
        size_t issued = 0, written = 0;
        size_t len[2] = {0, 0};
        auto issue = [&](int b) {
            len[b] = std::min(chunk, total - issued);
            ck(cudaMemcpyAsync(st.buf[b], reinterpret_cast<const char*>(band) + issued, len[b],
                               cudaMemcpyDeviceToHost, s),
               "spkb download");
            ck(cudaEventRecord(st.ev[b], s), "event");
            issued += len[b];
        };
        issue(0);
        for (int c = 0; written < total; ++c) {
            const int b = c & 1;
            if (issued < total) issue(b ^ 1);
            ck(cudaEventSynchronize(st.ev[b]), "spkb_store");
            full_write(f.fd, st.buf[b], len[b], p);
            written += len[b];
        }
    });
}

spk_status spk_generate_band(uint64_t seed, int64_t n, int32_t kl, int32_t ku, double dd, double* d_band,
                             void* stream) {
    return guarded([&] {
        launch_generate_band(seed, n, kl, ku, dd, 0, n, d_band, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "generate_band");
    });
}

spk_status spk_generate_rhs(uint64_t seed, int64_t n, int32_t ncols, double* d_F, int64_t ldf, void* stream) {
    return guarded([&] {
        if (ncols == 0) return;
        launch_generate_rhs(seed, 0, n, ncols, d_F, ldf, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "generate_rhs");
    });
}

spk_status spk_generate_band_cols(uint64_t seed, int64_t n, int32_t kl, int32_t ku, double dd, int64_t col0,
                                  int64_t ncols, double* d_band, void* stream) {
    return guarded([&] {
        if (ncols <= 0) return;
        launch_generate_band(seed, n, kl, ku, dd, col0, ncols, d_band, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "generate_band");
    });
}

spk_status spk_generate_rhs_rows(uint64_t seed, int64_t row0, int64_t nrows, int32_t ncols, double* d_F,
                                 int64_t ldf, void* stream) {
    return guarded([&] {
        if (ncols == 0 || nrows <= 0) return;
        launch_generate_rhs(seed, row0, nrows, ncols, d_F, ldf, static_cast<cudaStream_t>(stream));
        ck(cudaGetLastError(), "generate_rhs");
    });
}

}  // extern "C"
