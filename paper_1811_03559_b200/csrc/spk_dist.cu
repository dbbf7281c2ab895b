// spk_dist.cu — the multi-GPU data plane in the C++ host: one slab of rows
// per GPU (spk_factorize_slab), only the reduced-system tip blocks cross GPUs,
// by NCCL all-gathers over NVLink.
//
// The reference has no multi-GPU path (proj/include/spike/parallel_util.hpp:
// 13-45 is a single-node fork-join); the slab protocol extends its recursive
// reduction by one level: the G slab units form a reduced system of the
// reference's own shape (reduce_factorize, factorize.cpp:46-120, p = G), held
// redundantly on every GPU, assembled on the device from the gathered tips.
//
//   factorize: all-gather of each slab unit's tips [vt; vb; wt; wb] (4 k^2).
//   solve:     all-gather of [y_top; y_bot] (2k x nrhs), the slab-level
//              reduced solve, each GPU's import [x_top(g+1); x_bot(g-1)].
//   transpose: all-gather of the edge G-tip terms (2k x nrhs), then of
//              [t_top; t_bot; V_int^T t; W_int^T t] (4k x nrhs), the slab-level
//              transposed reduced solve, each GPU's [z_top; z_bot].
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the copy torch
// already loaded, or the system one; SPK_NCCL_LIB overrides): the library has
// no link-time NCCL dependency, and a missing NCCL is SPK_ENCCL, not a crash.
// The exchange arithmetic between the collectives (permutations of the
// gathered blocks, the transposed right-hand side's neighbour terms) is one
// small kernel, also exported (spk_dist_exchange) so the G-slab protocol can be
// run as virtual ranks in one process by the tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "spike_b200.h"
#include "spk_launch.h"

namespace {

// ---------------------------------------------------------------------------
// NCCL entry points (dlopen)
struct Nccl {
    bool tried = false;
    std::string err;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (n.tried) return n;
    n.tried = true;
    const char* path = getenv("SPK_NCCL_LIB");
    void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        n.err = std::string("NCCL not available: ") + dlerror();
        return n;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.comm_destroy || !n.error_string) {
        n.err = "NCCL library lacks an entry point";
        n.get_unique_id = nullptr;
    }
    return n;
}

struct Fail {
    spk_status st;
    std::string msg;
};
thread_local std::string g_dist_err;

template <class F>
spk_status run(F&& f) {
    try {
        f();
        return SPK_OK;
    } catch (const Fail& e) {
        g_dist_err = e.msg;
        return e.st;
    }
}
void need_nccl() {
    if (!nccl().get_unique_id) throw Fail{SPK_ENCCL, nccl().err};
}
void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Fail{SPK_ENCCL, std::string(what) + ": " + nccl().error_string(r)};
}
void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail{SPK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
void sck(spk_status st, const char* what) {
    if (st != SPK_OK) throw Fail{st, std::string(what) + ": " + spk_last_error()};
}

// ---------------------------------------------------------------------------
// exchange arithmetic (distributed.py's tensor formulas, on the device)
__global__ void k_dist_exchange(int op, const double* __restrict__ src, double* __restrict__ dst, int G, int rank,
                                int k, int nrhs) {
    const long long H2 = 2LL * G * k;  // slab-level reduced rows
    long long total = 0;
    switch (op) {
        case SPK_XCH_FWD_TOP_RHS: total = H2 * nrhs; break;
        case SPK_XCH_TR_TOP_RHS: total = H2 * nrhs; break;
        default: total = 2LL * k * nrhs; break;
    }
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        if (op == SPK_XCH_FWD_TOP_RHS) {
            // (G, nrhs, 2k) -> z (2Gk x nrhs): z[c][g 2k + r] = a[g][c][r]
            const long long c = e / H2, gr = e - c * H2, g = gr / (2 * k), r = gr - g * 2 * k;
            v = src[(g * nrhs + c) * 2 * k + r];
        } else if (op == SPK_XCH_FWD_IMPORT) {
            // z (2Gk x nrhs) -> [x_top(rank+1); x_bot(rank-1)] (2k x nrhs)
            const long long c = e / (2 * k), r = e - c * 2 * k;
            if (r < k) {
                if (rank + 1 < G) v = src[c * H2 + (long long)(rank + 1) * 2 * k + r];
            } else if (rank > 0) {
                v = src[c * H2 + (long long)(rank - 1) * 2 * k + r];
            }
        } else if (op == SPK_XCH_TR_IMPORT1) {
            // (G, nrhs, 2, k) -> [left slab's bhat^T tau_b; right slab's chat^T tau_t]
            const long long c = e / (2 * k), r = e - c * 2 * k;
            if (r < k) {
                if (rank > 0) v = src[((long long)(rank - 1) * nrhs + c) * 2 * k + k + r];
            } else if (rank + 1 < G) {
                v = src[((long long)(rank + 1) * nrhs + c) * 2 * k + (r - k)];
            }
        } else if (op == SPK_XCH_TR_TOP_RHS) {
            // (G, nrhs, 4, k) -> (2Gk x nrhs): top(g) = t_top(g) - V_int^T t(g-1),
            // bot(g) = t_bot(g) - W_int^T t(g+1)
            const long long c = e / H2, gr = e - c * H2, g = gr / (2 * k), r = gr - g * 2 * k;
            const double* b = src + (g * nrhs + c) * 4 * k;
            if (r < k) {
                v = b[r];
                if (g > 0) v -= src[((g - 1) * nrhs + c) * 4 * k + 2 * k + r];
            } else {
                v = b[r];
                if (g + 1 < G) v -= src[((g + 1) * nrhs + c) * 4 * k + 3 * k + (r - k)];
            }
        } else {  // SPK_XCH_TR_IMPORT2: z (2Gk x nrhs) -> this slab's [z_top; z_bot]
            const long long c = e / (2 * k), r = e - c * 2 * k;
            v = src[c * H2 + (long long)rank * 2 * k + r];
        }
        dst[e] = v;
    }
}

void exchange(int op, const double* src, double* dst, int G, int rank, int k, int nrhs, cudaStream_t s) {
    const long long total = (op == SPK_XCH_FWD_TOP_RHS || op == SPK_XCH_TR_TOP_RHS) ? 2LL * G * k * nrhs
                                                                                       : 2LL * k * nrhs;
    if (total <= 0) return;
    const int grid = (int)std::min<long long>((total + 255) / 256, 1184);
    k_dist_exchange<<<grid, 256, 0, s>>>(op, src, dst, G, rank, k, nrhs);
    cck(cudaGetLastError(), "exchange kernel");
}

struct Scratch {  // stream-ordered device scratch owned by one call
    cudaStream_t s;
    void* p = nullptr;
    Scratch(size_t bytes, cudaStream_t st) : s(st) { cck(cudaMallocAsync(&p, bytes ? bytes : 8, s), "alloc"); }
    ~Scratch() { cudaFreeAsync(p, s); }
    double* d() const { return static_cast<double*>(p); }
};

}  // namespace

struct spk_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    bool owned = false;
};

struct spk_dist {
    spk_fact* slab = nullptr;
    spk_reduced* top = nullptr;
    spk_comm* comm = nullptr;
    int k = 0;
    double boost_eps = 0.0;
    ~spk_dist() {
        if (top) spk_reduced_destroy(top);
        if (slab) spk_fact_destroy(slab);
    }
};

extern "C" {

const char* spk_dist_last_error(void) { return g_dist_err.c_str(); }

spk_status spk_comm_unique_id(uint8_t* id) {
    return run([&] {
        if (!id) throw Fail{SPK_EINVAL, "comm: null id buffer"};
        need_nccl();
        ncclUniqueId u;
        nck(nccl().get_unique_id(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == SPK_COMM_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id, &u, sizeof(u));
    });
}

spk_status spk_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, spk_comm** out) {
    return run([&] {
        if (!out || !id) throw Fail{SPK_EINVAL, "comm: null argument"};
        *out = nullptr;
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Fail{SPK_EINVAL, "comm: bad rank"};
        need_nccl();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto* c = new spk_comm;
        c->rank = rank;
        c->nranks = nranks;
        c->owned = true;
        const ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nck(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

spk_status spk_comm_wrap(void* nccl_comm, int32_t nranks, int32_t rank, spk_comm** out) {
    return run([&] {
        if (!out || !nccl_comm) throw Fail{SPK_EINVAL, "comm: null argument"};
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Fail{SPK_EINVAL, "comm: bad rank"};
        need_nccl();
        auto* c = new spk_comm;
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        c->rank = rank;
        c->nranks = nranks;
        *out = c;
    });
}

void spk_comm_destroy(spk_comm* c) {
    if (!c) return;
    if (c->owned && c->comm && nccl().comm_destroy) nccl().comm_destroy(c->comm);
    delete c;
}

spk_status spk_dist_exchange(int32_t op, const double* d_src, double* d_dst, int32_t G, int32_t rank, int32_t k,
                             int32_t nrhs, void* stream) {
    return run([&] {
        if (op < SPK_XCH_FWD_TOP_RHS || op > SPK_XCH_TR_IMPORT2) throw Fail{SPK_EINVAL, "exchange: bad op"};
        if (G < 1 || rank < 0 || rank >= G || k < 0 || nrhs < 0) throw Fail{SPK_EINVAL, "exchange: bad shape"};
        exchange(op, d_src, d_dst, G, rank, k, nrhs, static_cast<cudaStream_t>(stream));
    });
}

spk_status spk_dist_factorize(const double* d_band, int64_t n_local, int32_t kl, int32_t ku, const spk_plan* plan,
                              const spk_factor_options* opts, spk_comm* comm, void* stream, spk_dist** out) {
    return run([&] {
        if (!out || !comm) throw Fail{SPK_EINVAL, "dist_factorize: null argument"};
        *out = nullptr;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int G = comm->nranks, g = comm->rank;
        auto d = new spk_dist;
        try {
            d->comm = comm;
            d->k = kl > ku ? kl : ku;
            d->boost_eps = opts ? opts->boost_eps : 0.0;
            sck(spk_factorize_slab(d_band, SPK_MEM_DEVICE, n_local, kl, ku, plan, opts, g > 0, g + 1 < G, s, &d->slab),
                "slab factorization");
            if (G > 1) {
                const long long kk = (long long)d->k * d->k;
                Scratch tips(sizeof(double) * 4 * kk, s), all(sizeof(double) * 4 * kk * G, s);
                sck(spk_fact_unit_tips(d->slab, tips.d(), s), "unit tips");
                need_nccl();
                nck(nccl().all_gather(tips.d(), all.d(), 4 * kk, ncclFloat64, comm->comm, s), "tips all-gather");
                sck(spk_reduced_create_device(all.d(), G, d->k, d->boost_eps, s, &d->top), "slab-level system");
            }
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

spk_status spk_dist_solve(const spk_dist* d, int32_t transpose, const double* d_F, int64_t ldf, int32_t nrhs,
                          double* d_X, int64_t ldx, void* stream) {
    return run([&] {
        if (!d) throw Fail{SPK_EINVAL, "dist_solve: null handle"};
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const int G = d->comm->nranks, g = d->comm->rank, k = d->k;
        if (G == 1) {
            sck(spk_solve(d->slab, transpose, d_F, ldf, nrhs, d_X, ldx, SPK_MEM_DEVICE, s, nullptr), "solve");
            return;
        }
        if (nrhs == 0) return;
        need_nccl();
        const size_t blk = (size_t)2 * k * nrhs;  // 2k x nrhs
        Scratch exp(sizeof(double) * 2 * blk, s), all(sizeof(double) * 2 * blk * G, s),
            z(sizeof(double) * blk * G, s), imp(sizeof(double) * blk, s);
        spk_xsolve* x = nullptr;
        sck(spk_xsolve_begin(d->slab, transpose, d_F, ldf, nrhs, d_X, ldx, s, exp.d(), &x), "xsolve begin");
        try {
            nck(nccl().all_gather(exp.d(), all.d(), blk, ncclFloat64, d->comm->comm, s), "all-gather");
            if (!transpose) {
                exchange(SPK_XCH_FWD_TOP_RHS, all.d(), z.d(), G, g, k, nrhs, s);
                sck(spk_reduced_solve_device(d->top, 0, z.d(), nrhs, s), "slab-level solve");
                exchange(SPK_XCH_FWD_IMPORT, z.d(), imp.d(), G, g, k, nrhs, s);
                sck(spk_xsolve_step(x, imp.d(), nullptr), "xsolve step");
            } else {
                exchange(SPK_XCH_TR_IMPORT1, all.d(), imp.d(), G, g, k, nrhs, s);
                sck(spk_xsolve_step(x, imp.d(), exp.d()), "xsolve step 1");
                nck(nccl().all_gather(exp.d(), all.d(), 2 * blk, ncclFloat64, d->comm->comm, s), "all-gather");
                exchange(SPK_XCH_TR_TOP_RHS, all.d(), z.d(), G, g, k, nrhs, s);
                sck(spk_reduced_solve_device(d->top, 1, z.d(), nrhs, s), "slab-level solve");
                exchange(SPK_XCH_TR_IMPORT2, z.d(), imp.d(), G, g, k, nrhs, s);
                sck(spk_xsolve_step(x, imp.d(), nullptr), "xsolve step 2");
            }
        } catch (...) {
            spk_xsolve_end(x);
            throw;
        }
        spk_xsolve_end(x);
    });
}

const spk_fact* spk_dist_slab(const spk_dist* d) { return d ? d->slab : nullptr; }

void spk_dist_destroy(spk_dist* d) { delete d; }

}  // extern "C"
