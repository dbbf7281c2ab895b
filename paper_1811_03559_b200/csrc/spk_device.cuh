// spk_device.cuh — device-side data structures shared by the SPIKE kernels.
//
// Every stage of factorize / solve / transpose_solve is a batch of small
// "jobs" (one per partition, per coupling block, per boundary) executed by a
// single launch, so the host issues O(stages) launches, never O(p).
#pragma once

#include <cstdint>

namespace spk {

constexpr int kMaxBufs = 10;
// B_XCH / B_XIN: export / import blocks of a multi-GPU slab solve
enum BufId { B_X = 0, B_F = 1, B_S = 2, B_T = 3, B_AUX = 4, B_POOL = 5, B_FS = 6, B_FAC = 7, B_XCH = 8, B_XIN = 9 };

// Per call buffer table, passed by value.
struct Bufs {
    double* p[kMaxBufs];
    long long ld[kMaxBufs];
    const int* flags;  // per-pair coupling path flags (job guards)
};

// Job guard: -1 = unconditional, else run only if flags[g >> 1] == (g & 1).
__host__ __device__ __forceinline__ bool guard_ok(const int* flags, int g) {
    return g < 0 || flags[g >> 1] == (g & 1);
}

// Geometry of one band LU "unit": a SPIKE partition (kernels.cpp:29-42 layout:
// rows = ubw+kl+1 packed rows per column, diagonal at packed row d = ubw) or a
// dense 2k coupling block stored as a full band (kernels.cpp:67-77).
struct PartDev {
    long long r0;    // first system row (partitions) / unused (couplings)
    long long fofs;  // offset of the packed factor in the factor pool (doubles)
    long long bofs;  // offset of the backup copy (couplings; -1 if none)
    long long tofs;  // offset of the row-major factor copy (partitions; -1 if none)
    int m;           // order
    int kl, ku, ubw, d, rows;
    int rev;         // factors of Q A_i Q (UL via reversed LU, kernels.cpp:51-62)
    int trunc;       // trunc_start (block_util.hpp:13-16)
    int pivoting;
    int fallback;    // pivoted-with-boosted-fallback (coupling blocks)
    int rowsT;       // row-major copy: row i holds (i, i-kl .. i+ubw) at [kl + c - i]
    int guard;       // job guard for generic coupling units (-1: none)
    int pad;
};

// Row-mapped view of a column-major buffer.  Logical row L maps to physical
// row base + (rev ? mrows-1-(L-off) : L-off); column c adds c*ld.
struct View {
    long long base;
    long long ld;  // < 0: take Bufs.ld[buf]
    int buf;
    int rev;
    int off;
    int mrows;
};

enum SweepMode { SW_FWD_L = 0, SW_BWD_U = 1, SW_FWD_UT = 2, SW_BWD_LT = 3 };

struct SweepJob {
    View v;
    int part;  // PartDev index
    int mode;
    int lo, hi;
    int c0, nc;  // column range (nc < 0: all call columns)
    int guard;
};

enum CopyOp { CP_COPY = 0, CP_ADD = 1, CP_SUB = 2, CP_ZERO = 3, CP_IDENT = 4 };  // IDENT: dst = (L - L0 == c)

struct CopyJob {
    View src, dst;
    int L0, L1;  // logical rows [L0, L1) of both views
    int op;
    int c0, nc;  // nc < 0: call columns
    int guard;
};

enum GemmOp { GM_SET = 0, GM_SUB = 1 };

// C[crow0 + i, c] (op)= sum_l opA(A)[i, l] * B[brow0 + l, c],
// i < r, l < kk, c < nc.  opA(A) = A (r x kk) or A^T (A is kk x r).
struct GemmJob {
    View a, b, c;
    int transA;
    int brow0, crow0;
    int r, kk, nc;  // nc < 0: call columns
    int op;
    int guard;
};

// Coupling construction for one pair of reduced units (factorize.cpp:94-101):
// C = [[I, vl[hL-k:hL]], [wr[0:k], I]] written as a full band into the factor
// pool (and its backup) of PartDev `part`.
struct CouplingJob {
    long long vl_off, wr_off;  // pool offsets of the h x k spike columns
    int hL, hR;
    int part;
    int k;
    int guard;  // flag index (pair)
    int pad;
    long long aux;  // ST_SCHUR_INV: pool offset of S^-1 (k x k, ld k)
};

}  // namespace spk
