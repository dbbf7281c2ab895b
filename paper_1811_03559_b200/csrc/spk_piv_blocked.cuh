// spk_piv_blocked.cuh — the blocked form of a pivoted partition's L factor.
//
// The pivoted band LU (spk_lu_piv_dmma.cu) factors 8 columns per step; for
// each such panel it also writes one record that lets the forward L sweep
// (spk_sweep_piv_dmma.cu) advance 8 rows per step on the tensor cores instead
// of one row interchange + axpy per row (kernels.cpp:131-165):
//   [0, 64)          L11^-1 (unit lower, rows in the panel's final order), DMMA
//                    A-fragment layout;
//   [64, 64 TRW)     -L21, tile rows 1 .. TRW-1 of the window, A-fragment layout;
//   then int32       src[8 TRW]: window position -> position before the panel's
//                    interchanges; mv_out / mv_in[NSLW]: bit masks of the rows
//                    that leave / the positions that receive another row.
// Applying a record to the window rows j0 .. j0+8TRW-1 of B is exactly the 8
// reference steps j0 .. j0+7 (gbtf2: interchange, then axpy with column j):
// the interchanges of a panel only move rows between positions 0..7 and the
// pivot rows, and the panel's L columns in its final row order are L11, L21.
// Records of partition `part` start at panel index r0/8 + part (disjoint).
#pragma once

namespace spk {

template <int TRW>
struct PivRec {
    static constexpr int NSLW = (8 * TRW + 31) / 32;
    static constexpr int NINT = 8 * TRW + 2 * NSLW;
    static constexpr int SRC = 64 * TRW;                          // int offset base (in doubles)
    static constexpr int SIZE = (64 * TRW + (NINT + 1) / 2 + 1) / 2 * 2;  // doubles, even (16-B records)
};

// tile rows of the window for a band (the reversed UL partition swaps kl, ku)
inline int piv_trw(int kl, int ku) {
    const int kr = kl > ku ? kl : ku, kc = kl + ku;
    if (kr <= 32 && kc <= 64) return 5;
    if (kr <= 64 && kc <= 128) return 9;
    if (kr <= 96 && kc <= 192) return 13;
    return 0;
}

inline long long piv_rec_size(int trw) {
    switch (trw) {
        case 5: return PivRec<5>::SIZE;
        case 9: return PivRec<9>::SIZE;
        case 13: return PivRec<13>::SIZE;
        default: return 0;
    }
}

}  // namespace spk
