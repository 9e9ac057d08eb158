// Bit-exact float64 row dot products in numpy's pairwise order, for sm_100a.
//
// Reference arithmetic: csvd._linalg.gemv_rows = (rows*h).sum(axis=1)
// (/root/reference/pkg/src/csvd/_linalg.py:25-37): each product rounded to
// f64, then numpy's pairwise add-reduce, result = 0.0 + pw(row).  The tree
// (restated in oracle/pairwise.c) splits n>128 into n2 = n/2 - (n/2)%8 and
// n-n2; leaves of 8..128 elements run 8 interleaved accumulator chains
// (chain j sums elements j, j+8, j+16, ...), combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail sequentially.
//
// Two device paths:
//  * REGULAR (d = NL * L with NL = 2^m >= 4 leaves of equal length L, L%8==0:
//    d = 512..16384 step multiples such as 3584, 4096, 8192): one warp per
//    row, every lane owns CPL chains of one leaf (CPL = 8 when NL >= 32, so a
//    lane streams 8 consecutive elements per step with one 256-bit LDG), the
//    chain->leaf->row tree is a butterfly of __shfl_xor (IEEE add is
//    commutative, so both partners hold the identical bits).  h lives in
//    shared memory in a lane-interleaved layout so every LDS is
//    conflict-free: hs[((u*S + i)*CPL + c)*32 + lane].
//  * GENERIC (any other length, e.g. d+1 for bias_augmented): leaves are
//    host-enumerated; lanes evaluate leaves, lane 0 folds them with the
//    host-generated postfix program.
// Every product/sum uses __dmul_rn/__dadd_rn (no FMA contraction).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CSVD_FULL 0xffffffffu
#define CSVD_MAX_LEAVES 1024
#define CSVD_MAX_PROG 2048

struct PwPlan {
    int n;          // row length
    int regular;    // 1 -> regular path
    int cpl, q;     // chains per lane, slices (leaves per lane for cpl==8)
    int leaf_len;   // regular leaf length (multiple of 8, <= 128)
    int steps;      // leaf_len / 8
    int nleaf;      // generic: number of leaves
    int nprog;      // generic: program length
    const int2 *leaves;  // device: (offset, len) per leaf
    const short *prog;   // device: >=0 push leaf, -1 add
};

__device__ __forceinline__ double d_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double d_mul(double a, double b) { return __dmul_rn(a, b); }

// ---------------------------------------------------------------------------
// raw vector loads (read-only, streaming: rows are touched once per step)
// ---------------------------------------------------------------------------
template <typename ET, int CPL> struct Raw;

template <> struct Raw<float, 8> {
    float v[8];
    __device__ __forceinline__ void load(const float *p) {
        asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
              "=f"(v[6]), "=f"(v[7])
            : "l"(p));
    }
    __device__ __forceinline__ double get(int c) const { return (double)v[c]; }
};
template <> struct Raw<float, 4> {
    float4 v;
    __device__ __forceinline__ void load(const float *p) { v = __ldg(reinterpret_cast<const float4 *>(p)); }
    __device__ __forceinline__ double get(int c) const {
        return (double)(c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w);
    }
};
template <> struct Raw<float, 2> {
    float2 v;
    __device__ __forceinline__ void load(const float *p) { v = __ldg(reinterpret_cast<const float2 *>(p)); }
    __device__ __forceinline__ double get(int c) const { return (double)(c == 0 ? v.x : v.y); }
};
template <> struct Raw<float, 1> {
    float v;
    __device__ __forceinline__ void load(const float *p) { v = __ldg(p); }
    __device__ __forceinline__ double get(int) const { return (double)v; }
};

__device__ __forceinline__ double bf16lo(uint32_t u) { return (double)__uint_as_float(u << 16); }
__device__ __forceinline__ double bf16hi(uint32_t u) { return (double)__uint_as_float(u & 0xffff0000u); }

template <> struct Raw<uint16_t, 8> {
    uint4 v;
    __device__ __forceinline__ void load(const uint16_t *p) {
        asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
            : "l"(p));
    }
    __device__ __forceinline__ double get(int c) const {
        uint32_t w = (c >> 1) == 0 ? v.x : (c >> 1) == 1 ? v.y : (c >> 1) == 2 ? v.z : v.w;
        return (c & 1) ? bf16hi(w) : bf16lo(w);
    }
};
template <> struct Raw<uint16_t, 4> {
    uint2 v;
    __device__ __forceinline__ void load(const uint16_t *p) { v = __ldg(reinterpret_cast<const uint2 *>(p)); }
    __device__ __forceinline__ double get(int c) const {
        uint32_t w = (c >> 1) == 0 ? v.x : v.y;
        return (c & 1) ? bf16hi(w) : bf16lo(w);
    }
};
template <> struct Raw<uint16_t, 2> {
    uint32_t v;
    __device__ __forceinline__ void load(const uint16_t *p) { v = __ldg(reinterpret_cast<const unsigned int *>(p)); }
    __device__ __forceinline__ double get(int c) const { return c ? bf16hi(v) : bf16lo(v); }
};
template <> struct Raw<uint16_t, 1> {
    uint16_t v;
    __device__ __forceinline__ void load(const uint16_t *p) { v = __ldg(reinterpret_cast<const unsigned short *>(p)); }
    __device__ __forceinline__ double get(int) const { return bf16lo((uint32_t)v); }
};

template <> struct Raw<double, 8> {
    double v[8];
    __device__ __forceinline__ void load(const double *p) {
        asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
            : "l"(p));
        asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
            : "l"(p + 4));
    }
    __device__ __forceinline__ double get(int c) const { return v[c]; }
};
template <> struct Raw<double, 4> {
    double v[4];
    __device__ __forceinline__ void load(const double *p) {
        asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
            : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
            : "l"(p));
    }
    __device__ __forceinline__ double get(int c) const { return v[c]; }
};
template <> struct Raw<double, 2> {
    double2 v;
    __device__ __forceinline__ void load(const double *p) { v = __ldg(reinterpret_cast<const double2 *>(p)); }
    __device__ __forceinline__ double get(int c) const { return c ? v.y : v.x; }
};
template <> struct Raw<double, 1> {
    double v;
    __device__ __forceinline__ void load(const double *p) { v = __ldg(p); }
    __device__ __forceinline__ double get(int) const { return v; }
};

// loads in flight per lane per batch (register budget ~64 regs of raw data)
template <typename ET, int CPL> struct NBatch { static constexpr int value = 8; };
template <int CPL> struct NBatch<double, CPL> { static constexpr int value = 8; };
template <int CPL> struct NBatch<uint16_t, CPL> { static constexpr int value = 16; };

// ---------------------------------------------------------------------------
// REGULAR path: returns 0.0 + pw(row .* h) in every lane
//
// h layout in shared memory:
//  * CPL == 8 (lane = leaf): natural order with a 2-double pad after every
//    leaf, hs[L*(leaf_len+2) + r] = h[L*leaf_len + r].  A lane reads its 8
//    values per step as 4 LDS.128; within a quarter-warp the 8 lanes start
//    4 banks apart ((2*leaf_len+4) mod 32 in {4, 20} for leaf_len % 8 == 0),
//    so every LDS.128 is conflict-free.
//  * CPL < 8 (lanes share a leaf): interleaved, hs[((u*S+i)*CPL+c)*32+lane],
//    built from a host-computed source-index table.
// ---------------------------------------------------------------------------
__host__ __device__ inline int pw_hs_size(const PwPlan &pl) {
    return (pl.regular && pl.cpl == 8) ? pl.n + 2 * pl.nleaf : pl.n;
}

// CPL = 8 (one leaf per lane): the leaf's loads double-buffered, so the next
// batch is in flight while the current one is multiplied and summed (the
// row's load latency overlaps the f64 work instead of alternating with it)
template <typename ET, int Q>
__device__ __forceinline__ double warp_dot_r8(const ET *__restrict__ row, const double *__restrict__ hs,
                                              int leaf_len, int lane) {
    constexpr int NB = NBatch<ET, 8>::value / 2;  // loads per buffer
    const int S = leaf_len >> 3;
    double slice[Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const ET *lp = row + (size_t)(u * 32 + lane) * leaf_len;
        const double *hp = hs + (size_t)(u * 32 + lane) * (leaf_len + 2);
        double r[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) r[c] = 0.0;
        Raw<ET, 8> A[NB], B[NB];
#pragma unroll
        for (int s = 0; s < NB; ++s)
            if (s < S) A[s].load(lp + s * 8);
        auto consume = [&](const Raw<ET, 8>(&buf)[NB], int i0) {
#pragma unroll
            for (int s = 0; s < NB; ++s) {
                const int i = i0 + s;
                if (i < S) {
                    const double2 *h2 = reinterpret_cast<const double2 *>(hp + 8 * i);
                    double hv[8];
#pragma unroll
                    for (int c2 = 0; c2 < 4; ++c2) {
                        const double2 t = h2[c2];
                        hv[2 * c2] = t.x;
                        hv[2 * c2 + 1] = t.y;
                    }
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const double p = d_mul(buf[s].get(c), hv[c]);
                        r[c] = (i == 0) ? p : d_add(r[c], p);
                    }
                }
            }
        };
#pragma unroll 1
        for (int i0 = 0; i0 < S; i0 += 2 * NB) {
#pragma unroll
            for (int s = 0; s < NB; ++s)
                if (i0 + NB + s < S) B[s].load(lp + (i0 + NB + s) * 8);
            consume(A, i0);
#pragma unroll
            for (int s = 0; s < NB; ++s)
                if (i0 + 2 * NB + s < S) A[s].load(lp + (i0 + 2 * NB + s) * 8);
            consume(B, i0 + NB);
        }
        double v = d_add(d_add(d_add(r[0], r[1]), d_add(r[2], r[3])), d_add(d_add(r[4], r[5]), d_add(r[6], r[7])));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
        slice[u] = v;
    }
    double tot;
    if constexpr (Q == 1)
        tot = slice[0];
    else if constexpr (Q == 2)
        tot = d_add(slice[0], slice[1]);
    else
        tot = d_add(d_add(slice[0], slice[1]), d_add(slice[2], slice[3]));
    return d_add(0.0, tot);
}

// Two rows per warp (CPL = 8): both rows' leaf loads in flight together and
// every staged h value read once for both (half the shared-memory reads of
// two single-row dots).  Same tree as warp_dot_r8 for each row.
template <typename ET, int Q>
__device__ __forceinline__ void warp_dot_r8_x2(const ET *__restrict__ rowA, const ET *__restrict__ rowB,
                                               const double *__restrict__ hs, int leaf_len, int lane, double &outA,
                                               double &outB) {
#ifndef CSVD_X2_DIV
#define CSVD_X2_DIV 4  // 2 (twice the loads in flight, 240 registers) measured no faster
#endif
    constexpr int NB = NBatch<ET, 8>::value / CSVD_X2_DIV;  // loads per row per buffer
    const int S = leaf_len >> 3;
    double slA[Q], slB[Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const ET *la = rowA + (size_t)(u * 32 + lane) * leaf_len;
        const ET *lb = rowB + (size_t)(u * 32 + lane) * leaf_len;
        const double *hp = hs + (size_t)(u * 32 + lane) * (leaf_len + 2);
        double ra[8], rb[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            ra[c] = 0.0;
            rb[c] = 0.0;
        }
        Raw<ET, 8> A0[NB], A1[NB], B0[NB], B1[NB];
        auto load = [&](Raw<ET, 8>(&xa)[NB], Raw<ET, 8>(&xb)[NB], int i0) {
#pragma unroll
            for (int s = 0; s < NB; ++s)
                if (i0 + s < S) {
                    xa[s].load(la + (i0 + s) * 8);
                    xb[s].load(lb + (i0 + s) * 8);
                }
        };
        auto consume = [&](const Raw<ET, 8>(&xa)[NB], const Raw<ET, 8>(&xb)[NB], int i0) {
#pragma unroll
            for (int s = 0; s < NB; ++s) {
                const int i = i0 + s;
                if (i < S) {
                    const double2 *h2 = reinterpret_cast<const double2 *>(hp + 8 * i);
                    double hv[8];
#pragma unroll
                    for (int c2 = 0; c2 < 4; ++c2) {
                        const double2 t = h2[c2];
                        hv[2 * c2] = t.x;
                        hv[2 * c2 + 1] = t.y;
                    }
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const double pa = d_mul(xa[s].get(c), hv[c]);
                        const double pb = d_mul(xb[s].get(c), hv[c]);
                        ra[c] = (i == 0) ? pa : d_add(ra[c], pa);
                        rb[c] = (i == 0) ? pb : d_add(rb[c], pb);
                    }
                }
            }
        };
        load(A0, B0, 0);
#pragma unroll 1
        for (int i0 = 0; i0 < S; i0 += 2 * NB) {
            load(A1, B1, i0 + NB);
            consume(A0, B0, i0);
            load(A0, B0, i0 + 2 * NB);
            consume(A1, B1, i0 + NB);
        }
        double va = d_add(d_add(d_add(ra[0], ra[1]), d_add(ra[2], ra[3])), d_add(d_add(ra[4], ra[5]), d_add(ra[6], ra[7])));
        double vb = d_add(d_add(d_add(rb[0], rb[1]), d_add(rb[2], rb[3])), d_add(d_add(rb[4], rb[5]), d_add(rb[6], rb[7])));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            va = d_add(va, __shfl_xor_sync(CSVD_FULL, va, o));
            vb = d_add(vb, __shfl_xor_sync(CSVD_FULL, vb, o));
        }
        slA[u] = va;
        slB[u] = vb;
    }
    double ta, tb;
    if constexpr (Q == 1) {
        ta = slA[0];
        tb = slB[0];
    } else if constexpr (Q == 2) {
        ta = d_add(slA[0], slA[1]);
        tb = d_add(slB[0], slB[1]);
    } else {
        ta = d_add(d_add(slA[0], slA[1]), d_add(slA[2], slA[3]));
        tb = d_add(d_add(slB[0], slB[1]), d_add(slB[2], slB[3]));
    }
    outA = d_add(0.0, ta);
    outB = d_add(0.0, tb);
}

template <typename ET, int CPL, int Q>
__device__ __forceinline__ double warp_dot_regular(const ET *__restrict__ row,
                                                   const double *__restrict__ hs,
                                                   int leaf_len, int lane) {
#ifndef CSVD_NO_PIPE
    if constexpr (CPL == 8) return warp_dot_r8<ET, Q>(row, hs, leaf_len, lane);
#endif
    constexpr int LPL = 8 / CPL;   // lanes per leaf
    constexpr int NLW = 32 / LPL;  // leaves per slice
    constexpr int NB = NBatch<ET, CPL>::value;
    const int S = leaf_len >> 3;
    const int lil = lane / LPL;
    const int j0 = (lane % LPL) * CPL;
    double slice[Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const ET *lp = row + (size_t)(u * NLW + lil) * leaf_len + j0;
        const double *hp = (CPL == 8) ? hs + (size_t)(u * 32 + lane) * (leaf_len + 2)
                                      : hs + (size_t)u * S * CPL * 32 + lane;
        double r[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) r[c] = 0.0;
        for (int i0 = 0; i0 < S; i0 += NB) {
            Raw<ET, CPL> raw[NB];
#pragma unroll
            for (int s = 0; s < NB; ++s)
                if (i0 + s < S) raw[s].load(lp + (i0 + s) * 8);
#pragma unroll
            for (int s = 0; s < NB; ++s) {
                if (i0 + s < S) {
                    const int i = i0 + s;
                    double hv[CPL];
                    if constexpr (CPL == 8) {
                        const double2 *h2 = reinterpret_cast<const double2 *>(hp + 8 * i);
#pragma unroll
                        for (int c2 = 0; c2 < 4; ++c2) {
                            double2 t = h2[c2];
                            hv[2 * c2] = t.x;
                            hv[2 * c2 + 1] = t.y;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) hv[c] = hp[(i * CPL + c) * 32];
                    }
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        double p = d_mul(raw[s].get(c), hv[c]);
                        r[c] = (i == 0) ? p : d_add(r[c], p);
                    }
                }
            }
        }
        double v;
        if constexpr (CPL == 8)
            v = d_add(d_add(d_add(r[0], r[1]), d_add(r[2], r[3])), d_add(d_add(r[4], r[5]), d_add(r[6], r[7])));
        else if constexpr (CPL == 4)
            v = d_add(d_add(r[0], r[1]), d_add(r[2], r[3]));
        else if constexpr (CPL == 2)
            v = d_add(r[0], r[1]);
        else
            v = r[0];
#pragma unroll
        for (int o = 1; o < LPL; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
#pragma unroll
        for (int o = LPL; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
        slice[u] = v;
    }
    double tot;
    if constexpr (Q == 1)
        tot = slice[0];
    else if constexpr (Q == 2)
        tot = d_add(slice[0], slice[1]);
    else
        tot = d_add(d_add(slice[0], slice[1]), d_add(slice[2], slice[3]));
    return d_add(0.0, tot);
}

// Same tree as warp_dot_regular<double, 8, Q>, for NR rows x NQ queries at
// once: every row element is loaded once and every staged query value is read
// once per NR rows (batched bounds: centroid reads shared by the queries,
// shared-memory reads of h shared by the rows).  out[r][j] = row r . query j.
template <int Q, int NQ, int NR>
__device__ __forceinline__ void warp_dot_regular_multi(const double *const (&rows)[NR],
                                                       const double *__restrict__ hs0, int hs_stride, int nq,
                                                       int leaf_len, int lane, double (&out)[NR][NQ]) {
    const int S = leaf_len >> 3;
    // slice totals combined as they complete, in the (s0+s1)+(s2+s3) tree of
    // warp_dot_regular: at most two partials per (row, query) stay live
    double part[NR][NQ], first[NR][NQ];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const double *hp = hs0 + (size_t)(u * 32 + lane) * (leaf_len + 2);
        double r[NR][NQ][8];
        // MB element steps of every row per buffer, the next buffer's loads
        // in flight while the current one is multiplied into every query
        constexpr int MB = NR == 1 ? 2 : 1;  // register budget: 2 steps for one row, 1 for two
        Raw<double, 8> A[MB][NR], B[MB][NR];
        auto load = [&](Raw<double, 8>(&buf)[MB][NR], int i0) {
#pragma unroll
            for (int m = 0; m < MB; ++m)
#pragma unroll
                for (int w = 0; w < NR; ++w)
                    if (i0 + m < S) buf[m][w].load(rows[w] + (size_t)(u * 32 + lane) * leaf_len + (i0 + m) * 8);
        };
        auto consume = [&](const Raw<double, 8>(&buf)[MB][NR], int i0) {
#pragma unroll
            for (int m = 0; m < MB; ++m) {
                const int i = i0 + m;
                if (i < S) {
#pragma unroll
                    for (int j = 0; j < NQ; ++j) {
                        if (j < nq) {
                            const double2 *h2 = reinterpret_cast<const double2 *>(hp + (size_t)j * hs_stride + 8 * i);
                            double hv[8];
#pragma unroll
                            for (int c2 = 0; c2 < 4; ++c2) {
                                const double2 t = h2[c2];
                                hv[2 * c2] = t.x;
                                hv[2 * c2 + 1] = t.y;
                            }
#pragma unroll
                            for (int w = 0; w < NR; ++w)
#pragma unroll
                                for (int c = 0; c < 8; ++c) {
                                    const double pr = d_mul(buf[m][w].get(c), hv[c]);
                                    r[w][j][c] = (i == 0) ? pr : d_add(r[w][j][c], pr);
                                }
                        }
                    }
                }
            }
        };
        load(A, 0);
#pragma unroll 1
        for (int i = 0; i < S; i += 2 * MB) {
            load(B, i + MB);
            consume(A, i);
            load(A, i + 2 * MB);
            consume(B, i + MB);
        }
#pragma unroll
        for (int w = 0; w < NR; ++w)
#pragma unroll
            for (int j = 0; j < NQ; ++j) {
                double v = d_add(d_add(d_add(r[w][j][0], r[w][j][1]), d_add(r[w][j][2], r[w][j][3])),
                                 d_add(d_add(r[w][j][4], r[w][j][5]), d_add(r[w][j][6], r[w][j][7])));
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
                if (u % 2 == 0) {
                    part[w][j] = v;
                } else {
                    v = d_add(part[w][j], v);  // s0+s1 or s2+s3
                    if (u == 1) first[w][j] = v;
                    else first[w][j] = d_add(first[w][j], v);
                }
            }
    }
#pragma unroll
    for (int w = 0; w < NR; ++w)
#pragma unroll
        for (int j = 0; j < NQ; ++j) out[w][j] = d_add(0.0, Q == 1 ? part[w][j] : first[w][j]);
}

// ||h||^2 in the CPL = 8 pairwise order with both operands from the staged
// shared-memory copy (same tree as warp_dot_regular<double, 8, Q>(h, hs)).
template <int Q>
__device__ __forceinline__ double warp_selfdot_smem(const double *__restrict__ hs, int leaf_len, int lane) {
    const int S = leaf_len >> 3;
    double slice[Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const double *hp = hs + (size_t)(u * 32 + lane) * (leaf_len + 2);
        double r[8];
        for (int i = 0; i < S; ++i) {
            const double2 *h2 = reinterpret_cast<const double2 *>(hp + 8 * i);
#pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) {
                const double2 t = h2[c2];
                const double p0 = d_mul(t.x, t.x), p1 = d_mul(t.y, t.y);
                r[2 * c2] = (i == 0) ? p0 : d_add(r[2 * c2], p0);
                r[2 * c2 + 1] = (i == 0) ? p1 : d_add(r[2 * c2 + 1], p1);
            }
        }
        double v = d_add(d_add(d_add(r[0], r[1]), d_add(r[2], r[3])), d_add(d_add(r[4], r[5]), d_add(r[6], r[7])));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
        slice[u] = v;
    }
    double tot;
    if constexpr (Q == 1)
        tot = slice[0];
    else if constexpr (Q == 2)
        tot = d_add(slice[0], slice[1]);
    else
        tot = d_add(d_add(slice[0], slice[1]), d_add(slice[2], slice[3]));
    return d_add(0.0, tot);
}

// host: source element of interleaved index idx (CPL < 8 plans)
__host__ __device__ inline int pw_hs_source(const PwPlan &pl, int idx) {
    // idx = ((u*S + i)*CPL + c)*32 + t
    const int t = idx & 31;
    int rest = idx >> 5;
    const int c = rest % pl.cpl;
    rest /= pl.cpl;
    const int i = rest % pl.steps;
    const int u = rest / pl.steps;
    const int lpl = 8 / pl.cpl;
    const int nlw = 32 / lpl;
    const int L = u * nlw + t / lpl;
    const int j0 = (t % lpl) * pl.cpl;
    return L * pl.leaf_len + 8 * i + j0 + c;
}

// Stage h (length n_src; elements n_src..pl.n-1 are the 1.0 of the
// bias-augmented [h,1]) into shared memory in the plan's layout.
// Block-cooperative; loads are independent so they overlap.
template <int CPL>
__device__ __forceinline__ void pw_stage(const PwPlan &pl, const double *__restrict__ h, int n_src, double *hs,
                                         const int *__restrict__ src) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if constexpr (CPL == 8) {
        const int L = pl.leaf_len;
        for (int leaf = warp; leaf < pl.nleaf; leaf += nw) {
            const double *g = h + (size_t)leaf * L;
            double *t = hs + (size_t)leaf * (L + 2);
#pragma unroll 4
            for (int r = lane; r < L; r += 32) t[r] = __ldcg(g + r);
        }
    } else if constexpr (CPL > 0) {
#pragma unroll 4
        for (int idx = threadIdx.x; idx < pl.n; idx += blockDim.x) hs[idx] = __ldcg(h + __ldg(src + idx));
    } else {
#pragma unroll 4
        for (int idx = threadIdx.x; idx < pl.n; idx += blockDim.x) hs[idx] = idx < n_src ? __ldcg(h + idx) : 1.0;
    }
}

// ---------------------------------------------------------------------------
// GENERIC path
// ---------------------------------------------------------------------------
template <typename F>
__device__ __forceinline__ double pw_leaf(const F &prod, int off, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = d_add(res, prod(off + i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = prod(off + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = d_add(r[j], prod(off + i + j));
    }
    double res = d_add(d_add(d_add(r[0], r[1]), d_add(r[2], r[3])), d_add(d_add(r[4], r[5]), d_add(r[6], r[7])));
    for (; i < n; ++i) res = d_add(res, prod(off + i));
    return res;
}

// scratch: per-warp shared buffer of >= pl.nleaf doubles
template <typename F>
__device__ __forceinline__ double warp_dot_generic(const F &prod, const PwPlan &pl, double *scratch, int lane) {
    for (int l = lane; l < pl.nleaf; l += 32) {
        int2 lf = pl.leaves[l];
        scratch[l] = pw_leaf(prod, lf.x, lf.y);
    }
    __syncwarp();
    double res = 0.0;
    if (lane == 0) {
        double st[48];
        int sp = 0;
        for (int i = 0; i < pl.nprog; ++i) {
            int op = pl.prog[i];
            if (op >= 0) {
                st[sp++] = scratch[op];
            } else {
                double b = st[--sp];
                double a = st[--sp];
                st[sp++] = d_add(a, b);
            }
        }
        res = d_add(0.0, st[0]);
    }
    res = __shfl_sync(CSVD_FULL, res, 0);
    __syncwarp();
    return res;
}

template <typename ET>
struct RowProd {
    const ET *row;
    const double *hs;
    __device__ __forceinline__ double load(int e) const;
    __device__ __forceinline__ double operator()(int e) const { return d_mul(load(e), hs[e]); }
};
template <> __device__ __forceinline__ double RowProd<float>::load(int e) const { return (double)__ldg(row + e); }
template <> __device__ __forceinline__ double RowProd<double>::load(int e) const { return __ldg(row + e); }
template <> __device__ __forceinline__ double RowProd<uint16_t>::load(int e) const {
    return bf16lo((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(row) + e));
}

// Row dot, plan fixed at compile time: CPL == 0 selects the generic path.
template <typename ET, int CPL, int Q>
__device__ __forceinline__ double warp_dot_t(const ET *__restrict__ row, const double *__restrict__ hs,
                                             const PwPlan &pl, double *scratch, int lane) {
    if constexpr (CPL > 0) {
        return warp_dot_regular<ET, CPL, Q>(row, hs, pl.leaf_len, lane);
    } else {
        RowProd<ET> f{row, hs};
        return warp_dot_generic(f, pl, scratch, lane);
    }
}

// Row dot dispatch.  `row` has pl.n elements (for the bias-augmented bound
// rows the centroid already carries the d+1 entry).
template <typename ET>
__device__ __forceinline__ double warp_dot(const ET *__restrict__ row, const double *__restrict__ hs,
                                           const PwPlan &pl, double *scratch, int lane) {
    if (pl.regular) {
        switch (pl.cpl * 8 + pl.q) {
            case 8 * 8 + 1: return warp_dot_regular<ET, 8, 1>(row, hs, pl.leaf_len, lane);
            case 8 * 8 + 2: return warp_dot_regular<ET, 8, 2>(row, hs, pl.leaf_len, lane);
            case 8 * 8 + 4: return warp_dot_regular<ET, 8, 4>(row, hs, pl.leaf_len, lane);
            case 4 * 8 + 1: return warp_dot_regular<ET, 4, 1>(row, hs, pl.leaf_len, lane);
            case 2 * 8 + 1: return warp_dot_regular<ET, 2, 1>(row, hs, pl.leaf_len, lane);
            default: return warp_dot_regular<ET, 1, 1>(row, hs, pl.leaf_len, lane);
        }
    }
    RowProd<ET> f{row, hs};
    return warp_dot_generic(f, pl, scratch, lane);
}
