// td_kernels.cu — sm_100a kernels behind include/td_api.h.
//
// Kernel 1 (k_segnorm): one persistent pass over a flat tile list.  Each tile
// is a fixed slice of one segment (a 2-D strided block read in lockstep from
// the reference side x, candidate copy 0 y and up to seven replica copies z).
// It accumulates, in fp64:
//     d2 = sum (x - y)^2      x2 = sum x^2                 (rel_err(ref, cand))
//     y2 = sum y^2            z2[j] = sum (y - z_j)^2       (rel_err(copy0, copy_j))
// and writes the tile's block-reduced partials; no atomics, so the result is
// bit-reproducible for a given plan, independent of grid size.
// Reference semantics: tensor.py:158-167 (norms), canonical.py:182-212 (merge,
// never materialised here), canonical.py:225-247 (replica rel_err),
// tracestore.py:84-86 (f32 -> f64 widening).
//
// Kernel 3 (k_reduce_slots + k_verdict): deterministic per-id / per-group sums
// of tile partials, then checker.check's verdict precedence (checker.py:328-354)
// and check_replicas' strict-> worst tracking (canonical.py:236-247).
//
// Kernel 2 (k_perturb): Emulator._apply_perturbation (engine.py:351-361):
// y = Q(x * (1 + u*eps)) with the splitmix64 stream of generation.py:49-78 and
// the RNE-to-p-bits quantiser of tensor.py:64-77, each fp64 op rounded
// separately (__dmul_rn / __dadd_rn: numpy never contracts to FMA).

#include "td_api.h"

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace {

thread_local char g_err[512] = "";

int fail(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return 1;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail("%s: %s", what, cudaGetErrorString(e));
    return 0;
}

#ifndef TD_LDG_STREAM
#define TD_LDG_STREAM "ld.global.nc.L1::no_allocate.L2::256B.v4.u32"
#endif

constexpr int BLOCK = 256;
constexpr int NWARP = BLOCK / 32;

// ---------------------------------------------------------------------------
// loads and widening

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile(TD_LDG_STREAM " {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// words (u32) per 8-element vector, and their widening to fp64
template <int DT> struct Vec;

template <> struct Vec<TD_BF16> {
    static constexpr int Q = 1;  // uint4 loads per 8 elements
    __device__ __forceinline__ static double at(const uint4* q, int e) {
        const uint32_t w = (&q[0].x)[e >> 1];
        const uint32_t b = (e & 1) ? (w & 0xffff0000u) : (w << 16);
        return (double)__uint_as_float(b);
    }
};
template <> struct Vec<TD_F16> {
    static constexpr int Q = 1;
    __device__ __forceinline__ static double at(const uint4* q, int e) {
        const uint32_t w = (&q[0].x)[e >> 1];
        const unsigned short h = (e & 1) ? (unsigned short)(w >> 16) : (unsigned short)(w & 0xffffu);
        return (double)__half2float(__ushort_as_half(h));
    }
};
template <> struct Vec<TD_F32> {
    static constexpr int Q = 2;
    __device__ __forceinline__ static double at(const uint4* q, int e) {
        return (double)__uint_as_float((&q[0].x)[e]);
    }
};

__device__ __forceinline__ double load_elem(const char* base, int dt, int64_t idx) {
    switch (dt) {
        case TD_F32: return (double)__ldg(reinterpret_cast<const float*>(base) + idx);
        case TD_BF16: {
            unsigned short h = __ldg(reinterpret_cast<const unsigned short*>(base) + idx);
            return (double)__uint_as_float(((uint32_t)h) << 16);
        }
        case TD_F16: {
            unsigned short h = __ldg(reinterpret_cast<const unsigned short*>(base) + idx);
            return (double)__half2float(__ushort_as_half(h));
        }
        default: return __ldg(reinterpret_cast<const double*>(base) + idx);
    }
}

constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;

// Replica digests: 8-byte word w_j (j = its word index in the record) with
// position key k_j = (j+1)*gamma goes into lane j & 1 as
//     z = (w_j ^ k_j) * M[j & 1],   h[j & 1] += z ^ (z >> 32)   (mod 2^64, M odd)
// — for a fixed key a bijection of w_j, so a changed word always changes its
// lane's sum; position-keyed (permuted shards differ); order-independent (any
// reduction order, atomics included, gives the same bits).  One 64-bit
// multiply per word.  The fold (one LOP3: hi ^= into lo) keeps the lane sum
// from being M * sum(w ^ k), a plain additive checksum in which two equal and
// opposite word changes (e.g. a swap of two values whose keys agree on the
// differing bits) cancel exactly; with it such a pair collides only if 32
// nonlinear low bits cancel too.  (The first version folded every word into
// both lanes, h0 += z, h1 += hi32(z) * lo32(z): ~12 instructions per word
// against 8, and the compare pass that digests its copy is issue bound.)
__device__ __forceinline__ void fp_key_word(uint64_t w, uint64_t key, uint64_t& h, uint64_t mult) {
    const uint64_t z = (w ^ key) * mult;
    h += z ^ (z >> 32);
}

__device__ __forceinline__ void fp_word(uint64_t w, uint64_t j, uint64_t& h0, uint64_t& h1) {
    if (j & 1) fp_key_word(w, (j + 1) * GAMMA, h1, MIX2);
    else fp_key_word(w, (j + 1) * GAMMA, h0, MIX1);
}

// a 16-byte vector at (even) word index j: words j -> lane 0, j+1 -> lane 1
__device__ __forceinline__ void fp_vec_key(const uint4& v, uint64_t k0, uint64_t& h0, uint64_t& h1) {
    fp_key_word(((uint64_t)v.y << 32) | v.x, k0, h0, MIX1);
    fp_key_word(((uint64_t)v.w << 32) | v.z, k0 + GAMMA, h1, MIX2);
}

__device__ __forceinline__ void fp_vec(const uint4& v, uint64_t j, uint64_t& h0, uint64_t& h1) {
    fp_vec_key(v, (j + 1) * GAMMA, h0, h1);
}

#ifndef TD_REPLICA_SKIP
#define TD_REPLICA_SKIP 1
#endif
#ifndef TD_FP_U
#define TD_FP_U 8
#endif
#ifndef TD_REPLICA_SKIP_MIN_NZ
#define TD_REPLICA_SKIP_MIN_NZ 3
#endif

template <int Q>
__device__ __forceinline__ bool same_bits(const uint4* a, const uint4* b) {
    uint32_t d = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) d |= (a[q].x ^ b[q].x) | (a[q].y ^ b[q].y) | (a[q].z ^ b[q].z) | (a[q].w ^ b[q].w);
    return d == 0;
}

struct Acc {
    double d2, x2, y2, z[TD_MAX_Z];
    __device__ __forceinline__ void zero() {
        d2 = x2 = y2 = 0.0;
#pragma unroll
        for (int j = 0; j < TD_MAX_Z; ++j) z[j] = 0.0;
    }
};

struct SegView {
    const char* x;
    const char* y;
    const char* z[TD_MAX_Z];
    int64_t xs, ys, cols;
    uint32_t vpr;      // units per row
    uint32_t div_m;
    int div_p;
};

__device__ __forceinline__ uint32_t udiv(uint32_t n, uint32_t m, int p) {
    return (uint32_t)(((uint64_t)n * (uint64_t)m) >> p);
}

// Programmatic dependent launch (sm_90+): the slot reduction / verdict
// kernels are launched with programmatic stream serialisation and wait for
// their producer at entry, so their launch (and CTA rasterisation) overlaps
// the producer's tail instead of following its completion; the segnorm
// walkers signal once a CTA has written its last partial row.  Without the
// launch attribute (TD_PDL=0, or a non-kernel predecessor) both are no-ops.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------------------
// tile walkers.  Every (dtype, nz, has_x) class is its own __global__ so ptxas
// allocates registers for exactly one loop; the host launches one persistent
// kernel per class present in the plan (usually 1-3).

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


// Tiles are dealt to CTAs grid-stride (neighbouring CTAs stream neighbouring
// tiles: DRAM row locality; a contiguous share per CTA measured 17% slower).
// A class-list entry packs (segment << 32 | tile) so no tile->segment lookup
// is needed.  Warps are independent: each warp reduces its own slice of a
// tile and writes its own partial row, so there is no CTA barrier anywhere —
// a warp that finishes a tile starts loading the next one while its
// neighbours still drain theirs (a per-tile __syncthreads measured ~9% of
// the stream).  Rows: partials[(tile * TD_WARPS_PER_TILE + warp) * 10 + k].
__device__ __forceinline__ int entry_seg(int64_t e) { return (int)(e >> 32); }
__device__ __forceinline__ int64_t entry_tile(int64_t e) { return e & 0xffffffffll; }

// a segment-descriptor field: from the global table (read-only path), or —
// PARAM, a single-segment class — from the kernel's __grid_constant__
// parameter copy, so the first tile starts without two dependent DRAM round
// trips (tile list, then descriptor)
template <bool PARAM, typename T>
__device__ __forceinline__ T rd(const T* p) {
    if constexpr (PARAM) return *p;
    else return __ldg(p);
}

template <bool PARAM = false>
__device__ __forceinline__ int64_t tile_units(const td_segment* g) {
    const int sh = (rd<PARAM>(&g->flags) >> TD_SEG_TILE_SHIFT_POS) & 31;
    return sh ? (int64_t)1 << sh : (int64_t)TD_TILE_UNITS;
}

template <bool PARAM = false>
__device__ __forceinline__ void load_desc(const td_segment* __restrict__ g, SegView& S, int nz_max) {
    S.x = reinterpret_cast<const char*>(rd<PARAM>(&g->x));
    S.y = reinterpret_cast<const char*>(rd<PARAM>(&g->y));
#pragma unroll
    for (int j = 0; j < TD_MAX_Z; ++j)
        S.z[j] = j < nz_max ? reinterpret_cast<const char*>(rd<PARAM>(&g->z[j])) : nullptr;
    S.xs = rd<PARAM>(&g->x_stride);
    S.ys = rd<PARAM>(&g->y_stride);
    S.cols = rd<PARAM>(&g->cols);
    S.div_m = rd<PARAM>(&g->div_m);
    S.div_p = rd<PARAM>(&g->div_p);
}

// warp-level partial: lane 0 writes the first `used` fixed-order sums
__device__ __forceinline__ void write_warp_partial(const Acc& a, int used, double* __restrict__ out) {
    const double v[TD_PARTIAL_STRIDE] = {a.d2, a.x2, a.y2, a.z[0], a.z[1], a.z[2],
                                         a.z[3], a.z[4], a.z[5], a.z[6]};
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < TD_PARTIAL_STRIDE; ++k) {
        double s = 0.0;
        if (k < used) s = warp_sum(v[k]);
        if (lane == 0) out[k] = s;
    }
}

// vector class: every operand has dtype DT, rows 16-byte aligned, cols % 8 == 0
// DG: also digest y's bytes into digests[slot] (multi-GPU: the compare copy
// of a cross-GPU replica group is digested in the pass that compares it, so
// it is read once; the planner guarantees such a record's segments cover it
// exactly once, so the sum equals td_fingerprint's digest of the record).
// Hashing in the loads' registers needs U=2 to stay at 64 registers; a second
// pass over the warp's tile slice from L2 instead (U=4 compare loop) measured
// 18% slower on the config-4 share, U=4 at 3 CTAs/SM 5% slower.
// ONE: the class is one segment, passed by value (seg1) — tile i of the
// class is global tile seg1.tile_begin + i, no tile list, no descriptor load.
template <int DT, int NZ, bool HX, int U, int MINB, bool DG = false, bool ONE = false>
__global__ void __launch_bounds__(BLOCK, MINB)
k_segnorm_vec(const td_segment* __restrict__ segs, const int64_t* __restrict__ tiles, int64_t n,
              double* __restrict__ partials, unsigned long long* __restrict__ digests,
              const __grid_constant__ td_segment seg1) {
    constexpr int Q = Vec<DT>::Q;
    constexpr int ES = (DT == TD_F32) ? 4 : 2;
    constexpr int USED = NZ > 0 ? 3 + NZ : 2;
    // classes with >= 3 replicas (fewer: little XU work to save, more spills)
    // (2-byte payloads; f32 vectors need twice the registers)
    constexpr bool SKIP = TD_REPLICA_SKIP && NZ >= TD_REPLICA_SKIP_MIN_NZ && Q == 1;
    const int warp = threadIdx.x >> 5;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        int64_t t;
        const td_segment* g;
        if constexpr (ONE) {
            g = &seg1;
            t = seg1.tile_begin + i;
        } else {
            const int64_t e = __ldg(tiles + i);
            t = entry_tile(e);
            g = segs + entry_seg(e);
        }
        SegView S;
        load_desc<ONE>(g, S, NZ);
        const uint32_t vpr = (uint32_t)(S.cols >> 3);
        const int64_t tu = tile_units<ONE>(g);
        const int64_t first = (t - rd<ONE>(&g->tile_begin)) * tu;
        const uint32_t u0 = (uint32_t)first;
        const uint32_t u1 = (uint32_t)min(first + tu, rd<ONE>(&g->n_units));
        Acc a;
        a.zero();
        uint64_t h0 = 0, h1 = 0;
        const int64_t w0 = DG ? rd<ONE>(&g->y_word0) : 0;
        for (uint32_t base = u0 + threadIdx.x; base < u1; base += BLOCK * U) {
            uint4 xr[U][Q];
            uint4 yr[U][Q];
            uint4 zr[NZ > 0 ? NZ : 1][U][Q];
            bool ok[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint32_t u = base + k * BLOCK;
                ok[k] = u < u1;
                if (ok[k]) {
                    const uint32_t row = udiv(u, S.div_m, S.div_p);
                    const uint32_t cv = u - row * vpr;
                    const int64_t yo = ((int64_t)row * S.ys + (int64_t)cv * 8) * ES;
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        if (HX) xr[k][q] = ld_stream(S.x + ((int64_t)row * S.xs + (int64_t)cv * 8) * ES + 16 * q);
                        yr[k][q] = ld_stream(S.y + yo + 16 * q);
#pragma unroll
                        for (int j = 0; j < NZ; ++j) zr[j][k][q] = ld_stream(S.z[j] + yo + 16 * q);
                    }
                }
            }
            if constexpr (DG) {
                const bool flat = rd<ONE>(&g->rows) == 1;
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    if (!ok[k]) continue;
                    const uint32_t u = base + k * BLOCK;
                    uint64_t j;
                    if (flat) {
                        j = (uint64_t)w0 + (uint64_t)u * (2 * Q);       // one row: 2Q words per unit
                    } else {
                        const uint32_t row = udiv(u, S.div_m, S.div_p);
                        const uint32_t cv = u - row * vpr;
                        j = (uint64_t)(w0 + (((int64_t)row * S.ys + (int64_t)cv * 8) * ES >> 3));
                    }
#pragma unroll
                    for (int q = 0; q < Q; ++q) fp_vec(yr[k][q], j + 2 * q, h0, h1);
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (!ok[k]) continue;
#pragma unroll
                for (int e8 = 0; e8 < 8; ++e8) {
                    const double yv = Vec<DT>::at(yr[k], e8);
                    if (HX) {
                        const double xv = Vec<DT>::at(xr[k], e8);
                        const double d = xv - yv;
                        a.d2 = fma(d, d, a.d2);
                        a.x2 = fma(xv, xv, a.x2);
                    }
                    if (NZ > 0) a.y2 = fma(yv, yv, a.y2);
                    if constexpr (!SKIP) {
#pragma unroll
                        for (int j = 0; j < NZ; ++j) {
                            const double dz = yv - Vec<DT>::at(zr[j][k], e8);
                            a.z[j] = fma(dz, dz, a.z[j]);
                        }
                    }
                }
                if constexpr (SKIP) {
                    // a replica vector bit-identical to copy 0 adds exactly +0
                    // to its sum (or, for equal inf/NaN cells, turns a NaN
                    // error into 0 — neither ever wins check_replicas' strict
                    // max): skip its conversions, the bulk of the XU-pipe work
                    // in replica classes
#pragma unroll
                    for (int j = 0; j < NZ; ++j) {
                        if (!same_bits<Q>(zr[j][k], yr[k])) {
#pragma unroll
                            for (int e8 = 0; e8 < 8; ++e8) {
                                const double dz = Vec<DT>::at(yr[k], e8) - Vec<DT>::at(zr[j][k], e8);
                                a.z[j] = fma(dz, dz, a.z[j]);
                            }
                        }
                    }
                }
            }
        }
        write_warp_partial(a, USED, partials + (t * TD_WARPS_PER_TILE + warp) * TD_PARTIAL_STRIDE);
        if constexpr (DG) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                h0 += __shfl_xor_sync(0xffffffffu, h0, o);
                h1 += __shfl_xor_sync(0xffffffffu, h1, o);
            }
            const int slot = rd<ONE>(&g->digest_slot);
            if ((threadIdx.x & 31) == 0 && slot >= 0) {
                atomicAdd(digests + 2 * slot, (unsigned long long)h0);
                atomicAdd(digests + 2 * slot + 1, (unsigned long long)h1);
            }
        }
    }
    griddep_launch_dependents();
}

// generic class: per element, runtime dtypes, any alignment, any nz (<= 7).
// mode TD_MODE_STATIC replaces d2 by the count of cells failing
// |y - x| <= atol + rtol*|x| (numpy's elementwise test, each op rounded once;
// NaN fails) and leaves x2 at 0.
__global__ void __launch_bounds__(BLOCK, 4)
k_segnorm_generic(const td_segment* __restrict__ segs, const int64_t* __restrict__ tiles, int64_t n,
                  double* __restrict__ partials, int mode, double atol, double rtol) {
    const int warp = threadIdx.x >> 5;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const int64_t e = __ldg(tiles + i);
        const int64_t t = entry_tile(e);
        const td_segment* g = segs + entry_seg(e);
        const int nz = __ldg(&g->nz);
        const bool hx = (__ldg(&g->flags) & TD_SEG_HAS_X) != 0;
        const int xdt = __ldg(&g->x_dtype);
        const int ydt = __ldg(&g->y_dtype);
        SegView S;
        load_desc(g, S, nz);
        const uint32_t cols = (uint32_t)S.cols;
        const int64_t tu = tile_units(g);
        const int64_t first = (t - __ldg(&g->tile_begin)) * tu;
        const uint32_t u0 = (uint32_t)first;
        const uint32_t u1 = (uint32_t)min(first + tu, __ldg(&g->n_units));
        Acc a;
        a.zero();
        for (uint32_t u = u0 + threadIdx.x; u < u1; u += BLOCK) {
            const uint32_t row = udiv(u, S.div_m, S.div_p);
            const uint32_t col = u - row * cols;
            const int64_t yi = (int64_t)row * S.ys + col;
            const double yv = load_elem(S.y, ydt, yi);
            if (hx) {
                const double xv = load_elem(S.x, xdt, (int64_t)row * S.xs + col);
                if (mode == TD_MODE_STATIC) {
                    const double lim = __dadd_rn(atol, __dmul_rn(rtol, fabs(xv)));
                    if (!(fabs(__dsub_rn(yv, xv)) <= lim)) a.d2 += 1.0;
                } else {
                    const double d = xv - yv;
                    a.d2 = fma(d, d, a.d2);
                    a.x2 = fma(xv, xv, a.x2);
                }
            }
            if (nz > 0) {
                a.y2 = fma(yv, yv, a.y2);
#pragma unroll
                for (int j = 0; j < TD_MAX_Z; ++j) {
                    if (j < nz) {
                        const double dz = yv - load_elem(S.z[j], ydt, yi);
                        a.z[j] = fma(dz, dz, a.z[j]);
                    }
                }
            }
        }
        write_warp_partial(a, nz > 0 ? 3 + nz : 2,
                           partials + (t * TD_WARPS_PER_TILE + warp) * TD_PARTIAL_STRIDE);
    }
    griddep_launch_dependents();
}

typedef void (*segnorm_fn)(const td_segment*, const int64_t*, int64_t, double*, unsigned long long*, td_segment);

// ---------------------------------------------------------------------------
// Bulk-copy pipelined walker (compare classes, 2-byte payloads, nz = 0):
// a warp-specialised CTA — warp 8 is a producer that moves each tile's x and
// y bytes into a ring of shared-memory stages with cp.async.bulk (the TMA
// engine, SASS UBLKCP), each stage's bytes tracked by an mbarrier
// (complete_tx); warps 0-7 consume a stage from shared memory (fp64 norms,
// and for DG the 128-bit digest of y) and release it with one arrive per
// warp.  The loads hold no registers while in flight, so a CTA keeps
// STAGES x 2 x CH x 16 bytes in flight whatever the consumers' register
// budget — the LDG walker's digest class was latency-bound at 64 registers
// (ncu: 42% warps active, 4.3 long-scoreboard stalls per issue).
// Segment rows are cut into row pieces (16-B aligned, multiples of 16 B,
// guaranteed by the vector class), one bulk copy per piece and operand,
// issued by the producer warp's 32 lanes in parallel.  Partial rows and
// digest slots are written exactly as by k_segnorm_vec (warp w of a tile
// consumes units w*32+lane, +256, ... of every stage), so td_reduce_slots /
// td_finalize are unchanged.
#ifndef TD_BULK_CH
#define TD_BULK_CH 1024             // units (16 B of each operand) per stage
#endif
#ifndef TD_BULK_STAGES
#define TD_BULK_STAGES 3
#endif
#ifndef TD_BULK_MINB
#define TD_BULK_MINB 2              // CTAs per SM (16 consumer warps per SM; ncu, config-4
#endif                              // share: 4.58 ms vs 5.61 ms at 1 CTA x 6 stages)
constexpr int BULK_THREADS = BLOCK + 32;
constexpr uint32_t BULK_OPB = TD_BULK_CH * 16;   // bytes per operand per stage
constexpr size_t BULK_SMEM = (size_t)TD_BULK_STAGES * 2 * BULK_OPB + 2 * TD_BULK_STAGES * sizeof(uint64_t);

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "TD_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra TD_WAIT;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}

#ifndef TD_BULK_ACC
#define TD_BULK_ACC 2
#endif
#ifndef TD_BULK_ICONV
#define TD_BULK_ICONV 0
#endif

// bf16 element e of a 16-B vector as f64 without F2F: its bits placed under
// the f64 exponent field (value x * 2^-896, a double normal for bf16 normals
// and a double subnormal for bf16 subnormals, zero for zero), then one exact
// DMUL by 2^896.  Not for inf/NaN (exponent field 255): see bf16_any_infnan.
__device__ __forceinline__ double bf16_f64_int(const uint4* q, int e) {
    const uint32_t w = (&q[0].x)[e >> 1];
    const uint32_t f = (e & 1) ? (w & 0xffff0000u) : (w << 16);      // f32 bits
    const uint32_t hi = (f & 0x80000000u) | ((f & 0x7fffffffu) >> 3);
    return __dmul_rn(__hiloint2double((int)hi, 0), 0x1p896);
}

__device__ __forceinline__ bool bf16_any_infnan(const uint4& a, const uint4& b) {
    const uint32_t m = 0x7f807f80u;
    uint32_t r = __vcmpeq2(a.x & m, m) | __vcmpeq2(a.y & m, m) | __vcmpeq2(a.z & m, m) | __vcmpeq2(a.w & m, m);
    r |= __vcmpeq2(b.x & m, m) | __vcmpeq2(b.y & m, m) | __vcmpeq2(b.z & m, m) | __vcmpeq2(b.w & m, m);
    return r != 0;
}

template <int DT, bool DG>
__global__ void __launch_bounds__(BULK_THREADS, TD_BULK_MINB)
k_segnorm_bulk(const td_segment* __restrict__ segs, const int64_t* __restrict__ tiles, int64_t n,
               double* __restrict__ partials, unsigned long long* __restrict__ digests,
               const __grid_constant__ td_segment seg1) {
    static_assert(Vec<DT>::Q == 1, "2-byte payloads: 8 elements per 16-B unit");
    constexpr int ES = 2;
    constexpr int ST = TD_BULK_STAGES;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t base = smem_addr(smem);
    const uint32_t bars = base + ST * 2 * BULK_OPB;              // full[s], then empty[s]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(bars + 8 * s, 1);
            mbar_init(bars + 8 * (ST + s), NWARP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t stage = 0, phase = 0;
    if (warp == NWARP) {
        // ---- producer warp ----
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
        for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
            const int64_t e = __ldg(tiles + i);
            const int64_t t = entry_tile(e);
            const td_segment* g = segs + entry_seg(e);
            const char* x = reinterpret_cast<const char*>(__ldg(&g->x));
            const char* y = reinterpret_cast<const char*>(__ldg(&g->y));
            const int64_t xs = __ldg(&g->x_stride), ys = __ldg(&g->y_stride);
            const uint32_t vpr = (uint32_t)(__ldg(&g->cols) >> 3);
            const uint32_t dm = __ldg(&g->div_m);
            const int dp = __ldg(&g->div_p);
            const int64_t tu = tile_units(g);
            const int64_t first = (t - __ldg(&g->tile_begin)) * tu;
            const uint32_t u0 = (uint32_t)first;
            const uint32_t u1 = (uint32_t)min(first + tu, __ldg(&g->n_units));
            for (uint32_t c0 = u0; c0 < u1; c0 += TD_BULK_CH) {
                const uint32_t c1 = min(c0 + (uint32_t)TD_BULK_CH, u1);
                const uint32_t full = bars + 8 * stage;
                if (lane == 0) {
                    mbar_wait(bars + 8 * (ST + stage), phase ^ 1);   // consumers released the slot
                    mbar_expect_tx(full, 2u * (c1 - c0) * 16u);
                }
                __syncwarp();
                const uint32_t xd = base + stage * 2 * BULK_OPB, yd = xd + BULK_OPB;
                const uint32_t r0 = udiv(c0, dm, dp), r1 = udiv(c1 - 1, dm, dp);
                for (uint32_t r = r0 + lane; r <= r1; r += 32) {
                    const uint32_t a = max(c0, r * vpr), b = min(c1, (r + 1) * vpr);
                    const uint32_t cv = a - r * vpr, bytes = (b - a) * 16u, so = (a - c0) * 16u;
                    bulk_g2s(xd + so, x + ((int64_t)r * xs + (int64_t)cv * 8) * ES, bytes, full, policy);
                    bulk_g2s(yd + so, y + ((int64_t)r * ys + (int64_t)cv * 8) * ES, bytes, full, policy);
                }
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ---- consumer warps ----
        for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
            const int64_t e = __ldg(tiles + i);
            const int64_t t = entry_tile(e);
            const td_segment* g = segs + entry_seg(e);
            const int64_t tu = tile_units(g);
            const int64_t first = (t - __ldg(&g->tile_begin)) * tu;
            const uint32_t u0 = (uint32_t)first;
            const uint32_t u1 = (uint32_t)min(first + tu, __ldg(&g->n_units));
            const uint32_t vpr = (uint32_t)(__ldg(&g->cols) >> 3);
            const uint32_t dm = __ldg(&g->div_m);
            const int dp = __ldg(&g->div_p);
            const int64_t ys = __ldg(&g->y_stride);
            const int64_t w0 = DG ? __ldg(&g->y_word0) : 0;
            const bool flat = __ldg(&g->rows) == 1;
            const uint64_t key0 = (uint64_t)(w0 + 1) * GAMMA;
            // TD_BULK_ACC independent accumulator pairs (element e8 feeds pair
            // e8 % ACC): the DFMA chains, not the loads, bound a consumer warp
            constexpr int ACC = TD_BULK_ACC;
            double d2[ACC], x2[ACC];
#pragma unroll
            for (int q = 0; q < ACC; ++q) d2[q] = x2[q] = 0.0;
            uint64_t h0 = 0, h1 = 0;
            for (uint32_t c0 = u0; c0 < u1; c0 += TD_BULK_CH) {
                const uint32_t c1 = min(c0 + (uint32_t)TD_BULK_CH, u1);
                mbar_wait(bars + 8 * stage, phase);
                const unsigned char* xs_ = smem + stage * 2 * BULK_OPB;
                const uint4* xv = reinterpret_cast<const uint4*>(xs_);
                const uint4* yv = reinterpret_cast<const uint4*>(xs_ + BULK_OPB);
                for (uint32_t k = threadIdx.x; k < c1 - c0; k += BLOCK) {
                    const uint4 xr = xv[k], yr = yv[k];
                    if constexpr (DG) {
                        const uint32_t u = c0 + k;
                        if (flat) {                  // one row: word index w0 + 2u
                            fp_vec_key(yr, key0 + (uint64_t)u * (2 * GAMMA), h0, h1);
                        } else {
                            const uint32_t row = udiv(u, dm, dp);
                            const uint32_t cv = u - row * vpr;
                            fp_vec(yr, (uint64_t)(w0 + (((int64_t)row * ys + (int64_t)cv * 8) * ES >> 3)), h0, h1);
                        }
                    }
                    if (TD_BULK_ICONV && DT == TD_BF16 && !bf16_any_infnan(xr, yr)) {
                        // bf16 -> f64 on the integer pipe + one exact DMUL (no F2F on XU)
#pragma unroll
                        for (int e8 = 0; e8 < 8; ++e8) {
                            const double a = bf16_f64_int(&xr, e8);
                            const double d = a - bf16_f64_int(&yr, e8);
                            d2[e8 % ACC] = fma(d, d, d2[e8 % ACC]);
                            x2[e8 % ACC] = fma(a, a, x2[e8 % ACC]);
                        }
                    } else {
#pragma unroll
                        for (int e8 = 0; e8 < 8; ++e8) {
                            const double a = Vec<DT>::at(&xr, e8);
                            const double d = a - Vec<DT>::at(&yr, e8);
                            d2[e8 % ACC] = fma(d, d, d2[e8 % ACC]);
                            x2[e8 % ACC] = fma(a, a, x2[e8 % ACC]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bars + 8 * (ST + stage));
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            Acc a;
            a.zero();
#pragma unroll
            for (int q = 0; q < ACC; ++q) {
                a.d2 += d2[q];
                a.x2 += x2[q];
            }
            write_warp_partial(a, 2, partials + (t * TD_WARPS_PER_TILE + warp) * TD_PARTIAL_STRIDE);
            if constexpr (DG) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    h0 += __shfl_xor_sync(0xffffffffu, h0, o);
                    h1 += __shfl_xor_sync(0xffffffffu, h1, o);
                }
                const int slot = __ldg(&g->digest_slot);
                if (lane == 0 && slot >= 0) {
                    atomicAdd(digests + 2 * slot, (unsigned long long)h0);
                    atomicAdd(digests + 2 * slot + 1, (unsigned long long)h1);
                }
            }
        }
    }
    griddep_launch_dependents();
}

// TD_BULK bit 0: digest classes take the bulk walker; bit 1: plain nz = 0
// compare classes too (2-byte payloads).  Default: digest classes only.
int bulk_mode() {
    static const int m = [] {
        const char* e = getenv("TD_BULK");
        return e ? atoi(e) : 1;
    }();
    return m;
}

segnorm_fn pick_bulk(int dt, int nz, bool hx, bool dg) {
    if (nz != 0 || !hx || (dt != TD_BF16 && dt != TD_F16)) return nullptr;
    const int m = bulk_mode();
    if (!(dg ? (m & 1) : (m & 2))) return nullptr;
    if (dt == TD_BF16) return dg ? k_segnorm_bulk<TD_BF16, true> : k_segnorm_bulk<TD_BF16, false>;
    return dg ? k_segnorm_bulk<TD_F16, true> : k_segnorm_bulk<TD_F16, false>;
}

static_assert(sizeof(td_segment) == 160, "td_segment layout");
static_assert(BLOCK / 32 == TD_WARPS_PER_TILE, "one partial row per warp of a tile");
static_assert(sizeof(td_id_desc) == 56, "td_id_desc layout");
static_assert(sizeof(td_group_desc) == 24, "td_group_desc layout");
static_assert(sizeof(td_id_result) == 32, "td_id_result layout");
static_assert(sizeof(td_group_result) == 16, "td_group_result layout");
static_assert(sizeof(td_class) == 72, "td_class layout");
static_assert(sizeof(td_chunk) == 24, "td_chunk layout");

#ifndef TD_NZ7_U
#define TD_NZ7_U 1
#endif
#ifndef TD_NZ7_MINB
#define TD_NZ7_MINB 2
#endif
#ifndef TD_NZ3_U
#define TD_NZ3_U 1
#endif
#ifndef TD_NZ3_MINB
#define TD_NZ3_MINB 4
#endif
#ifndef TD_NZ0_U
#define TD_NZ0_U 4
#endif
#ifndef TD_NZ0_MINB
#define TD_NZ0_MINB 4
#endif

// U keeps ~4-8 16-byte loads in flight per thread; wide replica classes trade
// occupancy (2 CTAs/SM, 128 registers) for no spills.
#ifndef TD_DG_U
#define TD_DG_U 2
#endif
#ifndef TD_DG_MINB
#define TD_DG_MINB 4
#endif
template <int DT>
segnorm_fn pick_vec(int nz, bool hx, bool dg, bool one = false) {
    constexpr int Q = Vec<DT>::Q;
    constexpr int U4 = 4 / Q > 0 ? 4 / Q : 1;
    constexpr int U2 = 2 / Q > 0 ? 2 / Q : 1;
    if (one)   // single-segment compare classes (one tensor per side)
        return (hx && nz == 0 && !dg)
                   ? k_segnorm_vec<DT, 0, true, (TD_NZ0_U / Q > 0 ? TD_NZ0_U / Q : 1), TD_NZ0_MINB, false, true>
                   : nullptr;
    if (dg)   // compares of cross-GPU replica groups: copy 0 alone (nz = 0)
        return (hx && nz == 0)
                   ? k_segnorm_vec<DT, 0, true, (TD_DG_U / Q > 0 ? TD_DG_U / Q : 1), TD_DG_MINB, true>
                   : nullptr;
    if (hx) {
        switch (nz) {
            case 0: return k_segnorm_vec<DT, 0, true, (TD_NZ0_U / Q > 0 ? TD_NZ0_U / Q : 1), TD_NZ0_MINB>;
            case 1: return k_segnorm_vec<DT, 1, true, U2, 4>;
            case 2: return k_segnorm_vec<DT, 2, true, 1, 4>;
            case 3: return k_segnorm_vec<DT, 3, true, TD_NZ3_U, TD_NZ3_MINB>;
            case 4: return k_segnorm_vec<DT, 4, true, 1, 2>;
            case 5: return k_segnorm_vec<DT, 5, true, 1, 2>;
            case 6: return k_segnorm_vec<DT, 6, true, 1, 2>;
            case 7: return k_segnorm_vec<DT, 7, true, TD_NZ7_U, TD_NZ7_MINB>;
            default: return nullptr;
        }
    }
    switch (nz) {
        case 1: return k_segnorm_vec<DT, 1, false, U4, 4>;
        case 2: return k_segnorm_vec<DT, 2, false, U2, 4>;
        case 3: return k_segnorm_vec<DT, 3, false, 1, 4>;
        case 4: return k_segnorm_vec<DT, 4, false, 1, 2>;
        case 5: return k_segnorm_vec<DT, 5, false, 1, 2>;
        case 6: return k_segnorm_vec<DT, 6, false, 1, 2>;
        case 7: return k_segnorm_vec<DT, 7, false, 1, 2>;
        default: return nullptr;
    }
}

// ---------------------------------------------------------------------------
// slot reduction: one warp per id / group, fixed lane-strided order + butterfly

__global__ void k_reduce_slots(const td_id_desc* __restrict__ ids, int n_ids,
                               const td_group_desc* __restrict__ groups, int n_groups,
                               const double* __restrict__ partials,
                               double* __restrict__ id_sums, double* __restrict__ group_sums) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t slot = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (slot >= (int64_t)n_ids + n_groups) return;
    if (slot < n_ids) {
        const int64_t tb = ids[slot].tile_begin, te = ids[slot].tile_end;
        double d2 = 0.0, x2 = 0.0;
        for (int64_t r = tb * TD_WARPS_PER_TILE + lane; r < te * TD_WARPS_PER_TILE; r += 32) {
            d2 += partials[r * TD_PARTIAL_STRIDE + 0];
            x2 += partials[r * TD_PARTIAL_STRIDE + 1];
        }
        d2 = warp_sum(d2);
        x2 = warp_sum(x2);
        if (lane == 0) {
            id_sums[2 * slot + 0] = d2;
            id_sums[2 * slot + 1] = x2;
        }
    } else {
        const int64_t g = slot - n_ids;
        const int64_t tb = groups[g].tile_begin, te = groups[g].tile_end;
        const int nz = groups[g].nz;
        double s[TD_SLOT_STRIDE];
#pragma unroll
        for (int k = 0; k < TD_SLOT_STRIDE; ++k) s[k] = 0.0;
        for (int64_t r = tb * TD_WARPS_PER_TILE + lane; r < te * TD_WARPS_PER_TILE; r += 32) {
#pragma unroll
            for (int k = 0; k < TD_SLOT_STRIDE; ++k)
                if (k <= nz) s[k] += partials[r * TD_PARTIAL_STRIDE + 2 + k];
        }
#pragma unroll
        for (int k = 0; k < TD_SLOT_STRIDE; ++k) {
            const double v = warp_sum(s[k]);
            if (lane == 0) group_sums[g * TD_SLOT_STRIDE + k] = v;
        }
    }
}

// rel_err_arrays' tail (tensor.py:163-167): two square roots, then a divide
__device__ __forceinline__ double rel_from_sums(double d2, double r2) {
    const double diff = __dsqrt_rn(d2);
    const double ref = __dsqrt_rn(r2);
    if (ref == 0.0) return diff == 0.0 ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
    return __ddiv_rn(diff, ref);
}

// group result of check_replicas (canonical.py:236-247) from reduced sums
__device__ __forceinline__ int group_verdict(const double* s, int nz, double replica_eps,
                                             td_group_result* out) {
    double worst = 0.0;
    int widx = -1;
    for (int j = 0; j < nz && j < TD_MAX_Z; ++j) {
        const double err = rel_from_sums(s[1 + j], s[0]);
        if (err > worst) { worst = err; widx = j + 1; }   // NaN never wins
    }
    const int mm = worst > replica_eps;
    out->worst = worst;
    out->worst_index = widx;
    out->mismatch = mm;
    return mm;
}

// check()'s verdict precedence (checker.py:328-354) for id i
__device__ __forceinline__ void id_verdict(int i, const td_id_desc& D, const int any_rep[2], double d2, double x2,
                                           double kappa, double eps, td_id_result* __restrict__ id_out,
                                           unsigned long long* __restrict__ near_ties) {
    int kinds[2] = {D.cand_host, D.ref_host};
    for (int side = 0; side < 2; ++side)   // replica problems precede the merge problem
        if (kinds[side] != TD_REPLICA && any_rep[side]) kinds[side] = TD_REPLICA;
    const double m = (eps > D.tolerance) ? eps : D.tolerance;   // kappa * max(tol, eps)
    const double thr = __dmul_rn(kappa, m);
    double obs = __longlong_as_double(0x7ff8000000000000LL);
    int tie = 0;
    int verdict;
    if (D.has_compare) obs = rel_from_sums(d2, x2);
    if (kinds[0]) verdict = kinds[0];
    else if (kinds[1]) verdict = kinds[1];
    else if (!D.has_compare) verdict = TD_MERGE;
    else {
        verdict = (obs > thr) ? TD_FLAG : TD_PASS;   // NaN -> pass (reference quirk)
        if (fabs(obs - thr) <= 1e-12 * thr) {
            tie = 1;
            if (near_ties) atomicAdd(near_ties, 1ull);
        }
    }
    id_out[i].observed = obs;
    id_out[i].threshold = thr;
    id_out[i].verdict = verdict;
    id_out[i].cand_kind = kinds[0];
    id_out[i].ref_kind = kinds[1];
    id_out[i].near_tie = tie;
}

__global__ void k_verdict(const td_id_desc* __restrict__ ids, int n_ids,
                          const td_group_desc* __restrict__ groups,
                          const double* __restrict__ id_sums, const double* __restrict__ group_sums,
                          double kappa, double eps, double replica_eps,
                          td_id_result* __restrict__ id_out, td_group_result* __restrict__ group_out,
                          unsigned long long* __restrict__ near_ties) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_ids) return;
    const td_id_desc D = ids[i];
    int any[2] = {0, 0};
    const int gb[2] = {D.cgroup_begin, D.rgroup_begin};
    const int ge[2] = {D.cgroup_end, D.rgroup_end};
    for (int side = 0; side < 2; ++side)
        for (int g = gb[side]; g < ge[side]; ++g)
            any[side] |= group_verdict(group_sums + (int64_t)g * TD_SLOT_STRIDE, groups[g].nz, replica_eps,
                                       group_out + g);
    id_verdict(i, D, any, id_sums[2 * i + 0], id_sums[2 * i + 1], kappa, eps, id_out, near_ties);
}

// fixed-order CTA sum (warp butterfly, then warps 0..7 in order); all threads get it
__device__ __forceinline__ double cta_sum(double v, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) s += red[w];
    __syncthreads();
    return s;
}

// Single-GPU finalisation: td_reduce_slots + td_verdict in ONE launch, one
// CTA per id (threads stride the id's partial rows; fixed-order reduction).
__global__ void __launch_bounds__(BLOCK)
k_finalize(const td_id_desc* __restrict__ ids, const td_group_desc* __restrict__ groups,
           const double* __restrict__ partials, double* __restrict__ id_sums, double* __restrict__ group_sums,
           double kappa, double eps, double replica_eps, td_id_result* __restrict__ id_out,
           td_group_result* __restrict__ group_out, unsigned long long* __restrict__ near_ties) {
    __shared__ double red[NWARP];
    griddep_wait();
    const int i = blockIdx.x;
    const td_id_desc D = ids[i];
    // FIN_U rows per thread in flight (independent loads, summed in a fixed
    // order): one CTA walks up to ~8 k rows, so a load-add chain per row was
    // pure L2 latency (6 us for a 1 MiB check, as long as its td_segnorm)
    constexpr int FIN_U = 8;
    double d2 = 0.0, x2 = 0.0;
    const int64_t r1 = D.tile_end * TD_WARPS_PER_TILE;
    for (int64_t r0 = D.tile_begin * TD_WARPS_PER_TILE + threadIdx.x; r0 < r1; r0 += BLOCK * FIN_U) {
        double a[FIN_U], b[FIN_U];
#pragma unroll
        for (int k = 0; k < FIN_U; ++k) {
            const int64_t r = r0 + (int64_t)k * BLOCK;
            a[k] = r < r1 ? __ldg(partials + r * TD_PARTIAL_STRIDE + 0) : 0.0;
            b[k] = r < r1 ? __ldg(partials + r * TD_PARTIAL_STRIDE + 1) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < FIN_U; ++k) {
            d2 += a[k];
            x2 += b[k];
        }
    }
    d2 = cta_sum(d2, red);
    x2 = cta_sum(x2, red);
    int any[2] = {0, 0};
    const int gb[2] = {D.cgroup_begin, D.rgroup_begin};
    const int ge[2] = {D.cgroup_end, D.rgroup_end};
    for (int side = 0; side < 2; ++side) {
        for (int g = gb[side]; g < ge[side]; ++g) {
            const td_group_desc G = groups[g];
            double sums[TD_SLOT_STRIDE];
#pragma unroll
            for (int k = 0; k < TD_SLOT_STRIDE; ++k) sums[k] = 0.0;
            const int64_t g1 = G.tile_end * TD_WARPS_PER_TILE;
            for (int64_t r0 = G.tile_begin * TD_WARPS_PER_TILE + threadIdx.x; r0 < g1; r0 += BLOCK * 2) {
                double v[2][TD_SLOT_STRIDE];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int64_t r = r0 + (int64_t)u * BLOCK;
#pragma unroll
                    for (int k = 0; k < TD_SLOT_STRIDE; ++k)
                        v[u][k] = (r < g1 && k <= G.nz) ? __ldg(partials + r * TD_PARTIAL_STRIDE + 2 + k) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int k = 0; k < TD_SLOT_STRIDE; ++k) sums[k] += v[u][k];
            }
#pragma unroll
            for (int k = 0; k < TD_SLOT_STRIDE; ++k) sums[k] = (k <= G.nz) ? cta_sum(sums[k], red) : 0.0;
            if (threadIdx.x == 0) {
#pragma unroll
                for (int k = 0; k < TD_SLOT_STRIDE; ++k) group_sums[(int64_t)g * TD_SLOT_STRIDE + k] = sums[k];
                any[side] |= group_verdict(sums, G.nz, replica_eps, group_out + g);
            }
        }
    }
    if (threadIdx.x == 0) {
        id_sums[2 * i + 0] = d2;
        id_sums[2 * i + 1] = x2;
        id_verdict(i, D, any, d2, x2, kappa, eps, id_out, near_ties);
    }
}

// rel_err_arrays(a, b) of two contiguous arrays in ONE launch (tensor.py:
// 158-167, the reference's basic compare): a grid-stride stream of 16-byte
// vectors (U=4 per operand in flight), fp64 d2 / a2 per thread, CTA sums to
// per-CTA partials, and the last CTA to finish (atomic ticket) reduces the
// partials in CTA order and applies the reference's zero conventions.  No
// planner, no second launch: the public API's latency for one pair is one
// kernel + one 24-byte D2H.  Deterministic for a given (n, grid).
// U = 4 vectors per operand at 4 CTAs/SM; 8 at 2 or 3 CTAs/SM measured 7-15%
// slower on a 1 GiB pair (tools/bench_relerr.py)
#ifndef TD_RELERR_U
#define TD_RELERR_U 4
#endif
#ifndef TD_RELERR_MINB
#define TD_RELERR_MINB 4
#endif
template <int DT>
__global__ void __launch_bounds__(BLOCK, TD_RELERR_MINB)
k_rel_err(const char* __restrict__ a, const char* __restrict__ b, int64_t n, double* __restrict__ part,
          unsigned int* __restrict__ ticket, double* __restrict__ out) {
    __shared__ double red[NWARP];
    __shared__ bool last;
    constexpr int Q = DT == TD_F64 ? 1 : Vec<DT == TD_F64 ? TD_F32 : DT>::Q;
    constexpr int ES = DT == TD_F32 ? 4 : (DT == TD_F64 ? 8 : 2);
    constexpr int U = TD_RELERR_U / Q;
    double d2 = 0.0, a2 = 0.0;
    const bool vec = DT != TD_F64 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
    const int64_t nv = vec ? n / 8 : 0;
    if constexpr (DT != TD_F64) {
        const int64_t stride = (int64_t)gridDim.x * BLOCK;
        for (int64_t v0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x; v0 < nv; v0 += stride * U) {
            uint4 xr[U][Q], yr[U][Q];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t v = v0 + k * stride;
                if (v < nv) {
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        xr[k][q] = ld_stream(a + (v * 8) * ES + 16 * q);
                        yr[k][q] = ld_stream(b + (v * 8) * ES + 16 * q);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (v0 + k * stride >= nv) continue;
#pragma unroll
                for (int e8 = 0; e8 < 8; ++e8) {
                    const double xv = Vec<DT>::at(xr[k], e8);
                    const double d = xv - Vec<DT>::at(yr[k], e8);
                    d2 = fma(d, d, d2);
                    a2 = fma(xv, xv, a2);
                }
            }
        }
    }
    for (int64_t i = nv * 8 + (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
        const double xv = load_elem(a, DT, i);
        const double d = xv - load_elem(b, DT, i);
        d2 = fma(d, d, d2);
        a2 = fma(xv, xv, a2);
    }
    d2 = cta_sum(d2, red);
    a2 = cta_sum(a2, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = d2;
        part[2 * blockIdx.x + 1] = a2;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s0 = 0.0, s1 = 0.0;
    for (int c = threadIdx.x; c < (int)gridDim.x; c += BLOCK) {
        s0 += __ldcg(part + 2 * c);
        s1 += __ldcg(part + 2 * c + 1);
    }
    s0 = cta_sum(s0, red);
    s1 = cta_sum(s1, red);
    if (threadIdx.x == 0) {
        out[0] = s0;
        out[1] = s1;
        out[2] = rel_from_sums(s0, s1);
        *ticket = 0u;                     // ready for the next call
    }
}

// First level of the slot reduction (td_reduce_chunks): 320 threads = 10
// warps, thread t owns partial column t % 10 and walks the chunk's rows as
// one flat, fully coalesced double array (320 is a multiple of the row
// stride, so a thread's column never changes).  Column sums are then taken
// over the 32 owners of each column in thread order.
constexpr int CHUNK_BLOCK = 32 * TD_PARTIAL_STRIDE;

__global__ void __launch_bounds__(CHUNK_BLOCK)
k_reduce_chunks(const double* __restrict__ partials, const td_chunk* __restrict__ chunks, int64_t n,
                double* __restrict__ out) {
    __shared__ double red[CHUNK_BLOCK];
    griddep_wait();
    const int t = threadIdx.x;
    constexpr int ROW = TD_WARPS_PER_TILE * TD_PARTIAL_STRIDE;   // doubles per output "tile"
    for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
        const int64_t rb = __ldg(&chunks[c].row_begin), re = __ldg(&chunks[c].row_end);
        const int k0 = __ldg(&chunks[c].k0), nk = __ldg(&chunks[c].nk);
        const int64_t f1 = re * TD_PARTIAL_STRIDE;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t f = rb * TD_PARTIAL_STRIDE + t;
        for (; f + 3 * CHUNK_BLOCK < f1; f += 4 * CHUNK_BLOCK) {
            s0 += __ldg(partials + f);
            s1 += __ldg(partials + f + CHUNK_BLOCK);
            s2 += __ldg(partials + f + 2 * CHUNK_BLOCK);
            s3 += __ldg(partials + f + 3 * CHUNK_BLOCK);
        }
        for (; f < f1; f += CHUNK_BLOCK) s0 += __ldg(partials + f);
        red[t] = (s0 + s1) + (s2 + s3);
        __syncthreads();
        if (t < ROW) {
            double v = 0.0;
            if (t >= k0 && t < k0 + nk && t < TD_PARTIAL_STRIDE)
                for (int i = t; i < CHUNK_BLOCK; i += TD_PARTIAL_STRIDE) v += red[i];
            out[c * ROW + t] = v;
        }
        __syncthreads();
    }
    griddep_launch_dependents();
}

// ---------------------------------------------------------------------------
// RNG streams


// word k (0-based) of the splitmix64 stream: mix(seed + (k+1)*gamma)  (generation.py:67-78)
__device__ __forceinline__ uint64_t splitmix_word(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * GAMMA;
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

// Philox4x32-10 keyed by the seed: block b = Philox(counter = b) yields two
// 64-bit words, word 2b = (out1:out0) and word 2b+1 = (out3:out2)
__device__ __forceinline__ uint4 philox_block(uint64_t seed, uint64_t blk) {
    uint32_t c0 = (uint32_t)blk, c1 = (uint32_t)(blk >> 32), c2 = 0, c3 = 0;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ uint64_t philox_lane(const uint4& o, uint64_t k) {
    return (k & 1) ? (((uint64_t)o.w << 32) | o.z) : (((uint64_t)o.y << 32) | o.x);
}

// word k of the Philox stream
__device__ __forceinline__ uint64_t philox_word(uint64_t seed, uint64_t k) {
    return philox_lane(philox_block(seed, k >> 1), k);
}

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * MIX1;
    z = (z ^ (z >> 27)) * MIX2;
    return z ^ (z >> 31);
}

// 2u - 1 with u = (w >> 11) * 2^-53 (generation.py:74-78, 166), without an
// int->double conversion (XU pipe): t = 2u = m * 2^-52 for the 53-bit m is
// exact as (1.m52 as a double) - (m < 2^52 ? 1 : 0); then t - 1 rounds once,
// exactly like numpy's 2.0*u - 1.0.  Folded: (1.m52) - (m < 2^52 ? 2 : 1).
__device__ __forceinline__ double signed_uniform(uint64_t seed, uint64_t k, int gen) {
    const uint64_t w = gen == TD_GEN_PHILOX4x32 ? philox_word(seed, k) : splitmix_word(seed, k);
    const uint64_t m = w >> 11;
    const double one_m = __longlong_as_double((long long)(0x3FF0000000000000ull | (m & 0xFFFFFFFFFFFFFull)));
    return __dsub_rn(one_m, (m >> 52) ? 1.0 : 2.0);
}

// quantize_array (tensor.py:64-77): RNE to p significand bits, unbounded
// exponent, clip to +-max_finite.  Done on the fp64 bit pattern: never via f32.
__device__ __forceinline__ double quantize_p(double y, int p, double maxf) {
    double s = y;
    bool scaled = false;
    if (fabs(s) < 0x1p-1000 && s != 0.0) { s = s * 0x1p200; scaled = true; }   // exact
    long long b = __double_as_longlong(s);
    const int drop = 53 - p;
    const long long mask = (1ll << drop) - 1;
    const long long lsb = (b >> drop) & 1ll;
    const long long sign = b & (long long)0x8000000000000000ull;
    long long mag = b & 0x7fffffffffffffffll;
    mag = (mag + (mask >> 1) + lsb) & ~mask;
    double r = __longlong_as_double(mag | sign);
    if (scaled) r = r * 0x1p-200;   // one IEEE rounding, as numpy's ldexp
    if (fabs(r) > maxf) r = copysign(maxf, r);
    return r;
}

__device__ __forceinline__ double apply_format(double y, int fmt) {
    switch (fmt) {
        case TD_FMT_BF16: return quantize_p(y, 8, 0x1.fep127);
        case TD_FMT_FP8E4M3: return quantize_p(y, 4, 448.0);
        case TD_FMT_FP32: return quantize_p(y, 24, 0x1.fffffep127);
        default: return y;
    }
}

// bf16 bits of a double that already has <= 8 significant bits; integer ops
// only (no F2F) for the normal bf16 range, exact conversion otherwise
__device__ __forceinline__ unsigned short bf16_bits_q8(double v) {
    const uint32_t hi = (uint32_t)((unsigned long long)__double_as_longlong(v) >> 32);
    const uint32_t sign = (hi >> 16) & 0x8000u;
    const uint32_t e = (hi >> 20) & 0x7ffu;
    if (e >= 897u && e <= 1150u) return (unsigned short)(sign | ((e - 896u) << 7) | ((hi >> 13) & 0x7fu));
    if (v == 0.0) return (unsigned short)sign;
    return __bfloat16_as_ushort(__float2bfloat16_rn((float)v));
}

__device__ __forceinline__ void store_elem(void* base, int dt, int64_t idx, double v) {
    switch (dt) {
        case TD_F32: reinterpret_cast<float*>(base)[idx] = (float)v; break;
        case TD_BF16: {
            // round f64 straight to 8 significand bits (no f64->f32->bf16 double rounding);
            // only the bf16 subnormal range goes through f32
            const double q = (isfinite(v) && fabs(v) >= 0x1p-126) ? quantize_p(v, 8, __longlong_as_double(0x7ff0000000000000LL)) : v;
            reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn((float)q);
            break;
        }
        case TD_F16: reinterpret_cast<__half*>(base)[idx] = __double2half(v); break;
        default: reinterpret_cast<double*>(base)[idx] = v; break;
    }
}

// Q_bf16(v) (tensor.py:64-77: RNE to 8 significant bits, unbounded exponent,
// clamp to +-max_finite) straight to bf16 bits with 32-bit integer ops: the
// round bit is f64 mantissa bit 44 (hi word bit 12), sticky = hi[11:0] | lo.
// Exact for every f64 normal whose rounded value is a bf16 normal; anything
// else (zero, bf16-subnormal range, inf/NaN) takes the exact slow path.
__device__ __forceinline__ uint32_t bf16_q8_bits(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
    const uint32_t sticky = (hi & 0xfffu) | lo;
    const uint32_t up = ((hi >> 12) & 1u) & (((sticky != 0u) ? 1u : 0u) | ((hi >> 13) & 1u));
    const uint32_t h = ((hi & 0x7fffffffu) >> 13) + up;      // exp(11) | mant(7), carry-safe
    const uint32_t e = h >> 7;
    const uint32_t sign = (hi >> 16) & 0x8000u;
    if (e >= 897u && e <= 1150u) return sign | ((e - 896u) << 7) | (h & 0x7fu);
    if (e > 1150u && e < 2047u) return sign | 0x7f7fu;              // clamp to bf16 max_finite
    return (uint32_t)bf16_bits_q8(quantize_p(v, 8, 0x1.fep127));  // zero, tiny, inf/NaN
}

__device__ __forceinline__ double perturb_one(double xv, uint64_t seed, uint64_t k, double eps, int gen, int& bad) {
    const double u = signed_uniform(seed, k, gen);
    const double f = __dadd_rn(1.0, __dmul_rn(u, eps));   // 1.0 + u*eps
    const double v = __dmul_rn(xv, f);                     // x * factor
    bad |= !isfinite(v);
    return v;
}

// One thread per group of 8 consecutive elements of a row (cols % 8 == 0,
// 16-byte aligned rows): 16-byte loads/stores for bf16, one division per group.
__global__ void __launch_bounds__(256)
k_perturb_vec8(const char* x, char* y, int dt_in, int dt_out, int64_t rows, int64_t cols,
               int64_t full_cols, int64_t col0, const int64_t* __restrict__ row_pos, int64_t row0,
               uint64_t seed, double eps, int fmt, int gen, uint32_t div_m, int div_p,
               unsigned long long* __restrict__ nonfinite) {
    const int64_t groups = rows * (cols >> 3);
    const uint32_t gpr = (uint32_t)(cols >> 3);
    int bad = 0;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = groups < (1ll << 31) ? (int64_t)udiv((uint32_t)g, div_m, div_p) : g / gpr;
        const int64_t c = (g - r * gpr) * 8;
        const int64_t pos = row_pos ? __ldg(row_pos + r) : row0 + r;
        const uint64_t kb = (uint64_t)(pos * full_cols + col0 + c);
        const int64_t idx = r * cols + c;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const double v = perturb_one(load_elem(x, dt_in, idx + h), seed, kb + h, eps, gen, bad);
            store_elem(y, dt_out, idx + h, apply_format(v, fmt));
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1ull);
}

// bf16 -> bf16 with the bf16 policy, 16-B aligned rows, cols % 8 == 0: the
// common case (block inputs / embedding outputs of a bf16 model).  One thread
// per 8-element group; the generator is a template parameter so the loop has
// no stream switch, and the per-element work is branch-free:
//   * splitmix64 word kb+j = mix(z0 + j*gamma) (z0 = seed + (kb+1)*gamma);
//   * 2u-1 from the word's top 53 bits by exponent splice (no I2F);
//   * v = x * (1 + u*eps) in fp64, each op rounded (numpy's order);
//   * Q_bf16(v) as one 64-bit add of the RNE bias (2^44 - 1 + lsb) on |v|'s
//     bits, giving the bf16 pattern pre-shifted into the top half-word, and
//     a range test on the rounded exponent (bf16 normal range, finite).
// A group with any element outside that range (zero, bf16-subnormal range,
// overflow clamp, inf/NaN) is recomputed element by element with the exact
// general path (rare; zeros only cost a redo of their own group).
// The kernel is integer-issue bound (ncu: ALU pipe 80%, fmaheavy 44%).
// Moving the 64-bit right shifts to the FMA pipe as multiply-highs by
// 2^(32-s) (IMAD.HI + IMAD.WIDE instead of two SHF) was measured per shift
// site: every mix of sites lost 2-31% (fmaheavy saturates first; each
// IMAD.HI/WIDE costs ~2.6x the SHF it replaces), so the shifts stay on ALU.
#ifndef TD_PERTURB_CVT
#define TD_PERTURB_CVT 1        // 0: the integer RNE of round 1 (A/B)
#endif
template <int GEN>
__global__ void __launch_bounds__(256)
k_perturb_bf16(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t rows, uint32_t gpr,
               int64_t full_cols, int64_t col0, const int64_t* __restrict__ row_pos, int64_t row0,
               uint64_t seed, double eps, uint32_t div_m, int div_p,
               unsigned long long* __restrict__ nonfinite) {
    const int64_t groups = rows * (int64_t)gpr;
    int bad = 0;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = groups < (1ll << 31) ? (int64_t)udiv((uint32_t)g, div_m, div_p) : g / gpr;
        const int64_t c = (g - r * gpr) * 8;
        const int64_t pos = row_pos ? __ldg(row_pos + r) : row0 + r;
        const uint64_t kb = (uint64_t)(pos * full_cols + col0 + c);
        const uint4 in = __ldcs(x + g);
        const uint32_t iw[4] = {in.x, in.y, in.z, in.w};
        uint32_t ow[4];
        uint32_t out_of_range = 0;
        const uint64_t z0 = seed + (kb + 1) * GAMMA;
        uint4 blk;
#if TD_PERTURB_CVT
        uint32_t hlo = 0, emin = 0xffffffffu, emax = 0u;
#endif
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t xb = (j & 1) ? (iw[j >> 1] & 0xffff0000u) : (iw[j >> 1] << 16);
            const double xv = (double)__uint_as_float(xb);
            double u;
            {
                uint64_t w;
                if (GEN == TD_GEN_PHILOX4x32) {
                    // one Philox block per two words: recompute at even words (and word 0)
                    if (j == 0 || ((kb + j) & 1) == 0) blk = philox_block(seed, (kb + j) >> 1);
                    w = philox_lane(blk, kb + j);
                } else {
                    w = splitmix_mix(z0 + (uint64_t)j * GAMMA);
                }
                const uint64_t m = w >> 11;
                const double one_m = __longlong_as_double((long long)(0x3FF0000000000000ull | (m & 0xFFFFFFFFFFFFFull)));
                u = __dsub_rn(one_m, (m >> 52) ? 1.0 : 2.0);
            }
            const double v = __dmul_rn(xv, __dadd_rn(1.0, __dmul_rn(u, eps)));
#if TD_PERTURB_CVT
            // Q_bf16 as ONE XU conversion: F2F.BF16.F64 is IEEE round-to-nearest-
            // even from f64 straight to bf16 — the reference's quantizer wherever
            // the result is a bf16 normal.  The two halves of each packed pair
            // are range-tested together (16x2 min/max of the exponent fields):
            // a zero or subnormal result (exponent 0), an overflow to inf or a
            // NaN (exponent 0xff: the reference clamps to max_finite instead)
            // sends the group to the exact path below.
            {
                const uint32_t hb = __bfloat16_as_ushort(__double2bfloat16(v));
                if (j & 1) {
                    const uint32_t w = (hb << 16) | hlo;
                    const uint32_t t = w & 0x7f807f80u;
                    emin = __vminu2(emin, t);
                    emax = __vmaxu2(emax, t);
                    ow[j >> 1] = w;
                } else {
                    hlo = hb;
                }
            }
#else
            const uint64_t b = (uint64_t)__double_as_longlong(v);
            const uint32_t hi = (uint32_t)(b >> 32);
            const uint64_t rb = (b & 0x7fffffffffffffffull) + 0xfffffffffffull + ((hi >> 13) & 1u);
            const uint32_t rh = (uint32_t)(rb >> 32);      // rounded |v|: exp(11) at 30..20, mant7 at 19..13
            out_of_range |= (rh - (897u << 20)) < (254u << 20) ? 0u : 1u;
            const uint32_t t = (((rh << 3) - (896u << 23)) & 0x7fff0000u) | (hi & 0x80000000u);
            if (j & 1) ow[j >> 1] = __byte_perm(ow[j >> 1], t, 0x7632);
            else ow[j >> 1] = t;
#endif
        }
#if TD_PERTURB_CVT
        out_of_range = ((emin & 0xffffu) < 0x0080u) | ((emin >> 16) < 0x0080u) |
                       ((emax & 0xffffu) > 0x7f00u) | ((emax >> 16) > 0x7f00u);
#endif
        if (out_of_range) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t xb = (j & 1) ? (iw[j >> 1] & 0xffff0000u) : (iw[j >> 1] << 16);
                const double v = perturb_one((double)__uint_as_float(xb), seed, kb + j, eps, GEN, bad);
                const uint32_t q = bf16_q8_bits(v);
                ow[j >> 1] = (j & 1) ? ((ow[j >> 1] & 0xffffu) | (q << 16)) : ((ow[j >> 1] & 0xffff0000u) | q);
            }
        }
        __stcs(y + g, make_uint4(ow[0], ow[1], ow[2], ow[3]));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1ull);
}

__global__ void k_perturb(const char* x, char* y, int dt_in, int dt_out,
                          int64_t rows, int64_t cols, int64_t full_cols, int64_t col0,
                          const int64_t* __restrict__ row_pos, int64_t row0,
                          uint64_t seed, double eps, int fmt, int gen,
                          unsigned long long* __restrict__ nonfinite) {
    int bad = 0;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const int64_t pos = row_pos ? row_pos[r] : row0 + r;
        const uint64_t kbase = (uint64_t)(pos * full_cols + col0);
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (int64_t)gridDim.x * blockDim.x) {
            const int64_t idx = r * cols + c;
            const double v = perturb_one(load_elem(x, dt_in, idx), seed, kbase + (uint64_t)c, eps, gen, bad);
            store_elem(y, dt_out, idx, apply_format(v, fmt));
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1ull);
}

__global__ void k_signed_uniforms(double* __restrict__ out, int64_t n, uint64_t seed, int64_t k0, int gen) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = signed_uniform(seed, (uint64_t)(k0 + i), gen);
}

__global__ void k_quantize(const double* __restrict__ x, char* __restrict__ y, int dt_out, int64_t n,
                           int fmt, unsigned long long* __restrict__ nonfinite) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (!isfinite(v)) bad = 1;
        store_elem(y, dt_out, i, apply_format(v, fmt));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicAdd(nonfinite, 1ull);
}

// ---------------------------------------------------------------------------
// Replica digests (multi-GPU replica groups): for each item, an
// order-independent 128-bit digest of its bytes, sum over 8-byte words w_j
// (tail zero-padded) into two lanes by fp_word (see there).
// Position-keyed, so permuted shards differ.
// One launch covers every item: a flat list of 256 KB chunks (prefix sums of
// per-item chunk counts, binary-searched per chunk), 16-byte streaming loads,
// TD_FP_U = 8 vectors in flight per thread (4: 5.8 TB/s, 8: 6.7, 16: 6.4 —
// tools/bench_digest.py); warp sums are added atomically (wrapping
// u64 adds commute: the digest does not depend on the order).

__global__ void __launch_bounds__(BLOCK)
k_fingerprint(const td_fp_item* __restrict__ items, const int64_t* __restrict__ chunk_begin, int n_items,
              int64_t n_chunks, unsigned long long* __restrict__ out) {
    constexpr int U = TD_FP_U;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        int lo = 0, hi = n_items - 1;            // last item with chunk_begin[i] <= c
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(chunk_begin + mid) <= c) lo = mid;
            else hi = mid - 1;
        }
        const char* p = reinterpret_cast<const char*>(__ldg(reinterpret_cast<const unsigned long long*>(&items[lo].ptr)));
        const int64_t nb = __ldg(&items[lo].nbytes);
        const int64_t off0 = (c - __ldg(chunk_begin + lo)) * TD_FP_CHUNK;
        const int64_t off1 = min(off0 + (int64_t)TD_FP_CHUNK, nb);
        uint64_t h0 = 0, h1 = 0;
        int64_t scalar_from = off0;
        if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
            const int64_t vend = off1 & ~(int64_t)15;
            for (int64_t base = off0 + 16 * threadIdx.x; base < vend; base += 16 * BLOCK * U) {
                const uint64_t kbase = (uint64_t)((base >> 3) + 1) * GAMMA;
                uint4 v[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int64_t o = base + 16 * BLOCK * k;
                    if (o < vend) v[k] = ld_stream(p + o);
                }
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    const int64_t o = base + 16 * BLOCK * k;
                    if (o < vend) {
                        // key of word o/8: base key + k * (2 * BLOCK) * gamma (adds only)
                        const uint64_t key = kbase + (uint64_t)k * (2ull * BLOCK * GAMMA);
                        fp_vec_key(v[k], key, h0, h1);
                    }
                }
            }
            scalar_from = vend;
        }
        // unaligned items, and the last < 16 bytes of an item: whole words
        // assembled byte by byte, zero-padded past the end
        for (int64_t o = (scalar_from & ~(int64_t)7) + 8 * threadIdx.x; o < off1; o += 8 * BLOCK) {
            uint64_t w = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if (o + b < nb) w |= (uint64_t)(unsigned char)__ldg(p + o + b) << (8 * b);
            fp_word(w, (uint64_t)(o >> 3), h0, h1);
        }
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            h0 += __shfl_xor_sync(0xffffffffu, h0, s);
            h1 += __shfl_xor_sync(0xffffffffu, h1, s);
        }
        if ((threadIdx.x & 31) == 0 && (h0 | h1)) {
            atomicAdd(out + 2 * lo, (unsigned long long)h0);
            atomicAdd(out + 2 * lo + 1, (unsigned long long)h1);
        }
    }
}

__global__ void k_box_gather(const char* __restrict__ src, int dt, double* __restrict__ dst,
                             const int64_t* __restrict__ boxes) {
    const int64_t* b = boxes + 6 * (int64_t)blockIdx.y;
    const int64_t so = b[0], dof = b[1], rows = b[2], cols = b[3], ss = b[4], ds = b[5];
    const int64_t n = rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        dst[dof + r * ds + c] = load_elem(src, dt, so + r * ss + c);
    }
}

__device__ __forceinline__ double uniform53(uint64_t seed, uint64_t k) {
    return __dmul_rn((double)(splitmix_word(seed, k) >> 11), 0x1p-53);
}

// raw word index of the m-th word that survives the skip list (sorted)
__device__ __forceinline__ uint64_t skip_map(uint64_t m, const int64_t* __restrict__ skips, int n_skips) {
    for (int j = 0; j < n_skips; ++j)
        if ((uint64_t)skips[j] <= m) ++m;
    return m;
}

__global__ void k_generate(double* __restrict__ out, int64_t n, uint64_t seed, int dist, double a, double b,
                           int64_t vocab, const int64_t* __restrict__ skips, int n_skips,
                           unsigned long long* __restrict__ zero_count, int64_t* __restrict__ zero_pos,
                           int zero_cap) {
    const int64_t pairs = (n + 1) / 2;
    const int64_t words = dist == 0 ? 2 * pairs + n_skips : n;
    // zero census over the words the normal stream consumes
    if (dist == 0 && zero_count) {
        for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < words;
             k += (int64_t)gridDim.x * blockDim.x) {
            if ((splitmix_word(seed, (uint64_t)k) >> 11) == 0) {
                const unsigned long long slot = atomicAdd(zero_count, 1ull);
                if ((int64_t)slot < zero_cap) zero_pos[slot] = k;
            }
        }
    }
    if (dist == 0) {
        for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs;
             p += (int64_t)gridDim.x * blockDim.x) {
            const double u1 = uniform53(seed, skip_map(2 * p, skips, n_skips));
            const double u2 = uniform53(seed, skip_map(2 * p + 1, skips, n_skips));
            const double r = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
            const double th = __dmul_rn(2.0 * 3.141592653589793, u2);
            const double z0 = __dmul_rn(r, cos(th));
            out[2 * p] = __dadd_rn(__dmul_rn(z0, b), a);
            if (2 * p + 1 < n) out[2 * p + 1] = __dadd_rn(__dmul_rn(__dmul_rn(r, sin(th)), b), a);
        }
    } else {
        for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
             k += (int64_t)gridDim.x * blockDim.x) {
            const double u = uniform53(seed, (uint64_t)k);
            if (dist == 1) {
                out[k] = __dadd_rn(a, __dmul_rn(u, __dsub_rn(b, a)));
            } else {
                const double f = floor(__dmul_rn(u, (double)vocab));
                out[k] = f < (double)(vocab - 1) ? f : (double)(vocab - 1);
            }
        }
    }
}

// one CTA per range (grid-strided); bytes move 4 at a time when source and
// destination agree mod 4, else one at a time (file payloads are unaligned)
// Ranges are cut into TD_GATHER_PIECE-byte pieces dealt round-robin over the
// grid (every CTA walks the range table, ~6k rows for a large trace), so one
// 200 MB record spreads over every SM instead of serialising on one CTA.
// Each piece stores aligned uint4s: a few head bytes bring the destination to
// 16 B, then the source is read as uint4 (same alignment), as four u32
// (4-byte aligned), or as five aligned u32 funnel-shifted into place (any
// other offset: TTRC payload offsets are arbitrary, and the file writer
// scatters a 4-byte-aligned f32 arena to them).  The shifted path reads
// only aligned words holding at least one byte of the range (it stops 3
// bytes short of the end; the tail goes bytewise), so it never crosses an
// allocation boundary.
#define TD_GATHER_PIECE (64 << 10)
__global__ void __launch_bounds__(256) k_gather_bytes(const unsigned char* __restrict__ src,
                                                      unsigned char* __restrict__ dst,
                                                      const int64_t* __restrict__ ranges, int64_t n) {
    const int64_t grid = gridDim.x;
    int64_t base = 0;                                  // global index of range r's first piece
    for (int64_t r = 0; r < n; ++r) {
        const int64_t so = ranges[3 * r], dof = ranges[3 * r + 1], nb = ranges[3 * r + 2];
        const int64_t pieces = (nb + TD_GATHER_PIECE - 1) / TD_GATHER_PIECE;
        int64_t k = ((int64_t)blockIdx.x - base % grid + grid) % grid;
        base += pieces;
        for (; k < pieces; k += grid) {
            const int64_t lo = k * TD_GATHER_PIECE;
            const int64_t len = nb - lo < TD_GATHER_PIECE ? nb - lo : TD_GATHER_PIECE;
            const unsigned char* s = src + so + lo;
            unsigned char* d = dst + dof + lo;
            int64_t head = (16 - (int64_t)(reinterpret_cast<uintptr_t>(d) & 15)) & 15;
            if (head > len) head = len;
            for (int64_t i = threadIdx.x; i < head; i += blockDim.x) d[i] = s[i];
            const unsigned char* s1 = s + head;
            uint4* d16 = reinterpret_cast<uint4*>(d + head);
            const int64_t rest = len - head;
            const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(s1) & 15);
            int64_t v;
            if (mis == 0) {
                v = rest >> 4;
                const uint4* s16 = reinterpret_cast<const uint4*>(s1);
                for (int64_t i = threadIdx.x; i < v; i += blockDim.x) d16[i] = s16[i];
            } else if ((mis & 3) == 0) {
                v = rest >> 4;
                const uint32_t* s4 = reinterpret_cast<const uint32_t*>(s1);
                for (int64_t i = threadIdx.x; i < v; i += blockDim.x)
                    d16[i] = make_uint4(s4[4 * i], s4[4 * i + 1], s4[4 * i + 2], s4[4 * i + 3]);
            } else {
                const uint32_t sh = 8 * (mis & 3);
                v = rest >= 3 ? (rest - 3) >> 4 : 0;
                const uint32_t* sw = reinterpret_cast<const uint32_t*>(s1 - (mis & 3));
                for (int64_t i = threadIdx.x; i < v; i += blockDim.x) {
                    const uint32_t w0 = sw[4 * i], w1 = sw[4 * i + 1], w2 = sw[4 * i + 2],
                                   w3 = sw[4 * i + 3], w4 = sw[4 * i + 4];
                    d16[i] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh),
                                        __funnelshift_r(w2, w3, sh), __funnelshift_r(w3, w4, sh));
                }
            }
            unsigned char* d1 = d + head;
            for (int64_t i = 16 * v + threadIdx.x; i < rest; i += blockDim.x) d1[i] = s1[i];
        }
    }
}

// The same gather through shared memory: per 16 KiB piece one elected thread
// moves the piece's source bytes, widened to the enclosing aligned 16-byte
// blocks, with ONE cp.async.bulk (the TMA engine; 16-B aligned by
// construction whatever the record's offset) into a shared-memory stage,
// tracked by an mbarrier's transaction count; the CTA writes aligned uint4s
// built from 4-byte shared-memory words funnel-shifted into place (any source
// misalignment), with bytewise heads / tails.  Bulk copies hold no registers
// in flight, so the 8 resident CTAs of an SM keep 128 KiB of loads
// outstanding (a second stage per CTA, the next piece's copy overlapping
// this one's stores, measured slower: 33 KiB per CTA leaves 6 resident).
// The widened block never reaches past the 16-B block holding the range's
// last byte (same page), as the LDG kernel's aligned words.
#ifndef TD_GATHER_STAGE
#define TD_GATHER_STAGE (16 << 10)
#endif
constexpr int GATHER_SMEM = TD_GATHER_STAGE + 64 + 16;
__global__ void __launch_bounds__(256) k_gather_staged(const unsigned char* __restrict__ src,
                                                       unsigned char* __restrict__ dst,
                                                       const int64_t* __restrict__ ranges, int64_t n) {
    extern __shared__ __align__(128) unsigned char sm[];
    const uint32_t sbase = smem_addr(sm);
    const uint32_t sbar = smem_addr(sm + TD_GATHER_STAGE + 64);
    uint64_t policy = 0;
    if (threadIdx.x == 0) {
        mbar_init(sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    }
    __syncthreads();
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sm);
    uint32_t phase = 0;
    const int64_t grid = gridDim.x;
    int64_t base = 0;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t so = ranges[3 * r], dof = ranges[3 * r + 1], nb = ranges[3 * r + 2];
        const int64_t pieces = (nb + TD_GATHER_STAGE - 1) / TD_GATHER_STAGE;
        int64_t k = ((int64_t)blockIdx.x - base % grid + grid) % grid;
        base += pieces;
        for (; k < pieces; k += grid) {
            const int64_t lo = k * TD_GATHER_STAGE;
            const uint32_t len = (uint32_t)(nb - lo < TD_GATHER_STAGE ? nb - lo : TD_GATHER_STAGE);
            const unsigned char* s = src + so + lo;
            unsigned char* d = dst + dof + lo;
            const uint32_t mis0 = (uint32_t)(reinterpret_cast<uintptr_t>(s) & 15);
            const uint32_t bytes = (mis0 + len + 15u) & ~15u;
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier reads before the refill
                mbar_expect_tx(sbar, bytes);
                bulk_g2s(sbase, s - mis0, bytes, sbar, policy);
            }
            mbar_wait(sbar, phase);
            phase ^= 1u;
            uint32_t head = (16u - (uint32_t)(reinterpret_cast<uintptr_t>(d) & 15)) & 15u;
            if (head > len) head = len;
            if (threadIdx.x < head) d[threadIdx.x] = sm[mis0 + threadIdx.x];
            const uint32_t off = mis0 + head;               // staged byte of output byte `head`
            const uint32_t v = (len - head) >> 4;
            const uint32_t q = off >> 2, sh = 8u * (off & 3u);
            uint4* d16 = reinterpret_cast<uint4*>(d + head);
            for (uint32_t i = threadIdx.x; i < v; i += blockDim.x) {
                const uint32_t* w = sw + q + 4 * i;
                const uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3], w4 = w[4];
                d16[i] = make_uint4(__funnelshift_r(w0, w1, sh), __funnelshift_r(w1, w2, sh),
                                    __funnelshift_r(w2, w3, sh), __funnelshift_r(w3, w4, sh));
            }
            for (uint32_t i = head + 16 * v + threadIdx.x; i < len; i += blockDim.x) d[i] = sm[mis0 + i];
            __syncthreads();                                 // the stage is free again
        }
    }
}

// ---------------------------------------------------------------------------
// Multi-GPU combine, after ONE all-gather of every live rank's
// exchange buffer [slot sums: n_slots f64 | digest rows: 2 u64 each], rank r
// at gathered + r * stride:
//  * slot s = sum over ranks of gathered[r * stride + s], in rank order — a
//    fixed order, so every rank computes bit-identical sums (and verdicts)
//    whatever algorithm NCCL picks;
//  * copy c of a cross-GPU replica group: differs[c] = its 128-bit digest !=
//    copy 0's (first[c] = index of its group's copy 0; copies whose holder
//    is not live have off[c] < 0 and compare equal), n_differ += 1 per
//    differing copy.  Equal digests = identical copies (checker.py:184-191:
//    rel_err 0, the group's slot stays zero); a differing copy sends the
//    host down the exact bug path.
__global__ void __launch_bounds__(256)
k_combine(const double* __restrict__ gathered, int world, int64_t stride, int64_t n_slots,
          double* __restrict__ slots, const int64_t* __restrict__ off, const int32_t* __restrict__ first,
          int64_t n_copies, int32_t* __restrict__ differs, unsigned long long* __restrict__ n_differ) {
    const int64_t n = n_slots > n_copies ? n_slots : n_copies;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n_slots) {
            double s = gathered[i];
            for (int r = 1; r < world; ++r) s += gathered[(int64_t)r * stride + i];
            slots[i] = s;
        }
        if (i < n_copies) {
            const int64_t oc = off[i], o0 = off[first[i]];
            int d = 0;
            if (oc >= 0 && o0 >= 0) {
                const unsigned long long* a = reinterpret_cast<const unsigned long long*>(gathered + oc);
                const unsigned long long* b = reinterpret_cast<const unsigned long long*>(gathered + o0);
                d = (a[0] != b[0]) | (a[1] != b[1]);
            }
            differs[i] = d;
            if (d) atomicAdd(n_differ, 1ull);
        }
    }
}

// per-host-thread, per-device auxiliary streams for concurrent class launches
struct AuxStreams {
    static constexpr int N = 7;
    cudaStream_t stream[N];
    cudaEvent_t join[N];
    cudaEvent_t fork;
    int dev = -1;
};

// Auxiliary stream sets are per host thread (two threads' td_segnorm calls
// must not share fork/join events) but outlive it: a thread's sets go back
// to a process-wide free list when the thread exits and the next new thread
// on that device takes one, so services that run checks on short-lived
// threads hold at most one set per concurrently live thread instead of
// creating streams without bound.  Nothing is destroyed (no CUDA calls at
// thread or process exit); the list and its lock are never freed.
std::mutex& aux_lock() {
    static std::mutex* m = new std::mutex;
    return *m;
}
std::vector<AuxStreams*>& aux_free() {
    static std::vector<AuxStreams*>* v = new std::vector<AuxStreams*>;
    return *v;
}

struct AuxLocal {
    AuxStreams* per_dev[16] = {};
    ~AuxLocal() {
        std::lock_guard<std::mutex> g(aux_lock());
        for (AuxStreams* a : per_dev)
            if (a) aux_free().push_back(a);
    }
};

AuxStreams* aux_streams(int dev) {
    thread_local AuxLocal local;
    if (dev < 0 || dev >= 16) return nullptr;
    if (AuxStreams* a = local.per_dev[dev]) return a;
    {
        std::lock_guard<std::mutex> g(aux_lock());
        auto& pool = aux_free();
        for (size_t i = 0; i < pool.size(); ++i)
            if (pool[i]->dev == dev) {
                local.per_dev[dev] = pool[i];
                pool.erase(pool.begin() + i);
                return local.per_dev[dev];
            }
    }
    AuxStreams* a = new AuxStreams;
    int made = 0;
    bool ok = true;
    for (; made < AuxStreams::N && ok; ++made) {
        ok = cudaStreamCreateWithFlags(&a->stream[made], cudaStreamNonBlocking) == cudaSuccess;
        if (ok && cudaEventCreateWithFlags(&a->join[made], cudaEventDisableTiming) != cudaSuccess) {
            cudaStreamDestroy(a->stream[made]);
            ok = false;
        }
        if (!ok) break;
    }
    if (ok) ok = cudaEventCreateWithFlags(&a->fork, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {                                   // fall back to serial classes on this call
        for (int k = 0; k < made; ++k) {
            cudaStreamDestroy(a->stream[k]);
            cudaEventDestroy(a->join[k]);
        }
        delete a;
        cudaGetLastError();
        return nullptr;
    }
    a->dev = dev;
    local.per_dev[dev] = a;
    return a;
}

void join_aux(AuxStreams* a, int k, cudaStream_t main_stream) {
    cudaEventRecord(a->join[k], a->stream[k]);
    cudaStreamWaitEvent(main_stream, a->join[k], 0);
}

// TD_GATHER_STAGED=0: td_gather_bytes on the LDG walker instead of the
// shared-memory staged one (A/B)
bool gather_staged() {
    static const bool on = [] {
        const char* e = getenv("TD_GATHER_STAGED");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

bool serial_classes() {
    static const bool serial = [] {
        const char* e = getenv("TD_SERIAL_CLASSES");
        return e != nullptr && e[0] == '1';
    }();
    return serial;
}

// TD_BLOCKS_PER_SM=<n>: td_segnorm's resident CTAs per SM when the caller
// passes 0 (A/B knob; default 4)
int default_blocks_per_sm() {
    static const int n = [] {
        const char* e = getenv("TD_BLOCKS_PER_SM");
        const int v = e ? atoi(e) : 0;
        return v > 0 && v <= 8 ? v : 4;
    }();
    return n;
}

int grid_for(int64_t n, int per_block, int cap) {
    int64_t g = (n + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

// launch a consumer kernel with programmatic stream serialisation (PDL; see
// griddep_wait).  TD_PDL=0 disables it (A/B and debugging).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("TD_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_dependent(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace

// ===========================================================================
// C ABI

extern "C" {

int td_version(void) { return TD_ABI_VERSION; }

const char* td_last_error(void) { return g_err; }

int td_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return n;
}

int td_segnorm(const td_segment* segs, const td_class* classes, int32_t n_classes,
               double* partials, int32_t blocks_per_sm, void* stream) {
    if (n_classes == 0) return 0;
    if (!segs || !classes || !partials || n_classes < 0)
        return fail("td_segnorm: invalid arguments (n_classes=%d)", n_classes);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = blocks_per_sm > 0 ? blocks_per_sm : default_blocks_per_sm();
    // Classes run concurrently: the largest on the caller's stream, the others
    // forked onto this thread's auxiliary streams, so each kernel's tail is
    // filled by the next kernel's CTAs instead of idling SMs (joined below).
    int order[64];
    const int nc = n_classes < 64 ? n_classes : 64;
    for (int c = 0; c < nc; ++c) order[c] = c;
    for (int a = 1; a < nc; ++a)
        for (int b = a; b > 0 && classes[order[b]].n_tiles > classes[order[b - 1]].n_tiles; --b) {
            const int t = order[b]; order[b] = order[b - 1]; order[b - 1] = t;
        }
    AuxStreams* aux = (nc > 1 && !serial_classes()) ? aux_streams(dev) : nullptr;
    cudaStream_t main_stream = (cudaStream_t)stream;
    if (aux && cudaEventRecord(aux->fork, main_stream) != cudaSuccess) aux = nullptr;
    for (int k = 0; k < n_classes; ++k) {
        const int c = k < nc ? order[k] : k;
        const td_class& C = classes[c];
        cudaStream_t st = main_stream;
        if (aux && k > 0 && k <= AuxStreams::N) {
            st = aux->stream[k - 1];
            cudaStreamWaitEvent(st, aux->fork, 0);
        }
        if (C.n_tiles == 0) continue;
        if (!C.tiles || C.n_tiles < 0 || C.nz < 0 || C.nz > TD_MAX_Z)
            return fail("td_segnorm: invalid class %d", c);
        int64_t grid = (int64_t)sms * per_sm;
        if (grid > C.n_tiles) grid = C.n_tiles;
        if (!C.vec || C.mode != TD_MODE_NORMS) {
            if (C.digest) return fail("td_segnorm: digests need a vector class (class %d)", c);
            k_segnorm_generic<<<(unsigned)grid, BLOCK, 0, st>>>(
                segs, C.tiles, C.n_tiles, partials, C.mode, C.atol, C.rtol);
            if (int rc = check_launch("td_segnorm")) return rc;
            if (st != main_stream) join_aux(aux, k - 1, main_stream);
            continue;
        }
        segnorm_fn fn = nullptr;
        {
            const bool one = C.host_seg != nullptr && C.nz == 0 && C.has_x && !C.digest;
            switch (C.dtype) {
                case TD_BF16: fn = pick_vec<TD_BF16>(C.nz, C.has_x != 0, C.digest != 0, one); break;
                case TD_F16: fn = pick_vec<TD_F16>(C.nz, C.has_x != 0, C.digest != 0, one); break;
                case TD_F32: fn = pick_vec<TD_F32>(C.nz, C.has_x != 0, C.digest != 0, one); break;
                default: break;
            }
            if (!fn) return fail("td_segnorm: no vector walker for class %d (dtype=%d nz=%d has_x=%d digest=%d)",
                                 c, C.dtype, C.nz, C.has_x, C.digest);
        }
        if (C.digest && !C.digests) return fail("td_segnorm: digest class %d without a digest table", c);
        td_segment seg1;
        if (C.host_seg) seg1 = *C.host_seg;
        else memset(&seg1, 0, sizeof(seg1));
        if (segnorm_fn bulk = pick_bulk(C.dtype, C.nz, C.has_x != 0, C.digest != 0)) {
            static thread_local bool attr_set[2][2] = {{false, false}, {false, false}};
            bool& done = attr_set[C.dtype == TD_BF16][C.digest != 0];
            if (!done) {
                if (cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BULK_SMEM) !=
                    cudaSuccess)
                    return fail("td_segnorm: cannot reserve %zu bytes of shared memory", BULK_SMEM);
                done = true;
            }
            int64_t bgrid = (int64_t)sms * TD_BULK_MINB;
            if (bgrid > C.n_tiles) bgrid = C.n_tiles;
            bulk<<<(unsigned)bgrid, BULK_THREADS, BULK_SMEM, st>>>(segs, C.tiles, C.n_tiles, partials, C.digests,
                                                                   seg1);
        } else {
            fn<<<(unsigned)grid, BLOCK, 0, st>>>(segs, C.tiles, C.n_tiles, partials, C.digests, seg1);
        }
        if (int rc = check_launch("td_segnorm")) return rc;
        if (st != main_stream) join_aux(aux, k - 1, main_stream);
    }
    return 0;
}

int td_reduce_slots(const td_id_desc* ids, int32_t n_ids, const td_group_desc* groups, int32_t n_groups,
                    const double* partials, double* id_sums, double* group_sums, void* stream) {
    const int64_t slots = (int64_t)n_ids + n_groups;
    if (slots == 0) return 0;
    if (n_ids < 0 || n_groups < 0 || (n_ids && (!ids || !id_sums)) || (n_groups && (!groups || !group_sums)))
        return fail("td_reduce_slots: invalid arguments");
    const int threads = 256;
    const int64_t blocks = (slots * 32 + threads - 1) / threads;
    if (launch_dependent(k_reduce_slots, dim3((unsigned)blocks), dim3(threads), (cudaStream_t)stream, ids, n_ids,
                         groups, n_groups, partials, id_sums, group_sums) != cudaSuccess)
        return check_launch("td_reduce_slots");
    return check_launch("td_reduce_slots");
}

int td_verdict(const td_id_desc* ids, int32_t n_ids, const td_group_desc* groups, int32_t n_groups,
               const double* id_sums, const double* group_sums, double kappa, double eps,
               double replica_eps, td_id_result* id_out, td_group_result* group_out,
               unsigned long long* near_ties, void* stream) {
    if (n_ids == 0) return 0;
    if (n_ids < 0 || !ids || !id_sums || !id_out || (n_groups && (!groups || !group_sums || !group_out)))
        return fail("td_verdict: invalid arguments");
    const int threads = 128;
    if (near_ties && cudaMemsetAsync(near_ties, 0, sizeof(unsigned long long), (cudaStream_t)stream) != cudaSuccess)
        return fail("td_verdict: cannot reset the near-tie counter");
    launch_dependent(k_verdict, dim3((unsigned)((n_ids + threads - 1) / threads)), dim3(threads),
                     (cudaStream_t)stream, ids, n_ids, groups, id_sums, group_sums, kappa, eps, replica_eps,
                     id_out, group_out, near_ties);
    return check_launch("td_verdict");
}

int td_rel_err(const void* a, const void* b, int32_t dtype, int64_t n, void* work, double* out, void* stream) {
    if ((n > 0 && (!a || !b)) || !work || !out || n < 0 || dtype < 0 || dtype > 3)
        return fail("td_rel_err: invalid arguments");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t per = dtype == TD_F64 ? 1 : 8;            // elements per work item
    int64_t grid = (n / per + BLOCK - 1) / BLOCK;
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, std::min<int64_t>((int64_t)sms * 4, TD_REL_ERR_MAX_CTAS)));
    double* part = static_cast<double*>(work);
    unsigned int* ticket = reinterpret_cast<unsigned int*>(part + 2 * TD_REL_ERR_MAX_CTAS);
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case TD_BF16: k_rel_err<TD_BF16><<<(unsigned)grid, BLOCK, 0, st>>>(pa, pb, n, part, ticket, out); break;
        case TD_F16: k_rel_err<TD_F16><<<(unsigned)grid, BLOCK, 0, st>>>(pa, pb, n, part, ticket, out); break;
        case TD_F32: k_rel_err<TD_F32><<<(unsigned)grid, BLOCK, 0, st>>>(pa, pb, n, part, ticket, out); break;
        default: k_rel_err<TD_F64><<<(unsigned)grid, BLOCK, 0, st>>>(pa, pb, n, part, ticket, out); break;
    }
    return check_launch("td_rel_err");
}

int td_reduce_chunks(const double* partials, const td_chunk* chunks, int64_t n_chunks, double* out,
                     void* stream) {
    if (n_chunks == 0) return 0;
    if (n_chunks < 0 || !partials || !chunks || !out) return fail("td_reduce_chunks: invalid arguments");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(n_chunks, (int64_t)sms * 6);
    launch_dependent(k_reduce_chunks, dim3((unsigned)grid), dim3(CHUNK_BLOCK), (cudaStream_t)stream, partials,
                     chunks, n_chunks, out);
    return check_launch("td_reduce_chunks");
}

int td_finalize(const td_id_desc* ids, int32_t n_ids, const td_group_desc* groups, int32_t n_groups,
                const double* partials, double* id_sums, double* group_sums, double kappa, double eps,
                double replica_eps, td_id_result* id_out, td_group_result* group_out,
                unsigned long long* near_ties, void* stream) {
    if (n_ids == 0) return 0;
    if (n_ids < 0 || !ids || !partials || !id_sums || !id_out ||
        (n_groups && (!groups || !group_sums || !group_out)))
        return fail("td_finalize: invalid arguments");
    if (near_ties && cudaMemsetAsync(near_ties, 0, sizeof(unsigned long long), (cudaStream_t)stream) != cudaSuccess)
        return fail("td_finalize: cannot reset the near-tie counter");
    launch_dependent(k_finalize, dim3((unsigned)n_ids), dim3(BLOCK), (cudaStream_t)stream, ids, groups, partials,
                     id_sums, group_sums, kappa, eps, replica_eps, id_out, group_out, near_ties);
    return check_launch("td_finalize");
}

int td_perturb(const void* x, void* y, int32_t dtype_in, int32_t dtype_out, int64_t rows, int64_t cols,
               int64_t full_cols, int64_t col0, const int64_t* row_pos, int64_t row0, uint64_t seed,
               double eps, int32_t fmt, int32_t generator, unsigned long long* nonfinite, void* stream) {
    if (rows == 0 || cols == 0) return 0;
    if (!x || !y || !nonfinite || rows < 0 || cols < 0 || dtype_in < 0 || dtype_in > 3 || dtype_out < 0 ||
        dtype_out > 3 || fmt < 0 || fmt > 3 || col0 < 0 || col0 + cols > full_cols)
        return fail("td_perturb: invalid arguments");
    const int threads = 256;
    const int esz_in = dtype_in == TD_F32 ? 4 : (dtype_in == TD_F64 ? 8 : 2);
    const int esz_out = dtype_out == TD_F32 ? 4 : (dtype_out == TD_F64 ? 8 : 2);
    const bool vec = cols % 8 == 0 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)y % 16) == 0 &&
                     (cols * esz_in) % 16 == 0 && (cols * esz_out) % 16 == 0;
    if (vec) {
        const int64_t groups = rows * (cols / 8);
        const uint32_t gpr = (uint32_t)(cols / 8);
        const int l = gpr > 1 ? 32 - __builtin_clz(gpr - 1) : 0;
        const int p = 31 + l;
        const uint32_t m = (uint32_t)(((1ull << p) + gpr - 1) / gpr);
        const int grid = grid_for(groups, threads, 148 * 8);
        const bool q8 = dtype_in == TD_BF16 && dtype_out == TD_BF16 && fmt == TD_FMT_BF16;
        if (q8 && generator == TD_GEN_PHILOX4x32)
            k_perturb_bf16<TD_GEN_PHILOX4x32><<<grid, threads, 0, (cudaStream_t)stream>>>(
                static_cast<const uint4*>(x), static_cast<uint4*>(y), rows, gpr, full_cols, col0, row_pos, row0,
                seed, eps, m, p, nonfinite);
        else if (q8)
            k_perturb_bf16<TD_GEN_SPLITMIX64><<<grid, threads, 0, (cudaStream_t)stream>>>(
                static_cast<const uint4*>(x), static_cast<uint4*>(y), rows, gpr, full_cols, col0, row_pos, row0,
                seed, eps, m, p, nonfinite);
        else
            k_perturb_vec8<<<grid, threads, 0, (cudaStream_t)stream>>>(
                static_cast<const char*>(x), static_cast<char*>(y), dtype_in, dtype_out, rows, cols, full_cols,
                col0, row_pos, row0, seed, eps, fmt, generator, m, p, nonfinite);
    } else {
        dim3 grid((unsigned)grid_for(cols, threads, 64), (unsigned)(rows < 65535 ? rows : 65535));
        k_perturb<<<grid, threads, 0, (cudaStream_t)stream>>>(
            static_cast<const char*>(x), static_cast<char*>(y), dtype_in, dtype_out, rows, cols, full_cols, col0,
            row_pos, row0, seed, eps, fmt, generator, nonfinite);
    }
    return check_launch("td_perturb");
}

int td_signed_uniforms(double* out, int64_t n, uint64_t seed, int64_t k0, int32_t generator, void* stream) {
    if (n == 0) return 0;
    if (!out || n < 0) return fail("td_signed_uniforms: invalid arguments");
    k_signed_uniforms<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(out, n, seed, k0, generator);
    return check_launch("td_signed_uniforms");
}

int td_quantize(const double* x, void* y, int32_t dtype_out, int64_t n, int32_t fmt,
                unsigned long long* nonfinite, void* stream) {
    if (n == 0) return 0;
    if (!x || !y || !nonfinite || n < 0 || fmt < 0 || fmt > 3) return fail("td_quantize: invalid arguments");
    k_quantize<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(x, static_cast<char*>(y), dtype_out,
                                                                           n, fmt, nonfinite);
    return check_launch("td_quantize");
}

int td_fingerprint(const td_fp_item* items, const int64_t* chunk_begin, int32_t n_items, int64_t n_chunks,
                   unsigned long long* out, void* stream) {
    if (n_items == 0) return 0;
    if (!items || !chunk_begin || !out || n_items < 0 || n_chunks < 0)
        return fail("td_fingerprint: invalid arguments");
    if (cudaMemsetAsync(out, 0, sizeof(unsigned long long) * 2 * (size_t)n_items, (cudaStream_t)stream) != cudaSuccess)
        return fail("td_fingerprint: cannot clear the digests");
    if (n_chunks == 0) return 0;
    const int grid = (int)(n_chunks < 148 * 8 ? n_chunks : 148 * 8);
    k_fingerprint<<<grid, BLOCK, 0, (cudaStream_t)stream>>>(items, chunk_begin, n_items, n_chunks, out);
    return check_launch("td_fingerprint");
}

int td_box_gather(const void* src, int32_t src_dtype, double* dst, const int64_t* boxes, int32_t n_boxes,
                  void* stream) {
    if (n_boxes == 0) return 0;
    if (!src || !dst || !boxes || n_boxes < 0 || n_boxes > 65535) return fail("td_box_gather: invalid arguments");
    dim3 grid(64, (unsigned)n_boxes);
    k_box_gather<<<grid, 256, 0, (cudaStream_t)stream>>>(static_cast<const char*>(src), src_dtype, dst, boxes);
    return check_launch("td_box_gather");
}

int td_generate(double* out, int64_t n, uint64_t seed, int32_t dist, double a, double b, int64_t vocab,
                const int64_t* skips, int32_t n_skips, unsigned long long* zero_count, int64_t* zero_pos,
                int32_t zero_cap, void* stream) {
    if (n == 0) return 0;
    if (!out || n < 0 || dist < 0 || dist > 2 || n_skips < 0 || (n_skips && !skips) ||
        (zero_count && !zero_pos && zero_cap > 0) || (dist == 2 && vocab < 1))
        return fail("td_generate: invalid arguments");
    k_generate<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        out, n, seed, dist, a, b, vocab, skips, n_skips, zero_count, zero_pos, zero_cap);
    return check_launch("td_generate");
}

int td_combine(const double* gathered, int32_t world, int64_t stride, int64_t n_slots, double* slots,
               const int64_t* copy_off, const int32_t* copy_first, int64_t n_copies, int32_t* differs,
               unsigned long long* n_differ, void* stream) {
    if (world < 1 || stride < n_slots || n_slots < 0 || n_copies < 0 || (n_slots && (!gathered || !slots)) ||
        (n_copies && (!gathered || !copy_off || !copy_first || !differs)) || !n_differ)
        return fail("td_combine: invalid arguments");
    if (cudaMemsetAsync(n_differ, 0, sizeof(unsigned long long), (cudaStream_t)stream) != cudaSuccess)
        return fail("td_combine: cannot reset the mismatch counter");
    const int64_t n = n_slots > n_copies ? n_slots : n_copies;
    if (n == 0) return 0;
    k_combine<<<grid_for(n, 256, 148 * 4), 256, 0, (cudaStream_t)stream>>>(
        gathered, world, stride, n_slots, slots, copy_off, copy_first, n_copies, differs, n_differ);
    return check_launch("td_combine");
}

int td_gather_bytes(const void* src, void* dst, const int64_t* ranges, int64_t n, void* stream) {
    if (n == 0) return 0;
    if (!src || !dst || !ranges || n < 0) return fail("td_gather_bytes: invalid arguments");
    const int grid = 148 * 8;
    if (gather_staged()) {
        k_gather_staged<<<grid, 256, GATHER_SMEM, (cudaStream_t)stream>>>(
            static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst), ranges, n);
        return check_launch("td_gather_bytes");
    }
    k_gather_bytes<<<grid, 256, 0, (cudaStream_t)stream>>>(static_cast<const unsigned char*>(src),
                                                           static_cast<unsigned char*>(dst), ranges, n);
    return check_launch("td_gather_bytes");
}

}  // extern "C"

// ---- the cross-GPU exchange for hosts without torch.distributed ----
// NCCL is resolved at first use with dlopen (no link-time dependency: the
// library loads on hosts without NCCL, and inside a torch process it binds
// the libnccl.so.2 torch already loaded).  Enum values as in nccl.h.
namespace {
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
nccl_allreduce_fn nccl_allreduce() {
    static nccl_allreduce_fn fn = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        return h ? reinterpret_cast<nccl_allreduce_fn>(dlsym(h, "ncclAllReduce")) : nullptr;
    }();
    return fn;
}
constexpr int NCCL_INT64 = 4, NCCL_FLOAT64 = 8, NCCL_SUM = 0;

typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
nccl_allgather_fn nccl_allgather() {
    static nccl_allgather_fn fn = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        return h ? reinterpret_cast<nccl_allgather_fn>(dlsym(h, "ncclAllGather")) : nullptr;
    }();
    return fn;
}

int allreduce_sum(void* comm, void* buf, int64_t n, int dtype, void* stream, const char* what) {
    if (n == 0) return 0;
    if (!comm || !buf || n < 0) return fail("%s: invalid arguments", what);
    nccl_allreduce_fn fn = nccl_allreduce();
    if (!fn) return fail("%s: libnccl.so.2 not found", what);
    const int rc = fn(buf, buf, (size_t)n, dtype, NCCL_SUM, comm, (cudaStream_t)stream);
    return rc ? fail("%s: ncclAllReduce returned %d", what, rc) : 0;
}
}  // namespace

extern "C" {

int td_allreduce_partials(void* nccl_comm, double* slots, int64_t n, void* stream) {
    return allreduce_sum(nccl_comm, slots, n, NCCL_FLOAT64, stream, "td_allreduce_partials");
}

int td_allreduce_digests(void* nccl_comm, long long* table, int64_t n, void* stream) {
    return allreduce_sum(nccl_comm, table, n, NCCL_INT64, stream, "td_allreduce_digests");
}

int td_allgather_exchange(void* nccl_comm, const double* send, double* recv, int64_t n, void* stream) {
    if (n == 0) return 0;
    if (!nccl_comm || !send || !recv || n < 0) return fail("td_allgather_exchange: invalid arguments");
    nccl_allgather_fn fn = nccl_allgather();
    if (!fn) return fail("td_allgather_exchange: libnccl.so.2 not found");
    const int rc = fn(send, recv, (size_t)n, NCCL_FLOAT64, nccl_comm, (cudaStream_t)stream);
    return rc ? fail("td_allgather_exchange: ncclAllGather returned %d", rc) : 0;
}

}  // extern "C"
