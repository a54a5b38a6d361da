/*
 * td_api.h — C ABI of the B200-native tensor-comparison hot path.
 *
 * The reference (TTrace `traindiff`, pure Python/numpy) has no native
 * boundary; its hot path sits behind Python functions.  Each entry point
 * below replaces the arithmetic of one of those functions:
 *
 *   td_segnorm   replaces rel_err_arrays' two norms   (pkg/src/traindiff/tensor.py:158-167)
 *                fused with merge()'s box copies      (pkg/src/traindiff/canonical.py:182-212)
 *                and check_replicas' per-copy rel_err  (pkg/src/traindiff/canonical.py:225-247)
 *                and TraceRecord.values() widening     (pkg/src/traindiff/tracestore.py:84-86)
 *   td_reduce_slots + td_verdict (or fused: td_finalize)
 *                replace check()'s per-id loop         (pkg/src/traindiff/checker.py:312-365)
 *                and _merge_one's replica verdicts     (pkg/src/traindiff/checker.py:151-198)
 *   td_perturb   replaces Emulator._apply_perturbation (pkg/src/traindiff/engine.py:351-361)
 *                = signed_uniforms (generation.py:163-167) + 1+u*eps + quantize_array (tensor.py:64-77)
 *   td_quantize  replaces quantize_array               (pkg/src/traindiff/tensor.py:64-77)
 *   td_fingerprint
 *                order-independent 128-bit digest of a payload, used to decide
 *                replica equality across GPUs without moving data
 *   td_box_gather
 *                materialises merge()'s f64 output on the device (public merge API)
 *   td_generate  generate_full's Normal/Uniform/TokenIds streams (generation.py:81-160)
 *   td_gather_bytes
 *                unpacks TTRC payloads from a file image in HBM into an aligned
 *                arena (device-side trace reader, tracestore.py:225-284)
 *
 * Conventions: every function returns 0 on success and a nonzero status on
 * error (td_last_error() then describes it, thread-local).  All pointers to
 * bulk data are DEVICE pointers owned by the caller; no function allocates
 * device memory.  `stream` is a cudaStream_t passed as void*; all work is
 * stream-ordered and re-entrant per stream.  No C++ exceptions cross the ABI.
 */
#ifndef TD_API_H
#define TD_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TD_ABI_VERSION 2

/* element types of payload buffers */
enum td_dtype { TD_F32 = 0, TD_BF16 = 1, TD_F16 = 2, TD_F64 = 3 };

/* storage formats of the reference's FloatFormat (tensor.py:28-61) */
enum td_format { TD_FMT_NONE = 0, TD_FMT_FP32 = 1, TD_FMT_BF16 = 2, TD_FMT_FP8E4M3 = 3 };

/* verdict codes; order matches checker.VERDICTS (checker.py:36-42) */
enum td_verdict_code { TD_PASS = 0, TD_FLAG = 1, TD_REPLICA = 2, TD_MERGE = 3, TD_MISSING = 4, TD_NONE = 255 };

/* perturbation generators */
enum td_generator { TD_GEN_SPLITMIX64 = 0, TD_GEN_PHILOX4x32 = 1 };

#define TD_MAX_Z 7              /* replica copies beside copy 0 per segment */
#define TD_PARTIAL_STRIDE 10    /* doubles per partial row: d2, x2, y2, z2[7] */
#define TD_WARPS_PER_TILE 8     /* partial rows per tile (one per warp of a 256-thread CTA) */
#ifndef TD_TILE_UNITS
#define TD_TILE_UNITS 8192      /* units (8-element vectors or elements) per tile */
#endif
#define TD_SLOT_STRIDE 8        /* doubles per reduced slot */

/* segment flags */
#define TD_SEG_HAS_X 1u         /* x present: accumulate d2=sum (x-y)^2 and x2=sum x^2 */
#define TD_SEG_VEC 2u           /* 16-byte vector path legal (alignment + cols%8 proven by host) */
/* flags bits 8..12: log2 of the units per tile for this segment; 0 means
   TD_TILE_UNITS.  Small plans use smaller tiles so every SM gets work. */
#define TD_SEG_TILE_SHIFT_POS 8

/*
 * A segment is a 2-D strided block read in lockstep from x (the reference
 * side), y (candidate copy 0) and z[0..nz) (replica copies laid out like y).
 * rows x cols elements; row r of operand p starts at p + r*stride elements.
 * The host planner derives segments from the intersection of candidate and
 * reference global boxes (one per contiguous run), so the merged tensor is
 * never materialised.  144 bytes, all fields naturally aligned.
 */
typedef struct td_segment {
    uint64_t x;                 /* device address or 0 */
    uint64_t y;
    uint64_t z[TD_MAX_Z];
    int64_t  x_stride;          /* elements per row in x */
    int64_t  y_stride;          /* elements per row in y and every z */
    int64_t  rows;
    int64_t  cols;
    int64_t  tile_begin;        /* global index of this segment's first tile */
    int64_t  n_units;           /* rows*cols/8 (VEC) or rows*cols (scalar); < 2^31 */
    int32_t  x_dtype;
    int32_t  y_dtype;           /* dtype of y and of every z */
    int32_t  nz;
    uint32_t flags;
    uint32_t div_m;             /* magic divisor for units-per-row: q = (n*div_m) >> div_p */
    int32_t  div_p;
    int64_t  y_word0;           /* 8-byte word index of y's first element in its record (digests) */
    int32_t  digest_slot;       /* >= 0: also digest y's bytes into digests[2*slot..] (td_class.digests) */
    int32_t  pad;
} td_segment;                   /* 160 bytes */

/* per canonical id: where its partial sums live and what the host already knows */
typedef struct td_id_desc {
    int64_t tile_begin;         /* compare tiles [tile_begin, tile_end) */
    int64_t tile_end;
    int32_t cgroup_begin;       /* candidate replica-group slots [cgroup_begin, cgroup_end) */
    int32_t cgroup_end;
    int32_t rgroup_begin;       /* reference replica-group slots */
    int32_t rgroup_end;
    int32_t has_compare;        /* both merges succeed and merged shapes agree */
    int32_t cand_host;          /* host-known candidate problem: 0, TD_REPLICA (declared size), TD_MERGE */
    int32_t ref_host;           /* same for the reference side */
    int32_t pad;
    double  tolerance;          /* ToleranceMap.get(id) */
} td_id_desc;                   /* 56 bytes */

typedef struct td_group_desc {
    int64_t tile_begin;         /* tiles carrying this group's y2/z2 partials */
    int64_t tile_end;
    int32_t nz;                 /* copies beside copy 0 */
    int32_t pad;
} td_group_desc;                /* 24 bytes */

typedef struct td_id_result {
    double  observed;           /* rel_err(ref, cand) or NaN when not computed */
    double  threshold;          /* kappa * max(tol, eps) */
    int32_t verdict;            /* td_verdict_code */
    int32_t cand_kind;          /* 0, TD_REPLICA or TD_MERGE */
    int32_t ref_kind;
    int32_t near_tie;           /* |obs - thr| <= 1e-12 * thr */
} td_id_result;                 /* 32 bytes */

typedef struct td_group_result {
    double  worst;              /* max_i rel_err(copy0, copy_i), strict > (NaN ignored) */
    int32_t worst_index;        /* i of the worst copy, -1 when none exceeded 0 */
    int32_t mismatch;           /* worst > replica eps */
} td_group_result;              /* 16 bytes */

/* ---- library ---- */
int         td_version(void);
const char* td_last_error(void);
int         td_sm_count(int device);

/* A tile class: the tiles whose segments share one walker.  Each entry of
 * `tiles` (device) packs (segment index << 32) | global tile index.  Vector
 * classes (vec=1) require every operand to have `dtype` (bf16, f16 or f32);
 * everything else runs the generic walker. */
typedef struct td_class {
    const int64_t* tiles;       /* device, packed (segment << 32 | tile) */
    int64_t n_tiles;
    int32_t dtype;
    int32_t nz;
    int32_t has_x;
    int32_t vec;
    int32_t mode;               /* TD_MODE_NORMS, or TD_MODE_STATIC (generic walker only) */
    int32_t digest;             /* vector classes: segments carry digest slots (same hash as
                                   td_fingerprint, so a record covered exactly once by its
                                   segments gets the digest td_fingerprint would give it) */
    double  atol;               /* static mode: count |y - x| > atol + rtol*|x| into d2 */
    double  rtol;
    unsigned long long* digests; /* device, 2 u64 per digest slot, accumulated (caller zeroes) */
    const struct td_segment* host_seg; /* HOST copy of the class's only segment (its tiles are
                                   that segment's, in order), or NULL: passed to the kernel by
                                   value, so no tile list / descriptor load precedes the data */
} td_class;                     /* 72 bytes */

#define TD_MODE_NORMS 0
#define TD_MODE_STATIC 1        /* compare_static's elementwise test (checker.py:403-443) */

/* ---- kernel 1: fused canonicalise + relative-difference norms ----
 * One persistent launch per class (classes is a HOST array).  partials:
 * n_tiles_total * TD_WARPS_PER_TILE * TD_PARTIAL_STRIDE doubles; each warp
 * of a tile writes its own row (not accumulated).  blocks_per_sm <= 0 selects 4 CTAs of 256 threads per SM. */
int td_segnorm(const td_segment* segs, const td_class* classes, int32_t n_classes,
               double* partials, int32_t blocks_per_sm, void* stream);

/* deterministic per-slot sums of tile partials.
 * id_sums:    n_ids    * 2 doubles  (d2, x2)
 * group_sums: n_groups * TD_SLOT_STRIDE doubles (y2, z2[0..6]) */
int td_reduce_slots(const td_id_desc* ids, int32_t n_ids,
                    const td_group_desc* groups, int32_t n_groups,
                    const double* partials,
                    double* id_sums, double* group_sums, void* stream);

/* one chunk of a slot's partial rows for td_reduce_chunks */
typedef struct td_chunk {
    int64_t row_begin;          /* first partial row (tile * TD_WARPS_PER_TILE + warp) */
    int64_t row_end;            /* one past the last */
    int32_t k0;                 /* first partial column summed (0 for ids, 2 for groups) */
    int32_t nk;                 /* columns summed: 2 for ids, 1 + nz for groups */
} td_chunk;                     /* 24 bytes */

/* first level of the slot reduction for slots with many partial rows:
 * chunk c's sums go to row c * TD_WARPS_PER_TILE of `out` (columns
 * k0..k0+nk-1, every other cell of its TD_WARPS_PER_TILE rows zeroed), so
 * `out` is itself a partials array in which chunk c is "tile" c.  Id / group
 * descriptors whose tile ranges name chunk ranges then run td_reduce_slots /
 * td_finalize on `out` unchanged.  Fixed-order, deterministic.
 * (Replaces no reference code: the reference sums a whole tensor in numpy,
 * tensor.py:163-164.) */
int td_reduce_chunks(const double* partials, const td_chunk* chunks, int64_t n_chunks,
                     double* out, void* stream);

/* ---- rel_err_arrays for one pair, one launch ----
 * out[0] = sum (a-b)^2, out[1] = sum a^2, out[2] = rel_err with the
 * reference's conventions (0/0 -> 0, x/0 -> +inf; tensor.py:158-167), for two
 * contiguous device arrays of n elements of one dtype (16-byte-aligned bf16 /
 * f16 / f32 stream as vectors).  work: TD_REL_ERR_WORK_BYTES of device memory,
 * zeroed once before first use (its ticket is reset by every call); calls
 * sharing a work buffer must be stream-ordered. */
#define TD_REL_ERR_MAX_CTAS 1024
#define TD_REL_ERR_WORK_BYTES (16 * TD_REL_ERR_MAX_CTAS + 16)
int td_rel_err(const void* a, const void* b, int32_t dtype, int64_t n, void* work, double* out,
               void* stream);

/* ---- the cross-GPU exchange without torch.distributed ----
 * In-place sum over the ranks of an NCCL communicator (an ncclComm_t passed
 * as void*), enqueued on `stream`: the per-id / per-group slot sums between
 * td_reduce_slots and td_verdict (n doubles), and the replica digest table
 * (n int64, wrapping).  NCCL is loaded at first use (dlopen "libnccl.so.2");
 * without it these return non-zero with td_last_error() set. */
int td_allreduce_partials(void* nccl_comm, double* slots, int64_t n, void* stream);
int td_allreduce_digests(void* nccl_comm, long long* table, int64_t n, void* stream);

/* ---- the one-collective exchange (the distributed check's clean path) ----
 * Each rank's exchange buffer is [slot sums: n_slots doubles (td_reduce_slots'
 * id sums then group sums) | digest rows: 2 u64 per local copy of a cross-GPU
 * replica group], padded to a common length `stride` (doubles).
 * td_allgather_exchange: ncclAllGather of n = stride doubles per rank into
 * recv (world * stride), one NCCL call for sums and digests alike.
 * td_combine: slots[s] = sum over r < world of gathered[r*stride + s] in rank
 * order (identical on every rank, independent of NCCL's algorithm; slots may
 * alias gathered's own-rank row once the gather has completed); for copy c
 * of a cross-GPU replica group (n_copies in all, copy_first[c] = index of its
 * group's copy 0, copy_off[c] = offset in doubles of its digest row in
 * gathered, < 0 if its holder is not part of the gather), differs[c] = 1 iff
 * its 128-bit digest differs from copy 0's; *n_differ (reset here) counts
 * them.  Equal digests mean identical copies, i.e. rel_err 0 exactly
 * (canonical.py:236-242; the group's slot stays 0); a non-zero count sends
 * the caller down the exact bug path (point-to-point copy exchange).
 * Replaces the reference's emulated collectives (engine.py:100-142) on the
 * compare path. */
int td_allgather_exchange(void* nccl_comm, const double* send, double* recv, int64_t n, void* stream);
int td_combine(const double* gathered, int32_t world, int64_t stride, int64_t n_slots, double* slots,
               const int64_t* copy_off, const int32_t* copy_first, int64_t n_copies, int32_t* differs,
               unsigned long long* n_differ, void* stream);

/* ---- kernel 3: batched threshold compare -> per-id verdicts ----
 * eps = fmt.eps (threshold floor); replica_eps = fmt.eps for check_replicas.
 * near_ties: optional device uint64 counter, reset and then counted (NULL: per-id
 * near_tie flags only; callers that sum them keep the verdict kernel free to
 * launch programmatically behind its producer, PDL). */
int td_verdict(const td_id_desc* ids, int32_t n_ids,
               const td_group_desc* groups, int32_t n_groups,
               const double* id_sums, const double* group_sums,
               double kappa, double eps, double replica_eps,
               td_id_result* id_out, td_group_result* group_out,
               unsigned long long* near_ties, void* stream);

/* single-GPU finalisation: td_reduce_slots + td_verdict in one launch (one CTA
 * per id).  Multi-GPU callers keep the two steps apart and all-reduce the
 * slot sums between them. */
int td_finalize(const td_id_desc* ids, int32_t n_ids,
                const td_group_desc* groups, int32_t n_groups,
                const double* partials, double* id_sums, double* group_sums,
                double kappa, double eps, double replica_eps,
                td_id_result* id_out, td_group_result* group_out,
                unsigned long long* near_ties, void* stream);

/* ---- kernel 2: eps-scaled perturbation fused with the storage cast ----
 * y[i, j] = Q_fmt(x[i, j] * (1 + u_k * eps)),  k = pos(i) * full_cols + col0 + j,
 * u_k = 2 * U53(word k of the stream seeded by `seed`) - 1.
 * pos(i) = row_pos[i] when row_pos != NULL, else row0 + i.
 * x and y are contiguous (rows, cols); x == y (in place) is allowed.
 * nonfinite: device uint64 counter incremented for each non-finite product
 * (the reference raises NonFinite, tensor.py:66-67). */
int td_perturb(const void* x, void* y, int32_t dtype_in, int32_t dtype_out,
               int64_t rows, int64_t cols, int64_t full_cols, int64_t col0,
               const int64_t* row_pos, int64_t row0,
               uint64_t seed, double eps, int32_t fmt, int32_t generator,
               unsigned long long* nonfinite, void* stream);

/* raw stream words / signed uniforms for n consecutive counters from k0 */
int td_signed_uniforms(double* out, int64_t n, uint64_t seed, int64_t k0,
                       int32_t generator, void* stream);

/* quantize_array on the device: y = Q_fmt(x) elementwise (f64 in, dtype_out out) */
int td_quantize(const double* x, void* y, int32_t dtype_out, int64_t n, int32_t fmt,
                unsigned long long* nonfinite, void* stream);

/* ---- replica digests for multi-GPU replica groups ----
 * One launch for n_items byte ranges: out[2i], out[2i+1] += order-independent
 * 128-bit digest of item i's bytes (8-byte words keyed by their index, tail
 * zero-padded); the caller zeroes out first.  chunk_begin (device, n_items+1
 * int64) is the prefix sum of ceil(nbytes / TD_FP_CHUNK) per item and
 * n_chunks its last entry.  items and chunk_begin live in device memory. */
#define TD_FP_CHUNK (1 << 18)
typedef struct {
    const void* ptr;
    int64_t nbytes;
} td_fp_item;
int td_fingerprint(const td_fp_item* items, const int64_t* chunk_begin, int32_t n_items,
                   int64_t n_chunks, unsigned long long* out, void* stream);

/* ---- merge() materialisation: copy a strided box of src into dst (f64) ----
 * boxes: n_boxes rows of {src_off, dst_off, rows, cols, src_stride, dst_stride} int64 */
int td_box_gather(const void* src, int32_t src_dtype, double* dst,
                  const int64_t* boxes, int32_t n_boxes, void* stream);

/* ---- generate_full on the device (generation.py:81-160) ----
 * dist: 0 normal(mean=a, std=b) by Box-Muller on consecutive uniform pairs,
 *       1 uniform(low=a, high=b), 2 token ids floor(u*vocab) capped at vocab-1.
 * The reference drops exact-zero uniforms from the normal stream (a 2^-53
 * event per word, generation.py:94-103): `skips` lists the sorted raw word
 * indices to skip (NULL/0 normally); zero_count (device uint64) receives the
 * number of zero words seen in the first 2*ceil(n/2) + n_skips words, so the
 * caller can retry with the skip list.  Ops rounded separately (no FMA);
 * log/cos/sin are CUDA's (<= 2 ulp), sqrt is IEEE. */
int td_generate(double* out, int64_t n, uint64_t seed, int32_t dist, double a, double b,
                int64_t vocab, const int64_t* skips, int32_t n_skips,
                unsigned long long* zero_count, int64_t* zero_pos, int32_t zero_cap, void* stream);

/* ---- device TTRC reader / writer: byte-range scatter-gather in HBM ----
 * ranges: n rows of {src_off, dst_off, nbytes} int64 (device), any alignment
 * on either side, ranges must not overlap in dst.  Reader: file image ->
 * 256-B-aligned f32 arena (tracestore.trace_from_bytes); writer: f32 arena
 * and header blob -> file image (tracestore.write_trace).  Replaces the
 * reference's per-record np.frombuffer / tobytes (tracestore.py:155-289). */
int td_gather_bytes(const void* src, void* dst, const int64_t* ranges, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TD_API_H */
