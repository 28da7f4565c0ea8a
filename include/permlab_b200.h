/*
 * permlab-b200 C ABI: the drop-in boundary for the Store-zechin hot path.
 *
 * The reference ("permlab", arXiv 1802.02779) has no FFI layer; the path sits
 * behind free C++ functions in namespace permlab (reference
 * proj/include/permlab/permanent.hpp:77-100, proj/src/permanent.cpp:310-322).
 * This header is the thin C layer the B200 engine exports underneath the C++
 * host API in include/permlab/ (which keeps those signatures); plain pointers
 * and sizes only, no torch or CUDA types. Every entry point says which
 * reference interface it replaces.
 *
 * Data layout (all entry points):
 *   - a matrix is n*n entries, row-major (reference Matrix<T>::operator(),
 *     proj/include/permlab/matrix.hpp:80-82); a batch is `count` matrices
 *     stored contiguously;
 *   - PL_I64  entries are int64_t (the reference's exact Int ring,
 *     ring.hpp:31, restricted to values whose every intermediate fits int64 —
 *     guarded, never wrapped);
 *     PL_F64  entries are double (a real ring the reference lacks; it matches
 *     the reference's Complex ring with imag = 0 bit for bit);
 *     PL_C128 entries are interleaved (re, im) doubles, the layout of
 *     std::complex<double> (the reference's Cplx, ring.hpp:35).
 *
 * Errors: every call returns a pl_status and sets a thread-local message
 * readable with pl_last_error(). The C++ layer maps PL_ERR_LIMIT /
 * PL_ERR_OVERFLOW / PL_ERR_ARG to permlab::DomainError, the reference's error
 * type (proj/include/permlab/errors.hpp:24-27). There is no CPU fallback: with
 * no usable CUDA device every compute entry point returns PL_ERR_NODEVICE.
 */
#ifndef PERMLAB_B200_H
#define PERMLAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pl_status {
    PL_OK = 0,
    PL_ERR_ARG = 1,      /* malformed argument (null pointer, n < 1, ...)            */
    PL_ERR_LIMIT = 2,    /* order or scratch budget exceeds pl_limits               */
    PL_ERR_OVERFLOW = 3, /* an int64 intermediate would overflow (exact ring guard) */
    PL_ERR_NOMEM = 4,    /* device allocation failed                                 */
    PL_ERR_CUDA = 5,     /* CUDA runtime error                                       */
    PL_ERR_NODEVICE = 6, /* no CUDA device: the engine has no CPU fallback          */
    PL_ERR_NCCL = 7      /* NCCL unavailable or a collective failed (multi-GPU)     */
} pl_status;

typedef enum pl_dtype { PL_I64 = 0, PL_F64 = 1, PL_C128 = 2 } pl_dtype;

/* Resource guards (reference proj/include/permlab/limits.hpp:23-33).
 * subset_order_limit: reference default 30 with a hard mask cap of 31
 *   (permanent.cpp:51-53); the device engine uses 64-bit masks and uint32
 *   colex ranks, so its hard cap is PL_MAX_ORDER (C(34,17) < 2^32) and its
 *   default is PL_MAX_ORDER.
 * memo_budget_bytes: the reference caps its 2^n-slot memo table
 *   (permanent.cpp:143-149); the device engine caps its layer scratch
 *   (2 * max_k C(n,k) entries) instead. 0 = no cap beyond free device memory. */
typedef struct pl_limits {
    int32_t subset_order_limit;
    uint64_t memo_budget_bytes;
    /* Devices to run on (an addition: the reference is single-threaded).
     * 0 (default): the calling thread's current device, no collectives.
     * g >= 1: devices 0..g-1 of this process through the multi-GPU path --
     * a large-order matrix (n >= 15) runs its layer DP sharded over the g
     * devices with NCCL exchanges after every layer (single-process
     * communicators, pl_sz_permanent_multi); a batch of smaller orders is
     * split by matrix across them, with no collective. */
    int32_t num_gpus;
} pl_limits;

#define PL_MAX_ORDER 34

/* flags */
#define PL_FLAG_DEVICE_PTRS 0x1u /* `a` and `out` are device pointers (else host)           */
#define PL_FLAG_FMA 0x2u         /* allow fused multiply-add: faster, not the reference's   */
                                 /* bitwise rounding sequence (still <= 1e-9 relative)      */
#define PL_FLAG_ASYNC 0x4u       /* device pointers only: enqueue on `stream` and return;   */
                                 /* int64 overflow is reported into *status_dev instead     */

#define PL_FLAG_INPUT_READY 0x8u /* device pointers only: the caller states that `a` is not      */
                                 /* written by work still running on `stream` (it was uploaded   */
                                 /* or produced earlier and that work has completed, or on       */
                                 /* another stream the caller has already waited for). The batch */
                                 /* kernels of orders <= 5, the shared-memory kernels of orders  */
                                 /* 6..14 (warp / CTA per matrix, the int64 FP32 packs; not the  */
                                 /* two-matrix float packs) and the fused boson kernel           */
                                 /* (pl_boson_distribution) then start                           */
                                 /* loading while the previous kernel on the stream drains       */
                                 /* (programmatic dependent launch); their stores still wait for */
                                 /* it. Results are identical; other kernels ignore the flag.    */

/* Bits OR-ed into a caller-owned device status word by PL_FLAG_ASYNC calls. */
#define PL_STATUS_BIT_OVERFLOW 0x1
#define PL_STATUS_BIT_ROWS 0x2 /* boson: a malformed output row list (its probability is NaN) */

const char* pl_version(void);
const char* pl_last_error(void);
void pl_limits_default(pl_limits* out);
/* Number of CUDA devices visible (0 if none or the driver is unusable). */
int32_t pl_device_count(void);

/* Single permanent. Replaces permlab::store_zechin_permanent
 * (reference permanent.hpp:90, permanent.cpp:314-316). `out` receives one
 * entry of `dtype`. `stream` is a cudaStream_t (NULL = the calling thread's
 * default stream). Synchronous unless PL_FLAG_ASYNC. */
pl_status pl_sz_permanent(pl_dtype dtype, int32_t n, const void* a, void* out, uint32_t flags,
                          const pl_limits* limits, void* stream);

/* Batch of `count` permanents of order n. The reference has no batch entry
 * point: this replaces its callers' loops over store_zechin_permanent
 * (reference boson.cpp:262-265 via outcome_probability boson.cpp:229-240).
 * With PL_FLAG_ASYNC, `status_dev` (device int32, caller-zeroed) receives
 * PL_STATUS_BIT_* bits; otherwise it may be NULL. */
pl_status pl_sz_permanent_batch(pl_dtype dtype, int32_t n, int64_t count, const void* a, void* out,
                                uint32_t flags, const pl_limits* limits, void* stream, int32_t* status_dev);

/* Exact integer permanent of any magnitude. The reference's Int ring is
 * arbitrary precision (reference proj/include/permlab/ring.hpp:29-31), so its
 * store_zechin_permanent (permanent.cpp:314-316) never overflows; PL_I64 is
 * exact while every intermediate fits int64 and returns PL_ERR_OVERFLOW
 * otherwise. This entry point returns the reference's value in every case:
 * the layer DP runs on residues modulo K primes below 2^31 (K from the
 * row-sum bound |per(A)| <= prod_i sum_j |a_ij|) and the residues are
 * recombined on the host (CRT). `a`: n x n int64 entries (host). The result is
 * sign (*negative = 1 for a negative value) and magnitude as *nlimbs
 * little-endian 64-bit limbs (0 limbs = zero). If limb_cap is too small the
 * call returns PL_ERR_ARG with *nlimbs set to the size needed
 * (34 x 34 int64 entries need at most 37 limbs). Synchronous. */
pl_status pl_sz_permanent_bigint(int32_t n, const int64_t* a, uint64_t* limbs, size_t limb_cap, size_t* nlimbs,
                                 int32_t* negative, const pl_limits* limits, void* stream);

/* The residue passes on their own: out[i] = per(R_i) mod primes[i], where R_i
 * (n x n int64 entries in [0, primes[i]), host) is the matrix reduced modulo
 * primes[i] (any moduli in [2, 2^31); pairwise coprime for a CRT). For callers
 * whose entries exceed int64 and who recombine themselves (the Python API does,
 * for Python integers). pl_bigint_primes writes the first `count` primes the
 * engine itself uses (descending from 2^31 - 1) and returns count. */
pl_status pl_sz_permanent_modp(int32_t n, int32_t nprimes, const uint32_t* primes, const int64_t* residues,
                               uint32_t* out, const pl_limits* limits, void* stream);
int32_t pl_bigint_primes(int32_t count, uint32_t* out);

/* The same for Ryser's formula (reference permanent.hpp:84 on its Int ring,
 * permanent.cpp:85-136): pl_ryser_permanent reports PL_ERR_OVERFLOW where the
 * value or its guard bound leaves the 128-bit / int64 range; these return the
 * exact integer (sign + limbs as above) from inclusion-exclusion sums on
 * residues, and the residues alone. Any order up to PL_MAX_ORDER within
 * subset_order_limit. Synchronous. */
pl_status pl_ryser_permanent_bigint(int32_t n, const int64_t* a, uint64_t* limbs, size_t limb_cap, size_t* nlimbs,
                                    int32_t* negative, const pl_limits* limits, void* stream);
pl_status pl_ryser_permanent_modp(int32_t n, int32_t nprimes, const uint32_t* primes, const int64_t* residues,
                                  uint32_t* out, const pl_limits* limits, void* stream);

/* Operation counts of the Store-zechin recurrence (reference measures them
 * through Counted<T>, op_count.hpp:52-70; closed form cost_model.cpp:176-181):
 * n = 1 -> (0, 0); n = 2 -> (2, 1); n >= 3 -> (n*2^(n-1) - n, n*2^(n-1) - 2^n + 1). */
pl_status pl_sz_counts(int32_t n, uint64_t* multiplications, uint64_t* additions);

/* Memo diagnostics of permlab::store_zechin_run (reference permanent.hpp:66-73):
 * every subset of size 2..n-1 is evaluated exactly once, so
 * cache_misses = distinct_subsets = 2^n - n - 2 for n >= 3, 1 for n = 2, 0 for n = 1. */
pl_status pl_sz_diagnostics(int32_t n, uint64_t* cache_misses, uint64_t* distinct_subsets);

/* ---- Ryser engine (reference permanent.hpp:84, permanent.cpp:85-136) -----
 * permlab::ryser_permanent: inclusion-exclusion over the nonempty column
 * subsets, visited in the reference's depth-first (lexicographic preorder)
 * order. Float rings (PL_F64, PL_C128) reproduce the reference's rounding
 * sequence bit for bit: every row sum is the ascending left fold of its
 * columns, every product the left fold of the row sums, and the total the
 * left fold of the signed products in visit order (a sequential device
 * fold). PL_I64 is exact (wrapping 128-bit arithmetic, exact whenever
 * prod_i max(1, sum_j |a_ij|) < 2^126 and the permanent fits int64, else
 * PL_ERR_OVERFLOW). Synchronous;
 * host pointers, or device pointers with PL_FLAG_DEVICE_PTRS. PL_FLAG_FMA is
 * ignored (the engine has no multiply-add). Orders are limited as for
 * store-zechin (subset_order_limit, PL_MAX_ORDER). */
pl_status pl_ryser_permanent(pl_dtype dtype, int32_t n, const void* a, void* out, uint32_t flags,
                             const pl_limits* limits, void* stream);
/* Operation counts of Ryser (reference count_formula, cost_model.cpp:168-174,
 * equal to its instrumented counts): (2^n - 1)(n - 1) multiplications and
 * (2^n - n)(n + 1) - 2 additions (n >= 2; n = 1 -> (0, 0)). */
pl_status pl_ryser_counts(int32_t n, uint64_t* multiplications, uint64_t* additions);

/* ---- layer primitives (sharded multi-GPU driver, tests) -------------------
 * Layer k (2 <= k <= n-1) holds per(S) for every k-subset S of the columns
 * over the leading k rows, stored at its colex rank
 * rank(S) = sum_i C(s_i, i), s_1 < ... < s_k. */

/* Binomial coefficient C(s, k) (0 outside the table, s <= 64). */
uint64_t pl_binom(int32_t s, int32_t k);
/* Colex rank of a k-subset bitmask and its inverse. */
uint64_t pl_colex_rank(uint64_t mask);
uint64_t pl_colex_unrank(int32_t k, uint64_t rank);

/* Compute entries [rank_begin, rank_end) of layer k into cur_dev[rank] from
 * layer k-1 in prev_dev (ignored for k = 2). All pointers are device
 * pointers; `a_dev` is the n*n matrix; prev_dev must be 16-byte aligned and
 * readable for 16 bytes past its last entry (the kernel stages 16-byte
 * aligned spans). Asynchronous on `stream`. For PL_I64
 * the caller must have run pl_sz_guard_i64 on the same matrix first (its
 * device flag selects the checked path) and passes that flag in guard_dev. */
pl_status pl_sz_layer(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev,
                      void* cur_dev, uint64_t rank_begin, uint64_t rank_end, uint32_t flags,
                      const int32_t* guard_dev, int32_t* status_dev, void* stream);

/* Top level: out_dev[0] = sum_j a[n-1][j] * layer_{n-1}[n-1-j], j ascending
 * (reference permanent.cpp:184-198). n >= 3. Asynchronous. */
pl_status pl_sz_top(pl_dtype dtype, int32_t n, const void* a_dev, const void* last_layer_dev, void* out_dev,
                    uint32_t flags, const int32_t* guard_dev, int32_t* status_dev, void* stream);

/* int64 overflow guard for one matrix: guard_dev[0] = 1 when
 * prod_i max(1, sum_j |a_ij|) >= 2^63 (then kernels use checked arithmetic
 * and report PL_STATUS_BIT_OVERFLOW on an actual overflow). Asynchronous. */
pl_status pl_sz_guard_i64(int32_t n, const int64_t* a_dev, int32_t* guard_dev, void* stream);

/* Device scratch bytes a single-matrix run of order n needs (two layer
 * buffers of max_k C(n,k) entries). */
uint64_t pl_sz_scratch_bytes(pl_dtype dtype, int32_t n);

/* Large-order calls (n >= 15) keep their layer scratch (cudaMalloc blocks,
 * up to 2 x 9.6 GB at n = 32 complex) in a per-device cache for the next
 * call, as a caching allocator does; this frees every idle block (blocks of
 * calls still running on a stream are returned to the cache when their
 * stream finishes them) and the cached per-order tile lists of the layer
 * kernel (after synchronising the devices that hold them).
 * PL_SCRATCH_CACHE=0 frees the scratch after every synchronous call. */
void pl_release_scratch(void);

/* ---- multi-GPU inside one process ----------------------------------------
 * pl_limits.num_gpus = g >= 1 routes pl_sz_permanent / pl_sz_permanent_batch
 * here (synchronous; host or device pointers, UVA copies): a large order
 * (n >= 15) runs each matrix's layer DP sharded over devices 0..g-1 with
 * single-process NCCL communicators (ncclCommInitAll, cached per device set;
 * NCCL is loaded with dlopen) -- top-column blocks with ncclSend/ncclRecv
 * when g = 2^t (n - t >= 3), else equal slices with an in-place
 * ncclAllGather after every layer; smaller orders split the batch by matrix.
 * Results are bitwise those of the single-device path (same kernel on rank
 * ranges). The reference is single-threaded (permanent.cpp:310-316); this
 * is the engine's addition, the single-process counterpart of sharded.py. */
pl_status pl_sz_permanent_multi(pl_dtype dtype, int32_t n, int64_t count, const void* a, void* out, uint32_t flags,
                                const pl_limits* limits, int32_t num_gpus, const int32_t* devices);

/* The shard plans (shared with the torch.distributed driver, sharded.py). */
#define PL_SHARD_ALLGATHER 0 /* equal padded slices + in-place all-gather      */
#define PL_SHARD_BLOCKS 1    /* top-column blocks + point-to-point exchange    */
/* Plan of order n over `world` devices (-1 on bad arguments). */
int32_t pl_shard_plan(int32_t n, int32_t world);
/* Colex-rank range [r0, r1) of layer k computed by `rank`. */
pl_status pl_shard_range(int32_t n, int32_t world, int32_t rank, int32_t k, uint64_t* r0, uint64_t* r1);
/* Point-to-point operations of `rank` after layer k under the block plan
 * (0 under the all-gather plan; layer n-1 goes to rank 0): returns their
 * count and, if ops != NULL, writes up to max_ops quadruples
 * (recv ? 1 : 0, peer, r0, r1). -1 on bad arguments. */
int32_t pl_shard_exchange(int32_t n, int32_t world, int32_t rank, int32_t k, uint64_t* ops, int32_t max_ops);

/* Overlapped block plan (sharded.py, and pl_sz_permanent_multi by default;
 * PL_SHARD_OVERLAP=0 turns it off): `rank`'s block of layer k without the
 * terms of the top log2(world) columns, from its own block of layer k-1 only
 * -- so it can run while the exchange of layer k-1 is in flight -- then, once
 * the blocks P \ {c} of layer k-1 have been received, those top-column
 * terms. The top columns are the highest, so their terms come last in the
 * reference's ascending order (permanent.cpp:164-174): the two steps are the
 * same rounding sequence as pl_sz_layer. 3 <= k <= n-1; world = 2^t. */
pl_status pl_shard_block_partial(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev,
                                 void* cur_dev, int32_t world, int32_t rank, uint32_t flags, const int32_t* guard_dev,
                                 int32_t* status_dev, void* stream);
pl_status pl_shard_block_top_terms(pl_dtype dtype, int32_t n, const void* a_dev, int32_t k, const void* prev_dev,
                                   void* cur_dev, int32_t world, int32_t rank, uint32_t flags, int32_t* status_dev,
                                   void* stream);

/* ---- boson sampling (reference proj/include/permlab/boson.hpp:67-99) ------
 * An m-mode interferometer is its unitary U: m*m complex128 entries,
 * row-major, interleaved (re, im) (reference Interferometer, boson.hpp:40-56;
 * the unitarity check of its constructor stays with the host layer).
 * `input_modes` (always host memory) are n distinct modes in [0, m): the
 * submatrix columns. An output pattern with occupancy occ[0..m) is passed as
 * its n ROWS: mode i repeated occ[i] times in ascending mode order, exactly
 * the row list extract_submatrix builds (boson.cpp:213-219). The probability
 * of a pattern is |per(U[rows, input_modes])|^2 / prod_i occ[i]!
 * (outcome_probability, boson.cpp:229-240); in the default (non-FMA) mode it
 * is bitwise the reference's. Probabilities are computed on the device with
 * no submatrix in memory for n <= 6 (one fused kernel); larger n gathers the
 * submatrices and runs the batched permanent kernels. */

/* Number of output patterns of n photons over m modes, C(m+n-1, n)
 * (reference enumerate_patterns, boson.cpp:185-205); 0 on overflow. */
uint64_t pl_boson_pattern_count(int32_t m, int32_t n);

/* Rows of pattern `index` in enumerate_patterns(m, n) order (ascending mode
 * multisets: mode 0 takes the most photons first, boson.cpp:191-203) into
 * rows[0..n). Host-side helper; the device enumerator uses the same search. */
pl_status pl_boson_unrank_pattern(int32_t m, int32_t n, uint64_t index, int32_t* rows);

/* Probabilities of `count` output patterns given as row lists (count x n
 * int32, each nondecreasing in [0, m)). Replaces a loop over
 * permlab::outcome_probability (boson.hpp:73-76, boson.cpp:229-240).
 * Flags: PL_FLAG_DEVICE_PTRS (u, out_rows, probs are device pointers),
 * PL_FLAG_FMA, PL_FLAG_ASYNC (device pointers; a malformed row list sets
 * PL_STATUS_BIT_ROWS in *status_dev and gets a NaN probability; synchronous
 * calls return PL_ERR_ARG instead). `limits` applies the subset-order cap. */
pl_status pl_boson_probabilities(int32_t m, const void* u, int32_t n, const int32_t* input_modes, int64_t count,
                                 const int32_t* out_rows, double* probs, uint32_t flags, const pl_limits* limits,
                                 void* stream, int32_t* status_dev);

/* Probabilities of patterns [first, first + count) of enumerate_patterns(m, n)
 * order, the patterns enumerated on the device (nothing but U is read).
 * Replaces the probability loop of permlab::full_distribution
 * (boson.hpp:85-87, boson.cpp:250-269); n <= 6 as there (PL_ERR_LIMIT
 * otherwise, the reference's message). The enumeration_cap check stays with
 * the caller (the host layer applies Limits::enumeration_cap); a pattern
 * range lets callers chunk or shard a distribution. Flags as above. */
pl_status pl_boson_distribution(int32_t m, const void* u, int32_t n, const int32_t* input_modes, uint64_t first,
                                int64_t count, double* probs, uint32_t flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PERMLAB_B200_H */
