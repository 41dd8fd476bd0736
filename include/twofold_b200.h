/*
 * twofold_b200.h — C ABI of the B200 (sm_100a) twofold summation / dot library.
 *
 * The reference (arXiv 1401.0248 package `twofold`, pure Python + numba) has no
 * FFI: its hot-path boundary is the Python call
 *     run_flavor(method, flavor, data, b=None) -> SumResult     (pkg/src/twofold/kernels.py:591-640)
 * and the ten wrappers sum_* / dot_*                              (kernels.py:669-706).
 * Every entry point below replaces one piece of that boundary; the mapping is
 * given per function.  Python binds these with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers are CUDA device (or
 *     managed) addresses; `stream` is a cudaStream_t passed as void*.
 *   - No function allocates memory.  Scratch (leaf partials + retire
 *     counters) is owned by the caller; size it with tf_workspace_size().
 *     Counters must be zero on entry; every kernel leaves them zero.
 *   - All launches are stream-ordered and asynchronous; nothing synchronizes.
 *   - Return value: TF_OK (0) or a TF_E* code; tf_strerror() names it and
 *     tf_last_cuda_error() gives the CUDA error text of the calling thread.
 *   - Result pairs are (value, error) of the accumulator type: the data type,
 *     except TF_WIDE (float32 data, float64 accumulator; kernels.py:135-140).
 *     For TF_DIRECT / TF_WIDE the error slot is +0 (kernels.py:615-621).  For
 *     TF_KAHAN it carries the pending compensation c so that pairs stay
 *     mergeable across shards; the reference reports 0 there (kernels.py:627)
 *     and so does the Python shim.
 *   - Arithmetic is strict IEEE-754 round-to-nearest-even, no FMA contraction,
 *     no flush-to-zero (kernels.py:17-21); dot products round the
 *     product in the data precision before summing (kernels.py:23-26, :209).
 */
#ifndef TWOFOLD_B200_H
#define TWOFOLD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The Python shim maps them to the reference's exception
 * types: DTYPE -> TypeError (kernels.py:576-581, :600-601), SHAPE -> ValueError
 * (kernels.py:582-583), CANARY -> RuntimeError (kernels.py:559-565). */
#define TF_OK              0
#define TF_EINVAL_METHOD   1  /* unknown method id                                  */
#define TF_EINVAL_DTYPE    2  /* dtype not f32/f64, or WIDE on f64 data             */
#define TF_EINVAL_SHAPE    3  /* negative length, rows/cols/leading dim mismatch    */
#define TF_EINVAL_ARG      4  /* bad lane count / leaf size / distribution / null   */
#define TF_EWORKSPACE      5  /* workspace missing or too small                     */
#define TF_ECUDA           6  /* a CUDA runtime call failed (tf_last_cuda_error)    */
#define TF_ECANARY         7  /* device strict-rounding canary failed               */

/* Methods, in the order of twofold.kernels.Method (kernels.py:44-49). */
#define TF_DIRECT            0  /* sum / dot            kernels.py:127-132, :186-191 */
#define TF_WIDE              1  /* sumd / dotd          kernels.py:135-140, :194-200 */
#define TF_TWOFOLD_FAST      2  /* sumtf / dottf        kernels.py:143-154, :203-214 */
#define TF_TWOFOLD_RIGOROUS  3  /* sumt / dott          kernels.py:157-170, :217-230 */
#define TF_KAHAN             4  /* sumk / dotk          kernels.py:173-183, :233-243 */

/* Opt-in flag OR-ed into TF_TWOFOLD_FAST / TF_TWOFOLD_RIGOROUS for dot products:
 * TwoProduct — the product's exact round-off fma(a, b, -fl(a*b)) is added to the
 * error channel, so value + error tracks the exact dot of the TRUE products
 * (Ogita-Rump-Oishi Dot2 style).  Not in the reference, which rounds every
 * product and tracks only summation round-off (kernels.py:23-26).
 * Invalid (TF_EINVAL_ARG) for sums and other methods. */
#define TF_TRACK_PRODUCT 0x100

/* Data types. */
#define TF_F32 0
#define TF_F64 1

/* Distributions for tf_fill (BASELINE.json configs). */
#define TF_DIST_UNIFORM01   0  /* [0,1):  f32 (u32>>8)*2^-24, f64 (u64>>11)*2^-53        */
#define TF_DIST_UNIFORM_SYM 1  /* [-1,1): 2u-1, exact in T (lcg.py:58-59 convention)     */
#define TF_DIST_NORMAL      2  /* N(0,1) Box-Muller in f64, rounded to T                   */
#define TF_DIST_ILLCOND     3  /* cfg3: permuted +-U[p0,p0+p1) pairs + p2*U[0,1) half     */

/* Library build identity (bumps when the reduction tree changes). */
int tf_version(void);
const char* tf_strerror(int code);
/* Text of the last CUDA error seen by this thread ("" if none). */
const char* tf_last_cuda_error(void);
/* Number of kernels this library has launched in this process (all threads). */
uint64_t tf_launch_count(void);

/* Device strict-rounding canary: runs the kernels' own EFT and dot-step code on
 * runtime operands — fast_two_sum(1, 2^-53) must return (1, 2^-53) in f64 and
 * (1, 2^-24) in f32, and fl(fl(a*b) + s) must differ from fma(a, b, s).
 * Replaces the import-time canary kernels.py:545-568 (and eft.py:59-66).
 * Synchronous (one tiny launch + copy on the legacy default stream). */
int tf_canary(void);

/* Auto leaf size (log2 elements) the grid reduction uses for n = rows*cols
 * elements: clamp(ceil_log2(n * sizeof(T)) - 11, log2(256*V), 16) with
 * V = 16/sizeof(T) (about 2048 leaves; one 16-byte vector per thread at least).
 * A pure function of (dtype, n): results never depend on the SM count. */
int tf_leaf_log2(int dtype, int64_t n);

/* Tuning knob (process-wide): split every leaf's 256 chains over `split`
 * CTAs (1, 2 or 4; 0 = automatic, the default; env TFB_SPLIT sets the initial
 * value).  Result-neutral by construction: only the grid balance changes. */
int tf_set_leaf_split(int split);

/* Tuning knob (process-wide): tail of the fused reduction — 0 = automatic
 * (1-D inputs of <= 64 one-vector leaves: ONE thread-block-cluster launch whose
 * CTAs merge through distributed shared memory; otherwise PDL for the LDG
 * loader; the TMA loader keeps its single launch), 1 = last-CTA retire ticket
 * inside the single launch, 2 = partials-only launch + a programmatic-
 * dependent-launch (PDL) tree kernel.  Identical results; env TFB_TAIL sets
 * the initial value. */
int tf_set_tail(int tail);

/* Tuning knob (process-wide): L2 prefetch preamble of the streaming kernels (the
 * LDG leaves and single-cluster kernels, the one-CTA-per-SM TMA rings, the short-row
 * kernels up to 8 MiB).  The
 * kernel is launched as a programmatic dependent of whatever precedes it in the
 * stream; before it waits for that kernel's completion each CTA asks the L2 (bulk
 * prefetch, a hint: nothing is read into the SM, and the L2 is the point of
 * coherence) for the first `kib` KiB per operand of its first leaf, so HBM streams
 * the head of this call while the predecessor's tail retires.  -1 = automatic
 * (a 32 MiB budget shared by the grid), 0 = off, up to 512.  Result-neutral; env
 * TFB_PF_KB sets the initial value. */
int tf_set_prefetch(int kib);

/* Tuning knob (process-wide): kernel for tf_reduce_rows when every row fits one
 * leaf (cols <= 2^leaf_log2) — 0 = automatic (rows of <= 16 KiB per operand: a
 * group of 1..32 lanes per row, rows.cuh; longer rows: one CTA per row), 1 =
 * always one CTA per row, 2 = always lane groups.  Identical results; env
 * TFB_ROWS sets the initial value. */
int tf_set_rows_kernel(int kind);

/* Human-readable description of the calling thread's last grid-reduction
 * launch (kernel, template arguments, grid, block, units, leaf size). */
const char* tf_last_launch(void);

/* Tuning knob (process-wide): loader of the grid reduction for 16-byte aligned
 * inputs — 0 = automatic (default: TMA for >= 512 MiB dots and >= 4 GiB
 * twofold sums, else LDG), 1 = 128-bit streaming LDG, 2 = warp-
 * specialised bulk-copy (TMA engine) pipeline, 4 stages x 16 KiB per operand,
 * 3 = 8 x 8 KiB, 4 / 5 = experimental dot shapes (3 x 32 KiB, 6 x 16 KiB).
 * Results are bit-identical (same partition and trees); env TFB_LOADER sets
 * the initial value. */
int tf_set_loader(int loader);

/* Scratch for rows x cols (1-D: rows = 1, cols = n) at leaf_log2 (0 = auto):
 *   partials: rows * leaves(cols) (value, error) pairs, any contents on entry;
 *   counters: `rows` uint32 retire-tickets, ZERO on entry and left zero on exit
 *             (so a caller can keep one zeroed counter buffer per stream).
 * Only needed when a row spans more than one leaf (*leaves > 1): for rows > 1
 * and *leaves <= 1 both sizes are returned as 0 (a 1-D call with one leaf still
 * reports its pair slots, which the fused NVLink combine uses). */
int tf_workspace_size(int method, int dtype, int64_t rows, int64_t cols, int leaf_log2,
                      size_t* partials_bytes, int64_t* counters, int64_t* leaves);

/* Grid reduction ("cuda" flavor) of one contiguous array: one fused launch
 * (leaf partials -> last-CTA balanced tree).  y == NULL: sum of x; else dot.
 * out_pair: device, 2 accumulator elements.  Replaces run_flavor(method, <any
 * flavor>, x[, y]) (kernels.py:591-640) for the GPU flavor.  leaf_log2 = 0 picks
 * tf_leaf_log2(dtype, n); pass the GLOBAL array's leaf size when x is one shard
 * of a larger array so the shard's tree is a subtree of the whole. */
int tf_reduce(int method, int dtype, const void* x, const void* y, int64_t n,
              int leaf_log2, void* out_pair, void* partials, size_t partials_bytes,
              void* counters, int64_t counters_len, void* stream);

/* Batched row-wise reduction: rows x cols, row r at x + r*ldx (elements).
 * out_pairs: device, rows pairs.  Row r's pair is bit-identical to
 * tf_reduce(x + r*ldx, cols) with the same explicit leaf_log2 (the auto leaf
 * depends on rows*cols, so pass tf_leaf_log2(dtype, rows*cols)) (no reference analogue:
 * equals a per-row loop of dot_twofold_fast). */
int tf_reduce_rows(int method, int dtype, const void* x, const void* y,
                   int64_t rows, int64_t cols, int64_t ldx, int64_t ldy,
                   int leaf_log2, void* out_pairs, void* partials, size_t partials_bytes,
                   void* counters, int64_t counters_len, void* stream);

/* Fused cross-GPU combine over NVLink peer memory:
 * tf_reduce of this rank's shard whose final CTA publishes the shard's pair
 * into every peer's symmetric buffer, waits for all G pairs and runs the same
 * balanced merge as tf_merge_tree — one launch instead of reduce + NCCL
 * all-gather + merge; every rank gets the bit-identical global pair.
 * peer_ctx: device pointer to a PeerCtx (csrc/peer.cuh; tf_peer_ctx_size()
 * bytes): {int32 world, int32 rank, int32* error (2 words), void* bufs[16]
 * (peer r's [2][world] pair buffer), uint32* flags[16] (peer r's [world]
 * flags, zero at creation), uint64 timeout_ns}.  epoch: 1, 2, 3, ...
 * identical on all ranks for the same call.  If some peer's pair has not
 * arrived within timeout_ns, the call writes NaN, error[1] = bitmask of the
 * missing ranks and error[0] = epoch (per call, not sticky); the caller
 * checks error[0] == epoch after the stream completes.
 * Unlike tf_reduce, the partials scratch is required even for a single leaf. */
int tf_reduce_peer(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2,
                   void* out_pair, void* partials, size_t partials_bytes, void* counters,
                   int64_t counters_len, const void* peer_ctx, uint32_t epoch, void* stream);
int tf_peer_ctx_size(void);

/* Leaf partials only (no tree): partials_out[0 .. ceil(n/2^leaf_log2)) for an
 * n-element chunk whose first element starts a leaf.  Used for streamed
 * host->device inputs and by the shard layer; finish with tf_merge_tree. */
int tf_reduce_leaves(int method, int dtype, const void* x, const void* y, int64_t n,
                     int leaf_log2, void* partials_out, void* stream);

/* Balanced binary tree (padded to a power of two with (+0,+0)) over `count`
 * device pairs, using the method's merge: TwoSum + error fold for twofold
 * (kernels.py:310-317), Kahan feed (kernels.py:379-390), plain add otherwise.
 * Used after the NCCL all-gather of per-rank pairs.  count == 0 gives (+0,+0). */
int tf_merge_tree(int method, int dtype, const void* pairs, int64_t count,
                  void* out_pair, void* stream);

/* Sequential flavor on the GPU: one thread runs the reference recurrence left
 * to right — bit-identical to the reference `seq` kernels (kernels.py:127-243). */
int tf_reduce_seq(int method, int dtype, const void* x, const void* y, int64_t n,
                  void* out_pair, void* stream);

/* Lane flavor (unroll:k / vec:k) on the GPU: k lanes striding the array, merged
 * left to right, tail continued on the merged state — bit-identical to the
 * reference lane kernels (kernels.py:257-541).  lanes: power of two in [2,16]. */
int tf_reduce_lanes(int method, int dtype, const void* x, const void* y, int64_t n,
                    int lanes, void* out_pair, void* stream);

/* "noread" compute roof (the paper's p-functions): `blocks`
 * CTAs of 256 threads each run the method's per-element recurrence over
 * iters*8 register-resident addends (dot: products of register operands);
 * seed8 = 8 device values of the data type; out_pairs: blocks*256 pairs.
 * Throughput = blocks*256*iters*8 / time: the FP ceiling the memory-bound
 * kernels are compared against (bench.py:281-307 methodology). */
int tf_noread(int method, int dtype, int dot, const void* seed8, int64_t iters, int64_t blocks,
              void* out_pairs, void* stream);

/* Read roof (the paper's read1 / read2 rows): stream nbytes
 * (16-byte aligned) with an XOR fold only, `unroll` (2/4/8/16) 16-byte loads in
 * flight per thread, 8 CTAs x 256 threads per SM.  sink: one device uint32. */
int tf_read_roof(const void* data, int64_t nbytes, int unroll, void* sink, void* stream);

/* Elementwise EFTs on device arrays: kind 0 = fast_two_sum (eft.py:28-42),
 * kind 1 = two_sum (eft.py:45-56).  x_out = fl(a+b), y_out = round-off. */
int tf_eft(int kind, int dtype, const void* a, const void* b, int64_t n,
           void* x_out, void* y_out, void* stream);

/* Seeded Philox4x32-10 fill: element i of the stream uses counter
 * (offset+i, stream_id) and key = seed, so any shard [o, o+n) of a stream is
 * generated independently of the shard layout.  p0..p2: distribution
 * parameters (ILLCOND: p0 = 1e8, p1 = 9e8, p2 = 1e-3 for cfg3; total length
 * for the permutation is p3_total). */
int tf_fill(int dist, int dtype, uint64_t seed, uint64_t stream_id, uint64_t offset,
            int64_t n, double p0, double p1, double p2, int64_t total,
            void* out, void* stream);

/* Host twin of tf_fill for the integer-exact distributions (UNIFORM01,
 * UNIFORM_SYM, ILLCOND): fills a HOST buffer bit-identically to the device
 * stream (SURVEY.md §8(b) tf_philox_fill_host).  nthreads <= 0: all cores. */
int tf_fill_host(int dist, int dtype, uint64_t seed, uint64_t stream_id, uint64_t offset, int64_t n,
                 double p0, double p1, double p2, int64_t total, void* out, int nthreads);

/* The reference's LCG generators (lcg.py:75-116), bit-identical to
 * twofold.fill(kind, offset+n, seed, dtype, sym)[offset:]: kind 0 = Numerical
 * Recipes (32-bit), 1 = MMIX (64-bit); state jump-ahead makes any slice
 * independent, so the reference's accuracy experiments can run on GPU data. */
int tf_lcg_fill(int kind, int dtype, uint64_t seed, int sym, int64_t offset, int64_t n,
                void* out, void* stream);

/* Exact (correctly rounded) sum of addends on the GPU — the device counterpart
 * of the reference's expansion oracle (expansion.py:79-140).
 * Addends: x_i (y == NULL); fl_T(x_i*y_i) (the twofold dot kernels' addends);
 * or, with TF_EXACT_TRUE_PRODUCTS, the exact products x_i*y_i.  TF_EXACT_ABS
 * sums |addend| instead.  out2 (device, 2 doubles): hi = fl(S), lo = fl(S - hi).
 * limbs_out (device, optional, 73 int64): S = sum_k limbs[k] 2^(32k-1074) +
 * limbs[72] 2^(32*72-1074), for exact checks.  Non-finite addends give NaN.
 * Scratch: `records` (tf_exact_workspace bytes: the grid's integer accumulator)
 * and one uint32 counter, both ZERO on entry and left zero on exit.  *records
 * reports the grid size.  Integer accumulation makes the result independent of
 * the grid. */
#define TF_EXACT_ABS           1
#define TF_EXACT_TRUE_PRODUCTS 2
int tf_exact_workspace(int64_t* records, size_t* bytes);
int tf_exact(int dtype, const void* x, const void* y, int64_t n, int flags, void* out2,
             void* limbs_out, void* records, size_t records_bytes, void* counter, void* stream);

/* cfg4 rows: out[r*ld + c] = N(0,1)[stream_id, (row0+r)*cols + c] * 10^U_r with
 * U_r = lo + (hi-lo)*u(seed, scale_stream, row0+r), one scale per row. */
int tf_fill_rows_scaled(int dtype, uint64_t seed, uint64_t stream_id,
                        uint64_t scale_stream, int64_t row0, int64_t rows,
                        int64_t cols, int64_t ld, double lo, double hi,
                        void* out, void* stream);

/* Host-buffer engine — the reference's blocking call on HOST memory as one
 * native call: run_flavor(method, Flavor("cuda"), data, b) (kernels.py:591-640)
 * where data/b are numpy arrays.  An engine owns a stream, two staging slots
 * (pinned + device, chunk_bytes per operand; 0 = 16 MiB, min 1 MiB), grown-on-
 * demand scratch and a `threads`-wide memcpy pool (0 = min(8, cores/2)); it
 * allocates at creation and when the scratch grows — the one exception to "no
 * function allocates".  engine: out, an opaque handle. */
int tf_host_engine_create(int device, int threads, size_t chunk_bytes, void** engine);
int tf_host_engine_destroy(void* engine);
int tf_host_engine_threads(const void* engine);

/* (value, error) of x[, y] (n elements each) into out_pair_host (2 accumulator
 * elements, host memory); blocks until done.  Pageable inputs go through the
 * pinned slots (the pool copies chunk c+1 while chunk c is on the DMA engine
 * and its leaves reduce); page-locked inputs DMA directly; device pointers (of
 * the engine's device) reduce in place.  after_stream: the stream device /
 * page-locked operands are ordered on (NULL = the legacy default stream) —
 * the engine's work starts after that stream's pending work.  Leaf-aligned chunks: bit-identical
 * to tf_reduce.  Calls on one engine are serialised. */
int tf_host_reduce(void* engine, int method, int dtype, const void* hx, const void* hy, int64_t n,
                   int leaf_log2, void* out_pair_host, void* after_stream);

/* Hybrid host path of tf_host_reduce (1-D host operands, methods 0..4, no
 * TwoProduct, inputs >= min_bytes per operand): the engine's host workers
 * reduce full leaves from the back of the array while the GPU pipeline takes
 * chunks from the front; the host leaf pairs are uploaded and one tf_merge_tree
 * closes the tree — bit-identical to tf_reduce for every split.  threads: the
 * number of host workers (0 = GPU only; < 0 keeps the current pool).  Defaults
 * at creation: TFB_HYBRID_THREADS (the process's CPUs but one), TFB_HYBRID_MIN_MB (8). */
int tf_host_engine_hybrid(void* engine, int threads, size_t min_bytes);
/* Elements the last tf_host_reduce on this engine reduced on the GPU (these
 * crossed the link) and on the host workers. */
int tf_host_engine_last_split(const void* engine, int64_t* gpu_elems, int64_t* host_elems);
/* The host workers' leaf reducer itself (no GPU needed): pairs of the full
 * leaves [leaf_lo, leaf_hi) of x (and y) at leaf size 2^leaf_log2 (0 = auto for
 * n), exactly the device leaves' pairs (tf_reduce_leaves).  Methods 0..4. */
int tf_host_leaves(int method, int dtype, const void* x, const void* y, int64_t n, int leaf_log2, int64_t leaf_lo,
                   int64_t leaf_hi, void* out_pairs);

/* The host workers' row reducer (no GPU needed): pairs of rows [row_lo, row_hi)
 * of a (rows, cols) matrix with leading dimensions ldx / ldy at the matrix's leaf
 * size (0 = auto for rows * cols) — each row's leaves and row tree exactly as
 * tf_reduce_rows.  Used by tf_host_reduce_rows' hybrid path.  Methods 0..4. */
int tf_host_rows(int method, int dtype, const void* x, const void* y, int64_t rows, int64_t cols, int64_t ldx,
                 int64_t ldy, int leaf_log2, int64_t row_lo, int64_t row_hi, void* out_pairs);

/* Row-wise form (tf_reduce_rows on host matrices): rows x cols with leading
 * dimensions ldx / ldy (elements); out_pairs_host: rows (value, error) pairs.
 * Row blocks are packed into the staging slots (pitched DMA for page-locked
 * strided input) and reduced while the next block is in flight; the leaf size
 * is the whole matrix's, so every row is bit-identical to tf_reduce_rows on
 * the same matrix.  rows == 1 is the 1-D call. */
int tf_host_reduce_rows(void* engine, int method, int dtype, const void* hx, const void* hy, int64_t rows,
                        int64_t cols, int64_t ldx, int64_t ldy, int leaf_log2, void* out_pairs_host,
                        void* after_stream);

#ifdef __cplusplus
}
#endif

#endif /* TWOFOLD_B200_H */
