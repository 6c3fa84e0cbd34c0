/* bto_b200.h -- C ABI of libbto_b200.so, the B200 (sm_100a) drop-in for the
 * reference's generated-C kernels.
 *
 * Boundary being replaced.  The reference (matfuse) prints one C function per
 * kernel spec and calls it through ctypes:
 *   - signature rule ........ cemit.py:225-241 (kernel_params): inputs in
 *     declaration order (array -> const double*, scalar -> double by value),
 *     outputs in declaration order (double*; a scalar output is double*),
 *     then the extents in sorted order (M[, N]) as long; returns void;
 *   - symbol name ........... spec.name.lower()            (cemit.py:261)
 *   - caller ................ runtime.run_kernel            (runtime.py:99-150)
 *     which dlopens the library, looks the symbol up by kernel name and
 *     passes numpy (HOST) buffers; outputs arrive NaN-filled and must be
 *     fully overwritten (runtime.py:108,130);
 *   - layout ................ fp64, matrices dense row-major, i*N + j
 *     (cemit.py:54-72).
 *
 * Section 1 exports exactly those symbols, so the reference's own
 * `run_kernel(Path("libbto_b200.so"), kernel, graph, inputs, extents)` works
 * unchanged.  Every pointer argument may be a host pointer (pageable or
 * pinned) or a device pointer; the library asks the driver which.  If any
 * argument is host memory the call stages it through device memory and
 * returns when the outputs are back on the host; if all are device pointers
 * the kernels are enqueued on the library stream (bto_set_stream, default the
 * legacy default stream) and the call returns immediately.
 *
 * The functions return void like the reference's, so failures are reported
 * through bto_last_error(); nothing here falls back to the CPU.
 */
#ifndef BTO_B200_H
#define BTO_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define BTO_B200_ABI_VERSION 2

/* ---- error channel (thread-local; cleared at the start of every call) ---- */
enum {
    BTO_OK = 0,
    BTO_ERR_CUDA = 1,         /* a CUDA runtime call or launch failed         */
    BTO_ERR_INVALID = 2,      /* negative extent, null pointer, bad argument  */
    BTO_ERR_NO_DEVICE = 3,    /* no sm_100 device visible                     */
    BTO_ERR_ALLOC = 4,        /* workspace / staging allocation failed        */
    BTO_ERR_EXCHANGE = 5      /* fused cross-GPU exchange: a peer never arrived */
};
int         bto_last_error(void);
const char *bto_last_error_string(void);
void        bto_clear_error(void);

/* ---- 1. drop-in symbols: the reference's generated-C signatures ----------
 * Hot path (BASELINE.json north_star); replaces the functions cemit.py
 * prints for kernels/{axpydot,bicgk,atax,gesummv,gemver}.bto.              */
void axpydot(const double *w, const double *v, const double *u, double alpha,
             double *z, double *beta, long M);
void bicgk(const double *A, const double *p, const double *r,
           double *q, double *s, long M, long N);
void atax(const double *A, const double *x, double *y, long M, long N);
void gesummv(double alpha, double beta, const double *A, const double *B,
             const double *x, double *y, long M, long N);
void gemver(const double *A, const double *u1, const double *v1,
            const double *u2, const double *v2, double alpha, double beta,
            const double *y, const double *z,
            double *B, double *x, double *w, long M, long N);
/* Rest of the reference corpus (corpus.py:18-21 + BATAX), same primitives.  */
void vadd(const double *w, const double *y, const double *z, double *x, long M);
void waxpby(double alpha, const double *x, double beta, const double *y,
            double *w, long M);
void dgemv(double alpha, const double *A, const double *x, double beta,
           const double *y, double *z, long M, long N);
void dgemvt(double alpha, double beta, const double *A, const double *y,
            const double *z, double *x, double *w, long M, long N);
void batax(const double *x, double beta, const double *A, double *y,
           long M, long N);

/* ---- 2. asynchronous variants: DEVICE pointers only, explicit stream ------
 * Same argument order plus a cudaStream_t (as void*).  Return BTO_OK or an
 * error code (also left in bto_last_error).  These are what the timing loop
 * (the replacement for cost.py:163-208 / cemit.py:294-359) and the sharded
 * runtime call.
 *
 * Concurrency contract (the reference: "thread-safe to invoke once at a time
 * per output buffer"; its kernels malloc their partials per call,
 * cemit.py:183-202).  Here:
 *   - host-side the library is thread safe: every entry point takes one
 *     process-wide lock for the (microseconds of) launch planning;
 *   - device-side every CUDA stream has its OWN partial-sum workspace and
 *     ticket counters, so sequences enqueued on different streams may run
 *     concurrently; sequences on one stream run in order.  Output buffers must
 *     not be shared between calls that can overlap;
 *   - the entry points are legal under stream capture and the captured graphs
 *     stay valid: a stream's workspace grows by adding a chunk, and a chunk a
 *     captured kernel was given is never freed before bto_release_workspace()
 *     (growth itself allocates in relaxed capture mode; call
 *     bto_reserve_workspace(stream, bytes) once before capturing to avoid even
 *     that).  Replaying a graph concurrently with other work on the stream it
 *     was captured from shares that stream's workspace -- do not;
 *   - section-1 calls with host operands hold the lock until their outputs are
 *     back on the host (one at a time per process);
 *   - the sharded entry points of 3b share ONE exchange buffer per device:
 *     one stream at a time, every rank the same order.                       */
typedef void *bto_stream_t;

int bto_axpydot_async(const double *w, const double *v, const double *u,
                      double alpha, double *z, double *beta, long M,
                      bto_stream_t stream);
int bto_bicgk_async(const double *A, const double *p, const double *r,
                    double *q, double *s, long M, long N, bto_stream_t stream);
int bto_atax_async(const double *A, const double *x, double *y,
                   long M, long N, bto_stream_t stream);
int bto_gesummv_async(double alpha, double beta, const double *A,
                      const double *B, const double *x, double *y,
                      long M, long N, bto_stream_t stream);
int bto_gemver_async(const double *A, const double *u1, const double *v1,
                     const double *u2, const double *v2, double alpha,
                     double beta, const double *y, const double *z,
                     double *B, double *x, double *w, long M, long N,
                     bto_stream_t stream);
int bto_vadd_async(const double *w, const double *y, const double *z,
                   double *x, long M, bto_stream_t stream);
int bto_waxpby_async(double alpha, const double *x, double beta,
                     const double *y, double *w, long M, bto_stream_t stream);
int bto_dgemv_async(double alpha, const double *A, const double *x,
                    double beta, const double *y, double *z,
                    long M, long N, bto_stream_t stream);
int bto_dgemvt_async(double alpha, double beta, const double *A,
                     const double *y, const double *z, double *x, double *w,
                     long M, long N, bto_stream_t stream);
int bto_batax_async(const double *x, double beta, const double *A, double *y,
                    long M, long N, bto_stream_t stream);

/* ---- 3. row-sharded pieces (multi-GPU runtime) ------
 * A rank owning rows [M*g/G, M*(g+1)/G) calls the *_async entry points above
 * on its shard for AXPYDOT/BiCGK/ATAX/GESUMMV and all-reduces the column-
 * indexed result.  GEMVER and DGEMVT have a true grid-wide dependency (x needs
 * every row), so they are split at the exchange point:
 *   pass1: B = A + u1 v1' + u2 v2' (rows of the shard), colsum = B' y
 *          (A == B and u1 == NULL selects DGEMVT: colsum = A' y, nothing stored)
 *   -- all-reduce colsum over ranks --
 *   xupdate: x = colsum*beta + z
 *   pass2: w = alpha * B x  (rows of the shard)                              */
int bto_gemver_pass1_async(const double *A, const double *u1, const double *v1,
                           const double *u2, const double *v2, const double *y,
                           double *B, double *colsum, long M, long N,
                           bto_stream_t stream);
int bto_gemver_xupdate_async(const double *colsum, double beta, const double *z,
                             double *x, long N, bto_stream_t stream);
int bto_gemver_pass2_async(const double *B, const double *x, double alpha,
                           double *w, long M, long N, bto_stream_t stream);

/* ---- 3b. the exchange fused into the join (NVLink / NVSwitch peer memory) ---
 * Instead of "join locally, then all-reduce", the join kernel of a sharded
 * sequence writes this rank's partial of the column-indexed result into a
 * symmetric exchange buffer, publishes a flag in every peer's flag array, waits
 * for the peers' flags and adds all partials in rank order straight from peer
 * memory (one-shot; the payload is <= 256 KiB, so this is latency-optimal and
 * every rank gets bit-identical results).  GEMVER's x = beta*sum + z epilogue
 * runs in the same kernel.
 *   exch_ptrs[p]  : rank p's exchange buffer as mapped on THIS device,
 *                   capacity_doubles doubles (>= 2 * the longest reduced vector:
 *                   two halves alternate between consecutive exchanges)
 *   flag_ptrs[p]  : rank p's flag array, bto_exchange_flag_bytes(world) bytes,
 *                   zeroed before the first exchange
 *   epoch0        : exchanges already performed on these buffers (0 at start)
 * Every rank must call the same *_sharded_async sequence in the same order.
 * A waiter accepts any flag value that has REACHED its epoch (a fast peer may
 * already have published the next one; the two buffer halves make that safe). */
int bto_exchange_init(int rank, int world, void *const *exch_ptrs, void *const *flag_ptrs,
                      long capacity_doubles, unsigned int epoch0);
int bto_exchange_shutdown(void);
int bto_exchange_flag_bytes(int world);
/* Synchronises the device and reports the exchange's health: BTO_OK, or
 * BTO_ERR_EXCHANGE if a wait for a peer ran into the 20 s guard (the results of
 * that exchange were set to NaN instead of hanging the GPU).  *epoch (may be
 * NULL) receives the number of exchanges completed on this rank; the counter
 * lives on the device, so replaying a captured graph advances it like a call. */
int bto_exchange_status(unsigned int *epoch);
int bto_axpydot_sharded_async(const double *w, const double *v, const double *u,
                              double alpha, double *z, double *beta, long M,
                              bto_stream_t stream);
int bto_bicgk_sharded_async(const double *A, const double *p, const double *r,
                            double *q, double *s, long M, long N, bto_stream_t stream);
int bto_atax_sharded_async(const double *A, const double *x, double *y,
                           long M, long N, bto_stream_t stream);
int bto_gemver_sharded_async(const double *A, const double *u1, const double *v1,
                             const double *u2, const double *v2, double alpha,
                             double beta, const double *y, const double *z,
                             double *B, double *x, double *w, long M, long N,
                             bto_stream_t stream);

/* ---- 3c. unfused primitives --------------------------------------------------
 * Building blocks of the generic executor: a valid kernel spec with no
 * hand-written fused sequence is evaluated statement by statement with these
 * (what the reference's unfused organism does on the CPU).  Device pointers.
 *   matvec : out = A x (transposed = 0, out has M entries) or A' x (1, N entries),
 *            A row-major M x N
 *   axpby  : mode 0 out = x*alpha; 1 out = x*alpha + y*beta; 2 out = x + y;
 *            3 out = x - y  (n elements; every op rounded on its own)
 *   outer  : out[i,j] = u[i]*v[j]  (row-major M x N)
 *   dot    : *out = sum x[i]*y[i]  (device scalar)                             */
int bto_prim_matvec_async(const double *A, const double *x, double *out, long M, long N,
                          int transposed, bto_stream_t stream);
int bto_prim_axpby_async(double alpha, const double *x, double beta, const double *y,
                         double *out, long n, int mode, bto_stream_t stream);
int bto_prim_outer_async(const double *u, const double *v, double *out, long M, long N,
                         bto_stream_t stream);
int bto_prim_dot_async(const double *x, const double *y, double *out, long n,
                       bto_stream_t stream);

/* ---- 3d. fused passes for column-major operands -----------------------------
 * A `matrix(column)` operand (lang.py:17-31, runtime.py:92-95) reaches the
 * library as the row-major buffer S of its TRANSPOSE.  Every corpus sequence
 * then maps onto the row-major passes with the roles of the two products
 * swapped (A x = S' x is a column sum, A' r = S r a row dot); the two shapes
 * the row-major entry points do not offer are these (device pointers):
 *   colsum_axpz : out[c] = (sum_r S[r,c]*y[r])*scale (+ z[c] when z != NULL)
 *   rank2_rowdot: Sout[r,c] = (S[r,c] + a1[r]*b1[c]) + a2[r]*b2[c];
 *                 out[r] = (sum_c Sout[r,c]*wgt[c])*scale + add[r]
 * each product and sum rounded as in cemit.py:112-136; S is rows x cols.      */
int bto_colsum_axpz_async(const double *S, const double *y, double scale, const double *z,
                          double *out, long rows, long cols, bto_stream_t stream);
int bto_rank2_rowdot_async(const double *S, const double *a1, const double *b1,
                           const double *a2, const double *b2, const double *wgt,
                           double scale, const double *add, double *Sout, double *out,
                           long rows, long cols, bto_stream_t stream);

/* ---- 4. runtime control and introspection --------------------------------- */
int   bto_abi_version(void);
int   bto_set_stream(bto_stream_t stream);      /* stream for section-1 calls */
/* Tunables of the launch heuristics (what the GPU variant search explores):
 * "mv_rows" (8|16|32 rows per unit), "mv_vec" (1|2 double2 per thread per row),
 * "grid_per_sm" (0 = default), "mv_minb", "vec_unroll" (1|2|4), "atax_fused",
 * "atax_cluster" (0 = chosen by the cost model of host_sequences.cuh::plan_atax, or 1..10 | 16 CTAs
 * per cluster), "atax_rows", "atax_stages", "atax_per_sm" (1|2), "host_pipeline", "host_panel_mib",
 * "rowstream" (0|1|2: GESUMMV streams whole rows, rowstream_kernels.cuh, for N >= 4096 and -- with
 * "midsize" -- for N <= 2048; 2 also the single-matrix A x pass -- measured: no gain),
 * "midsize" (0|1: size-aware launch shapes below the bench sizes), "direct_cols" (0|1),
 * "skinny" (0|1: N <= 512 takes the shared-row kernels of skinny_kernels.cuh),
 * "host_bounce" (0|1: pageable host operands of 16 MiB and more go through pinned
 * bounce slots), "host_threads" (host threads filling the slots, 0 = auto),
 * "exchange_phases", "pdl", "debug".  Unknown key or an
 * unsupported value returns BTO_ERR_INVALID.  bto_get_tuning returns -1 for
 * an unknown key.                                                           */
int   bto_set_tuning(const char *key, long value);
long  bto_get_tuning(const char *key);
/* Kernels launched by this library since load (bench.py's gpu_launches).    */
long  bto_kernel_launches(void);
/* Hash of the kernel entry points (template instances) the calling thread's LAST
 * library call launched, in order; 0 if it launched nothing.  Two calls with equal
 * signatures took the same dispatch -- the empirical timer uses it to prove that the
 * variant it validated is the variant it times.                              */
unsigned long long bto_last_launch_signature(void);
/* The same launches by name with their template arguments, '+'-separated, e.g.
 * "mv_tile_kernel<5,8,2,1,2>+finalize_kernel" (valid until the thread's next call). */
const char *bto_last_launch_plan(void);
/* Minimum HBM traffic of one call in bytes (SURVEY.md section 8d formulas);
 * negative for an unknown kernel name.  N is ignored for vector kernels.    */
double bto_bytes_min(const char *kernel, long M, long N);
/* Device facts the cost model needs: SM count, max resident threads per SM,
 * L2 bytes, total global memory bytes.  Returns BTO_OK or an error.         */
int   bto_device_info(int *sm_count, int *max_threads_per_sm,
                      long *l2_bytes, long *global_bytes);
/* Bytes currently held in the partial-sum workspace and the host staging
 * arena (both cached between calls); bto_release_workspace frees them.      */
long  bto_workspace_bytes(void);
int   bto_release_workspace(void);
/* Make `stream`'s workspace at least `bytes` large now (e.g. before capturing a graph
 * on it), so that later calls on that stream do not allocate.                 */
int   bto_reserve_workspace(bto_stream_t stream, long bytes);
/* Host <-> device copies with the staging the section-1 entry points use (pageable
 * buffers of 16 MiB and more go through the pinned bounce slots at 45-50 GB/s instead of
 * ~11 GB/s); synchronous: the data has arrived when the call returns.          */
int   bto_copy_to_device(void *device_dst, const void *host_src, long bytes);
int   bto_copy_to_host(void *host_dst, const void *device_src, long bytes);
/* Testing hook: fills every SM's shared memory with the all-ones bit pattern (NaN as a double) on
 * `stream`.  The library's kernels must not depend on shared memory they did not write in their own
 * launch; the GPU tests call this before ragged-shape runs to make such a read loud.            */
int   bto_debug_poison_shared_memory(bto_stream_t stream);
/* Testing hook: `stream`'s partial-sum workspace := NaN patterns (stream-ordered), so that a join
 * reading a partial nobody produced in the same call is loud.                                    */
int   bto_debug_poison_workspace(bto_stream_t stream);
/* Both of the above for the host-pointer entry points of section 1: shared memory on the library's
 * own stream, and the workspace of every stream the library has seen.                            */
int   bto_debug_poison_all(void);
/* host_dst[0 .. count) = value with the copy threads (first touch of fresh pages in
 * parallel: the NaN prefill of a large output, runtime.py:99-150, at 30+ GB/s).   */
int   bto_fill_host(double *host_dst, long count, double value);

#ifdef __cplusplus
}
#endif
#endif /* BTO_B200_H */
