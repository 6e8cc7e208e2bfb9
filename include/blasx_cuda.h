/* blasx_cuda.h — C ABI of the B200 tile engine (libblasx_cuda.so).
 *
 * The Python host runtime (paper_1510_05041_b200/, loaded with ctypes) keeps the
 * reference's planner, scheduler and cache bookkeeping; everything that touches a GPU
 * goes through these entry points.  Each one replaces a seam of the reference
 * (paths relative to /root/reference/pkg/src/tileblas):
 *
 *   bx_init / bx_shutdown      memory.py:50-51 (one backing reservation per device),
 *                              devices.py:102-118 (engines = streams), peer enablement
 *   bx_host_register           (new) page-locking of caller operands, excluded from
 *                              timing like the paper
 *   bx_h2d_tile                tiling.py:192-204 tile_host_copy_in + scheduler.py:248-258
 *   bx_d2h_tile                tiling.py:207-215 tile_host_copy_out + scheduler.py:488-505
 *   bx_p2p_tile                scheduler.py:260-270 copy_from_peer / cache.py:312-322
 *   bx_gemm_task               kernels.py:49-58 gemm_update (+ the k-loop of one task,
 *                              routines.py:227-236), syrk/syr2k_update (kernels.py:67-102)
 *                              via the triangle epilogue
 *   bx_trsm_tile               kernels.py:105-161 trsm_solve
 *   bx_materialize             kernels.py:164-211 (_masked_triangle / _symmetrized)
 *   bx_axpy_tile               kernels.py:40-41 _accumulate's beta*C term, applied late
 *   bx_event_*                 devices.py:150-166 sync_streams / drain_time; trace times
 *   bx_last_error              errors.py exception messages
 *
 * Conventions: every call returns int status (BX_OK = 0; BX_EINVAL = 5 invalid argument,
 * BX_ESINGULAR = 6, BX_ENOMEM = 7, BX_ECUDA = -1 any CUDA runtime error — message in
 * bx_last_error).  No exception crosses the ABI.  Device memory is addressed as
 * (device index, byte offset into that device's arena); the Python Arena is the
 * authority for offsets.  Host pointers are borrowed and should be registered.  Every
 * enqueue is asynchronous: it waits on `n_wait` event ids first and returns a completion
 * event id through `ev_out` (pass NULL to skip).  Event ids are owned by the caller until
 * bx_event_release.  Any host thread may call; ctypes drops the GIL for the call.
 */
#ifndef BLASX_CUDA_H
#define BLASX_CUDA_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define BX_OK 0
#define BX_EINVAL 5
#define BX_ESINGULAR 6
#define BX_ENOMEM 7
#define BX_ECUDA (-1)

/* stream lanes per device: 0..n_compute-1 compute, then these */
#define BX_LANE_H2D (-1)
#define BX_LANE_D2H (-2)
#define BX_LANE_P2P (-3)

int bx_version(void);
int bx_device_count(int* n);
/* name (>=64 bytes), SM count, total and free HBM bytes */
int bx_device_info(int dev, char* name, int name_len, int* sms, uint64_t* total_bytes,
                   uint64_t* free_bytes);
/* free / total HBM of engine slot `dev` (cudaMemGetInfo only; cheap) */
int bx_mem_info(int dev, uint64_t* free_bytes, uint64_t* total_bytes);
/* Create per-device engines: streams, event pool, singular flag, arena of arena_bytes[i]
 * (0 = keep current), enable peer access between all pairs.  Idempotent; re-init with a
 * larger arena grows the reservation. */
int bx_init(int ndev, const int* device_ids, const uint64_t* arena_bytes, int n_compute);
int bx_shutdown(void);
int bx_arena_base(int dev, uint64_t* base);
int bx_peer_enabled(int dev_a, int dev_b, int* enabled);

int bx_host_register(void* ptr, uint64_t bytes);
int bx_host_unregister(void* ptr);
int bx_host_is_registered(const void* ptr, int* yes);

/* strided host tile (column-major, host ld in elements) <-> contiguous device tile
 * (column-major, device ld in elements) */
int bx_h2d_tile(int dev, uint64_t dst_off, int dst_ld, const void* src, int64_t src_ld, int h,
                int w, int elem_bytes, int n_wait, const int* wait, int* ev_out);
int bx_d2h_tile(int dev, uint64_t src_off, int src_ld, void* dst, int64_t dst_ld, int h, int w,
                int elem_bytes, int n_wait, const int* wait, int* ev_out);
/* device->device copy over NVLink/NVSwitch (dst device's P2P lane) */
int bx_p2p_tile(int dst_dev, uint64_t dst_off, int src_dev, uint64_t src_off, uint64_t bytes,
                int n_wait, const int* wait, int* ev_out);

/* one tile task: C = alpha * sum_s op(A_s) op(B_s) + beta * C on compute lane `stream`.
 * ta/tb: operands stored transposed; tri: 0 full, 1 lower, 2 upper (diagonal tiles).
 * Offsets in bytes into the arena; lds in elements; depth[s] = reduction extent of step s. */
int bx_gemm_task(int dev, int stream, int ta, int tb, int tri, int h, int w, int nsteps,
                 const uint64_t* a_off, const int* lda, const uint64_t* b_off, const int* ldb,
                 const int* depth, double alpha, double beta, uint64_t c_off, int ldc, int n_wait,
                 const int* wait, int* ev_out);
/* fp32 task GEMM (SGEMM) on tcgen05.mma.kind::tf32 with TMEM accumulators and TMA operand
 * staging; same operands/semantics as bx_gemm_task (no triangle mode). Leading dimensions
 * must be multiples of 4 elements and operands 16-byte aligned. */
int bx_sgemm_task(int dev, int stream, int ta, int tb, int h, int w, int nsteps, const uint64_t* a_off,
                  const int* lda, const uint64_t* b_off, const int* ldb, const int* depth, float alpha,
                  float beta, uint64_t c_off, int ldc, int n_wait, const int* wait, int* ev_out);
/* the same task GEMM (f32 = 0: bx_gemm_task, 1: bx_sgemm_task) with the steps packed as
 * nsteps rows of 6 int64 {a_off, lda, b_off, ldb, depth, kmode}: one host array per launch
 * (the runtime's issue path marshals one buffer instead of five).  kmode (FP64 only;
 * 0 none, 1/2 A lower/upper, 3/4 B upper/lower triangular) lets each CTA skip the k-range
 * where that step's triangular operand is zero (TRMM diagonal steps, kernels.py:173-185) */
int bx_gemm_task_packed(int dev, int stream, int f32, int ta, int tb, int tri, int h, int w, int nsteps,
                        const int64_t* steps, double alpha, double beta, uint64_t c_off, int ldc, int n_wait,
                        const int* wait, int* ev_out);
/* a launch group's tile fetches in one call (resident issue path): n rows of 8 int64
 * {kind | eb << 8, dst_off, dst_ld, src, src_ld | src_off, h | bytes, w, wait_ev};
 * kind 0 = 2-d H2D tile (src = pinned host address), 1 = peer copy (src = device slot);
 * records one event per lane used (ev_h2d / ev_p2p, -1 if unused): in-order lanes, so it
 * marks every tile of the batch on that lane (replaces per-tile bx_h2d_tile/bx_p2p_tile
 * calls and events: scheduler.py:248-281 fetch, cache.py:312-322 copy_from_peer) */
int bx_copy_batch(int dev, int n, const int64_t* ops, int n_wait, const int* wait, int* ev_h2d,
                  int* ev_p2p);
/* in-place triangular solve of B (h x w) against the diagonal tile A */
int bx_trsm_tile(int dev, int stream, int side_right, int upper, int trans, int unit, int h,
                 int w, double alpha, uint64_t a_off, int lda, uint64_t b_off, int ldb, int n_wait,
                 const int* wait, int* ev_out);
/* inverse-based TRSM diagonal step (kernels.py:105-161 restated as X = alpha inv(E) B):
 * inv (n x n) = inv(E), E = op(tri(A)) of the diagonal tile, by the substitution solve
 * E Z = I (same division rule and singular flag as bx_trsm_tile); computed once per
 * diagonal tile and reused by every task of that tile row (left) / column (right) */
int bx_trsm_inverse(int dev, int stream, int upper, int trans, int unit, int n, uint64_t a_off,
                    int lda, uint64_t inv_off, int ldi, int n_wait, const int* wait, int* ev_out);
/* x (h x w) = alpha inv(E) B (left) / alpha B inv(E) (right); eff_upper = upper ^ trans;
 * the FP64 task GEMM reading only the k-range where the triangular inv(E) is non-zero */
int bx_trsm_apply(int dev, int stream, int side_right, int eff_upper, int h, int w, double alpha,
                  uint64_t inv_off, int ldi, uint64_t b_off, int ldb, uint64_t x_off, int ldx,
                  int n_wait, const int* wait, int* ev_out);
/* dst (n x n) = op(tri(A)) [mode 0, unit diag substituted] or sym(A) [mode 1] */
int bx_materialize(int dev, int stream, int mode_sym, int upper, int trans, int unit, int n,
                   uint64_t a_off, int lda, uint64_t dst_off, int ldd, int n_wait, const int* wait,
                   int* ev_out);
/* dst (h x w) += beta * src (fp64 or fp32 by elem_bytes): the deferred beta*C term of a
 * task whose first GEMM launch ran with beta = 0, so the C tile's host copy is needed only
 * by this last kernel (kernels.py:49-58 applies beta once; same value, C0 read late) */
int bx_axpy_tile(int dev, int stream, int elem_bytes, int h, int w, double beta, uint64_t src_off,
                 int src_ld, uint64_t dst_off, int dst_ld, int n_wait, const int* wait, int* ev_out);
/* singular flag set by bx_trsm_tile kernels of this device since the last reset */
int bx_singular_flag(int dev, int reset, int* flag);

/* events */
int bx_event_record(int dev, int stream, int timing, int* ev_out);
int bx_event_query(int ev);  /* 0 complete, 1 pending, <0 error */
int bx_event_sync(int ev);
int bx_event_wait_any(int n, const int* evs, int* index, int spin_us);
int bx_event_elapsed(int ev0, int ev1, float* ms);
int bx_event_release(int ev);
int bx_event_release_many(int n, const int* evs); /* a retired task's events in one call */
int bx_stream_wait(int dev, int stream, int ev);
int bx_device_sync(int dev);
int bx_launch_count(uint64_t* n); /* kernels launched by this library since load */

/* raw device buffers + device-resident GEMM (the HBM-resident bench leg) */
int bx_dev_alloc(int dev, uint64_t bytes, uint64_t* ptr);
int bx_dev_free(int dev, uint64_t ptr);
int bx_dev_fill_uniform(int dev, uint64_t ptr, uint64_t n, uint64_t seed, int stream);
int bx_dev_fill_uniform_f32(int dev, uint64_t ptr, uint64_t n, uint64_t seed, int stream);
int bx_dev_copy_h2d(int dev, uint64_t dst, const void* src, uint64_t bytes);
int bx_dev_copy_d2h(int dev, void* dst, uint64_t src, uint64_t bytes);
int bx_dgemm_device(int dev, int stream, int ta, int tb, int m, int n, int k, double alpha,
                    uint64_t a, int lda, uint64_t b, int ldb, double beta, uint64_t c, int ldc);
/* tuning knob: tile configuration of the FP64 task GEMM: 0 (default) mbarrier ring, 16 warps
 * of 32x32; 9 the same ring with 8 warps of 64x32; 1 wide, 2 deep (__syncthreads rings);
 * 3 slack-2, 5 two CTAs/SM, 6 BK 32, 7 no slack; 8 TMA-fed */
int bx_set_gemm_variant(int variant);
/* tuning knob: raster group (consecutive m-tiles per grid column group) of the FP64 task
 * GEMM, default 8 */
int bx_set_gemm_group(int group);
/* tuning knob: largest triangle order solved by a TRSM leaf kernel (default 256); larger
 * diagonal tiles recurse (two half solves + a DMMA GEMM update) */
int bx_set_trsm_leaf(int n);
/* tuning knob: right-hand sides per CTA of the TRSM panel kernel (8, 16, 32 or 64; default 32) */
int bx_set_trsm_rhs(int nr);
/* tuning knob: SGEMM kernel, 0 = 1-SM 128x256 tile, 1 = 2-SM (cta_group::2) 256x256 tile,
 * 2 = persistent 2-SM with double-buffered TMEM accumulators (static round robin),
 * 3 = the same persistent kernel taking tiles by cluster launch control (launch order;
 * default) */
int bx_set_sgemm_variant(int variant);
/* tuning knob: load MN-major SGEMM operands with one 3-d TMA box per stage (1, default) or
 * one 2-d box per 32-wide group (0) */
int bx_set_sgemm_mn3d(int on);
/* SGEMM accuracy mode: 0 (default) TF32 inputs; 1 = 3xTF32 (hi*hi + hi*lo + lo*hi of a
 * TF32 hi/lo split of each operand): ~fp32 accuracy at a third of the tensor rate */
int bx_set_sgemm_precise(int on);
/* diagnostic: SGEMM ablation bits 0-7 (1 = skip TMA loads after the first ring fill, 2 =
 * skip the MMAs, 8 = skip the C stores; results are garbage while set — timing experiments
 * only) and, in bits 8-15, the raster group (m-tiles) of the 2-SM kernels (0 = default 4) */
int bx_set_sgemm_debug(int bits);
int bx_sgemm_device(int dev, int stream, int ta, int tb, int m, int n, int k, float alpha,
                    uint64_t a, int lda, uint64_t b, int ldb, float beta, uint64_t c, int ldc);
/* register-only DMMA loop: measured FP64 tensor peak for the roofline denominator */
int bx_fp64_peak_probe(int dev, int iters, double* tflops);

int bx_last_error(char* buf, int len);

/* ---- one process per GPU (spmd.py) ---------------------------------------------------
 * The reference drives every device from one process (scheduler.py:597-663); on B200 the
 * host side runs one process per GPU, so the L2 tile cache reaches peer arenas through
 * CUDA IPC, tile arrival is signalled through device-written flags in node-shared pinned
 * host memory (stream memory operations: a peer's copy waits on the flag on the GPU, no
 * host round trip), and the shared scheduler state uses host atomics. */
/* IPC handle (64 bytes) of this slot's arena, and the arena size */
int bx_ipc_arena_handle(int dev, void* handle64, uint64_t* arena_bytes);
/* open a peer process's arena in this slot's context; *base = its device address */
int bx_ipc_open(int dev, const void* handle64, uint64_t* base);
int bx_ipc_close(int dev, uint64_t base);
/* page-lock + map host memory (flags); *dev_ptr = the address kernels / stream ops use */
int bx_host_register_mapped(void* ptr, uint64_t bytes, uint64_t* dev_ptr);
/* copy_from_peer across processes (replaces cache.py:312-322 for a remote holder): on the
 * P2P lane, optionally wait until the 32-bit flag at flag_dptr >= flag_min, then copy
 * `bytes` from the device address src_ptr (an IPC-opened peer arena) into this arena */
int bx_copy_remote(int dst_dev, uint64_t dst_off, uint64_t src_ptr, uint64_t bytes, uint64_t flag_dptr,
                   uint32_t flag_min, int n_wait, const int* wait, int* ev_out);
/* on `lane`, after the waits, write `value` to the flag at flag_dptr (arrival signal) */
int bx_write_flag(int dev, int lane, uint64_t flag_dptr, uint32_t value, int n_wait, const int* wait);
/* host atomics on node-shared memory (64-bit, sequentially consistent) */
int bx_atomic_add(int64_t* p, int64_t v, int64_t* old);
int bx_atomic_cas(int64_t* p, int64_t expected, int64_t desired, int64_t* old);

/* ---- resident issue engine (one routine call; replaces the per-tile translate/fetch of
 * scheduler.py:426-461 + cache.py:97-113 and the per-launch kernel dispatch of
 * routines.py:456-479 for resident arenas, in one C call per launch) ----
 * tiles: ntiles rows of 6 int64 {host address, host ld (elements), h, w, element bytes,
 * device ld}; each GPU d (engine slot slots[d], peer group groups[d]) places tiles in its
 * arena region [region_off[d], +region_bytes[d]).  A missing tile is copied from the
 * lowest-id GPU of the same group that holds it (l2 != 0; the copy waits on the holder's
 * arrival event) or from the host; copies of one call share one arrival event per lane. */
int bx_ic_create(int ndev, const int* slots, const int* groups, int ntiles, const int64_t* tiles,
                 const uint64_t* region_off, const uint64_t* region_bytes, int l2, int* id);
/* releases the call's arrival events (the caller drains its GPUs first) */
int bx_ic_destroy(int id);
/* the tile table, valid until bx_ic_destroy: off[d*ntiles+t] (-1 = absent), ev[d*ntiles+t]
 * (pending arrival event, -1 = landed), holders[t] (bit d), metrics[d*8+k] (k: H2D bytes,
 * d2d-in bytes, host fetches, L2 hits, d2d-out bytes, tile references served) */
int bx_ic_state(int id, int64_t** off, int32_t** ev, uint32_t** holders, int64_t** metrics);
/* make tiles present on GPU d; their offsets / device lds and the distinct arrival
 * events (<= wait_cap) a consumer must wait on */
int bx_ic_resolve(int id, int d, int n, const int32_t* tids, int64_t* off_out, int32_t* ld_out, int* n_wait,
                  int* wait_out, int wait_cap);
/* bx_gemm_task_packed with tile-id operands: nsteps rows of 4 int32 {a, b, depth, kmode};
 * an id < 0 names raw[2*(-id-1)..] = (arena offset, ld) (scratch tiles) */
int bx_ic_gemm(int id, int d, int stream, int f32, int ta, int tb, int tri, int h, int w, int nsteps,
               const int32_t* steps, const int64_t* raw, int nraw, double alpha, double beta, uint64_t c_off,
               int ldc, int n_wait, const int* wait, int* ev_out);

#ifdef __cplusplus
}
#endif
#endif
