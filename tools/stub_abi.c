/* TEST/TOOL STUB (never shipped): the libblasx_cuda.so ABI with every call a no-op that
 * completes immediately.  tools/host_cost.py loads it in place of the real library to time
 * the Python runtime + ctypes marshalling per task without a GPU. */
#include <stdint.h>
#include <string.h>
static int ev_next = 0;
static uint64_t launches = 0;
#define EV(p) ((p) ? (*(p) = ev_next++) : 0, 0)
int bx_version(void) { return 1; }
int bx_device_count(int *n) { *n = 8; return 0; }
int bx_device_info(int dev, char *name, int len, int *sms, uint64_t *tot, uint64_t *fr) {
    strncpy(name, "stub", len); *sms = 148; *tot = 180ull << 30; *fr = 170ull << 30; return 0; }
int bx_mem_info(int dev, uint64_t *fr, uint64_t *tot) { *fr = 170ull << 30; *tot = 180ull << 30; return 0; }
int bx_init() { return 0; }
int bx_shutdown() { return 0; }
int bx_arena_base(int d, uint64_t *b) { *b = 0; return 0; }
int bx_peer_enabled(int a, int b, int *e) { *e = 1; return 0; }
int bx_host_register() { return 0; }
int bx_host_unregister() { return 0; }
int bx_host_is_registered(const void *p, int *yes) { *yes = 1; return 0; }
int bx_h2d_tile(int d, uint64_t o, int ld, const void *s, int64_t sl, int h, int w, int e, int n, const int *wt, int *ev) { return EV(ev); }
int bx_d2h_tile(int d, uint64_t o, int ld, void *s, int64_t sl, int h, int w, int e, int n, const int *wt, int *ev) { return EV(ev); }
int bx_p2p_tile(int d, uint64_t o, int s, uint64_t so, uint64_t b, int n, const int *wt, int *ev) { return EV(ev); }
int bx_gemm_task(int d, int s, int ta, int tb, int tri, int h, int w, int ns, const uint64_t *a, const int *la,
                 const uint64_t *b, const int *lb, const int *dp, double al, double be, uint64_t c, int lc,
                 int n, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_sgemm_task(int d, int s, int ta, int tb, int h, int w, int ns, const uint64_t *a, const int *la,
                  const uint64_t *b, const int *lb, const int *dp, double al, double be, uint64_t c, int lc,
                  int n, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_gemm_task_packed(int d, int s, int f, int ta, int tb, int tr, int h, int w, int ns, const int64_t *st,
                        double al, double be, uint64_t c, int lc, int n, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_trsm_tile(int d, int s, int r, int u, int t, int un, int h, int w, double al, uint64_t a, int la,
                 uint64_t b, int lb, int n, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_copy_batch(int d, int n, const int64_t *ops, int nw, const int *wt, int *eh, int *ep) {
  *eh = -1; *ep = -1; for (int i = 0; i < n; ++i) { if ((ops[8*i] & 0xff) == 0) EV(eh); else EV(ep); } return 0; }
int bx_trsm_inverse(int d, int s, int u, int t, int un, int n, uint64_t a, int la, uint64_t o, int lo,
                    int nw, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_trsm_apply(int d, int s, int r, int eu, int h, int w, double al, uint64_t i, int li, uint64_t b, int lb,
                  uint64_t x, int lx, int nw, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_materialize(int d, int s, int m, int u, int t, int un, int n, uint64_t a, int la, uint64_t o, int lo,
                   int nw, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_axpy_tile(int d, int s, int e, int h, int w, double be, uint64_t a, int la, uint64_t o, int lo,
                 int nw, const int *wt, int *ev) { launches++; return EV(ev); }
int bx_singular_flag(int d, int r, int *f) { *f = 0; return 0; }
int bx_event_record(int d, int s, int t, int *ev) { return EV(ev); }
int bx_event_query(int ev) { return 0; }
int bx_event_sync() { return 0; }
int bx_event_wait_any(int n, const int *evs, int *idx, int spin) { *idx = 0; return 0; }
int bx_event_elapsed(int a, int b, float *ms) { *ms = 1.0f; return 0; }
int bx_event_release() { return 0; }
int bx_event_release_many() { return 0; }
int bx_stream_wait() { return 0; }
int bx_device_sync() { return 0; }
int bx_launch_count(uint64_t *n) { *n = launches; return 0; }
int bx_dev_alloc(int d, uint64_t b, uint64_t *p) { *p = 0; return 0; }
int bx_dev_free() { return 0; }
int bx_dev_fill_uniform() { return 0; }
int bx_dev_fill_uniform_f32() { return 0; }
int bx_dev_copy_h2d() { return 0; }
int bx_dev_copy_d2h() { return 0; }
int bx_dgemm_device() { return 0; }
int bx_set_gemm_variant() { return 0; }
int bx_set_trsm_leaf() { return 0; }
int bx_set_trsm_rhs() { return 0; }
int bx_set_sgemm_debug() { return 0; }
int bx_set_sgemm_mn3d() { return 0; }
int bx_set_sgemm_precise() { return 0; }
int bx_set_gemm_group() { return 0; }
int bx_set_sgemm_variant() { return 0; }
int bx_sgemm_device() { return 0; }
int bx_fp64_peak_probe(int d, int it, double *tf) { *tf = 37.0; return 0; }
int bx_last_error(char *buf, int len) { if (len) buf[0] = 0; return 0; }
/* one process per GPU (spmd.py) */
int bx_ipc_arena_handle(int d, void *h, uint64_t *b) { *b = 0; return 0; }
int bx_ipc_open(int d, const void *h, uint64_t *b) { *b = 0; return 0; }
int bx_ipc_close(int d, uint64_t b) { return 0; }
int bx_host_register_mapped(void *p, uint64_t n, uint64_t *dp) { *dp = (uint64_t)p; return 0; }
int bx_copy_remote(int d, uint64_t o, uint64_t s, uint64_t n, uint64_t f, uint32_t m, int nw, const int *w,
                   int *ev) { return EV(ev); }
int bx_write_flag(int d, int l, uint64_t f, uint32_t v, int nw, const int *w) { return 0; }
int bx_atomic_add(int64_t *p, int64_t v, int64_t *old) { *old = __atomic_fetch_add(p, v, __ATOMIC_SEQ_CST); return 0; }
int bx_atomic_cas(int64_t *p, int64_t e, int64_t d, int64_t *old) {
  int64_t x = e; __atomic_compare_exchange_n(p, &x, d, 0, __ATOMIC_SEQ_CST, __ATOMIC_SEQ_CST); *old = x; return 0; }
