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
/* resident issue engine: the table bookkeeping of the real library (bump allocation,
 * holder masks, one arrival event per lane and batch), no CUDA */
#include <stdlib.h>
typedef struct { int ndev, nt; int64_t *off; int32_t *ev; uint32_t *hold; int64_t *met; uint64_t *cur;
                 int64_t *tiles; uint32_t *stamp; uint32_t epoch; } IcStub;
static IcStub *ics[64];
int bx_ic_create(int ndev, const int *slots, const int *groups, int nt, const int64_t *tiles,
                 const uint64_t *roff, const uint64_t *rb, int l2, int *id) {
    IcStub *c = calloc(1, sizeof(IcStub)); c->ndev = ndev; c->nt = nt;
    c->off = malloc(sizeof(int64_t) * ndev * nt); for (int i = 0; i < ndev * nt; ++i) c->off[i] = -1;
    c->ev = malloc(sizeof(int32_t) * ndev * nt); for (int i = 0; i < ndev * nt; ++i) c->ev[i] = -1;
    c->hold = calloc(nt, 4); c->met = calloc(ndev * 8, 8); c->cur = malloc(8 * ndev);
    c->tiles = malloc(48 * (size_t)nt); memcpy(c->tiles, tiles, 48 * (size_t)nt);
    c->stamp = calloc(nt, 4);
    for (int d = 0; d < ndev; ++d) c->cur[d] = roff[d];
    for (int i = 0; i < 64; ++i) if (!ics[i]) { ics[i] = c; *id = i; return 0; }
    return 7; }
int bx_ic_destroy(int id) { IcStub *c = ics[id]; free(c->off); free(c->ev); free(c->hold); free(c->met);
    free(c->cur); free(c->tiles); free(c->stamp); free(c); ics[id] = 0; return 0; }
int bx_ic_state(int id, int64_t **o, int32_t **e, uint32_t **h, int64_t **m) {
    *o = ics[id]->off; *e = ics[id]->ev; *h = ics[id]->hold; *m = ics[id]->met; return 0; }
static void ic_res(IcStub *c, int d, int n, const int32_t *t) {
    int nh = 0, np = 0; ++c->epoch;
    for (int i = 0; i < n; ++i) {
        int x = t[i]; if (c->stamp[x] == c->epoch) continue; c->stamp[x] = c->epoch;
        size_t idx = (size_t)d * c->nt + x;
        if (c->off[idx] >= 0) continue;
        const int64_t *r = c->tiles + 6 * x; uint64_t b = (uint64_t)r[5] * r[3] * r[4];
        c->off[idx] = (int64_t)((c->cur[d] + 255) & ~255ull); c->cur[d] = c->off[idx] + b;
        int src = -1; for (int e = 0; e < c->ndev; ++e) if (e != d && ((c->hold[x] >> e) & 1)) { src = e; break; }
        if (src >= 0) { c->met[d * 8 + 1] += r[2] * r[3] * r[4]; c->met[d * 8 + 3]++; c->met[src * 8 + 4] += r[2] * r[3] * r[4]; ++np; }
        else { c->met[d * 8] += r[2] * r[3] * r[4]; c->met[d * 8 + 2]++; ++nh; }
        c->hold[x] |= 1u << d;
    }
    if (nh) ev_next++;
    if (np) ev_next++; }
int bx_ic_resolve(int id, int d, int n, const int32_t *t, int64_t *o, int32_t *l, int *nw, int *w, int cap) {
    IcStub *c = ics[id]; ic_res(c, d, n, t);
    for (int i = 0; i < n; ++i) { o[i] = c->off[(size_t)d * c->nt + t[i]]; l[i] = (int)c->tiles[6 * t[i] + 5]; }
    *nw = 0; return 0; }
int bx_ic_gemm(int id, int d, int s, int f, int ta, int tb, int tr, int h, int w, int ns, const int32_t *st,
               const int64_t *raw, int nraw, double al, double be, uint64_t co, int lc, int n, const int *wt, int *ev) {
    int32_t t[8192]; int k = 0; IcStub *c = ics[id];
    for (int i = 0; i < ns; ++i) { if (st[4 * i] >= 0) t[k++] = st[4 * i]; if (st[4 * i + 1] >= 0) t[k++] = st[4 * i + 1]; }
    ic_res(c, d, k, t); launches++; return EV(ev); }
