/*
 * oracle.c -- CPU restatement of the reference reshard path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker.  The product never links it.
 *
 * Parity pin: every function below is checked against the reference itself
 * (oracle/_ref, compiled from /root/reference/proj/src by oracle/Makefile) on
 * the committed golden fixtures in tests/golden/ (tests/test_oracle.py).
 *
 * Restates, with per-tensor element size as the only extension:
 *   tp_block / view / owners          proj/src/topology.cpp:8-47
 *   default_layer_assignment, coords  proj/src/parallel_config.cpp:19-71
 *   validate_config                   proj/src/parallel_config.cpp:73-123
 *   compute_transfer_plan             proj/src/planner.cpp:57-192
 *   layout_identical                  proj/src/planner.cpp:31-42
 *   verify_plan                       proj/src/planner.cpp:194-303
 *   write_plan / read_plan            proj/src/transfer_plan.cpp:73-141
 *   slice_local / scatter_local       proj/src/executor.cpp:23-93
 *   chunk_bounds                      proj/src/executor.cpp:95-126
 *   execute_plan (loopback)           proj/src/executor.cpp:128-220,
 *                                     proj/src/transport.cpp:6-19
 *   splitmix64 / pattern_byte / fill  proj/src/shard_store.cpp:12-85
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>
#include <time.h>

#define MAXD 8

typedef struct { int64_t lo, hi; } iv_t;
typedef struct { int nd; iv_t b[MAXD]; } box_t;

typedef struct {
  char id[128];
  int layer, nd, axis, bpe;       /* axis -1: replicated */
  int dp_axis;                    /* extension: -1, or the distributed-optimizer DP split axis */
  char role[16];                  /* param / m1 / m2: flat buckets are per role */
  int64_t shape[MAXD];
} tspec_t;

typedef struct {
  char name[128];
  int L, bpe, nt;
  tspec_t* t;
} spec_t;

/* C-ABI config record shared with the ctypes side. */
typedef struct {
  uint64_t gen;
  int32_t tp, pp, dp, nranks;
  const int32_t* ranks;
  const int32_t* layer_stage; /* NULL: default ceil split */
  int32_t dist_opt;           /* extension (no reference counterpart): DP-shard dp_axis tensors,
                                 1 dim chunks, 2 Megatron flat buckets */
  int32_t bucket_elems;       /* flat buckets: bucket size in elements (0: max(40M, 1M x dp)) */
} orc_config;

typedef struct {
  uint64_t gen;
  int tp, pp, dp, n, L, dist_opt;
  int64_t bucket;
  int* ranks;
  int* stage;
} cfg_t;

typedef struct { uint32_t ti; int layer, src, dst; box_t bx; int64_t bytes; int64_t seq; } task_t;
typedef struct { uint32_t ti; int layer, rank; box_t bx; int64_t bytes; int64_t seq; } keep_t;

typedef struct {
  uint64_t sg, dg;
  int ntid; char** tids;
  task_t* tasks; int64_t ntask, cap_task;
  keep_t* keeps; int64_t nkeep, cap_keep;
} plan_t;

/* ------------------------------------------------------------------ text */

typedef struct { char* s; size_t n, cap; } sbuf;

static void sb_printf(sbuf* b, const char* fmt, ...) {
  va_list ap;
  for (;;) {
    size_t room = b->cap - b->n;
    va_start(ap, fmt);
    int k = vsnprintf(b->s ? b->s + b->n : NULL, b->s ? room : 0, fmt, ap);
    va_end(ap);
    if (b->s && (size_t)k < room) { b->n += (size_t)k; return; }
    size_t nc = b->cap ? b->cap * 2 : 4096;
    while (nc - b->n <= (size_t)k) nc *= 2;
    b->s = (char*)realloc(b->s, nc);
    b->cap = nc;
  }
}

static char* sb_take(sbuf* b) {
  if (!b->s) { b->s = (char*)malloc(1); b->s[0] = 0; }
  return b->s;
}

static void box_text(sbuf* b, const box_t* x, int brackets) {
  for (int i = 0; i < x->nd; ++i) {
    if (brackets)
      sb_printf(b, "%s[%lld,%lld)", i ? "x" : "", (long long)x->b[i].lo, (long long)x->b[i].hi);
    else
      sb_printf(b, "%s%lld:%lld", i ? "," : "", (long long)x->b[i].lo, (long long)x->b[i].hi);
  }
}

/* -------------------------------------------------------------- parsing */

static int parse_spec(const char* text, spec_t* sp, char* err, size_t errn) {
  memset(sp, 0, sizeof(*sp));
  int cap = 64, have_model = 0;
  sp->t = (tspec_t*)calloc((size_t)cap, sizeof(tspec_t));
  const char* p = text;
  char line[4096];
  while (*p) {
    size_t k = strcspn(p, "\n");
    size_t m = k < sizeof(line) - 1 ? k : sizeof(line) - 1;
    memcpy(line, p, m); line[m] = 0;
    p += k; if (*p == '\n') ++p;
    char* hash = strchr(line, '#'); if (hash) *hash = 0;
    char kind[32] = {0};
    if (sscanf(line, "%31s", kind) != 1) continue;
    if (!strcmp(kind, "model")) {
      if (sscanf(line, "model %127s layers %d bpe %d", sp->name, &sp->L, &sp->bpe) != 3) {
        snprintf(err, errn, "spec parse: bad model line"); return 1;
      }
      have_model = 1;
    } else if (!strcmp(kind, "tensor")) {
      if (sp->nt == cap) { cap *= 2; sp->t = (tspec_t*)realloc(sp->t, (size_t)cap * sizeof(tspec_t)); }
      tspec_t* t = &sp->t[sp->nt];
      memset(t, 0, sizeof(*t));
      char shape[512], axis[16], role[16];
      if (sscanf(line, "tensor %127s %d %511s %15s %15s %d", t->id, &t->layer, shape, axis,
                 role, &t->bpe) != 6) {
        snprintf(err, errn, "spec parse: bad tensor line"); return 1;
      }
      t->axis = (axis[0] == '-') ? -1 : atoi(axis);
      snprintf(t->role, sizeof t->role, "%s", role);
      t->dp_axis = -1;
      {
        const char* dpo = strstr(line, " dp=");  /* optional extension token */
        if (dpo) t->dp_axis = atoi(dpo + 4);
      }
      char* q = shape;
      while (*q && t->nd < MAXD) {
        t->shape[t->nd++] = strtoll(q, &q, 10);
        if (*q == ',') ++q;
      }
      sp->nt++;
    } else {
      snprintf(err, errn, "spec parse: unknown record '%s'", kind); return 1;
    }
  }
  if (!have_model) { snprintf(err, errn, "spec parse: missing model record"); return 1; }
  return 0;
}

static void free_spec(spec_t* sp) { free(sp->t); sp->t = NULL; }

/* default_layer_assignment: parallel_config.cpp:19-29 */
static void load_cfg(const orc_config* c, int L, cfg_t* out) {
  out->gen = c->gen; out->tp = c->tp; out->pp = c->pp; out->dp = c->dp;
  out->n = c->nranks; out->L = L; out->dist_opt = c->dist_opt;
  out->bucket = c->bucket_elems > 0 ? c->bucket_elems : (c->dp * 1000000LL > 40000000LL ? c->dp * 1000000LL : 40000000LL);
  out->ranks = (int*)malloc(sizeof(int) * (size_t)(c->nranks > 0 ? c->nranks : 1));
  for (int i = 0; i < c->nranks; ++i) out->ranks[i] = c->ranks[i];
  out->stage = (int*)malloc(sizeof(int) * (size_t)(L > 0 ? L : 1));
  if (c->layer_stage) {
    for (int l = 0; l < L; ++l) out->stage[l] = c->layer_stage[l];
  } else {
    int base = c->pp > 0 ? L / c->pp : 0, extra = c->pp > 0 ? L % c->pp : 0, layer = 0;
    for (int s = 0; s < c->pp; ++s) {
      int take = base + (s < extra ? 1 : 0);
      for (int k = 0; k < take && layer < L; ++k) out->stage[layer++] = s;
    }
  }
}

static void free_cfg(cfg_t* c) { free(c->ranks); free(c->stage); }

static int cfg_index(const cfg_t* c, int rank) {
  for (int i = 0; i < c->n; ++i) if (c->ranks[i] == rank) return i;
  return -1;
}

/* coord rule: tp = i % tp, dp = (i / tp) % dp, pp = i / (tp*dp)  (parallel_config.cpp:42-49) */
static void coord_of(const cfg_t* c, int idx, int* tp, int* pp, int* dp) {
  *tp = idx % c->tp; *dp = (idx / c->tp) % c->dp; *pp = idx / (c->tp * c->dp);
}

static int rank_at(const cfg_t* c, int tp, int dp, int pp) {
  return c->ranks[tp + c->tp * (dp + c->dp * pp)];
}

/* tp_block: topology.cpp:8-14 */
static int tp_block(int64_t len, int tp, int idx, iv_t* out) {
  int64_t blk = (len + tp - 1) / tp;
  int64_t lo = (int64_t)idx * blk, hi = lo + blk < len ? lo + blk : len;
  if (lo >= hi) return 0;
  out->lo = lo; out->hi = hi;
  return 1;
}

/* Extension (distributed optimizer; no reference counterpart, parity
 * unpinned): ceil chunk idx of parts over [iv.lo, iv.hi). */
static int dp_chunk(iv_t iv, int parts, int idx, iv_t* out) {
  int64_t len = iv.hi - iv.lo, blk = (len + parts - 1) / parts;
  int64_t lo = iv.lo + (int64_t)idx * blk, hi = lo + blk < iv.hi ? lo + blk : iv.hi;
  if (lo >= hi) return 0;
  out->lo = lo; out->hi = hi;
  return 1;
}

static int dp_sharded(const tspec_t* t, const cfg_t* c) { return c->dist_opt && t->dp_axis >= 0; }
static int flat_sharded(const tspec_t* t, const cfg_t* c) { return c->dist_opt == 2 && t->dp_axis >= 0; }

/* view: topology.cpp:16-37 (rank given by its index in the rank list),
 * plus the DP chunk of the TP block for distributed-optimizer tensors */
static int view_coord(const tspec_t* t, const cfg_t* c, int tp, int dp, box_t* out) {
  out->nd = t->nd;
  for (int i = 0; i < t->nd; ++i) { out->b[i].lo = 0; out->b[i].hi = t->shape[i]; }
  if (t->axis >= 0) {
    iv_t b;
    if (!tp_block(t->shape[t->axis], c->tp, tp, &b)) return 0;
    out->b[t->axis] = b;
  }
  if (dp_sharded(t, c) && !flat_sharded(t, c)) {
    iv_t ch;
    if (!dp_chunk(out->b[t->dp_axis], c->dp, dp, &ch)) return 0;
    out->b[t->dp_axis] = ch;
  }
  return 1;
}

/* Extension (parity unpinned): Megatron's flat-bucket distributed optimizer
 * (megatron/core/distributed/param_and_grad_buffer.py: parameters laid out
 * in reverse order, each start padded to 64 elements, a bucket closed once it
 * reaches the bucket size and its end padded to lcm(dp, 128);
 * megatron/core/optimizer/distrib_optimizer.py: DP rank d owns the d-th of dp
 * equal parts of each bucket).  One flat buffer per (stage, role, TP index)
 * over the dp_axis tensors, in global buffer positions.  Returns the element
 * range [lo, hi) of tensor ti's TP block held by (tp, dp); empty = 0, 0. */
static int64_t round_up64(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static int64_t tp_local_numel(const tspec_t* t, const cfg_t* c, int tp) {
  int64_t n = 1;
  for (int i = 0; i < t->nd; ++i) {
    if (i == t->axis) {
      iv_t b;
      if (!tp_block(t->shape[i], c->tp, tp, &b)) return 0;
      n *= b.hi - b.lo;
    } else {
      n *= t->shape[i];
    }
  }
  return n;
}

static void flat_range(const spec_t* sp, int ti, const cfg_t* c, int tp, int dp, int64_t* lo, int64_t* hi) {
  const tspec_t* t = &sp->t[ti];
  int st = c->stage[t->layer];
  int64_t a = c->dp, b = 128;
  while (b) { int64_t r = a % b; a = b; b = r; }
  int64_t align = c->dp / a * 128;  /* lcm(dp, 128) */
  int64_t bucket_start = 0, pos = 0, mine = -1, mine_n = 0, mine_bucket = 0, mine_end = -1;
  for (int k = sp->nt - 1; k >= 0; --k) {
    const tspec_t* u = &sp->t[k];
    if (u->dp_axis < 0 || strcmp(u->role, t->role) || c->stage[u->layer] != st) continue;
    int64_t n = tp_local_numel(u, c, tp);
    if (!n) continue;
    pos = round_up64(pos, 64);
    if (k == ti) { mine = pos; mine_n = n; mine_bucket = bucket_start; }
    pos += n;
    if (pos - bucket_start >= c->bucket) {
      int64_t end = round_up64(pos, align);
      if (mine >= 0 && mine_end < 0) mine_end = end;
      bucket_start = pos = end;
    }
  }
  *lo = *hi = 0;
  if (mine < 0) return;
  if (mine_end < 0) mine_end = round_up64(pos, align);
  int64_t part = (mine_end - mine_bucket) / c->dp;
  int64_t r0 = mine_bucket + part * dp, r1 = r0 + part;
  int64_t l = mine > r0 ? mine : r0, h = mine + mine_n < r1 ? mine + mine_n : r1;
  if (l < h) { *lo = l - mine; *hi = h - mine; }
}

/* The boxes of elements [lo, hi) of v's row-major order, recursively: within
 * axis d the range splits into a partial first step, whole steps, and a
 * partial last step; partial steps recurse into axis d + 1 with axis d fixed. */
static int range_boxes_rec(const box_t* v, int d, int64_t lo, int64_t hi, box_t pre, box_t* out, int n) {
  if (lo >= hi) return n;
  int64_t inner = 1;
  for (int i = d + 1; i < v->nd; ++i) inner *= v->b[i].hi - v->b[i].lo;
  int64_t a = lo / inner, b = hi / inner;
  if (a == b) {  /* inside one step of axis d */
    pre.b[d].lo = v->b[d].lo + a; pre.b[d].hi = pre.b[d].lo + 1;
    return range_boxes_rec(v, d + 1, lo - a * inner, hi - a * inner, pre, out, n);
  }
  int64_t full0 = a;
  if (lo % inner) {
    pre.b[d].lo = v->b[d].lo + a; pre.b[d].hi = pre.b[d].lo + 1;
    n = range_boxes_rec(v, d + 1, lo - a * inner, inner, pre, out, n);
    full0 = a + 1;
  }
  if (b > full0) {
    box_t x = pre;
    x.b[d].lo = v->b[d].lo + full0; x.b[d].hi = v->b[d].lo + b;
    for (int i = d + 1; i < v->nd; ++i) x.b[i] = v->b[i];
    out[n++] = x;
  }
  if (hi % inner) {
    pre.b[d].lo = v->b[d].lo + b; pre.b[d].hi = pre.b[d].lo + 1;
    n = range_boxes_rec(v, d + 1, 0, hi - b * inner, pre, out, n);
  }
  return n;
}

static int range_boxes(const box_t* v, int64_t lo, int64_t hi, box_t* out) {
  box_t pre = *v;
  return range_boxes_rec(v, 0, lo, hi, pre, out, 0);
}

/* what (tp, dp) holds of tensor ti: its view, or the boxes of its flat range */
static int held_coord(const spec_t* sp, int ti, const cfg_t* c, int tp, int dp, box_t* out) {
  box_t v;
  if (!view_coord(&sp->t[ti], c, tp, dp, &v)) return 0;
  if (!flat_sharded(&sp->t[ti], c)) { out[0] = v; return 1; }
  int64_t lo, hi;
  flat_range(sp, ti, c, tp, dp, &lo, &hi);
  return range_boxes(&v, lo, hi, out);
}

static int view_at(const tspec_t* t, const cfg_t* c, int idx, box_t* out) {
  int tp, pp, dp;
  coord_of(c, idx, &tp, &pp, &dp);
  if (c->stage[t->layer] != pp) return 0;
  return view_coord(t, c, tp, dp, out);
}

/* validate_config: parallel_config.cpp:73-123 (first violation only is needed) */
static int validate(const cfg_t* c, const spec_t* sp, char* msg, size_t n) {
  if (c->tp < 1 || c->pp < 1 || c->dp < 1) { snprintf(msg, n, "tp/pp/dp degrees must be positive"); return 1; }
  long long prod = (long long)c->tp * c->pp * c->dp;
  if (prod != c->n) { snprintf(msg, n, "tp*pp*dp = %lld != world size %d", prod, c->n); return 1; }
  for (int i = 0; i < c->n; ++i) {
    for (int j = 0; j < i; ++j)
      if (c->ranks[j] == c->ranks[i]) { snprintf(msg, n, "duplicate rank id %d", c->ranks[i]); return 1; }
    if (c->ranks[i] < 0) { snprintf(msg, n, "negative rank id %d", c->ranks[i]); return 1; }
  }
  /* layer_assignment always covers the model's layers here (built from L) */
  int prev = 0;
  int* count = (int*)calloc((size_t)c->pp, sizeof(int));
  for (int l = 0; l < sp->L; ++l) {
    int s = c->stage[l];
    if (s < 0 || s >= c->pp) {
      snprintf(msg, n, "layer %d assigned to stage %d outside [0,%d)", l, s, c->pp);
      free(count); return 1;
    }
    if (s < prev || s > prev + 1) {
      snprintf(msg, n, "layer assignment not contiguous at layer %d", l); free(count); return 1;
    }
    prev = s; count[s]++;
  }
  for (int s = 0; s < c->pp; ++s)
    if (count[s] == 0) { snprintf(msg, n, "pipeline stage %d receives no layers", s); free(count); return 1; }
  free(count);
  for (int i = 0; i < sp->nt; ++i) {
    const tspec_t* t = &sp->t[i];
    if (t->axis >= 0 && t->shape[t->axis] < c->tp) {
      snprintf(msg, n, "tensor %s: sharded axis length %lld < tp %d", t->id,
               (long long)t->shape[t->axis], c->tp);
      return 1;
    }
  }
  return 0;
}

/* ------------------------------------------------------------- planner */

static void push_task(plan_t* p, task_t t) {
  if (p->ntask == p->cap_task) {
    p->cap_task = p->cap_task ? p->cap_task * 2 : 256;
    p->tasks = (task_t*)realloc(p->tasks, (size_t)p->cap_task * sizeof(task_t));
  }
  t.seq = p->ntask;
  p->tasks[p->ntask++] = t;
}

static void push_keep(plan_t* p, keep_t k) {
  if (p->nkeep == p->cap_keep) {
    p->cap_keep = p->cap_keep ? p->cap_keep * 2 : 256;
    p->keeps = (keep_t*)realloc(p->keeps, (size_t)p->cap_keep * sizeof(keep_t));
  }
  k.seq = p->nkeep;
  p->keeps[p->nkeep++] = k;
}

static int cmp_task(const void* a, const void* b) {
  const task_t *x = (const task_t*)a, *y = (const task_t*)b;
  if (x->layer != y->layer) return x->layer < y->layer ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

static int cmp_keep(const void* a, const void* b) {
  const keep_t *x = (const keep_t*)a, *y = (const keep_t*)b;
  if (x->layer != y->layer) return x->layer < y->layer ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

static int64_t box_count(const box_t* b) {
  int64_t n = 1;
  for (int i = 0; i < b->nd; ++i) n *= b->b[i].hi - b->b[i].lo;
  return n;
}

/* layout_identical: planner.cpp:31-42 */
static int layout_identical(const box_t* vo, const box_t* vn, const box_t* r) {
  int64_t so[MAXD], sn[MAXD];
  int nd = r->nd;
  so[nd - 1] = sn[nd - 1] = 1;
  for (int i = nd - 2; i >= 0; --i) {
    so[i] = so[i + 1] * (vo->b[i + 1].hi - vo->b[i + 1].lo);
    sn[i] = sn[i + 1] * (vn->b[i + 1].hi - vn->b[i + 1].lo);
  }
  int64_t oo = 0, on = 0;
  for (int i = 0; i < nd; ++i) {
    oo += (r->b[i].lo - vo->b[i].lo) * so[i];
    on += (r->b[i].lo - vn->b[i].lo) * sn[i];
  }
  if (oo != on) return 0;
  for (int i = 0; i < nd; ++i)
    if (r->b[i].hi - r->b[i].lo > 1 && so[i] != sn[i]) return 0;
  return 1;
}

/* compute_transfer_plan: planner.cpp:57-192 */
static int compute_plan(const spec_t* sp, const cfg_t* co, const cfg_t* cn, int balance,
                        plan_t* plan, int64_t* pairs_out, char* err, size_t errn) {
  memset(plan, 0, sizeof(*plan));
  if (co->gen == cn->gen) { snprintf(err, errn, "compute_transfer_plan: identical generation ids"); return 1; }
  char msg[512];
  if (validate(co, sp, msg, sizeof msg)) { snprintf(err, errn, "compute_transfer_plan: invalid source config: %s", msg); return 1; }
  if (validate(cn, sp, msg, sizeof msg)) { snprintf(err, errn, "compute_transfer_plan: invalid destination config: %s", msg); return 1; }
  plan->sg = co->gen; plan->dg = cn->gen;
  plan->ntid = sp->nt;
  plan->tids = (char**)calloc((size_t)(sp->nt ? sp->nt : 1), sizeof(char*));
  int64_t pairs = 0, cursor = 0;
  for (int ti = 0; ti < sp->nt; ++ti) {
    const tspec_t* t = &sp->t[ti];
    plan->tids[ti] = strdup(t->id);
    int so = co->stage[t->layer], sn = cn->stage[t->layer];
    int sharded = t->axis >= 0, ax = t->axis;
    int64_t alen = sharded ? t->shape[ax] : 0;
    int nblk = 0, btp[4096]; iv_t biv[4096];
    if (sharded) {
      for (int i = 0; i < co->tp; ++i) { iv_t b; if (tp_block(alen, co->tp, i, &b)) { btp[nblk] = i; biv[nblk] = b; ++nblk; } }
    } else { btp[0] = -1; biv[0].lo = 0; biv[0].hi = 1; nblk = 1; }
    if (t->dp_axis >= 0 && (co->dist_opt == 2 || cn->dist_opt == 2)) {
      /* extension: a flat-bucket side (parity unpinned).  Every box the new
         (tp, dp) holds, tiled by every box an old holder holds: all dp
         indices when the old state is DP-sharded, dp 0 otherwise; tensors
         without a TP axis from old TP index 0 (each TP index cuts them
         differently).  Self-held boxes keep in place when block and flat
         offset are unchanged. */
      int osh = co->dist_opt != 0, ntp = t->axis >= 0 ? co->tp : 1;
      static box_t db[2 * MAXD], sb[2 * MAXD];
      for (int dtp = 0; dtp < cn->tp; ++dtp)
        for (int ddp = 0; ddp < cn->dp; ++ddp) {
          int dst = rank_at(cn, dtp, ddp, sn);
          int ndb = held_coord(sp, ti, cn, dtp, ddp, db);
          if (!ndb) continue;
          box_t vdn; view_coord(t, cn, dtp, ddp, &vdn);
          int64_t lon = 0, hin = 0;
          if (flat_sharded(t, cn)) flat_range(sp, ti, cn, dtp, ddp, &lon, &hin);
          int have_old = 0, otp = -1, odp = -1; box_t vdo; int64_t loo = 0, hio = 0;
          int oidx = cfg_index(co, dst);
          if (oidx >= 0) {
            int a, b, c; coord_of(co, oidx, &a, &b, &c);
            if (b == so && view_coord(t, co, a, c, &vdo)) {
              have_old = 1; otp = a; odp = c;
              if (flat_sharded(t, co)) flat_range(sp, ti, co, a, c, &loo, &hio);
            }
          }
          for (int i = 0; i < ndb; ++i)
            for (int stp = 0; stp < ntp; ++stp)
              for (int sdp = 0; sdp < (osh ? co->dp : 1); ++sdp) {
                int nsb = held_coord(sp, ti, co, stp, sdp, sb);
                int src = rank_at(co, stp, sdp, so);
                for (int j = 0; j < nsb; ++j) {
                  ++pairs;
                  box_t r; r.nd = t->nd;
                  int empty = 0;
                  for (int x = 0; x < t->nd; ++x) {
                    r.b[x].lo = db[i].b[x].lo > sb[j].b[x].lo ? db[i].b[x].lo : sb[j].b[x].lo;
                    r.b[x].hi = db[i].b[x].hi < sb[j].b[x].hi ? db[i].b[x].hi : sb[j].b[x].hi;
                    if (r.b[x].lo >= r.b[x].hi) empty = 1;
                  }
                  if (empty) continue;
                  int64_t bytes = box_count(&r) * t->bpe;
                  if (have_old && otp == stp && (!osh || odp == sdp)) {
                    int same = loo == lon && !memcmp(vdo.b, vdn.b, sizeof(iv_t) * (size_t)t->nd) &&
                               layout_identical(&vdo, &vdn, &r);
                    if (same) { keep_t kk = { (uint32_t)ti, t->layer, dst, r, bytes, 0 }; push_keep(plan, kk); }
                    else { task_t tt = { (uint32_t)ti, t->layer, dst, dst, r, bytes, 0 }; push_task(plan, tt); }
                    continue;
                  }
                  task_t tt = { (uint32_t)ti, t->layer, src, dst, r, bytes, 0 };
                  push_task(plan, tt);
                }
              }
        }
      continue;
    }
    /* extension: distributed-optimizer DP chunks (parity unpinned) */
    int dpo = dp_sharded(t, co), dpn = dp_sharded(t, cn), dax = t->dp_axis;
    for (int dtp = 0; dtp < cn->tp; ++dtp) {
      box_t vdt; vdt.nd = t->nd;
      for (int i = 0; i < t->nd; ++i) { vdt.b[i].lo = 0; vdt.b[i].hi = t->shape[i]; }
      if (sharded) { iv_t b; if (!tp_block(alen, cn->tp, dtp, &b)) continue; vdt.b[ax] = b; }
      for (int ddp = 0; ddp < cn->dp; ++ddp) {
        box_t vd = vdt;
        if (dpn) { iv_t ch; if (!dp_chunk(vdt.b[dax], cn->dp, ddp, &ch)) continue; vd.b[dax] = ch; }
        int dst = rank_at(cn, dtp, ddp, sn);
        int have_old = 0, otp = -1, odp = -1; box_t vdo;
        int oidx = cfg_index(co, dst);
        if (oidx >= 0) {
          int a, b, c; coord_of(co, oidx, &a, &b, &c);
          if (b == so) {
            otp = a; odp = c;
            have_old = view_coord(t, co, a, c, &vdo) ? 1 : 2;  /* 2: on the stage, empty view */
          }
        }
        for (int k = 0; k < nblk; ++k) {
          box_t rt = vd;
          if (sharded) {
            iv_t iv = { vd.b[ax].lo > biv[k].lo ? vd.b[ax].lo : biv[k].lo,
                        vd.b[ax].hi < biv[k].hi ? vd.b[ax].hi : biv[k].hi };
            if (iv.lo >= iv.hi) { ++pairs; continue; }
            rt.b[ax] = iv;
          }
          int nsrc_dp = dpo ? co->dp : 1;
          for (int s = 0; s < nsrc_dp; ++s) {
            ++pairs;
            box_t r = rt;
            if (dpo) {
              box_t sv;
              if (!view_coord(t, co, sharded ? btp[k] : 0, s, &sv)) continue;
              iv_t iv = { rt.b[dax].lo > sv.b[dax].lo ? rt.b[dax].lo : sv.b[dax].lo,
                          rt.b[dax].hi < sv.b[dax].hi ? rt.b[dax].hi : sv.b[dax].hi };
              if (iv.lo >= iv.hi) continue;
              r.b[dax] = iv;
            }
            int64_t bytes = box_count(&r) * t->bpe;
            int self = have_old == 1 && (!sharded || otp == btp[k]) && (!dpo || odp == s);
            if (self) {
              if (layout_identical(&vdo, &vd, &r)) {
                keep_t kk = { (uint32_t)ti, t->layer, dst, r, bytes, 0 };
                push_keep(plan, kk);
              } else {
                task_t tt = { (uint32_t)ti, t->layer, dst, dst, r, bytes, 0 };
                push_task(plan, tt);
              }
              continue;
            }
            int sdp = dpo ? s : (balance ? (int)(cursor++ % co->dp) : 0);
            int src;
            if (sharded) src = rank_at(co, btp[k], sdp, so);
            else {
              src = rank_at(co, 0, sdp, so);
              for (int x = 1; x < co->tp; ++x) { int q = rank_at(co, x, sdp, so); if (q < src) src = q; }
            }
            task_t tt = { (uint32_t)ti, t->layer, src, dst, r, bytes, 0 };
            push_task(plan, tt);
          }
        }
      }
    }
  }
  qsort(plan->tasks, (size_t)plan->ntask, sizeof(task_t), cmp_task);
  qsort(plan->keeps, (size_t)plan->nkeep, sizeof(keep_t), cmp_keep);
  if (pairs_out) *pairs_out = pairs;
  return 0;
}

static void free_plan(plan_t* p) {
  for (int i = 0; i < p->ntid; ++i) free(p->tids[i]);
  free(p->tids); free(p->tasks); free(p->keeps);
  memset(p, 0, sizeof(*p));
}

/* write_plan: transfer_plan.cpp:73-89 */
static char* plan_to_text(const plan_t* p) {
  sbuf b = {0};
  sb_printf(&b, "plan src_gen=%llu dst_gen=%llu\n", (unsigned long long)p->sg, (unsigned long long)p->dg);
  for (int64_t i = 0; i < p->ntask; ++i) {
    const task_t* t = &p->tasks[i];
    sb_printf(&b, "task %s %d %d %d ", p->tids[t->ti], t->layer, t->src, t->dst);
    box_text(&b, &t->bx, 0);
    sb_printf(&b, " %lld%s\n", (long long)t->bytes, t->src == t->dst ? " local" : "");
  }
  for (int64_t i = 0; i < p->nkeep; ++i) {
    const keep_t* k = &p->keeps[i];
    sb_printf(&b, "keep %s %d %d ", p->tids[k->ti], k->layer, k->rank);
    box_text(&b, &k->bx, 0);
    sb_printf(&b, " %lld\n", (long long)k->bytes);
  }
  return sb_take(&b);
}

static int parse_bounds(const char* s, box_t* b) {
  b->nd = 0;
  while (*s && b->nd < MAXD) {
    char* e;
    long long lo = strtoll(s, &e, 10);
    if (*e != ':') return 1;
    long long hi = strtoll(e + 1, &e, 10);
    b->b[b->nd].lo = lo; b->b[b->nd].hi = hi; b->nd++;
    if (lo < 0 || lo >= hi) return 2;  /* ShardView ctor rejects */
    s = e;
    if (*s == ',') ++s; else break;
  }
  return 0;
}

/* read_plan: transfer_plan.cpp:91-141 (tensor ids interned in first-appearance order) */
static int plan_from_text(const char* text, plan_t* p, char* err, size_t errn) {
  memset(p, 0, sizeof(*p));
  int cap_tid = 0;
  const char* s = text;
  char line[4096];
  while (*s) {
    size_t k = strcspn(s, "\n");
    size_t m = k < sizeof(line) - 1 ? k : sizeof(line) - 1;
    memcpy(line, s, m); line[m] = 0;
    s += k; if (*s == '\n') ++s;
    if (!line[0]) continue;
    char kind[16] = {0};
    sscanf(line, "%15s", kind);
    if (!strcmp(kind, "plan")) {
      unsigned long long a = 0, b = 0;
      char* q = strstr(line, "src_gen="); if (q) a = strtoull(q + 8, NULL, 10);
      q = strstr(line, "dst_gen="); if (q) b = strtoull(q + 8, NULL, 10);
      p->sg = a; p->dg = b;
      continue;
    }
    char id[256], bounds[1024];
    int layer, src = 0, dst = 0;
    long long bytes;
    int is_task = !strcmp(kind, "task");
    if (!is_task && strcmp(kind, "keep")) { snprintf(err, errn, "plan parse: unknown record '%s'", kind); return 1; }
    int ok = is_task ? sscanf(line, "task %255s %d %d %d %1023s %lld", id, &layer, &src, &dst, bounds, &bytes) == 6
                     : sscanf(line, "keep %255s %d %d %1023s %lld", id, &layer, &src, bounds, &bytes) == 5;
    if (!ok) { snprintf(err, errn, "plan parse: bad %s line '%.900s'", kind, line); return 1; }
    int ti = -1;
    for (int i = 0; i < p->ntid; ++i) if (!strcmp(p->tids[i], id)) { ti = i; break; }
    if (ti < 0) {
      if (p->ntid == cap_tid) { cap_tid = cap_tid ? cap_tid * 2 : 64; p->tids = (char**)realloc(p->tids, sizeof(char*) * (size_t)cap_tid); }
      p->tids[p->ntid] = strdup(id); ti = p->ntid++;
    }
    box_t bx;
    if (parse_bounds(bounds, &bx)) { snprintf(err, errn, "plan parse: bad bounds '%.900s'", bounds); return 1; }
    if (is_task) { task_t t = { (uint32_t)ti, layer, src, dst, bx, bytes, 0 }; push_task(p, t); }
    else { keep_t kk = { (uint32_t)ti, layer, src, bx, bytes, 0 }; push_keep(p, kk); }
  }
  qsort(p->tasks, (size_t)p->ntask, sizeof(task_t), cmp_task);
  qsort(p->keeps, (size_t)p->nkeep, sizeof(keep_t), cmp_keep);
  return 0;
}

/* ------------------------------------------------------------ verify_plan */

static int box_contains(const box_t* outer, const box_t* inner) {
  if (outer->nd != inner->nd) return 0;
  for (int i = 0; i < outer->nd; ++i)
    if (inner->b[i].lo < outer->b[i].lo || inner->b[i].hi > outer->b[i].hi) return 0;
  return 1;
}

typedef struct { sbuf b; int n; } vlist;

static void complain(vlist* v, const char* fmt, ...) {
  if (v->n >= 64) return;
  char tmp[1024];
  va_list ap; va_start(ap, fmt); vsnprintf(tmp, sizeof tmp, fmt, ap); va_end(ap);
  sb_printf(&v->b, "%s\n", tmp);
  v->n++;
}

static int cmp_int(const void* a, const void* b) { int x = *(const int*)a, y = *(const int*)b; return (x > y) - (x < y); }

/* owners in ascending rank order (std::map<int, ShardView>), topology.cpp:39-47 */
static int owners(const tspec_t* t, const cfg_t* c, int* ranks_out, box_t* views_out) {
  int st = c->stage[t->layer], per = c->tp * c->dp, n = 0;
  int idx[4096];
  for (int i = st * per; i < (st + 1) * per; ++i) idx[n++] = i;
  int m = 0;
  int tmp_r[4096];
  for (int k = 0; k < n; ++k) tmp_r[k] = c->ranks[idx[k]];
  qsort(tmp_r, (size_t)n, sizeof(int), cmp_int);
  for (int k = 0; k < n; ++k) {
    box_t v;
    if (view_at(t, c, cfg_index(c, tmp_r[k]), &v)) { ranks_out[m] = tmp_r[k]; views_out[m] = v; ++m; }
  }
  return m;
}

/* the element range of its view a rank holds: [0, count) unless flat */
static void held_range(const spec_t* sp, int ti, const cfg_t* c, int rank, const box_t* v, int64_t* lo, int64_t* hi) {
  *lo = 0; *hi = box_count(v);
  if (!flat_sharded(&sp->t[ti], c)) return;
  int tp, pp, dp;
  coord_of(c, cfg_index(c, rank), &tp, &pp, &dp);
  flat_range(sp, ti, c, tp, dp, lo, hi);
}

/* row-major positions of a region's first and last elements in view v */
static void region_span(const box_t* v, const box_t* r, int64_t* first, int64_t* last) {
  *first = *last = 0;
  for (int i = 0; i < v->nd; ++i) {
    int64_t len = v->b[i].hi - v->b[i].lo;
    *first = *first * len + (r->b[i].lo - v->b[i].lo);
    *last = *last * len + (r->b[i].hi - 1 - v->b[i].lo);
  }
}

static int held_contains(const box_t* v, int64_t lo, int64_t hi, const box_t* r) {
  if (!box_contains(v, r)) return 0;
  int64_t f, l;
  region_span(v, r, &f, &l);
  return f >= lo && l < hi;
}

/* verify_plan: planner.cpp:194-303 (flat-bucket holders: an element range of the view) */
static char* verify(const plan_t* p, const cfg_t* co, const cfg_t* cn, const spec_t* sp) {
  vlist v = {{0}, 0};
  int* p2m = (int*)malloc(sizeof(int) * (size_t)(p->ntid ? p->ntid : 1));
  for (int pi = 0; pi < p->ntid; ++pi) {
    p2m[pi] = -1;
    for (int mi = 0; mi < sp->nt; ++mi) if (!strcmp(sp->t[mi].id, p->tids[pi])) p2m[pi] = mi;
    if (p2m[pi] < 0) complain(&v, "plan references unknown tensor %s", p->tids[pi]);
  }
  static int dr[4096], sr[4096];
  static box_t dv[4096], sv[4096];
  for (int mi = 0; mi < sp->nt; ++mi) {
    const tspec_t* t = &sp->t[mi];
    int nd_ = owners(t, cn, dr, dv);
    int ns_ = owners(t, co, sr, sv);
    for (int d = 0; d < nd_; ++d) {
      const box_t* vd = &dv[d];
      int64_t dlo, dhi;
      held_range(sp, mi, cn, dr[d], vd, &dlo, &dhi);
      if (dlo >= dhi) continue;  /* an empty flat-bucket range */
      int64_t n = box_count(vd), str[MAXD];
      uint8_t* cover = (uint8_t*)calloc((size_t)n, 1);
      str[vd->nd - 1] = 1;
      for (int i = vd->nd - 2; i >= 0; --i) str[i] = str[i + 1] * (vd->b[i + 1].hi - vd->b[i + 1].lo);
      #define MARK(region, what) do {                                                  \
        const box_t* R = (region);                                                     \
        if (!held_contains(vd, dlo, dhi, R)) {                                         \
          complain(&v, "%s for tensor %s rank %d escapes destination view", what, t->id, dr[d]); \
        } else {                                                                       \
          int64_t pt[MAXD];                                                            \
          for (int i = 0; i < R->nd; ++i) pt[i] = R->b[i].lo;                          \
          for (;;) {                                                                   \
            int64_t off = 0;                                                           \
            for (int i = 0; i < R->nd; ++i) off += (pt[i] - vd->b[i].lo) * str[i];     \
            if (cover[off] < 255) cover[off]++;                                        \
            int dd = R->nd - 1;                                                        \
            while (dd >= 0) { if (++pt[dd] < R->b[dd].hi) break; pt[dd] = R->b[dd].lo; --dd; } \
            if (dd < 0) break;                                                         \
          }                                                                            \
        }                                                                              \
      } while (0)
      for (int64_t i = 0; i < p->ntask; ++i) {
        const task_t* tk = &p->tasks[i];
        if (tk->layer != t->layer || tk->dst != dr[d]) continue;
        if (p2m[tk->ti] != mi) continue;
        if (box_count(&tk->bx) <= 0 || tk->bytes <= 0) { complain(&v, "empty task for tensor %s", t->id); continue; }
        int si = -1;
        for (int s = 0; s < ns_; ++s) if (sr[s] == tk->src) si = s;
        int64_t slo = 0, shi = 0;
        if (si >= 0) held_range(sp, mi, co, sr[si], &sv[si], &slo, &shi);
        if (si < 0 || slo >= shi) complain(&v, "task source rank %d owns nothing of tensor %s", tk->src, t->id);
        else if (!held_contains(&sv[si], slo, shi, &tk->bx))
          complain(&v, "task bounds escape source view for tensor %s src %d", t->id, tk->src);
        MARK(&tk->bx, "task");
      }
      for (int64_t i = 0; i < p->nkeep; ++i) {
        const keep_t* kp = &p->keeps[i];
        if (kp->layer != t->layer || kp->rank != dr[d]) continue;
        if (p2m[kp->ti] != mi) continue;
        int si = -1;
        for (int s = 0; s < ns_; ++s) if (sr[s] == kp->rank) si = s;
        int64_t slo = 0, shi = 0;
        if (si >= 0) held_range(sp, mi, co, sr[si], &sv[si], &slo, &shi);
        if (si < 0 || !held_contains(&sv[si], slo, shi, &kp->bx))
          complain(&v, "carryover not resident in old view for tensor %s rank %d", t->id, kp->rank);
        MARK(&kp->bx, "carryover");
      }
      #undef MARK
      int64_t gaps = 0, over = 0;
      for (int64_t i = 0; i < n; ++i) {
        if (i >= dlo && i < dhi && !cover[i]) ++gaps;
        if (cover[i] > 1) ++over;
      }
      if (gaps) complain(&v, "coverage gap: tensor %s rank %d missing %lld elements", t->id, dr[d], (long long)gaps);
      if (over) complain(&v, "coverage overlap: tensor %s rank %d has %lld doubly-covered elements", t->id, dr[d], (long long)over);
      free(cover);
    }
  }
  free(p2m);
  return sb_take(&v.b);
}

/* ----------------------------------------------------- pattern + stores */

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* pattern_byte: shard_store.cpp:51-56 */
uint8_t orc_pattern_byte(uint32_t ti, int64_t element, int64_t b, uint64_t seed) {
  uint64_t h = splitmix64(seed ^ (0x1000003ULL * ti) ^ (uint64_t)element);
  return (uint8_t)(h >> ((b % 8) * 8));
}

typedef struct { int rank; box_t view; uint8_t* bytes; int64_t n; int flat; int64_t flo; } entry_t;
typedef struct { int nt; int* cnt; entry_t** e; int bpe_dummy; } store_t;

static int owners(const tspec_t* t, const cfg_t* c, int* ranks_out, box_t* views_out);

static store_t* store_alloc(const spec_t* sp, const cfg_t* c) {
  store_t* s = (store_t*)calloc(1, sizeof(store_t));
  s->nt = sp->nt;
  s->cnt = (int*)calloc((size_t)(sp->nt ? sp->nt : 1), sizeof(int));
  s->e = (entry_t**)calloc((size_t)(sp->nt ? sp->nt : 1), sizeof(entry_t*));
  static int rk[4096]; static box_t vw[4096];
  for (int ti = 0; ti < sp->nt; ++ti) {
    int m = owners(&sp->t[ti], c, rk, vw);
    s->cnt[ti] = m;
    s->e[ti] = (entry_t*)calloc((size_t)(m ? m : 1), sizeof(entry_t));
    for (int k = 0; k < m; ++k) {
      entry_t* e = &s->e[ti][k];
      e->rank = rk[k]; e->view = vw[k];
      e->n = box_count(&vw[k]) * sp->t[ti].bpe;
      e->flat = 0; e->flo = 0;
      if (flat_sharded(&sp->t[ti], c)) {  /* a flat-bucket shard holds an element range of its view */
        int tp, pp, dp;
        int64_t lo, hi;
        coord_of(c, cfg_index(c, rk[k]), &tp, &pp, &dp);
        flat_range(sp, ti, c, tp, dp, &lo, &hi);
        e->flat = 1; e->flo = lo;
        e->n = (hi - lo) * sp->t[ti].bpe;
      }
      e->bytes = (uint8_t*)calloc((size_t)(e->n ? e->n : 1), 1);
    }
  }
  return s;
}

void orc_store_free(store_t* s) {
  if (!s) return;
  for (int ti = 0; ti < s->nt; ++ti) {
    for (int k = 0; k < s->cnt[ti]; ++k) free(s->e[ti][k].bytes);
    free(s->e[ti]);
  }
  free(s->e); free(s->cnt); free(s);
}

static entry_t* store_at(store_t* s, int rank, uint32_t ti) {
  if ((int)ti >= s->nt) return NULL;
  for (int k = 0; k < s->cnt[ti]; ++k) if (s->e[ti][k].rank == rank) return &s->e[ti][k];
  return NULL;
}

/* fill_pattern: shard_store.cpp:58-85, one hash per element (bytes identical) */
static void store_fill(store_t* s, const spec_t* sp, uint64_t seed) {
  for (int ti = 0; ti < s->nt; ++ti) {
    const tspec_t* t = &sp->t[ti];
    int64_t gs[MAXD];
    gs[t->nd - 1] = 1;
    for (int i = t->nd - 2; i >= 0; --i) gs[i] = gs[i + 1] * t->shape[i + 1];
    for (int k = 0; k < s->cnt[ti]; ++k) {
      entry_t* e = &s->e[ti][k];
      if (e->flat) {  /* element j of the range: decode its coordinates in the view */
        uint8_t* out = e->bytes;
        uint64_t base = seed ^ (0x1000003ULL * (uint32_t)ti);
        for (int64_t j = e->flo; j < e->flo + e->n / t->bpe; ++j) {
          int64_t rem = j, g = 0;
          for (int i = t->nd - 1; i >= 0; --i) {
            int64_t len = e->view.b[i].hi - e->view.b[i].lo;
            g += (e->view.b[i].lo + rem % len) * gs[i];
            rem /= len;
          }
          uint64_t h = splitmix64(base ^ (uint64_t)g);
          for (int b = 0; b < t->bpe; ++b) *out++ = (uint8_t)(h >> ((b % 8) * 8));
        }
        continue;
      }
      int64_t pt[MAXD];
      for (int i = 0; i < t->nd; ++i) pt[i] = e->view.b[i].lo;
      uint8_t* out = e->bytes;
      for (;;) {
        int64_t g = 0;
        for (int i = 0; i < t->nd; ++i) g += pt[i] * gs[i];
        uint64_t base = seed ^ (0x1000003ULL * (uint32_t)ti);
        int64_t rowlen = e->view.b[t->nd - 1].hi - e->view.b[t->nd - 1].lo;
        for (int64_t j = 0; j < rowlen; ++j) {
          uint64_t h = splitmix64(base ^ (uint64_t)(g + j));
          for (int b = 0; b < t->bpe; ++b) *out++ = (uint8_t)(h >> ((b % 8) * 8));
        }
        int dd = t->nd - 2;
        while (dd >= 0) { if (++pt[dd] < e->view.b[dd].hi) break; pt[dd] = e->view.b[dd].lo; --dd; }
        if (dd < 0) break;
      }
    }
  }
}

/* for_each_row + slice_local / scatter_local: executor.cpp:23-93.
 * dir 0: buffer -> payload (slice), dir 1: payload -> buffer (scatter). */
static int move_rows_at(uint8_t* buf, int64_t buflen, const box_t* owner, int flat, int64_t flo,
                        const box_t* region, uint8_t* payload, int64_t paylen, int64_t bpe, int dir, char* err,
                        size_t errn);

static int move_rows(uint8_t* buf, int64_t buflen, const box_t* owner, const box_t* region,
                     uint8_t* payload, int64_t paylen, int64_t bpe, int dir, char* err, size_t errn) {
  return move_rows_at(buf, buflen, owner, 0, 0, region, payload, paylen, bpe, dir, err, errn);
}

static int move_entry(entry_t* e, const box_t* region, uint8_t* payload, int64_t paylen, int64_t bpe, int dir,
                      char* err, size_t errn) {
  return move_rows_at(e->bytes, e->n, &e->view, e->flat, e->flo, region, payload, paylen, bpe, dir, err, errn);
}

/* flat = 1: the buffer holds elements [flo, flo + buflen / bpe) of the
 * owner's row-major order (a flat-bucket shard) */
static int move_rows_at(uint8_t* buf, int64_t buflen, const box_t* owner, int flat, int64_t flo,
                        const box_t* region, uint8_t* payload, int64_t paylen, int64_t bpe, int dir, char* err,
                        size_t errn) {
  const char* who = dir ? "scatter_local" : "slice_local";
  int escapes = !box_contains(owner, region);
  if (!escapes && flat) {  /* first and last region elements inside the held range */
    int64_t first = 0, last = 0;
    for (int i = 0; i < owner->nd; ++i) {
      int64_t len = owner->b[i].hi - owner->b[i].lo;
      first = first * len + (region->b[i].lo - owner->b[i].lo);
      last = last * len + (region->b[i].hi - 1 - owner->b[i].lo);
    }
    escapes = first < flo || last >= flo + buflen / bpe;
  }
  if (escapes) {
    sbuf b = {0};
    sb_printf(&b, "%s: bounds ", who); box_text(&b, region, 1);
    sb_printf(&b, " escape owner view "); box_text(&b, owner, 1);
    snprintf(err, errn, "%s", b.s); free(b.s);
    return 1;
  }
  if (dir && paylen != box_count(region) * bpe) { snprintf(err, errn, "scatter_local: payload length mismatch"); return 1; }
  if (!flat && buflen != box_count(owner) * bpe) { snprintf(err, errn, "%s: buffer size does not match owner view", who); return 1; }
  int nd = owner->nd;
  int64_t st[MAXD];
  st[nd - 1] = 1;
  for (int i = nd - 2; i >= 0; --i) st[i] = st[i + 1] * (owner->b[i + 1].hi - owner->b[i + 1].lo);
  int64_t rowb = (region->b[nd - 1].hi - region->b[nd - 1].lo) * bpe, cur = 0, pt[MAXD];
  for (int i = 0; i < nd; ++i) pt[i] = region->b[i].lo;
  for (;;) {
    int64_t off = 0;
    for (int i = 0; i < nd; ++i) off += (pt[i] - owner->b[i].lo) * st[i];
    off -= flo;
    if (dir) memcpy(buf + off * bpe, payload + cur, (size_t)rowb);
    else memcpy(payload + cur, buf + off * bpe, (size_t)rowb);
    cur += rowb;
    int dd = nd - 2;
    while (dd >= 0) { if (++pt[dd] < region->b[dd].hi) break; pt[dd] = region->b[dd].lo; --dd; }
    if (dd < 0) break;
  }
  return 0;
}

/* chunk_bounds: executor.cpp:95-126 */
typedef struct { box_t* v; int64_t n, cap; } boxes;
static void boxes_push(boxes* b, box_t x) {
  if (b->n == b->cap) { b->cap = b->cap ? b->cap * 2 : 16; b->v = (box_t*)realloc(b->v, sizeof(box_t) * (size_t)b->cap); }
  b->v[b->n++] = x;
}

static int chunk(const box_t* bx, int64_t maxb, int64_t bpe, boxes* out, char* err, size_t errn) {
  int64_t total = box_count(bx) * bpe;
  if (total <= maxb) { boxes_push(out, *bx); return 0; }
  if (bpe > maxb) { snprintf(err, errn, "chunk_bounds: one element exceeds the staging budget"); return 1; }
  int d = 0;
  while (d < bx->nd && bx->b[d].hi - bx->b[d].lo <= 1) ++d;
  if (d == bx->nd) { snprintf(err, errn, "chunk_bounds: single-element region over budget"); return 1; }
  int64_t unit = total / (bx->b[d].hi - bx->b[d].lo);
  int64_t step = maxb / (unit > 1 ? unit : 1);
  if (step < 1) step = 1;
  for (int64_t lo = bx->b[d].lo; lo < bx->b[d].hi; lo += step) {
    box_t piece = *bx;
    piece.b[d].lo = lo;
    piece.b[d].hi = lo + step < bx->b[d].hi ? lo + step : bx->b[d].hi;
    if (box_count(&piece) * bpe <= maxb) boxes_push(out, piece);
    else if (chunk(&piece, maxb, bpe, out, err, errn)) return 1;
  }
  return 0;
}

typedef struct {
  int32_t ok;
  int32_t failed_layer;       /* -1: none */
  int64_t peak_staging_bytes;
  int64_t bytes_moved;
  int64_t local_copy_bytes;
  int32_t layers_processed;
  int32_t pad;
  double seconds;
  char error[512];
} orc_report;

typedef struct { int src, dst; uint32_t ti; box_t bx; uint8_t* data; int64_t n; } frame_t;

static const frame_t* g_frames;
static int cmp_frame(const void* a, const void* b) {
  const frame_t *x = &g_frames[*(const int64_t*)a], *y = &g_frames[*(const int64_t*)b];
  if (x->dst != y->dst) return x->dst < y->dst ? -1 : 1;
  if (x->src != y->src) return x->src < y->src ? -1 : 1;
  int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  return (i > j) - (i < j);
}

static int flush_frames(frame_t* q, const int64_t* order, int64_t lo, int64_t hi, store_t* dst,
                        const spec_t* sp, char* err, size_t errn) {
  for (int64_t k = lo; k < hi; ++k) {
    frame_t* f = &q[order[k]];
    entry_t* de = store_at(dst, f->dst, f->ti);
    if (!de) { snprintf(err, errn, "shard store: no buffer for rank %d tensor %u", f->dst, f->ti); return 1; }
    if (move_entry(de, &f->bx, f->data, f->n, sp->t[f->ti].bpe, 1, err, errn)) return 1;
  }
  return 0;
}

/* execute_plan over a loopback transport: executor.cpp:128-220 */
static void execute(const plan_t* p, const spec_t* sp, store_t* src, store_t* dst,
                    int64_t staging, orc_report* rep) {
  memset(rep, 0, sizeof(*rep));
  rep->failed_layer = -1;
  int64_t it = 0, ik = 0;
  char err[512];
  frame_t* q = NULL; int64_t nq = 0, capq = 0;
  boxes pcs = {0};
  while (it < p->ntask || ik < p->nkeep) {
    int layer = 0x7fffffff;
    if (it < p->ntask) layer = p->tasks[it].layer;
    if (ik < p->nkeep && p->keeps[ik].layer < layer) layer = p->keeps[ik].layer;
    int64_t te = it, ke = ik;
    while (te < p->ntask && p->tasks[te].layer == layer) ++te;
    while (ke < p->nkeep && p->keeps[ke].layer == layer) ++ke;
    int failed = 0;
    for (int64_t k = ik; k < ke && !failed; ++k) {
      const keep_t* kp = &p->keeps[k];
      entry_t* s = store_at(src, kp->rank, kp->ti);
      entry_t* d = s ? store_at(dst, kp->rank, kp->ti) : NULL;
      if (!s || !d) { snprintf(err, sizeof err, "shard store: no buffer for rank %d tensor %u", kp->rank, kp->ti); failed = 1; break; }
      int64_t bpe = sp->t[kp->ti].bpe, n = box_count(&kp->bx) * bpe;
      uint8_t* tmp = (uint8_t*)malloc((size_t)(n ? n : 1));
      failed = move_entry(s, &kp->bx, tmp, n, bpe, 0, err, sizeof err) ||
               move_entry(d, &kp->bx, tmp, n, bpe, 1, err, sizeof err);
      free(tmp);
    }
    for (int64_t k = it; k < te && !failed; ++k) {
      const task_t* tk = &p->tasks[k];
      entry_t* s = store_at(src, tk->src, tk->ti);
      if (!s) { snprintf(err, sizeof err, "shard store: no buffer for rank %d tensor %u", tk->src, tk->ti); failed = 1; break; }
      if (!box_contains(&s->view, &tk->bx)) { snprintf(err, sizeof err, "integrity: task bounds escape source view"); failed = 1; break; }
      int64_t bpe = sp->t[tk->ti].bpe;
      pcs.n = 0;
      if (chunk(&tk->bx, staging, bpe, &pcs, err, sizeof err)) { failed = 1; break; }
      for (int64_t c = 0; c < pcs.n && !failed; ++c) {
        int64_t n = box_count(&pcs.v[c]) * bpe;
        uint8_t* tmp = (uint8_t*)malloc((size_t)(n ? n : 1));
        if (move_entry(s, &pcs.v[c], tmp, n, bpe, 0, err, sizeof err)) { free(tmp); failed = 1; break; }
        if (tk->src == tk->dst) {
          entry_t* d = store_at(dst, tk->dst, tk->ti);
          if (!d) { snprintf(err, sizeof err, "shard store: no buffer for rank %d tensor %u", tk->dst, tk->ti); free(tmp); failed = 1; break; }
          rep->local_copy_bytes += n;
          if (move_entry(d, &pcs.v[c], tmp, n, bpe, 1, err, sizeof err)) failed = 1;
          free(tmp);
        } else {
          if (nq == capq) { capq = capq ? capq * 2 : 64; q = (frame_t*)realloc(q, sizeof(frame_t) * (size_t)capq); }
          frame_t f = { tk->src, tk->dst, tk->ti, pcs.v[c], tmp, n };
          q[nq++] = f;
        }
      }
    }
    /* receivers ascending; per receiver lowest source first, per-link FIFO
       (all sends of a layer precede its receives, so this is a stable sort) */
    if (!failed && nq) {
      int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)nq);
      for (int64_t i = 0; i < nq; ++i) order[i] = i;
      g_frames = q;
      qsort(order, (size_t)nq, sizeof(int64_t), cmp_frame);
      int64_t i = 0;
      while (i < nq && !failed) {
        int d = q[order[i]].dst;
        int64_t j = i, occ = 0, fl = i;  /* staged frames: order[fl, j) */
        for (; j < nq && q[order[j]].dst == d; ++j) {
          int64_t sz = q[order[j]].n;
          if (sz > staging) { snprintf(err, sizeof err, "integrity: chunk larger than staging buffer"); failed = 1; break; }
          if (occ + sz > staging) {
            if (flush_frames(q, order, fl, j, dst, sp, err, sizeof err)) { failed = 1; break; }
            fl = j; occ = 0;
          }
          occ += sz;
          rep->bytes_moved += sz;
          if (occ > rep->peak_staging_bytes) rep->peak_staging_bytes = occ;
        }
        if (!failed && flush_frames(q, order, fl, j, dst, sp, err, sizeof err)) failed = 1;
        i = j;
      }
      free(order);
    }
    for (int64_t i = 0; i < nq; ++i) free(q[i].data);
    nq = 0;
    if (failed) {
      rep->ok = 0;
      snprintf(rep->error, sizeof rep->error, "%s", err);
      rep->failed_layer = layer;
      free(q); free(pcs.v);
      return;
    }
    rep->layers_processed++;
    it = te; ik = ke;
  }
  free(q); free(pcs.v);
  rep->ok = 1;
}

/* ---------------------------------------------------------------- C ABI */

void orc_free(char* p) { free(p); }

static int setup(const char* spec_text, const orc_config* o, const orc_config* n, spec_t* sp,
                 cfg_t* co, cfg_t* cn, char** out) {
  char err[512];
  if (parse_spec(spec_text, sp, err, sizeof err)) { *out = strdup(err); return 1; }
  load_cfg(o, sp->L, co);
  load_cfg(n, sp->L, cn);
  return 0;
}

/* Plan text (write_plan format); returns 0, or 1 with the error in *out. */
int orc_plan_text(const char* spec_text, const orc_config* o, const orc_config* n, int balance,
                  char** out, int64_t* pairs) {
  spec_t sp; cfg_t co, cn; plan_t p;
  if (setup(spec_text, o, n, &sp, &co, &cn, out)) return 1;
  char err[1024];
  int rc = compute_plan(&sp, &co, &cn, balance, &p, pairs, err, sizeof err);
  *out = rc ? strdup(err) : plan_to_text(&p);
  if (!rc) free_plan(&p);
  free_cfg(&co); free_cfg(&cn); free_spec(&sp);
  return rc;
}

/* verify_plan over a plan given as text; *out = newline-joined violations. */
int orc_verify_plan(const char* spec_text, const orc_config* o, const orc_config* n,
                    const char* plan_text, char** out) {
  spec_t sp; cfg_t co, cn; plan_t p;
  if (setup(spec_text, o, n, &sp, &co, &cn, out)) return 1;
  char err[1024];
  if (plan_from_text(plan_text, &p, err, sizeof err)) { *out = strdup(err); free_cfg(&co); free_cfg(&cn); free_spec(&sp); return 1; }
  *out = verify(&p, &co, &cn, &sp);
  free_plan(&p); free_cfg(&co); free_cfg(&cn); free_spec(&sp);
  return 0;
}

/* Allocate a pattern-filled store for a config (seed) -- the analytic
 * gather-reslice oracle when built for C_new. */
store_t* orc_store_pattern(const char* spec_text, const orc_config* c, uint64_t seed, int fill) {
  spec_t sp; char err[256];
  if (parse_spec(spec_text, &sp, err, sizeof err)) return NULL;
  cfg_t cc; load_cfg(c, sp.L, &cc);
  store_t* s = store_alloc(&sp, &cc);
  if (fill) store_fill(s, &sp, seed);
  free_cfg(&cc); free_spec(&sp);
  return s;
}

int orc_store_count(store_t* s, int ti) { return (s && ti < s->nt) ? s->cnt[ti] : 0; }

/* k-th entry of tensor ti in ascending-rank order */
int orc_store_entry(store_t* s, int ti, int k, int* rank, uint8_t** bytes, int64_t* n) {
  if (!s || ti >= s->nt || k >= s->cnt[ti]) return 1;
  entry_t* e = &s->e[ti][k];
  *rank = e->rank; *bytes = e->bytes; *n = e->n;
  return 0;
}

/* execute_plan: fills a source store with the pattern, runs the plan text
 * through the loopback executor, returns the destination store. */
store_t* orc_execute(const char* spec_text, const orc_config* o, const orc_config* n,
                     const char* plan_text, uint64_t seed, int64_t staging, orc_report* rep) {
  spec_t sp; cfg_t co, cn; plan_t p; char* msg = NULL;
  memset(rep, 0, sizeof(*rep));
  rep->failed_layer = -1;
  if (setup(spec_text, o, n, &sp, &co, &cn, &msg)) { snprintf(rep->error, sizeof rep->error, "%s", msg); free(msg); return NULL; }
  char err[512];
  if (plan_from_text(plan_text, &p, err, sizeof err)) {
    snprintf(rep->error, sizeof rep->error, "%s", err);
    free_cfg(&co); free_cfg(&cn); free_spec(&sp); return NULL;
  }
  /* re-index the parsed plan by tensor name (read_plan interns in appearance order) */
  for (int64_t i = 0; i < p.ntask; ++i)
    for (int mi = 0; mi < sp.nt; ++mi) if (!strcmp(sp.t[mi].id, p.tids[p.tasks[i].ti])) { p.tasks[i].ti = (uint32_t)mi; break; }
  for (int64_t i = 0; i < p.nkeep; ++i)
    for (int mi = 0; mi < sp.nt; ++mi) if (!strcmp(sp.t[mi].id, p.tids[p.keeps[i].ti])) { p.keeps[i].ti = (uint32_t)mi; break; }
  store_t* src = store_alloc(&sp, &co);
  store_fill(src, &sp, seed);
  store_t* dst = store_alloc(&sp, &cn);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  execute(&p, &sp, src, dst, staging, rep);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  rep->seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  orc_store_free(src);
  free_plan(&p); free_cfg(&co); free_cfg(&cn); free_spec(&sp);
  return dst;
}

/* chunk_bounds over one box; writes up to cap boxes as lo/hi pairs. */
int orc_chunk_bounds(int nd, const int64_t* lo, const int64_t* hi, int64_t maxb, int64_t bpe,
                     int64_t* out_lo, int64_t* out_hi, int64_t cap, int64_t* count, char** err_out) {
  box_t b; b.nd = nd;
  for (int i = 0; i < nd; ++i) { b.b[i].lo = lo[i]; b.b[i].hi = hi[i]; }
  boxes out = {0};
  char err[256];
  if (chunk(&b, maxb, bpe, &out, err, sizeof err)) { *err_out = strdup(err); free(out.v); return 1; }
  *count = out.n;
  for (int64_t i = 0; i < out.n && i < cap; ++i)
    for (int k = 0; k < nd; ++k) { out_lo[i * nd + k] = out.v[i].b[k].lo; out_hi[i * nd + k] = out.v[i].b[k].hi; }
  free(out.v);
  return 0;
}

/* slice_local on a raw buffer (1 on error, message in *err_out) */
int orc_slice_local(const uint8_t* buf, int64_t buflen, int nd, const int64_t* olo, const int64_t* ohi,
                    const int64_t* rlo, const int64_t* rhi, int64_t bpe, uint8_t* out, char** err_out) {
  box_t o, r; o.nd = r.nd = nd;
  for (int i = 0; i < nd; ++i) { o.b[i].lo = olo[i]; o.b[i].hi = ohi[i]; r.b[i].lo = rlo[i]; r.b[i].hi = rhi[i]; }
  char err[512];
  if (move_rows((uint8_t*)buf, buflen, &o, &r, out, box_count(&r) * bpe, bpe, 0, err, sizeof err)) { *err_out = strdup(err); return 1; }
  return 0;
}
