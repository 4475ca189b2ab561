/*
 * dsd_oracle.c — TEST INFRASTRUCTURE ONLY (see dsd_oracle.h).
 *
 * A plain-C restatement of the reference's single-replica engine, written in
 * the reference's own shape (one (time, seq) heap holding every event
 * including arrivals, array-backed FIFO work queues, per-request state
 * structs) so it shares no structure with the GPU engine it checks.
 * Each function names the reference code it follows (paths relative to
 * /root/reference/proj).
 */
#define _GNU_SOURCE
#include "dsd_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------------ */
/* RNG: src/sim/rng.cpp:11-77, include/specsim/util/fnv.hpp:10-18           */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint64_t s[4];
} rng_t;

static uint64_t fnv1a(const char* p) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *p; ++p) {
        h ^= (unsigned char)*p;
        h *= 0x100000001b3ULL;
    }
    return h;
}

static uint64_t splitmix(uint64_t* st) {
    uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static void rng_init(rng_t* r, uint64_t seed, const char* label) {
    uint64_t st = seed ^ fnv1a(label);
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix(&st);
    if ((r->s[0] | r->s[1] | r->s[2] | r->s[3]) == 0) r->s[0] = 1;
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_next(rng_t* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

static double rng_unit(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static uint64_t rng_below(rng_t* r, uint64_t n) {
    if (n <= 1) return 0;
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        uint64_t v = rng_next(r);
        if (v >= threshold) return v % n;
    }
}

static double rng_exponential(rng_t* r, double mean) { return -mean * log(1.0 - rng_unit(r)); }

static double rng_lognormal(rng_t* r, double mu, double sigma) {
    double u1 = 1.0 - rng_unit(r);
    double u2 = rng_unit(r);
    double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
    return exp(mu + sigma * z);
}

static int64_t ms_to_us(double ms) { return (int64_t)llround(ms * 1000.0); }

/* ------------------------------------------------------------------------ */
/* state                                                                    */
/* ------------------------------------------------------------------------ */
enum { EV_ARRIVAL, EV_BATCH_READY, EV_COMPUTE_DONE, EV_NET_ARRIVE, EV_ITER_START };
enum { OP_PREFILL, OP_DECODE, OP_VERIFY };
enum { MSG_PROMPT, MSG_PROPOSAL, MSG_RESULT };
enum { PH_ARRIVED, PH_ROUTED, PH_QUEUED, PH_SPEC, PH_TO_TARGET, PH_VERIFYING, PH_TO_DRAFT, PH_DONE };
#define DRAFT_FLAG (1ULL << 32)

typedef struct {
    int64_t time;
    uint64_t seq;
    int kind;
    uint64_t a, b;
} event_t;

typedef struct {
    int op;
    int64_t req;
    int tokens;
    int64_t context;
    int64_t enq;
    int via;
} item_t;

typedef struct {
    int is_draft, id, grid_pre, grid_dec;
    item_t* q;
    int64_t qn, qcap;
    item_t* run;
    int64_t rn, rcap;
    int busy;
    int64_t busy_us;
    int armed;
    uint64_t gen;
    int64_t* sess; /* session FIFO (ring) */
    int64_t s_head, s_n, s_cap;
    int64_t active;
} server_t;

typedef struct {
    int64_t prompt, output, arrival_tr, drafter;
    const uint8_t* bits;
    int64_t nbits;
    int phase, draft_id, target_id;
    int64_t tokens_done;
    uint64_t cursor;
    int64_t arrival, first, completion;
    int dpd, tpd, fused, pending_gamma, lcr;
    int64_t out_d, back_d, prop, acc;
    int32_t* gseq;
    int32_t* cseq;
    int64_t ng, nc, scap;
} req_t;

typedef struct {
    int acc_ex[20], acc_ac[20], acc_n, acc_pos;
    double rtt[20];
    int rtt_n, rtt_pos, gamma_prev, dyn_gamma;
    int sm_init, sm_low, sm_fused;
    double sm_ema;
} pair_t;

typedef struct {
    double tpot[50];
    int tpot_n, tpot_pos, open;
} tstat_t;

typedef struct {
    const dsd_scenario* S;
    int T, D, fused_everything;
    int64_t N;
    rng_t routing, jitter;
    uint64_t rr;
    event_t* heap;
    int64_t hn, hcap;
    uint64_t next_seq, processed;
    int64_t now;
    server_t* tg;
    server_t* dr;
    req_t* rq;
    pair_t* pairs;
    tstat_t* ts;
    int64_t first_arrival, last_completion, net_total, net_count, completed;
    uint8_t* gen_bits; /* synthetic acceptance bits (owned) */
    int failed;
    char err[256];
} sim_t;

static void* xrealloc(void* p, size_t n) {
    void* q = realloc(p, n ? n : 1);
    if (!q) abort();
    return q;
}

/* ------------------------------------------------------------------------ */
/* SimKernel (src/sim/event_queue.cpp:20-42): binary heap on (time, seq)    */
/* ------------------------------------------------------------------------ */
static int ev_later(const event_t* x, const event_t* y) {
    if (x->time != y->time) return x->time > y->time;
    return x->seq > y->seq;
}

static void schedule(sim_t* m, int64_t t, int kind, uint64_t a, uint64_t b) {
    if (m->hn == m->hcap) {
        m->hcap = m->hcap ? 2 * m->hcap : 64;
        m->heap = xrealloc(m->heap, sizeof(event_t) * m->hcap);
    }
    event_t e = {t, m->next_seq++, kind, a, b};
    int64_t i = m->hn++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!ev_later(&m->heap[p], &e)) break;
        m->heap[i] = m->heap[p];
        i = p;
    }
    m->heap[i] = e;
}

static event_t pop(sim_t* m) {
    event_t top = m->heap[0];
    event_t last = m->heap[--m->hn];
    int64_t i = 0;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= m->hn) break;
        if (c + 1 < m->hn && ev_later(&m->heap[c], &m->heap[c + 1])) ++c;
        if (!ev_later(&last, &m->heap[c])) break;
        m->heap[i] = m->heap[c];
        i = c;
    }
    if (m->hn > 0) m->heap[i] = last;
    return top;
}

/* ------------------------------------------------------------------------ */
/* network, acceptance (src/engine/engine.cpp:10-32)                        */
/* ------------------------------------------------------------------------ */
static const dsd_link* link_of(sim_t* m, int d, int t) {
    const dsd_scenario* S = m->S;
    return &S->links[S->draft_group[d] * S->n_target_groups + S->target_group[t]];
}

static int64_t net_delay(sim_t* m, int d, int t) {
    const dsd_link* l = link_of(m, d, t);
    double lo = -l->jitter_ms / 2.0, hi = l->jitter_ms / 2.0;
    double j = lo + (hi - lo) * rng_unit(&m->jitter);
    double ms = l->rtt_ms / 2.0 + j;
    if (ms < 0.0) ms = 0.0;
    return ms_to_us(ms);
}

static void consume_acceptance(req_t* r, int gamma, int* accepted, int* consumed) {
    *accepted = 0;
    *consumed = 0;
    while (*consumed < gamma) {
        uint8_t bit = r->bits[r->cursor % (uint64_t)r->nbits];
        ++r->cursor;
        ++*consumed;
        if (bit) ++*accepted;
        else break;
    }
}

/* ------------------------------------------------------------------------ */
/* latency profile (src/latency/profile.cpp:20-27,57-88,129-151)            */
/* ------------------------------------------------------------------------ */
static size_t seg_index(const double* axis, size_t n, double q) {
    if (n == 1) return 0;
    size_t hi = 0;
    while (hi < n && !(q < axis[hi])) ++hi; /* upper_bound */
    if (hi == 0) return 0;
    if (hi >= n) return n - 2;
    return hi - 1;
}

static double interpolate(const dsd_grid* g, double batch, double context) {
    double b = batch, c = context;
    if (b < g->batch_axis[0]) b = g->batch_axis[0];
    else if (b > g->batch_axis[g->n_batch - 1]) b = g->batch_axis[g->n_batch - 1];
    if (c < g->context_axis[0]) c = g->context_axis[0];
    else if (c > g->context_axis[g->n_context - 1]) c = g->context_axis[g->n_context - 1];
    size_t bi = seg_index(g->batch_axis, (size_t)g->n_batch, b);
    size_t ci = seg_index(g->context_axis, (size_t)g->n_context, c);
    size_t bj = bi + 1 < (size_t)g->n_batch - 1 ? bi + 1 : (size_t)g->n_batch - 1;
    size_t cj = ci + 1 < (size_t)g->n_context - 1 ? ci + 1 : (size_t)g->n_context - 1;
    double tb = bj == bi ? 0.0 : (b - g->batch_axis[bi]) / (g->batch_axis[bj] - g->batch_axis[bi]);
    double tc = cj == ci ? 0.0 : (c - g->context_axis[ci]) / (g->context_axis[cj] - g->context_axis[ci]);
    size_t n = (size_t)g->n_context;
    const double* v = g->values_ms;
    double r = (1.0 - tb) * (1.0 - tc) * v[bi * n + ci] + (1.0 - tb) * tc * v[bi * n + cj] +
               tb * (1.0 - tc) * v[bj * n + ci] + tb * tc * v[bj * n + cj];
    return r * g->calibration;
}

static double predict(sim_t* m, server_t* s, int op, int batch, int tokens, int64_t context) {
    const dsd_grid* grids = m->S->grids;
    switch (op) {
        case OP_PREFILL: return interpolate(&grids[s->grid_pre], batch, (double)tokens);
        case OP_DECODE: {
            double r = interpolate(&grids[s->grid_dec], batch, (double)context);
            r *= tokens;
            return r;
        }
        default: return interpolate(&grids[s->grid_dec], (double)batch * tokens, (double)context);
    }
}

/* ------------------------------------------------------------------------ */
/* AWC: features.cpp:5-13, mlp.cpp:83-97,163-176, smoother.cpp:8-37,        */
/* matvec in the AVX2 order (kernels_avx2.cpp:17-40)                        */
/* ------------------------------------------------------------------------ */
static void matvec4(const double* w, const double* x, const double* b, double* y, int rows, int cols) {
    int tail = cols & ~3;
    for (int r = 0; r < rows; ++r) {
        const double* row = w + (size_t)r * cols;
        double l[4] = {0, 0, 0, 0};
        int c = 0;
        for (; c < tail; c += 4)
            for (int k = 0; k < 4; ++k) l[k] = l[k] + row[c + k] * x[c + k];
        double s = (l[0] + l[2]) + (l[1] + l[3]);
        for (; c < cols; ++c) s += row[c] * x[c];
        y[r] = b[r] + s;
    }
}

static double awc_forward(const dsd_awc_model* M, const double raw[5]) {
    double x[5];
    for (int f = 0; f < 5; ++f) {
        double v = M->log_scale[f] ? log1p(raw[f]) : raw[f];
        double span = M->norm_hi[f] - M->norm_lo[f];
        x[f] = span > 0.0 ? (v - M->norm_lo[f]) / span : 0.0;
    }
    int H = M->hidden, I = M->input;
    double* h = malloc(sizeof(double) * H);
    double* u = malloc(sizeof(double) * H);
    double* s = malloc(sizeof(double) * H);
    const double* p = M->params;
    matvec4(p, x, p + (size_t)H * I, h, H, I);
    p += (size_t)H * I + H;
    for (int blk = 0; blk < M->blocks; ++blk) {
        const double* w1 = p;
        const double* b1 = w1 + (size_t)H * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + (size_t)H * H;
        matvec4(w1, h, b1, u, H, H);
        for (int i = 0; i < H; ++i) s[i] = u[i] * (1.0 / (1.0 + exp(-u[i])));
        matvec4(w2, s, b2, u, H, H);
        for (int i = 0; i < H; ++i) h[i] += u[i];
        p = b2 + H;
    }
    double out = p[H];
    for (int i = 0; i < H; ++i) out += p[i] * h[i];
    free(h);
    free(u);
    free(s);
    return out;
}

static double acceptance_recent(const pair_t* p) {
    int64_t ex = 0, ac = 0;
    for (int k = 0; k < p->acc_n; ++k) {
        ex += p->acc_ex[k];
        ac += p->acc_ac[k];
    }
    return ex == 0 ? 0.5 : (double)ac / (double)ex;
}

typedef struct {
    int fused, gamma;
} decision_t;

static decision_t decide_window(sim_t* m, req_t* r) {
    const dsd_scenario* S = m->S;
    decision_t fz = {1, 1};
    if (r->draft_id < 0) return fz;
    pair_t* p = &m->pairs[(size_t)r->draft_id * m->T + r->target_id];
    decision_t d = {0, S->gamma};
    switch (S->window_kind) {
        case DSD_WINDOW_STATIC: return d;
        case DSD_WINDOW_DYNAMIC: { /* policies.cpp:60-68 */
            double a = acceptance_recent(p);
            if (a > 0.75 && p->dyn_gamma < S->gamma_max) ++p->dyn_gamma;
            else if (a < 0.25 && p->dyn_gamma > S->gamma_min) --p->dyn_gamma;
            d.gamma = p->dyn_gamma;
            return d;
        }
        case DSD_WINDOW_AWC: {
            double f[5];
            double q = (double)m->ts[r->target_id].open / (double)S->queue_capacity;
            f[0] = q < 0.0 ? 0.0 : (q > 1.0 ? 1.0 : q);
            f[1] = acceptance_recent(p);
            if (p->rtt_n == 0) {
                f[2] = link_of(m, r->draft_id, r->target_id)->rtt_ms;
            } else {
                double sum = 0.0;
                for (int k = 0; k < p->rtt_n; ++k) sum += p->rtt[k];
                f[2] = sum / (double)p->rtt_n;
            }
            tstat_t* t = &m->ts[r->target_id];
            if (t->tpot_n == 0) {
                f[3] = 0.0;
            } else {
                double sum = 0.0;
                for (int k = 0; k < t->tpot_n; ++k) sum += t->tpot[k];
                f[3] = sum / (double)t->tpot_n;
            }
            f[4] = (double)p->gamma_prev;
            double raw = awc_forward(S->awc, f);
            double gmin = (double)S->gamma_min, gmax = (double)S->gamma_max;
            double cl = raw < gmin ? gmin : (gmax < raw ? gmax : raw);
            if (!p->sm_init) {
                p->sm_ema = cl;
                p->sm_init = 1;
            } else {
                p->sm_ema = 0.4 * cl + (1.0 - 0.4) * p->sm_ema;
            }
            if (!p->sm_fused) {
                if (p->sm_ema <= 1.5) ++p->sm_low;
                else p->sm_low = 0;
                if (p->sm_low >= 2) p->sm_fused = 1;
            } else if (p->sm_ema > 1.5) {
                p->sm_fused = 0;
                p->sm_low = 0;
            }
            int g = (int)floor(p->sm_ema + 0.5);
            if (g < (int)gmin) g = (int)gmin;
            if (g > (int)gmax) g = (int)gmax;
            if (p->sm_fused && g <= 1) return fz;
            d.gamma = g > 1 ? g : 1;
            return d;
        }
        default: return fz;
    }
}

/* ------------------------------------------------------------------------ */
/* engine (src/engine/engine.cpp:289-669)                                   */
/* ------------------------------------------------------------------------ */
static void try_dispatch(sim_t* m, server_t* s, int expired);

static void push_gamma(req_t* r, int g) {
    if (r->ng < r->scap) r->gseq[r->ng] = g;
    ++r->ng;
}

static void push_commit(req_t* r, int c) {
    if (r->nc < r->scap) r->cseq[r->nc] = c;
    ++r->nc;
}

static void push_work(sim_t* m, server_t* s, item_t it) {
    if (s->qn == s->qcap) {
        s->qcap = s->qcap ? 2 * s->qcap : 8;
        s->q = xrealloc(s->q, sizeof(item_t) * s->qcap);
    }
    s->q[s->qn++] = it;
    try_dispatch(m, s, 0);
}

static uint64_t server_code(const server_t* s) { return s->is_draft ? ((uint64_t)s->id | DRAFT_FLAG) : (uint64_t)s->id; }

static int eligible(sim_t* m, const server_t* s, const item_t* it) {
    if (s->is_draft) return 1;
    if (it->op == OP_PREFILL) return 1;
    return m->rq[it->req].tpd;
}

static void try_dispatch(sim_t* m, server_t* s, int expired) {
    const dsd_scenario* S = m->S;
    if (s->busy || s->qn == 0) return;
    int64_t* cand = malloc(sizeof(int64_t) * s->qn);
    int64_t* wl = malloc(sizeof(int64_t) * s->qn);
    int64_t nc = 0;
    int kind = -1;
    for (int64_t i = 0; i < s->qn; ++i) {
        item_t* it = &s->q[i];
        if (!eligible(m, s, it)) continue;
        if (kind < 0) kind = it->op;
        if (it->op != kind) continue;
        cand[nc] = i;
        wl[nc] = it->op == OP_PREFILL ? it->tokens : m->rq[it->req].output - m->rq[it->req].tokens_done;
        ++nc;
    }
    if (nc == 0) {
        free(cand);
        free(wl);
        return;
    }
    int max_batch = s->is_draft ? S->draft_max_batch : S->max_batch_size;
    if (!s->is_draft && S->batching_window_us > 0 && !expired && nc < max_batch) {
        if (!s->armed) {
            s->armed = 1;
            ++s->gen;
            schedule(m, m->now + S->batching_window_us, EV_BATCH_READY, server_code(s), s->gen);
        }
        free(cand);
        free(wl);
        return;
    }
    s->armed = 0;
    char* take = calloc((size_t)s->qn, 1);
    int64_t picked = 0;
    if (s->is_draft || S->batching == DSD_BATCH_FIFO) { /* batch_fifo, policies.cpp:30-38 */
        for (int64_t k = 0; k < nc && picked < max_batch; ++k, ++picked) take[cand[k]] = 1;
    } else { /* batch_lab, policies.cpp:40-53 */
        double band = S->similarity_fraction * (double)wl[0];
        take[cand[0]] = 1;
        picked = 1;
        for (int64_t k = 1; k < nc; ++k) {
            if (picked >= max_batch) break;
            if (fabs((double)(wl[k] - wl[0])) <= band) {
                take[cand[k]] = 1;
                ++picked;
            }
        }
    }
    if (s->rcap < picked) {
        s->rcap = picked;
        s->run = xrealloc(s->run, sizeof(item_t) * s->rcap);
    }
    s->rn = 0;
    int64_t keep = 0;
    int tokens = 1;
    int64_t context = 0;
    for (int64_t i = 0; i < s->qn; ++i) {
        if (take[i]) {
            item_t it = s->q[i];
            s->run[s->rn++] = it;
            if (it.tokens > tokens) tokens = it.tokens;
            if (it.context > context) context = it.context;
            if (it.via) {
                m->net_total += m->now - it.enq;
                ++m->net_count;
            }
        } else {
            s->q[keep++] = s->q[i];
        }
    }
    s->qn = keep;
    free(take);
    free(cand);
    free(wl);
    int64_t lat = ms_to_us(predict(m, s, kind, (int)s->rn, tokens, context));
    if (lat < 1) lat = 1;
    s->busy = 1;
    s->busy_us += lat;
    schedule(m, m->now + lat, EV_COMPUTE_DONE, server_code(s), 0);
}

static void activate_next_session(sim_t* m, server_t* d) {
    if (d->active >= 0 || d->s_n == 0) return;
    d->active = d->sess[d->s_head];
    d->s_head = (d->s_head + 1) % d->s_cap;
    --d->s_n;
    req_t* r = &m->rq[d->active];
    item_t it = {OP_PREFILL, d->active, (int)r->prompt, 0, m->now, 0};
    push_work(m, d, it);
}

static int route(sim_t* m) {
    switch (m->S->routing) {
        case DSD_ROUTE_RANDOM: return (int)rng_below(&m->routing, (uint64_t)m->T);
        case DSD_ROUTE_ROUND_ROBIN: return (int)(m->rr++ % (uint64_t)m->T);
        default: {
            int best = 0;
            for (int t = 1; t < m->T; ++t)
                if (m->ts[t].open < m->ts[best].open) best = t;
            return best;
        }
    }
}

static void finish_request(sim_t* m, req_t* r) {
    r->completion = m->now;
    if (r->first < 0) r->first = r->completion;
    r->phase = PH_DONE;
    /* MetricsCollector::add_record (metrics.cpp:74-89) */
    tstat_t* t = &m->ts[r->target_id];
    --t->open;
    if (r->output >= 2) {
        double tpot = ((double)(r->completion - r->first) / 1000.0) / (double)(r->output - 1);
        if (t->tpot_n < 50) t->tpot[t->tpot_n++] = tpot;
        else {
            t->tpot[t->tpot_pos] = tpot;
            t->tpot_pos = (t->tpot_pos + 1) % 50;
        }
    }
    if (r->completion > m->last_completion) m->last_completion = r->completion;
    ++m->completed;
    if (r->draft_id >= 0) {
        server_t* d = &m->dr[r->draft_id];
        if (d->active == (int64_t)(r - m->rq)) {
            d->active = -1;
            activate_next_session(m, d);
        }
    }
}

static void commit_tokens(sim_t* m, req_t* r, int raw) {
    int64_t remaining = r->output - r->tokens_done;
    int c = (int)((int64_t)raw < remaining ? (int64_t)raw : remaining);
    r->tokens_done += c;
    push_commit(r, c);
    if (r->first < 0) r->first = m->now;
    if (r->tokens_done >= r->output) finish_request(m, r);
}

static void begin_iteration(sim_t* m, req_t* r, decision_t d) {
    if (r->phase == PH_DONE) return;
    int64_t id = r - m->rq;
    if (r->draft_id >= 0 && r->target_id >= 0)
        m->pairs[(size_t)r->draft_id * m->T + r->target_id].gamma_prev = d.fused ? 1 : d.gamma;
    item_t it = {OP_DECODE, id, 1, r->prompt + r->tokens_done, m->now, 0};
    if (d.fused) {
        r->fused = 1;
        push_gamma(r, 0);
        push_work(m, &m->tg[r->target_id], it);
    } else {
        r->fused = 0;
        push_gamma(r, d.gamma);
        r->pending_gamma = d.gamma;
        r->phase = PH_SPEC;
        it.tokens = d.gamma;
        push_work(m, &m->dr[r->draft_id], it);
    }
}

static void on_arrival(sim_t* m, int64_t i) {
    req_t* r = &m->rq[i];
    r->arrival = m->now;
    r->phase = PH_ROUTED;
    if (m->D > 0) r->draft_id = (int)r->drafter;
    r->target_id = route(m);
    ++m->ts[r->target_id].open;
    if (m->first_arrival < 0 || r->arrival < m->first_arrival) m->first_arrival = r->arrival;
    r->phase = PH_QUEUED;
    if (m->fused_everything) {
        r->fused = 1;
        item_t it = {OP_PREFILL, i, (int)r->prompt, 0, m->now, 0};
        push_work(m, &m->tg[r->target_id], it);
    } else {
        server_t* d = &m->dr[r->draft_id];
        if (d->s_n == d->s_cap) { /* grow the ring, keeping FIFO order */
            int64_t nc = d->s_cap ? 2 * d->s_cap : 8;
            int64_t* ns = malloc(sizeof(int64_t) * nc);
            for (int64_t k = 0; k < d->s_n; ++k) ns[k] = d->sess[(d->s_head + k) % d->s_cap];
            free(d->sess);
            d->sess = ns;
            d->s_cap = nc;
            d->s_head = 0;
        }
        d->sess[(d->s_head + d->s_n) % d->s_cap] = i;
        ++d->s_n;
        activate_next_session(m, d);
        int64_t delay = net_delay(m, r->draft_id, r->target_id);
        schedule(m, m->now + delay, EV_NET_ARRIVE, (uint64_t)i, MSG_PROMPT);
    }
}

static void on_target_item_done(sim_t* m, req_t* r, const item_t* it) {
    int64_t id = r - m->rq;
    if (it->op == OP_PREFILL) {
        r->tpd = 1;
        if (r->output == 0) {
            if (r->phase != PH_DONE) finish_request(m, r);
            return;
        }
        if (r->fused && m->fused_everything) begin_iteration(m, r, (decision_t){1, 1});
    } else if (it->op == OP_VERIFY) {
        int acc, cons;
        consume_acceptance(r, it->tokens, &acc, &cons);
        r->lcr = acc + 1;
        r->prop += cons;
        r->acc += acc;
        pair_t* p = &m->pairs[(size_t)r->draft_id * m->T + r->target_id];
        if (p->acc_n < 20) {
            p->acc_ex[p->acc_n] = cons;
            p->acc_ac[p->acc_n] = acc;
            ++p->acc_n;
        } else {
            p->acc_ex[p->acc_pos] = cons;
            p->acc_ac[p->acc_pos] = acc;
            p->acc_pos = (p->acc_pos + 1) % 20;
        }
        r->back_d = net_delay(m, r->draft_id, r->target_id);
        r->phase = PH_TO_DRAFT;
        schedule(m, m->now + r->back_d, EV_NET_ARRIVE, (uint64_t)id, MSG_RESULT);
    } else {
        commit_tokens(m, r, 1);
        if (r->phase == PH_DONE) return;
        if (m->fused_everything || r->draft_id < 0) begin_iteration(m, r, (decision_t){1, 1});
        else begin_iteration(m, r, decide_window(m, r));
    }
}

static void on_compute_done(sim_t* m, server_t* s) {
    s->busy = 0;
    int64_t n = s->rn;
    item_t* batch = malloc(sizeof(item_t) * (n ? n : 1));
    memcpy(batch, s->run, sizeof(item_t) * n);
    s->rn = 0;
    for (int64_t k = 0; k < n; ++k) {
        req_t* r = &m->rq[batch[k].req];
        if (s->is_draft) {
            if (batch[k].op == OP_PREFILL) {
                r->dpd = 1;
                if (r->output > 0) schedule(m, m->now, EV_ITER_START, (uint64_t)batch[k].req, 0);
            } else {
                r->phase = PH_TO_TARGET;
                r->out_d = net_delay(m, r->draft_id, r->target_id);
                schedule(m, m->now + r->out_d, EV_NET_ARRIVE, (uint64_t)batch[k].req, MSG_PROPOSAL);
            }
        } else {
            on_target_item_done(m, r, &batch[k]);
        }
    }
    free(batch);
    try_dispatch(m, s, 0);
}

static void on_net_arrive(sim_t* m, uint64_t msg, int64_t i) {
    req_t* r = &m->rq[i];
    if (msg == MSG_PROMPT) {
        item_t it = {OP_PREFILL, i, (int)r->prompt, 0, m->now, 1};
        push_work(m, &m->tg[r->target_id], it);
    } else if (msg == MSG_PROPOSAL) {
        r->phase = PH_VERIFYING;
        item_t it = {OP_VERIFY, i, r->pending_gamma, r->prompt + r->tokens_done, m->now, 1};
        push_work(m, &m->tg[r->target_id], it);
    } else {
        pair_t* p = &m->pairs[(size_t)r->draft_id * m->T + r->target_id];
        double rtt = (double)(r->out_d + r->back_d) / 1000.0;
        if (p->rtt_n < 20) p->rtt[p->rtt_n++] = rtt;
        else {
            p->rtt[p->rtt_pos] = rtt;
            p->rtt_pos = (p->rtt_pos + 1) % 20;
        }
        commit_tokens(m, r, r->lcr);
        if (r->phase != PH_DONE) schedule(m, m->now, EV_ITER_START, (uint64_t)i, 0);
    }
}

/* ------------------------------------------------------------------------ */
/* setup: generate_synthetic (src/workload/trace.cpp:145-187) and           */
/* schedule_arrivals (engine.cpp:224-244)                                   */
/* ------------------------------------------------------------------------ */
int64_t oracle_request_count(const dsd_scenario* s) {
    return s->workload == DSD_WORKLOAD_SYNTHETIC ? s->n_requests : (s->trace ? s->trace->n : 0);
}

static void setup(sim_t* m, const dsd_scenario* S, const dsd_replica* rep, int64_t seq_cap_per_req_hint) {
    (void)seq_cap_per_req_hint;
    m->S = S;
    m->T = S->n_targets;
    m->D = S->n_drafts;
    m->fused_everything = S->window_kind == DSD_WINDOW_FUSED || S->n_drafts == 0;
    m->N = oracle_request_count(S);
    rng_init(&m->routing, rep->seed, "routing");
    rng_init(&m->jitter, rep->seed, "jitter");
    m->first_arrival = m->last_completion = -1;
    m->rq = calloc((size_t)(m->N ? m->N : 1), sizeof(req_t));
    if (S->workload == DSD_WORKLOAD_SYNTHETIC) {
        rng_t ar, bits, len, dra;
        rng_init(&ar, rep->gen_seed, "arrivals");
        rng_init(&bits, rep->gen_seed, "accept-bits");
        rng_init(&len, rep->gen_seed, "lengths");
        rng_init(&dra, rep->gen_seed, "drafter-assign");
        double gap = 1000.0 / S->rate_rps, p_mu = log(S->prompt_median), o_mu = log(S->output_median);
        double clock_ms = 0.0;
        int64_t total = 0, cap = 0;
        for (int64_t n = 0; n < m->N; ++n) {
            req_t* r = &m->rq[n];
            clock_ms += rng_exponential(&ar, gap);
            r->arrival_tr = ms_to_us(clock_ms);
            int64_t p = llround(rng_lognormal(&len, p_mu, S->prompt_sigma));
            r->prompt = p < 1 ? 1 : (p > S->prompt_cap ? S->prompt_cap : p);
            int64_t o = llround(rng_lognormal(&len, o_mu, S->output_sigma));
            r->output = o < 1 ? 1 : (o > S->output_cap ? S->output_cap : o);
            r->drafter = (int64_t)rng_below(&dra, (uint64_t)S->gen_n_drafts);
            if (total + r->output > cap) {
                cap = 2 * (total + r->output) + 64;
                m->gen_bits = xrealloc(m->gen_bits, (size_t)cap);
            }
            for (int64_t k = 0; k < r->output; ++k) m->gen_bits[total + k] = rng_unit(&bits) < S->acceptance_rate;
            r->nbits = total; /* offset for now */
            total += r->output;
        }
        for (int64_t n = 0; n < m->N; ++n) {
            req_t* r = &m->rq[n];
            r->bits = m->gen_bits + r->nbits;
            r->nbits = r->output;
        }
    } else {
        const dsd_trace* t = S->trace;
        rng_t ar;
        rng_init(&ar, rep->seed, "arrivals");
        double clock_ms = 0.0;
        for (int64_t n = 0; n < m->N; ++n) {
            req_t* r = &m->rq[n];
            r->prompt = t->prompt_length[n];
            r->output = t->output_length[n];
            r->drafter = t->drafter_id[n];
            r->bits = t->acceptance_bits + t->bits_offset[n];
            r->nbits = t->bits_offset[n + 1] - t->bits_offset[n];
            if (S->workload == DSD_WORKLOAD_TRACE_POISSON) {
                clock_ms += rng_exponential(&ar, 1000.0 / S->rate_rps);
                r->arrival_tr = ms_to_us(clock_ms);
            } else {
                r->arrival_tr = t->arrival_us[n];
            }
        }
    }
    for (int64_t n = 0; n < m->N; ++n) {
        req_t* r = &m->rq[n];
        r->draft_id = -1;
        r->target_id = -1;
        r->arrival = r->first = r->completion = -1;
        r->scap = r->output;
        r->gseq = malloc(sizeof(int32_t) * (size_t)(r->scap ? r->scap : 1));
        r->cseq = malloc(sizeof(int32_t) * (size_t)(r->scap ? r->scap : 1));
        schedule(m, r->arrival_tr, EV_ARRIVAL, (uint64_t)n, 0);
    }
    m->tg = calloc((size_t)m->T, sizeof(server_t));
    m->dr = calloc((size_t)(m->D ? m->D : 1), sizeof(server_t));
    for (int t = 0; t < m->T; ++t) {
        m->tg[t].id = t;
        m->tg[t].active = -1;
        m->tg[t].grid_pre = S->target_grids[2 * t];
        m->tg[t].grid_dec = S->target_grids[2 * t + 1];
    }
    for (int d = 0; d < m->D; ++d) {
        m->dr[d].is_draft = 1;
        m->dr[d].id = d;
        m->dr[d].active = -1;
        m->dr[d].grid_pre = S->draft_grids[2 * d];
        m->dr[d].grid_dec = S->draft_grids[2 * d + 1];
    }
    size_t np = (size_t)m->T * (size_t)(m->D ? m->D : 1);
    m->pairs = calloc(np, sizeof(pair_t));
    for (size_t p = 0; p < np; ++p) m->pairs[p].gamma_prev = m->pairs[p].dyn_gamma = S->gamma;
    m->ts = calloc((size_t)m->T, sizeof(tstat_t));
}

static void teardown(sim_t* m) {
    for (int64_t n = 0; n < m->N; ++n) {
        free(m->rq[n].gseq);
        free(m->rq[n].cseq);
    }
    for (int t = 0; t < m->T; ++t) {
        free(m->tg[t].q);
        free(m->tg[t].run);
        free(m->tg[t].sess);
    }
    for (int d = 0; d < m->D; ++d) {
        free(m->dr[d].q);
        free(m->dr[d].run);
        free(m->dr[d].sess);
    }
    free(m->rq);
    free(m->tg);
    free(m->dr);
    free(m->pairs);
    free(m->ts);
    free(m->heap);
    free(m->gen_bits);
}

int64_t oracle_sequence_bound(const dsd_scenario* s, const dsd_replica* r) {
    (void)r;
    if (s->workload == DSD_WORKLOAD_SYNTHETIC) return s->n_requests * s->output_cap;
    int64_t tot = 0;
    for (int64_t i = 0; i < s->trace->n; ++i) tot += s->trace->output_length[i];
    return tot;
}

int oracle_run(const dsd_scenario* S, const dsd_replica* rep, dsd_replica_summary* sum, dsd_request_record* recs,
               int32_t* gseq, int32_t* cseq, int64_t seq_cap, int64_t* busy_us, char* err, size_t errlen) {
    sim_t m;
    memset(&m, 0, sizeof(m));
    setup(&m, S, rep, 0);
    /* SimKernel::run_until (event_queue.cpp:28-42) */
    while (m.hn > 0) {
        event_t ev = pop(&m);
        m.now = ev.time;
        ++m.processed;
        switch (ev.kind) {
            case EV_ARRIVAL: on_arrival(&m, (int64_t)ev.a); break;
            case EV_ITER_START: begin_iteration(&m, &m.rq[ev.a], decide_window(&m, &m.rq[ev.a])); break;
            case EV_NET_ARRIVE: on_net_arrive(&m, ev.b, (int64_t)ev.a); break;
            case EV_COMPUTE_DONE: {
                server_t* s = (ev.a & DRAFT_FLAG) ? &m.dr[ev.a & ~DRAFT_FLAG] : &m.tg[ev.a];
                on_compute_done(&m, s);
                break;
            }
            case EV_BATCH_READY: {
                server_t* s = (ev.a & DRAFT_FLAG) ? &m.dr[ev.a & ~DRAFT_FLAG] : &m.tg[ev.a];
                if (s->armed && s->gen == ev.b) {
                    s->armed = 0;
                    try_dispatch(&m, s, 1);
                }
                break;
            }
        }
    }
    /* Engine::finish + aggregate_run (engine.cpp:648-669, runner.cpp:153-169) */
    dsd_replica_summary s;
    memset(&s, 0, sizeof(s));
    s.events_processed = m.processed;
    s.end_time_us = m.now;
    s.completed = m.completed;
    s.first_arrival_us = m.first_arrival;
    s.last_completion_us = m.last_completion;
    s.net_queue_wait_total_us = m.net_total;
    s.net_queue_wait_count = m.net_count;
    s.n_requests = m.N;
    s.has_duration = m.completed > 0 && m.last_completion > m.first_arrival;
    if (s.has_duration)
        s.throughput_rps = (double)m.completed / ((double)(m.last_completion - m.first_arrival) / 1e6);
    double ttft = 0.0, tpot = 0.0;
    int64_t ntp = 0, nrec = 0, w = 0;
    for (int64_t i = 0; i < m.N; ++i) {
        req_t* r = &m.rq[i];
        if (recs) {
            dsd_request_record* o = &recs[i];
            o->drafter_id = m.D > 0 ? r->drafter : -1;
            o->prompt_length = r->prompt;
            o->output_length = r->output;
            o->arrival_us = r->arrival;
            o->first_token_us = r->first;
            o->completion_us = r->completion;
            o->proposed = r->prop;
            o->accepted = r->acc;
            o->target_id = r->target_id;
            o->n_iterations = (int32_t)r->ng;
        }
        for (int64_t k = 0; k < r->ng && w < seq_cap; ++k, ++w) {
            if (gseq) gseq[w] = r->gseq[k];
            if (cseq) cseq[w] = r->cseq[k];
        }
        if (r->completion < 0) continue;
        ++nrec;
        ttft += (double)(r->first - r->arrival) / 1000.0;
        if (r->output >= 2) {
            tpot += ((double)(r->completion - r->first) / 1000.0) / (double)(r->output - 1);
            ++ntp;
        }
    }
    s.mean_ttft_ms = nrec > 0 ? ttft / (double)nrec : 0.0;
    s.mean_tpot_ms = ntp > 0 ? tpot / (double)ntp : 0.0;
    s.status = DSD_OK;
    if (busy_us)
        for (int t = 0; t < m.T; ++t) busy_us[t] = m.tg[t].busy_us;
    if (sum) *sum = s;
    teardown(&m);
    if (err && errlen) err[0] = '\0';
    return DSD_OK;
}

/* ------------------------------------------------------------------------ */
/* multi-threaded batch (the CPU baseline's shape: sweep.cpp:109-160)       */
/* ------------------------------------------------------------------------ */
typedef struct {
    const dsd_scenario* sc;
    const dsd_replica* reps;
    dsd_replica_summary* out;
    size_t n;
    size_t next;
    pthread_mutex_t mu;
} batch_t;

static void* batch_worker(void* arg) {
    batch_t* b = arg;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        size_t i = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (i >= b->n) return NULL;
        oracle_run(&b->sc[b->reps[i].scenario], &b->reps[i], &b->out[i], NULL, NULL, NULL, 0, NULL, NULL, 0);
    }
}

int oracle_run_batch(const dsd_scenario* scenarios, const dsd_replica* replicas, size_t n, int threads,
                     dsd_replica_summary* summaries, char* err, size_t errlen) {
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    batch_t b = {scenarios, replicas, summaries, n, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &b);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    if (err && errlen) err[0] = '\0';
    return DSD_OK;
}
