/*
 * oracle/vcs_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU oracle of the solver path.
 *
 * A plain-C restatement of the reference algorithm, used by tests/ (parity checker),
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, and by nothing in the product.
 * Parity of THIS file is pinned against (a) the unmodified reference compiled from
 * /root/reference by oracle/Makefile into oracle/_ref/libvcsref.so and (b) the reference's
 * golden values (tests/golden/) — see tests/test_oracle.py.
 *
 * Restated functions (reference paths relative to /root/reference/proj):
 *   orc_build        core/src/mdp.cpp:81-214   StateSpace::build (layered BFS, first-insertion
 *                                              order, reduced keys, retirement charge)
 *   orc_backup       core/src/mdp.cpp:245-263  StateSpace::backup (strict '>' argmax)
 *   orc_vi           core/src/parallel_vi.cpp:48-116  Jacobi sweeps, sup-norm residual,
 *                                              `delta < eps`, extraction (:109-111)
 *   orc_greedy       core/src/greedy.cpp:5-30 + workload.cpp:22-26 feasible()
 *   orc_hidden_penalty core/src/mdp.cpp:236-243
 * Compile with -ffp-contract=off and without -march=native: the reward is a separate multiply
 * and subtract (SURVEY §7.2 hard part 1).
 */
#include "../include/vcs_gpu.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

static int orc_fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

typedef struct orc_space {
    int n_clouds;
    int H;
    uint64_t S, E;
    uint64_t* layer_off; /* H+2 */
    uint64_t* row_ptr;   /* S+1 */
    uint32_t* succ;
    double* reward;
    int32_t* action;
    int* last_use;       /* per cloud, -1 if never eligible */
    double gamma;
    int owns;            /* 0 when the CSR arrays are borrowed (orc_space_wrap) */
} orc_space;

/* ---------------------------------------------------------------------------------------- */
/* growable arrays                                                                           */
/* ---------------------------------------------------------------------------------------- */

typedef struct { void* p; size_t n, cap, elem; } vec_t;

static void vec_init(vec_t* v, size_t elem) { v->p = NULL; v->n = v->cap = 0; v->elem = elem; }

static void* vec_grow(vec_t* v, size_t add) {
    if (v->n + add > v->cap) {
        size_t c = v->cap ? v->cap : 1024;
        while (c < v->n + add) c *= 2;
        void* np = realloc(v->p, c * v->elem);
        if (!np) return NULL;
        v->p = np;
        v->cap = c;
    }
    void* at = (char*)v->p + v->n * v->elem;
    v->n += add;
    return at;
}

/* ---------------------------------------------------------------------------------------- */
/* per-layer key map: key (u16 x klen) -> local index, first-insertion order (mdp.cpp:157-165) */
/* ---------------------------------------------------------------------------------------- */

typedef struct {
    uint32_t* slots; /* local index + 1, 0 = empty */
    size_t cap;
    size_t count;
    int klen;
    vec_t* keys;     /* next frontier keys, klen u16 each, in insertion order */
} keymap_t;

static uint64_t key_hash(const uint16_t* k, int klen) {
    uint64_t h = 1469598103934665603ull; /* FNV-1a, as KeyHash (mdp.cpp:71-79) */
    for (int i = 0; i < klen; ++i) {
        h ^= k[i];
        h *= 1099511628211ull;
    }
    return h ^ (h >> 29);
}

static int keymap_init(keymap_t* m, int klen, vec_t* keys) {
    m->cap = 1024;
    m->count = 0;
    m->klen = klen;
    m->keys = keys;
    m->slots = (uint32_t*)calloc(m->cap, sizeof(uint32_t));
    return m->slots ? 0 : -1;
}

static int keymap_rehash(keymap_t* m) {
    size_t nc = m->cap * 2;
    uint32_t* ns = (uint32_t*)calloc(nc, sizeof(uint32_t));
    if (!ns) return -1;
    const uint16_t* base = (const uint16_t*)m->keys->p;
    for (size_t i = 0; i < m->cap; ++i) {
        if (!m->slots[i]) continue;
        const uint16_t* k = base + (size_t)(m->slots[i] - 1) * (size_t)m->klen;
        size_t j = (size_t)key_hash(k, m->klen) & (nc - 1);
        while (ns[j]) j = (j + 1) & (nc - 1);
        ns[j] = m->slots[i];
    }
    free(m->slots);
    m->slots = ns;
    m->cap = nc;
    return 0;
}

/* Returns the local index of `k`, inserting it at the end when new (*inserted = 1). */
static int64_t keymap_intern(keymap_t* m, const uint16_t* k, int* inserted) {
    if ((m->count + 1) * 2 > m->cap && keymap_rehash(m) != 0) return -1;
    size_t j = (size_t)key_hash(k, m->klen) & (m->cap - 1);
    const int klen = m->klen;
    while (m->slots[j]) {
        const uint16_t* other = (const uint16_t*)m->keys->p + (size_t)(m->slots[j] - 1) * klen;
        if (klen == 0 || memcmp(other, k, (size_t)klen * sizeof(uint16_t)) == 0) {
            *inserted = 0;
            return (int64_t)m->slots[j] - 1;
        }
        j = (j + 1) & (m->cap - 1);
    }
    uint16_t* dst = (uint16_t*)vec_grow(m->keys, (size_t)(klen > 0 ? klen : 0));
    if (klen > 0 && !dst) return -1;
    if (klen > 0) memcpy(dst, k, (size_t)klen * sizeof(uint16_t));
    m->slots[j] = (uint32_t)(++m->count);
    *inserted = 1;
    return (int64_t)m->count - 1;
}

/* ---------------------------------------------------------------------------------------- */
/* StateSpace::build restated (mdp.cpp:81-214)                                               */
/* ---------------------------------------------------------------------------------------- */

void orc_space_free(orc_space* sp) {
    if (!sp) return;
    if (sp->owns) {
        free(sp->layer_off);
        free(sp->row_ptr);
        free(sp->succ);
        free(sp->reward);
        free(sp->action);
    }
    free(sp->last_use);
    free(sp);
}

int orc_build(const vcs_instance* in, uint64_t state_cap, orc_space** out) {
    const int K = in->n_clouds;
    const int H = in->n_tasks;
    for (int i = 0; i < K; ++i) /* mdp.cpp:90-92 */
        if (in->cloud_vm_free[i] > 0xffff)
            return orc_fail(VCS_EINVAL, "cloud free counts above 65535 are not supported");

    orc_space* sp = (orc_space*)calloc(1, sizeof(orc_space));
    sp->n_clouds = K;
    sp->H = H;
    sp->owns = 1;
    sp->gamma = in->gamma_vc;

    /* attr_ok and last_use (mdp.cpp:94-109): capacity against the INITIAL free count. */
    char* attr_ok = (char*)calloc((size_t)(K > 0 ? K : 1) * (size_t)(H > 0 ? H : 1), 1);
    sp->last_use = (int*)malloc(sizeof(int) * (size_t)(K > 0 ? K : 1));
    for (int i = 0; i < K; ++i) {
        sp->last_use[i] = -1;
        for (int j = 0; j < H; ++j) {
            const int ok = in->cloud_delay_ms[i] <= in->task_max_delay_ms[j] &&
                           in->cloud_thr_kbps[i] >= in->task_min_thr_kbps[j] &&
                           in->task_demand[j] <= in->cloud_vm_free[i];
            attr_ok[(size_t)i * H + j] = (char)ok;
            if (ok) sp->last_use[i] = j;
        }
    }
    /* active clouds per layer (mdp.cpp:111-116) */
    int* act = (int*)malloc(sizeof(int) * (size_t)(K > 0 ? K : 1) * (size_t)(H + 1));
    int* n_act = (int*)calloc((size_t)H + 1, sizeof(int));
    for (int t = 0; t <= H; ++t)
        for (int i = 0; i < K; ++i)
            if (sp->last_use[i] >= t) act[(size_t)t * K + n_act[t]++] = i;

    sp->layer_off = (uint64_t*)calloc((size_t)H + 2, sizeof(uint64_t));
    vec_t row_ptr, succ, reward, action;
    vec_init(&row_ptr, sizeof(uint64_t));
    vec_init(&succ, sizeof(uint32_t));
    vec_init(&reward, sizeof(double));
    vec_init(&action, sizeof(int32_t));

    vec_t frontier, next;
    vec_init(&frontier, sizeof(uint16_t));
    vec_init(&next, sizeof(uint16_t));
    uint64_t n_frontier = 1;
    {
        uint16_t* k0 = (uint16_t*)vec_grow(&frontier, (size_t)n_act[0]);
        for (int p = 0; p < n_act[0]; ++p) k0[p] = (uint16_t)in->cloud_vm_free[act[p]];
    }
    uint64_t n_states = 1;
    *(uint64_t*)vec_grow(&row_ptr, 1) = 0;

    const double beta_vc = in->beta_vc, beta_tc = in->beta_tc, gamma = in->gamma_vc;
    int rc = VCS_OK;
    uint16_t* succ_key = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(K > 0 ? K : 1));
    int* keep = (int*)malloc(sizeof(int) * (size_t)(K > 0 ? K : 1));
    int* retire = (int*)malloc(sizeof(int) * (size_t)(K > 0 ? K : 1));

    for (int t = 0; t < H && rc == VCS_OK; ++t) {
        const int* active = act + (size_t)t * K;
        const int na = n_act[t];
        const int demand = in->task_demand[t];
        sp->layer_off[t + 1] = n_states;
        int nk = 0, nr = 0;
        for (int p = 0; p < na; ++p) {
            if (sp->last_use[active[p]] >= t + 1) keep[nk++] = p;
            else retire[nr++] = p;
        }
        next.n = 0;
        keymap_t map;
        keymap_init(&map, nk, &next);
        const uint64_t next_base = n_states;
        for (uint64_t si = 0; si < n_frontier && rc == VCS_OK; ++si) {
            const uint16_t* key = (const uint16_t*)frontier.p + si * (size_t)na;
            /* cloud actions ascending, then paid (mdp.cpp:169-204) */
            for (int p = 0; p <= na; ++p) {
                const int paid = p == na;
                int32_t cloud = VCS_PAID_CLOUD;
                if (!paid) {
                    cloud = active[p];
                    if (!attr_ok[(size_t)cloud * H + t]) continue;
                    if (key[p] < demand) continue;
                }
                double retired_free = 0.0;
                for (int q = 0; q < nk; ++q) {
                    uint16_t v = key[keep[q]];
                    if (!paid && keep[q] == p) v = (uint16_t)(v - demand);
                    succ_key[q] = v;
                }
                for (int q = 0; q < nr; ++q) {
                    double v = key[retire[q]];
                    if (!paid && retire[q] == p) v -= demand;
                    retired_free += v;
                }
                int inserted = 0;
                const int64_t local = keymap_intern(&map, succ_key, &inserted);
                if (local < 0) { rc = orc_fail(1, "out of memory"); break; }
                if (inserted) {
                    ++n_states;
                    if (n_states > state_cap) {
                        char msg[128];
                        snprintf(msg, sizeof msg, "reachable state space exceeds cap of %llu states",
                                 (unsigned long long)state_cap);
                        rc = orc_fail(VCS_ECAP, msg);
                        break;
                    }
                }
                *(uint32_t*)vec_grow(&succ, 1) = (uint32_t)(next_base + (uint64_t)local);
                const double n = (double)demand;
                const double r = paid ? -beta_tc * n - gamma * retired_free
                                      : beta_vc * n - gamma * retired_free;
                *(double*)vec_grow(&reward, 1) = r;
                *(int32_t*)vec_grow(&action, 1) = cloud;
            }
            *(uint64_t*)vec_grow(&row_ptr, 1) = (uint64_t)succ.n;
        }
        free(map.slots);
        /* swap frontier <- next */
        vec_t tmp = frontier;
        frontier = next;
        next = tmp;
        n_frontier = map.count;
    }
    if (rc == VCS_OK) {
        for (uint64_t i = 0; i < n_frontier; ++i) *(uint64_t*)vec_grow(&row_ptr, 1) = (uint64_t)succ.n;
        sp->layer_off[H + 1] = n_states;
        sp->layer_off[0] = 0;
        if (H == 0) sp->layer_off[1] = n_states;
    }
    free(succ_key);
    free(keep);
    free(retire);
    free(frontier.p);
    free(next.p);
    free(attr_ok);
    free(act);
    free(n_act);
    sp->S = n_states;
    sp->E = succ.n;
    sp->row_ptr = (uint64_t*)row_ptr.p;
    sp->succ = (uint32_t*)succ.p;
    sp->reward = (double*)reward.p;
    sp->action = (int32_t*)action.p;
    if (rc != VCS_OK) {
        orc_space_free(sp);
        return rc;
    }
    *out = sp;
    return VCS_OK;
}

/* Borrow an external CSR (e.g. the product's, downloaded) so the oracle sweep can be timed or
 * cross-checked on it.  Arrays must outlive the handle. */
int orc_space_wrap(uint64_t S, uint64_t E, int32_t H, uint64_t* layer_off, uint64_t* row_ptr,
                   uint32_t* succ, double* reward, int32_t* action, orc_space** out) {
    orc_space* sp = (orc_space*)calloc(1, sizeof(orc_space));
    sp->S = S;
    sp->E = E;
    sp->H = H;
    sp->layer_off = layer_off;
    sp->row_ptr = row_ptr;
    sp->succ = succ;
    sp->reward = reward;
    sp->action = action;
    sp->owns = 0;
    *out = sp;
    return VCS_OK;
}

void orc_space_info(const orc_space* sp, uint64_t* S, uint64_t* E, int32_t* H) {
    *S = sp->S;
    *E = sp->E;
    *H = sp->H;
}

void orc_space_csr(const orc_space* sp, uint64_t* layer_off, uint64_t* row_ptr, uint32_t* succ,
                   double* reward, int32_t* action) {
    if (layer_off) memcpy(layer_off, sp->layer_off, sizeof(uint64_t) * (size_t)(sp->H + 2));
    if (row_ptr) memcpy(row_ptr, sp->row_ptr, sizeof(uint64_t) * (size_t)(sp->S + 1));
    if (succ) memcpy(succ, sp->succ, sizeof(uint32_t) * (size_t)sp->E);
    if (reward) memcpy(reward, sp->reward, sizeof(double) * (size_t)sp->E);
    if (action) memcpy(action, sp->action, sizeof(int32_t) * (size_t)sp->E);
}

/* ---------------------------------------------------------------------------------------- */
/* StateSpace::backup (mdp.cpp:245-263) and the Jacobi driver (parallel_vi.cpp:48-116)       */
/* ---------------------------------------------------------------------------------------- */

static inline double orc_backup(const orc_space* sp, uint64_t s, const double* prev,
                                int32_t* best_action, double discount) {
    const uint64_t first = sp->row_ptr[s], last = sp->row_ptr[s + 1];
    if (first == last) {
        if (best_action) *best_action = VCS_PAID_CLOUD;
        return 0.0;
    }
    double best = -INFINITY;
    int32_t a = VCS_PAID_CLOUD;
    for (uint64_t e = first; e < last; ++e) {
        const double v = prev[sp->succ[e]];
        const double q = discount == 1.0 ? sp->reward[e] + v : sp->reward[e] + discount * v;
        if (q > best) {
            best = q;
            a = sp->action[e];
        }
    }
    if (best_action) *best_action = a;
    return best;
}

typedef struct {
    const orc_space* sp;
    double* bufs[2];
    uint64_t begin, end;
    double discount;
    double eps;
    int max_sweeps;
    int w, nw;
    double* block_delta;
    pthread_barrier_t* bar;
    int* stop;
    int* sweeps;
    int* cur; /* index of the buffer holding the previous iterate */
} orc_worker_t;

static void* orc_worker(void* arg) {
    orc_worker_t* a = (orc_worker_t*)arg;
    for (;;) {
        const double* prev = a->bufs[*a->cur];
        double* next = a->bufs[*a->cur ^ 1];
        double delta = 0.0;
        for (uint64_t s = a->begin; s < a->end; ++s) {
            const double v = orc_backup(a->sp, s, prev, NULL, a->discount);
            const double d = fabs(v - prev[s]);
            delta = delta < d ? d : delta; /* std::max(delta, d) */
            next[s] = v;
        }
        a->block_delta[a->w] = delta;
        pthread_barrier_wait(a->bar);
        if (a->w == 0) {
            double g = 0.0;
            for (int i = 0; i < a->nw; ++i) g = g < a->block_delta[i] ? a->block_delta[i] : g;
            *a->cur ^= 1;
            ++*a->sweeps;
            *a->stop = g < a->eps || (a->max_sweeps > 0 && *a->sweeps >= a->max_sweeps);
        }
        pthread_barrier_wait(a->bar);
        if (*a->stop) return NULL;
    }
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

/* Jacobi value iteration from V=0 until delta < eps, then argmax extraction.  `workers` > 1
 * uses contiguous equal row blocks (BlockPartition::even, parallel_vi.cpp:11-24); results are
 * identical for any worker count.  max_sweeps > 0 bounds the run (timing samples only). */
int orc_vi(const orc_space* sp, double eps, int workers, double discount, int max_sweeps,
           double* values_out, int32_t* actions_out, int32_t* sweeps_out, double* sweep_ms,
           double* extract_ms) {
    if (workers < 1) return orc_fail(VCS_EINVAL, "n_workers must be >= 1");
    const uint64_t n = sp->S;
    double* b0 = (double*)calloc(n ? n : 1, sizeof(double));
    double* b1 = (double*)calloc(n ? n : 1, sizeof(double));
    int sweeps = 0, cur = 0, stop = 0;
    const double t0 = now_ms();
    if (workers == 1) {
        for (;;) {
            const double* prev = cur ? b1 : b0;
            double* next = cur ? b0 : b1;
            double delta = 0.0;
            for (uint64_t s = 0; s < n; ++s) {
                const double v = orc_backup(sp, s, prev, NULL, discount);
                const double d = fabs(v - prev[s]);
                delta = delta < d ? d : delta;
                next[s] = v;
            }
            cur ^= 1;
            ++sweeps;
            if (delta < eps || (max_sweeps > 0 && sweeps >= max_sweeps)) break;
        }
    } else {
        pthread_barrier_t bar;
        pthread_barrier_init(&bar, NULL, (unsigned)workers);
        double* block_delta = (double*)calloc((size_t)workers, sizeof(double));
        orc_worker_t* args = (orc_worker_t*)calloc((size_t)workers, sizeof(orc_worker_t));
        pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
        const uint64_t base = n / (uint64_t)workers, extra = n % (uint64_t)workers;
        uint64_t begin = 0;
        for (int w = 0; w < workers; ++w) {
            const uint64_t len = base + ((uint64_t)w < extra ? 1 : 0);
            args[w] = (orc_worker_t){sp, {b0, b1}, begin, begin + len, discount, eps, max_sweeps,
                                     w, workers, block_delta, &bar, &stop, &sweeps, &cur};
            begin += len;
        }
        for (int w = 1; w < workers; ++w) pthread_create(&th[w], NULL, orc_worker, &args[w]);
        orc_worker(&args[0]);
        for (int w = 1; w < workers; ++w) pthread_join(th[w], NULL);
        pthread_barrier_destroy(&bar);
        free(block_delta);
        free(args);
        free(th);
    }
    const double t1 = now_ms();
    const double* prev = cur ? b1 : b0;
    if (actions_out)
        for (uint64_t s = 0; s < n; ++s) {
            actions_out[s] = VCS_PAID_CLOUD;
            orc_backup(sp, s, prev, &actions_out[s], discount);
        }
    const double t2 = now_ms();
    if (values_out) memcpy(values_out, prev, sizeof(double) * (size_t)n);
    if (sweeps_out) *sweeps_out = sweeps;
    if (sweep_ms) *sweep_ms = t1 - t0;
    if (extract_ms) *extract_ms = t2 - t1;
    free(b0);
    free(b1);
    return VCS_OK;
}

/* Row-range pieces of the same sweep, for the CPU backend of the sharded-driver tests:
 * one Jacobi sweep over rows [rb, re) (returns the block residual) and the argmax extraction. */
double orc_sweep_rows(const orc_space* sp, const double* prev, double* next, uint64_t rb,
                      uint64_t re, double discount) {
    double delta = 0.0;
    for (uint64_t s = rb; s < re; ++s) {
        const double v = orc_backup(sp, s, prev, NULL, discount);
        const double d = fabs(v - prev[s]);
        delta = delta < d ? d : delta;
        next[s] = v;
    }
    return delta;
}

void orc_extract_rows(const orc_space* sp, const double* v, int32_t* act, uint64_t rb, uint64_t re,
                      double discount) {
    for (uint64_t s = rb; s < re; ++s) {
        act[s] = VCS_PAID_CLOUD;
        orc_backup(sp, s, v, &act[s], discount);
    }
}

/* hidden_penalty (mdp.cpp:236-243): gamma * free VMs of clouds retired at the state's layer. */
double orc_hidden_penalty(const orc_space* sp, const int32_t* free_vms, int32_t t, uint8_t terminal) {
    if (sp->H == 0) return 0.0;
    const int layer = terminal ? sp->H : t;
    double retired = 0.0;
    for (int i = 0; i < sp->n_clouds; ++i)
        if (sp->last_use[i] < layer) retired += free_vms[i];
    return sp->gamma * retired;
}

/* ---------------------------------------------------------------------------------------- */
/* greedy_schedule (greedy.cpp:5-30) and greedy_reward (greedy.cpp:32-36)                    */
/* ---------------------------------------------------------------------------------------- */

int orc_greedy(const vcs_instance* in, int32_t* target_idx, int64_t* per_cloud_used, int64_t* paid,
               int64_t* unused, double* ms) {
    const int K = in->n_clouds;
    int32_t* free_vms = (int32_t*)malloc(sizeof(int32_t) * (size_t)(K > 0 ? K : 1));
    int64_t* used = (int64_t*)calloc((size_t)(K > 0 ? K : 1), sizeof(int64_t));
    memcpy(free_vms, in->cloud_vm_free, sizeof(int32_t) * (size_t)K);
    int64_t p = 0, placed = 0, cap = 0;
    const double t0 = now_ms();
    for (int j = 0; j < in->n_tasks; ++j) {
        const int d = in->task_demand[j];
        int hit = VCS_PAID_CLOUD;
        for (int i = 0; i < K; ++i) {
            if (free_vms[i] >= d && in->cloud_delay_ms[i] <= in->task_max_delay_ms[j] &&
                in->cloud_thr_kbps[i] >= in->task_min_thr_kbps[j]) {
                hit = i;
                break;
            }
        }
        if (hit >= 0) {
            free_vms[hit] -= d;
            used[hit] += d;
            placed += d;
        } else {
            p += d;
        }
        target_idx[j] = hit;
    }
    const double t1 = now_ms();
    for (int i = 0; i < K; ++i) cap += in->cloud_vm_total[i];
    *paid = p;
    *unused = cap - placed;
    if (per_cloud_used) memcpy(per_cloud_used, used, sizeof(int64_t) * (size_t)K);
    if (ms) *ms = t1 - t0;
    free(free_vms);
    free(used);
    return VCS_OK;
}

double orc_greedy_reward(const vcs_instance* in, int64_t placed, int64_t paid, int64_t unused) {
    return in->beta_vc * (double)placed - in->beta_tc * (double)paid - in->gamma_vc * (double)unused;
}
