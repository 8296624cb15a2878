/*
 * orc.c -- CPU ORACLE for the B200 list-ranking / connected-components path.
 *
 * TEST INFRASTRUCTURE ONLY.  Restates, in plain C, the reference's
 * sequential algorithms (/root/reference/pkg/src/simtgraph/core.py and
 * gen.py).  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * / reference arm may load this library -- as the checker and as the timed
 * CPU baseline, never as part of the product path.
 *
 * Parity of this restatement is pinned against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py -> tests/golden/*.npz)
 * and the reference's own known-answer tests (tests/test_oracle.py).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- KISS64: gen.py:51-64 (_kiss_batch) ------------------------------- */
void orc_kiss_batch(uint64_t* st, uint64_t n, uint64_t* out) {
    uint64_t x = st[0], y = st[1], z = st[2], c = st[3];
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t t = (x << 58) + c; /* multiply-with-carry */
        c = x >> 6;
        x = x + t;
        if (x < t) c = c + 1;
        y ^= y << 13; /* xorshift */
        y ^= y >> 17;
        y ^= y << 43;
        z = 6906969069ull * z + 1234567ull; /* congruential */
        out[i] = x + y + z;
    }
    st[0] = x;
    st[1] = y;
    st[2] = z;
    st[3] = c;
}

/* ---- _chain_positions: core.py:122-145 ----------------------------------
 * pos[i] = hops from the head, -1 if never reached.  Returns 1 (ok) or 0,
 * with *bad = first unreached index. */
int orc_chain_positions(const int64_t* succ, int64_t n, int64_t* pos, int64_t* bad) {
    for (int64_t i = 0; i < n; ++i) pos[i] = -1;
    int64_t cur = 0;
    for (int64_t step = 0; step < n; ++step) {
        if (pos[cur] >= 0) break; /* re-entered a visited node */
        pos[cur] = step;
        int64_t nxt = succ[cur];
        if (nxt == cur) break;
        cur = nxt;
    }
    for (int64_t i = 0; i < n; ++i) {
        if (pos[i] < 0) {
            *bad = i;
            return 0;
        }
    }
    *bad = -1;
    return 1;
}

/* ---- validate_list: core.py:148-167 --------------------------------------
 * kind: 0 ok, 1 out-of-range, 2 no-tail, 3 multiple-self-loops, 4 unreachable */
int orc_validate_list(const int64_t* succ, int64_t n, int64_t* index, int64_t* scratch_pos) {
    for (int64_t i = 0; i < n; ++i) {
        if (succ[i] < 0 || succ[i] >= n) {
            *index = i;
            return 1;
        }
    }
    int64_t loops = 0, second = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (succ[i] == i && ++loops == 2) second = i;
    }
    if (loops == 0) {
        *index = -1;
        return 2;
    }
    if (loops > 1) {
        *index = second;
        return 3;
    }
    int64_t bad;
    if (!orc_chain_positions(succ, n, scratch_pos, &bad)) {
        *index = bad;
        return 4;
    }
    *index = -1;
    return 0;
}

/* ---- seq_rank: core.py:179-186 (validate, positions, rank = n-1-pos) ---- */
int orc_seq_rank(const int64_t* succ, int64_t n, int64_t* rank, int64_t* index) {
    int kind = orc_validate_list(succ, n, index, rank); /* rank doubles as scratch */
    if (kind) return kind;
    int64_t bad;
    orc_chain_positions(succ, n, rank, &bad);
    for (int64_t i = 0; i < n; ++i) rank[i] = (n - 1) - rank[i];
    return 0;
}

/* ---- seq_components: core.py:209-248 (_uf_min_labels) --------------------
 * union-find with path halving, union keeps the smaller root; labels are
 * the find roots, i.e. the component minima. */
void orc_seq_components(int64_t n, const int64_t* edges, int64_t m, int64_t* label, int64_t* parent) {
    for (int64_t i = 0; i < n; ++i) parent[i] = i;
    for (int64_t k = 0; k < m; ++k) {
        int64_t a = edges[2 * k], b = edges[2 * k + 1];
        while (parent[a] != a) {
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        while (parent[b] != b) {
            parent[b] = parent[parent[b]];
            b = parent[b];
        }
        if (a < b)
            parent[b] = a;
        else if (b < a)
            parent[a] = b;
    }
    for (int64_t i = 0; i < n; ++i) {
        int64_t r = i;
        while (parent[r] != r) r = parent[r];
        label[i] = r;
        int64_t j = i;
        while (parent[j] != r) {
            int64_t nxt = parent[j];
            parent[j] = r;
            j = nxt;
        }
    }
}

/* ---- validate_graph: core.py:196-206 --------------------------------------
 * kind: 0 ok, 1 out-of-range (index = row), 2 self-loop (index = row) */
int orc_validate_graph(int64_t n, const int64_t* edges, int64_t m, int64_t* index) {
    for (int64_t f = 0; f < 2 * m; ++f) {
        if (edges[f] < 0 || edges[f] >= n) {
            *index = f / 2;
            return 1;
        }
    }
    for (int64_t k = 0; k < m; ++k) {
        if (edges[2 * k] == edges[2 * k + 1]) {
            *index = k;
            return 2;
        }
    }
    *index = -1;
    return 0;
}

/* ---- CPU-baseline samples (bench.py) --------------------------------------
 * Bounded samples of the same workloads, timed by the caller.
 *
 * seq_rank's per-node work is two dependent walks over the full-size arrays
 * (core.py:164 via validate_list, and core.py:175), each reading succ[cur]
 * and testing / writing pos[cur].  orc_rank_walk_sample runs `threads`
 * independent copies of that walk (pthreads) from distinct start nodes for
 * up to `hops` hops each, twice (validation walk + position walk), over a
 * shared n-sized pos array.  Returns the hops actually walked. */
typedef struct {
    const int64_t* succ;
    int64_t* pos;
    int64_t start, hops, done;
} walk_arg;

static void* walk_thread(void* p) {
    walk_arg* a = (walk_arg*)p;
    int64_t cur = a->start, step = 0;
    for (; step < a->hops; ++step) {
        if (a->pos[cur] >= 0) break;
        a->pos[cur] = step;
        int64_t nxt = a->succ[cur];
        if (nxt == cur) break;
        cur = nxt;
    }
    a->done = step;
    return NULL;
}

int64_t orc_rank_walk_sample(const int64_t* succ, int64_t n, int64_t* pos, int64_t hops, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    walk_arg args[256];
    pthread_t tid[256];
    int64_t total = 0;
    for (int pass = 0; pass < 2; ++pass) {
        memset(pos, 0xff, sizeof(int64_t) * (size_t)n); /* pos = -1 */
        for (int t = 0; t < threads; ++t) {
            args[t].succ = succ;
            args[t].pos = pos;
            args[t].start = (int64_t)(((unsigned __int128)(uint64_t)t * (uint64_t)n) / (uint64_t)threads);
            args[t].hops = hops;
            args[t].done = 0;
            pthread_create(&tid[t], NULL, walk_thread, &args[t]);
        }
        for (int t = 0; t < threads; ++t) {
            pthread_join(tid[t], NULL);
            total += args[t].done;
        }
    }
    return total / 2;
}

/* union-find over every `stride`-th stored edge (a G(n, m/stride) sample of
 * the same graph), then the labelling pass over all n vertices; returns the
 * two phase times in seconds through t_union / t_label. */
static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int64_t orc_uf_sample(int64_t n, const int64_t* edges, int64_t m, int64_t stride, int64_t* parent, int64_t* label,
                      double* t_union, double* t_label) {
    if (stride < 1) stride = 1;
    double t0 = now_s();
    for (int64_t i = 0; i < n; ++i) parent[i] = i;
    int64_t used = 0;
    for (int64_t k = 0; k < m; k += stride, ++used) {
        int64_t a = edges[2 * k], b = edges[2 * k + 1];
        while (parent[a] != a) {
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        while (parent[b] != b) {
            parent[b] = parent[parent[b]];
            b = parent[b];
        }
        if (a < b)
            parent[b] = a;
        else if (b < a)
            parent[a] = b;
    }
    double t1 = now_s();
    for (int64_t i = 0; i < n; ++i) {
        int64_t r = i;
        while (parent[r] != r) r = parent[r];
        label[i] = r;
        int64_t j = i;
        while (parent[j] != r) {
            int64_t nxt = parent[j];
            parent[j] = r;
            j = nxt;
        }
    }
    double t2 = now_s();
    *t_union = t1 - t0;
    *t_label = t2 - t1;
    return used;
}
