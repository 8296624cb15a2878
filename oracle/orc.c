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
 * the reference itself (tests/golden/make_golden.py -> tests/golden/golden.npz)
 * and the reference's own known-answer tests (tests/test_oracle.py).
 */
#define _GNU_SOURCE
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

/* ---- generators at full size (gen.py:110-127, :183-218) -------------------
 * Plain-C restatements of gen_list and gen_random_graph, so the reference
 * arm and the tests can build the 2^28-node list and the 2^26 / 2^28 graph
 * on the host in seconds instead of minutes.  Same KISS stream, same
 * draw-order rules; the sorts are LSD radix sorts (stable, as np.argsort's
 * kind="stable" and np.sort on distinct keys). */

/* stable LSD radix argsort of keys[0..n) -> idx (0-based), 11-bit digits;
 * passes whose digit is constant are skipped. */
static int radix_argsort_u64(const uint64_t* keys_in, int64_t n, uint32_t* idx_out) {
    enum { B = 11, NB = 1 << B };
    uint64_t* ka = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
    uint64_t* kb = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
    uint32_t* ib = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * NB);
    if (!ka || !kb || !ib || !cnt) {
        free(ka), free(kb), free(ib), free(cnt);
        return -1;
    }
    memcpy(ka, keys_in, sizeof(uint64_t) * (size_t)n);
    uint32_t* ia = idx_out;
    for (int64_t i = 0; i < n; ++i) ia[i] = (uint32_t)i;
    for (int shift = 0; shift < 64; shift += B) {
        memset(cnt, 0, sizeof(int64_t) * NB);
        for (int64_t i = 0; i < n; ++i) cnt[(ka[i] >> shift) & (NB - 1)]++;
        int constant = 0;
        for (int d = 0; d < NB; ++d)
            if (cnt[d] == n) constant = 1;
        if (constant) continue;
        int64_t s = 0;
        for (int d = 0; d < NB; ++d) {
            int64_t c = cnt[d];
            cnt[d] = s;
            s += c;
        }
        for (int64_t i = 0; i < n; ++i) {
            int64_t o = cnt[(ka[i] >> shift) & (NB - 1)]++;
            kb[o] = ka[i];
            ib[o] = ia[i];
        }
        uint64_t* tk = ka;
        ka = kb;
        kb = tk;
        uint32_t* ti = ia;
        ia = ib;
        ib = ti;
    }
    if (ia != idx_out) {
        memcpy(idx_out, ia, sizeof(uint32_t) * (size_t)n);
        ib = ia; /* the malloc'd one */
    }
    free(ka), free(kb), free(ib), free(cnt);
    return 0;
}

/* gen_list (gen.py:110-127): keys = n-1 KISS draws from kiss_seed(seed)
 * (passed in as the state); order = [0] + 1 + argsort(keys, stable);
 * succ[order[k]] = order[k+1], tail self-loop.  n < 2^32. */
int orc_gen_list(int64_t n, const uint64_t* state, int64_t* succ) {
    if (n == 1) {
        succ[0] = 0;
        return 0;
    }
    uint64_t st[4] = {state[0], state[1], state[2], state[3]};
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n - 1));
    uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n - 1));
    if (!keys || !idx) {
        free(keys), free(idx);
        return -1;
    }
    orc_kiss_batch(st, (uint64_t)(n - 1), keys);
    if (radix_argsort_u64(keys, n - 1, idx)) {
        free(keys), free(idx);
        return -1;
    }
    free(keys);
    int64_t prev = 0;
    for (int64_t k = 0; k < n - 1; ++k) {
        int64_t nxt = 1 + (int64_t)idx[k];
        succ[prev] = nxt;
        prev = nxt;
    }
    succ[prev] = prev;
    free(idx);
    return 0;
}

/* gen_random_graph (gen.py:183-218) for m = round(d * n(n-1)/2) given by
 * the caller: batches of 2*(need + need/4 + 16) draws, u = even draws % n,
 * v = odd draws % n, loops dropped, key = min*n + max; keys are taken in
 * draw order, skipping repeats within the batch and keys already kept
 * (np.unique(return_index) + isin), at most `need` per batch; the rest of
 * a batch is drawn and discarded.  Output rows sorted.  Returns 0, or -1
 * on allocation failure. */
int orc_gen_random_graph(int64_t n, int64_t m, const uint64_t* state, int64_t* edges) {
    uint64_t st[4] = {state[0], state[1], state[2], state[3]};
    uint64_t un = (uint64_t)n;
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * m + 16)) cap <<= 1;
    int shift = 64 - __builtin_ctzll(cap);
    uint64_t* table = (uint64_t*)calloc((size_t)cap, sizeof(uint64_t)); /* key + 1, 0 = empty */
    uint64_t* seen = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m ? m : 1));
    enum { CH = 1 << 16 };
    uint64_t* draws = (uint64_t*)malloc(sizeof(uint64_t) * CH);
    if (!table || !seen || !draws) {
        free(table), free(seen), free(draws);
        return -1;
    }
    int64_t got = 0;
    while (got < m) {
        int64_t need = m - got, taken = 0;
        uint64_t left = 2 * (uint64_t)(need + need / 4 + 16);
        while (left) {
            uint64_t c = left < CH ? left : CH;
            orc_kiss_batch(st, c, draws);
            left -= c;
            if (taken == need) continue;
            for (uint64_t j = 0; j + 1 < c && taken < need; j += 2) {
                uint64_t u = draws[j] % un, v = draws[j + 1] % un;
                if (u == v) continue;
                uint64_t key = (u < v ? u : v) * un + (u < v ? v : u);
                uint64_t h = (key * 0x9E3779B97F4A7C15ull) >> shift;
                for (;;) {
                    if (table[h] == 0) {
                        table[h] = key + 1;
                        seen[got + taken++] = key;
                        break;
                    }
                    if (table[h] == key + 1) break;
                    h = (h + 1) & (cap - 1);
                }
            }
        }
        got += taken;
    }
    free(table), free(draws);
    uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m ? m : 1));
    if (!idx || radix_argsort_u64(seen, m, idx)) {
        free(idx), free(seen);
        return -1;
    }
    for (int64_t k = 0; k < m; ++k) {
        uint64_t key = seen[idx[k]];
        edges[2 * k] = (int64_t)(key / un);
        edges[2 * k + 1] = (int64_t)(key % un);
    }
    free(idx), free(seen);
    return 0;
}

/* ---- CPU-baseline / reference-arm timing ------------------------------------
 * orc_seq_rank_sample: a bounded sample of seq_rank (core.py:179-186) on the
 * full-size list: the same per-node work for the first `hops` nodes of the
 * chain -- range and self-loop scans over `hops` entries (core.py:151-160),
 * the validation walk (core.py:164 -> _chain_positions), the position walk
 * (core.py:175) and the rank fill -- each walk starting at the head and
 * reading succ[cur], testing and writing pos[cur] over the full n-sized
 * arrays.  Visited marks carry an epoch in bits 40+ so the n-sized pos array
 * is not re-initialised per sample (one memset when epoch == 1).  Returns
 * the nodes ranked; *anomalies counts range / self-loop findings. */
int64_t orc_seq_rank_sample(const int64_t* succ, int64_t n, int64_t* pos, int64_t* rank, int64_t hops,
                            int64_t epoch, int64_t* anomalies) {
    if (hops > n) hops = n;
    int64_t bad = 0, loops = 0;
    for (int64_t i = 0; i < hops; ++i) {
        bad += (succ[i] < 0) | (succ[i] >= n);
        loops += succ[i] == i;
    }
    int64_t walked[2];
    for (int pass = 0; pass < 2; ++pass) {
        const int64_t tag = (epoch * 2 + pass) << 40;
        int64_t cur = 0, step = 0;
        for (; step < hops; ++step) {
            if ((pos[cur] & ~((1ll << 40) - 1)) == tag) break;
            pos[cur] = tag | step;
            int64_t nxt = succ[cur];
            if (nxt == cur) break;
            cur = nxt;
        }
        walked[pass] = step;
    }
    for (int64_t i = 0; i < hops; ++i) rank[i] = (n - 1) - (pos[i] & ((1ll << 40) - 1));
    *anomalies = bad + loops; /* range violations + self-loops in the scanned prefix */
    return walked[0] < walked[1] ? walked[0] : walked[1];
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

double orc_now(void) { return now_s(); }
