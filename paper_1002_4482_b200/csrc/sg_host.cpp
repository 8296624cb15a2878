// sg_host.cpp -- host-side helpers of libsg: the KISS64 recurrence for host
// generation (gen.py:51-64) and the error-path list validation that builds
// the reference's exact InvalidListError message (core.py:113-167).  Neither
// computes a ranking or a labelling: the product path has no CPU fallback.
#include <stdint.h>
#include <stdlib.h>

#include <vector>

#include "sg.h"

extern "C" {

int sg_kiss_batch_host(uint64_t* state, uint64_t n, uint64_t* out) {
    uint64_t x = state[0], y = state[1], z = state[2], c = state[3];
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t t = (x << 58) + c;
        c = x >> 6;
        x += t;
        c += x < t;
        y ^= y << 13;
        y ^= y >> 17;
        y ^= y << 43;
        z = 6906969069ull * z + 1234567ull;
        out[i] = x + y + z;
    }
    state[0] = x;
    state[1] = y;
    state[2] = z;
    state[3] = c;
    return SG_OK;
}

// First violation in the reference's report order: out-of-range, tail count,
// reachability of every node from the head (core.py:148-167).
int sg_list_violation_host(const int64_t* succ, uint64_t n, sg_violation* v) {
    v->kind = SG_LIST_OK;
    v->index = -1;
    v->pad = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (succ[i] < 0 || (uint64_t)succ[i] >= n) {
            v->kind = SG_LIST_OUT_OF_RANGE;
            v->index = (int64_t)i;
            return SG_OK;
        }
    }
    int64_t loops = 0, second = -1;
    for (uint64_t i = 0; i < n; ++i) {
        if ((uint64_t)succ[i] == i) {
            if (++loops == 2) second = (int64_t)i;
        }
    }
    if (loops == 0) {
        v->kind = SG_LIST_NO_TAIL;
        return SG_OK;
    }
    if (loops > 1) {
        v->kind = SG_LIST_MULTIPLE_SELF_LOOPS;
        v->index = second;
        return SG_OK;
    }
    std::vector<uint8_t> seen(n, 0);
    uint64_t cur = 0;
    for (uint64_t step = 0; step < n; ++step) {
        if (seen[cur]) break;
        seen[cur] = 1;
        const uint64_t nxt = (uint64_t)succ[cur];
        if (nxt == cur) break;
        cur = nxt;
    }
    for (uint64_t i = 0; i < n; ++i) {
        if (!seen[i]) {
            v->kind = SG_LIST_UNREACHABLE;
            v->index = (int64_t)i;
            return SG_OK;
        }
    }
    return SG_OK;
}

}  // extern "C"
