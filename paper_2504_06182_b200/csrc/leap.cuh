// Space-time meetings of one-bend routes (leap mode, batching.cu; window
// mode, batch_wide.cu).  A path with k of its len moves done at offset s is at
// P(t) = v(k + t - s), two linear pieces (horizontal, then vertical;
// virtual_line.cpp:150-173).
#pragma once

#include <climits>

namespace rb {

struct Seg {
    int x0, y0, vx, vy, t0, t1;  // position (x0 + vx t, y0 + vy t) for t in [t0, t1]
};

__device__ __forceinline__ void lane_segs(int k, int len, int xs, int ys, int xt, int yt, Seg &h, Seg &v) {
    const int dx = abs(xt - xs), sx = xt > xs ? 1 : -1, sy = yt > ys ? 1 : -1;
    h = Seg{xs + sx * k, ys, sx, 0, 0, dx - k};
    v = Seg{xt, ys + sy * (k - dx), 0, sy, max(0, dx - k), len - k};
}

// t / c for c in {+-1, +-2}; false when not an integer
__device__ __forceinline__ bool div12(int r, int c, int *t) {
    if (c & 1) {
        *t = r * c;
        return true;
    }
    if (r & 1) return false;
    *t = (r >> 1) * (c >> 1);
    return true;
}

// min t in [lo, hi] with (ax + avx t, ay + avy t) == (bx + bvx t, by + bvy t)
__device__ __forceinline__ int meet(int ax, int ay, int avx, int avy, int bx, int by, int bvx, int bvy, int lo,
                                    int hi) {
    const int cx = avx - bvx, rx = bx - ax, cy = avy - bvy, ry = by - ay;
    int t;
    if (cx == 0) {
        if (rx != 0) return INT_MAX;
    } else {
        if (!div12(rx, cx, &t)) return INT_MAX;
        lo = max(lo, t);
        hi = min(hi, t);
    }
    if (cy == 0) {
        if (ry != 0) return INT_MAX;
    } else {
        if (!div12(ry, cy, &t)) return INT_MAX;
        lo = max(lo, t);
        hi = min(hi, t);
    }
    return lo <= hi ? lo : INT_MAX;
}

// first offset t in [lo0, T] at which p (pieces a) is blocked by q (pieces b):
// P(t+1) == Q(t) (q's pre-batch vertex) or P(t+1) == Q(t+1) (same destination)
__device__ __forceinline__ int pair_event(const Seg *a, const Seg *b, int lo0, int T) {
    int best = INT_MAX;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            const Seg &A = a[u], &B = b[w];
            int lo = max(max(A.t0 - 1, B.t0), lo0), hi = min(min(A.t1 - 1, B.t1), T);
            if (lo <= hi) best = min(best, meet(A.x0 + A.vx, A.y0 + A.vy, A.vx, A.vy, B.x0, B.y0, B.vx, B.vy, lo, hi));
            lo = max(max(A.t0, B.t0), lo0 + 1);
            hi = min(min(A.t1, B.t1), T + 1);
            if (lo <= hi) {
                const int s = meet(A.x0, A.y0, A.vx, A.vy, B.x0, B.y0, B.vx, B.vy, lo, hi);
                if (s != INT_MAX) best = min(best, s - 1);
            }
        }
    return best;
}

// the pieces of a path that starts moving at offset s (absolute offsets)
__device__ __forceinline__ void shift_segs(Seg *g, int s) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        g[u].x0 -= g[u].vx * s;
        g[u].y0 -= g[u].vy * s;
        g[u].t0 += s;
        g[u].t1 += s;
    }
}

}  // namespace rb
