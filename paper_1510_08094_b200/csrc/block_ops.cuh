// Block-wide scans and reductions (warp shuffles + one shared-memory slot per
// warp).  Used by the partitioned tridiagonal solve of the theta stage.
#pragma once

#include <cuda_runtime.h>

namespace sk {

struct V4 {
    double a, b, c, d;
};

__device__ __forceinline__ V4 shfl_up4(V4 v, int delta) {
    V4 r;
    r.a = __shfl_up_sync(0xffffffffu, v.a, delta);
    r.b = __shfl_up_sync(0xffffffffu, v.b, delta);
    r.c = __shfl_up_sync(0xffffffffu, v.c, delta);
    r.d = __shfl_up_sync(0xffffffffu, v.d, delta);
    return r;
}
__device__ __forceinline__ V4 shfl_down4(V4 v, int delta) {
    V4 r;
    r.a = __shfl_down_sync(0xffffffffu, v.a, delta);
    r.b = __shfl_down_sync(0xffffffffu, v.b, delta);
    r.c = __shfl_down_sync(0xffffffffu, v.c, delta);
    r.d = __shfl_down_sync(0xffffffffu, v.d, delta);
    return r;
}

// Exclusive scan over the CTA in thread order (REV = false) or reverse thread
// order (REV = true).  Op::combine(earlier, later) composes two elements,
// Op::identity() is its neutral element.  blockDim.x must be a multiple of 32
// and <= 1024; `wsc` needs 32 V4 slots.  Ends with a barrier.
template <class Op, bool REV>
__device__ V4 block_exclusive_scan(V4 v, V4* wsc) {
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int nw = nthr >> 5;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // position of this thread in scan order
    const int vlane = REV ? 31 - lane : lane;
    const int vwarp = REV ? nw - 1 - warp : warp;
    // inclusive warp scan in scan order
    V4 inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const V4 o = REV ? shfl_down4(inc, off) : shfl_up4(inc, off);
        if (vlane >= off) inc = Op::combine(o, inc);
    }
    if (vlane == 31) wsc[vwarp] = inc;
    __syncthreads();
    if (warp == 0) {
        V4 t = lane < nw ? wsc[lane] : Op::identity();
        // inclusive scan of warp totals (natural lane order = scan order here)
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const V4 o = shfl_up4(t, off);
            if (lane >= off) t = Op::combine(o, t);
        }
        // exclusive warp prefixes
        const V4 prev = shfl_up4(t, 1);
        if (lane < nw) wsc[lane] = lane == 0 ? Op::identity() : prev;
    }
    __syncthreads();
    const V4 wpre = wsc[vwarp];
    // exclusive within the warp
    V4 ex = REV ? shfl_down4(inc, 1) : shfl_up4(inc, 1);
    if (vlane == 0) ex = Op::identity();
    const V4 res = Op::combine(wpre, ex);
    __syncthreads();
    return res;
}

// 2x2 Moebius matrices [[a, b], [c, d]]; later * earlier, rescaled.
struct MobOp {
    __device__ static V4 identity() { return V4{1.0, 0.0, 0.0, 1.0}; }
    __device__ static V4 combine(V4 e, V4 l) {
        V4 r{l.a * e.a + l.b * e.c, l.a * e.b + l.b * e.d, l.c * e.a + l.d * e.c, l.c * e.b + l.d * e.d};
        const double m = fmax(fmax(fabs(r.a), fabs(r.b)), fmax(fabs(r.c), fabs(r.d)));
        if (m > 0.0 && (m > 1e150 || m < 1e-150)) {
            const double s = 1.0 / m;
            r.a *= s;
            r.b *= s;
            r.c *= s;
            r.d *= s;
        }
        return r;
    }
};

// Affine maps x -> a x + (b + i c) with real a: later o earlier.
struct AffOp {
    __device__ static V4 identity() { return V4{1.0, 0.0, 0.0, 0.0}; }
    __device__ static V4 combine(V4 e, V4 l) { return V4{l.a * e.a, fma(l.a, e.b, l.b), fma(l.a, e.c, l.c), 0.0}; }
};

// Affine maps x -> a x + (b + i c) with real a, three doubles (the scans of
// the chain solve shuffle 3 instead of 4 doubles per step).
struct Aff3 {
    double a, b, c;
};
__device__ __forceinline__ Aff3 aff_identity() { return Aff3{1.0, 0.0, 0.0}; }
// later o earlier
__device__ __forceinline__ Aff3 aff_combine(Aff3 e, Aff3 l) {
    return Aff3{l.a * e.a, fma(l.a, e.b, l.b), fma(l.a, e.c, l.c)};
}
template <bool UP>
__device__ __forceinline__ Aff3 shfl_aff(Aff3 v, int delta) {
    Aff3 r;
    if constexpr (UP) {
        r.a = __shfl_up_sync(0xffffffffu, v.a, delta);
        r.b = __shfl_up_sync(0xffffffffu, v.b, delta);
        r.c = __shfl_up_sync(0xffffffffu, v.c, delta);
    } else {
        r.a = __shfl_down_sync(0xffffffffu, v.a, delta);
        r.b = __shfl_down_sync(0xffffffffu, v.b, delta);
        r.c = __shfl_down_sync(0xffffffffu, v.c, delta);
    }
    return r;
}

// Exclusive scan of affine maps over the CTA in thread order (REV = false) or
// reverse thread order (REV = true); `wsc` needs 32 slots.  Ends with a barrier.
template <bool REV>
__device__ __forceinline__ Aff3 block_scan_aff(Aff3 v, Aff3* wsc) {
    const int tid = threadIdx.x;
    const int nw = blockDim.x >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    const int vlane = REV ? 31 - lane : lane;
    const int vwarp = REV ? nw - 1 - warp : warp;
    Aff3 inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const Aff3 o = shfl_aff<!REV>(inc, off);
        if (vlane >= off) inc = aff_combine(o, inc);
    }
    if (vlane == 31) wsc[vwarp] = inc;
    __syncthreads();
    if (warp == 0) {
        Aff3 t = lane < nw ? wsc[lane] : aff_identity();
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const Aff3 o = shfl_aff<true>(t, off);
            if (lane >= off) t = aff_combine(o, t);
        }
        const Aff3 prev = shfl_aff<true>(t, 1);
        if (lane < nw) wsc[lane] = lane == 0 ? aff_identity() : prev;
    }
    __syncthreads();
    const Aff3 wpre = wsc[vwarp];
    Aff3 ex = shfl_aff<!REV>(inc, 1);
    if (vlane == 0) ex = aff_identity();
    const Aff3 res = aff_combine(wpre, ex);
    __syncthreads();
    return res;
}

// Segmented variant: the CTA's warps form 2 equal segments (warps
// [0, nw/2) and [nw/2, nw)), each scanned independently in thread order
// (REV = false) or reverse thread order (REV = true) within the segment.
template <bool REV>
__device__ __forceinline__ Aff3 block_scan_aff_seg2(Aff3 v, Aff3* wsc) {
    const int tid = threadIdx.x;
    const int nw = blockDim.x >> 5;
    const int segw = nw >> 1;
    const int lane = tid & 31, warp = tid >> 5;
    const int seg = warp / segw, wi = warp - seg * segw;
    const int vlane = REV ? 31 - lane : lane;
    const int slot = seg * segw + (REV ? segw - 1 - wi : wi);
    Aff3 inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const Aff3 o = shfl_aff<!REV>(inc, off);
        if (vlane >= off) inc = aff_combine(o, inc);
    }
    if (vlane == 31) wsc[slot] = inc;
    __syncthreads();
    if (warp == 0) {
        Aff3 t = lane < nw ? wsc[lane] : aff_identity();
        const int li = lane % segw;
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const Aff3 o = shfl_aff<true>(t, off);
            if (li >= off) t = aff_combine(o, t);
        }
        const Aff3 prev = shfl_aff<true>(t, 1);
        if (lane < nw) wsc[lane] = li == 0 ? aff_identity() : prev;
    }
    __syncthreads();
    const Aff3 wpre = wsc[slot];
    Aff3 ex = shfl_aff<!REV>(inc, 1);
    if (vlane == 0) ex = aff_identity();
    const Aff3 res = aff_combine(wpre, ex);
    __syncthreads();
    return res;
}

// One-barrier variant: after the warp totals are published, every warp scans
// them itself (lanes < nw) instead of waiting for warp 0, and there is no
// trailing barrier — callers alternate two `slots` arrays (nw entries each)
// between consecutive scans so that a fast warp's next publication cannot
// overwrite totals a slow warp is still reading.  The barrier orders every
// shared-memory access made before the call against those made after it.
template <bool REV>
__device__ __forceinline__ Aff3 block_scan_aff1(Aff3 v, Aff3* slots) {
    const int tid = threadIdx.x;
    const int nw = blockDim.x >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    const int vlane = REV ? 31 - lane : lane;
    const int vwarp = REV ? nw - 1 - warp : warp;
    Aff3 inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const Aff3 o = shfl_aff<!REV>(inc, off);
        if (vlane >= off) inc = aff_combine(o, inc);
    }
    if (vlane == 31) slots[vwarp] = inc;
    __syncthreads();
    Aff3 t = lane < nw ? slots[lane] : aff_identity();
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        if (off >= nw) break;
        const Aff3 o = shfl_aff<true>(t, off);
        if (lane >= off) t = aff_combine(o, t);
    }
    Aff3 pre;
    pre.a = __shfl_sync(0xffffffffu, t.a, vwarp > 0 ? vwarp - 1 : 0);
    pre.b = __shfl_sync(0xffffffffu, t.b, vwarp > 0 ? vwarp - 1 : 0);
    pre.c = __shfl_sync(0xffffffffu, t.c, vwarp > 0 ? vwarp - 1 : 0);
    if (vwarp == 0) pre = aff_identity();
    Aff3 ex = shfl_aff<!REV>(inc, 1);
    if (vlane == 0) ex = aff_identity();
    return aff_combine(pre, ex);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// Sum of (x, y) pairs over the CTA; result valid in every thread. `red` needs
// 64 doubles.  Ends with a barrier.
__device__ __forceinline__ double2 block_sum2(double2 v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    if (lane == 0) {
        red[2 * warp] = v.x;
        red[2 * warp + 1] = v.y;
    }
    __syncthreads();
    double2 t = make_double2(0.0, 0.0);
    for (int w = 0; w < nw; ++w) {
        t.x += red[2 * w];
        t.y += red[2 * w + 1];
    }
    __syncthreads();
    return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t = fmax(t, red[w]);
    __syncthreads();
    return t;
}

// atomic max of a non-negative double (IEEE order == unsigned order)
// (the maximum only grows: a plain read first spares the atomic whenever the
// stored value already dominates — hundreds of thousands of CTAs update one
// address in the multi-pass theta stage, and same-address atomics serialise)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    if (bits > *reinterpret_cast<volatile unsigned long long*>(addr))
        atomicMax(reinterpret_cast<unsigned long long*>(addr), bits);
}

}  // namespace sk
