// Double-double arithmetic (value = hi + lo, |lo| <= ulp(hi)/2).
//
// Why: the O(1) filter cancels running sums of magnitude ~D^{4r} down to an
// output of magnitude ~1; the taps, interpolation
// weights and the signed accumulation carry ~106 bits.  Error-free
// transformations use the _rn intrinsics so nvcc never contracts them.
#pragma once
#include <cuda_runtime.h>

namespace bsf {

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_make(double a) { return {a, 0.0}; }

__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dadd_rn(s, -a);
    double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
    return {s, e};
}

__device__ __forceinline__ dd fast_two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double e = __dadd_rn(b, -__dadd_rn(s, -a));
    return {s, e};
}

__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    double e = __fma_rn(a, b, -p);
    return {p, e};
}

// accurate addition (Shewchuk/QD "ieee add")
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = fast_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return fast_two_sum(s.hi, s.lo);
}

// addition for operands of the same sign (no cancellation): 11 flops instead
// of 20, relative error <= 3u^2 (QD's "sloppy" add is accurate in this case).
// Used by the running sums of non-negative images.
__device__ __forceinline__ dd dd_add_same_sign(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    s.lo = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
    return fast_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__device__ __forceinline__ dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo = __dadd_rn(s.lo, a.lo);
    return fast_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, p.lo);
    p.lo = __fma_rn(a.lo, b.hi, p.lo);
    return fast_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return fast_two_sum(p.hi, p.lo);
}

// a*b + c
__device__ __forceinline__ dd dd_fma(dd a, dd b, dd c) { return dd_add(dd_mul(a, b), c); }

__device__ __forceinline__ double dd_to_d(dd a) { return __dadd_rn(a.hi, a.lo); }

// floor of a double-double (integral double) and the fractional part in [0,1)
__device__ __forceinline__ double dd_floor(dd a, dd *frac) {
    double f = floor(a.hi);
    if (f == a.hi && a.lo < 0.0) f -= 1.0;
    // a.hi - f is not exact for a.hi in (-1, 0) (no Sterbenz), so keep its error
    dd t = two_sum(a.hi, -f);
    t.lo = __dadd_rn(t.lo, a.lo);
    *frac = fast_two_sum(t.hi, t.lo);
    return f;
}

}  // namespace bsf
