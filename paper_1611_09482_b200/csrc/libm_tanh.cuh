// Double-precision tanh with the host libm's exact rounding, for the plain-mode kernels.
//
// The reference's node kernel ends with libm's tanh (numba lowers np.tanh / math.tanh to a
// call into the platform libm, kernel.py:54-55). CUDA's tanh() differs from it in the last
// ulp for some arguments, and a deep tanh stack amplifies one ulp into a visible deviation.
// This restates the published algorithm the host libm (glibc, x86-64) uses: fdlibm's tanh
// over expm1 (Sun Microsystems, 1993) with glibc's Estrin evaluation of expm1's rational
// correction, compiled -- as glibc's build is -- with a*b+c contracted to fused
// multiply-adds. Every operation below is an explicit IEEE intrinsic (__fma_rn, __dmul_rn,
// __dadd_rn, __ddiv_rn, ...) so nvcc cannot re-associate or contract anything else.
// Checked bit-for-bit against the host's math.tanh on 2.4M arguments spanning 1e-20..40
// (tests/test_oracle_plain.py::test_libm_tanh_restatement runs the same algorithm in Python
// against math.tanh; tests/test_gpu_plain.py checks the device copy).
#pragma once

namespace fw {

__device__ __forceinline__ double fw_expm1(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
               invln2 = 1.44269504088896338700e+00;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  const unsigned hx0 = (unsigned)__double2hiint(x);
  const unsigned xsb = hx0 & 0x80000000u;
  const unsigned hx = hx0 & 0x7fffffffu;
  // tanh calls this with |x| <= 44 and x = -2|y| for |y| < 1: no overflow or NaN branches
  if (hx >= 0x4043687Au && xsb) return -1.0;  // x < -56 ln2
  double hi, lo, c = 0.0;
  int k = 0;
  if (hx > 0x3fd62e42u) {    // |x| > 0.5 ln2
    if (hx < 0x3FF0A2B2u) {  // and < 1.5 ln2
      if (!xsb) {
        hi = __dsub_rn(x, ln2_hi);
        lo = ln2_lo;
        k = 1;
      } else {
        hi = __dadd_rn(x, ln2_hi);
        lo = -ln2_lo;
        k = -1;
      }
    } else {
      k = (int)__fma_rn(invln2, x, xsb ? -0.5 : 0.5);  // truncation, as C's conversion
      const double t = (double)k;
      hi = __fma_rn(-t, ln2_hi, x);  // exact
      lo = __dmul_rn(t, ln2_lo);
    }
    x = __dsub_rn(hi, lo);
    c = __dsub_rn(__dsub_rn(hi, x), lo);
  } else if (hx < 0x3c900000u) {  // |x| < 2^-54
    return x;
  }
  const double hfx = __dmul_rn(0.5, x);
  const double hxs = __dmul_rn(x, hfx);
  const double R1 = __fma_rn(hxs, Q1, 1.0);
  const double h2 = __dmul_rn(hxs, hxs);
  const double R2 = __fma_rn(hxs, Q3, Q2);
  const double h4 = __dmul_rn(h2, h2);
  const double R3 = __fma_rn(hxs, Q5, Q4);
  const double r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
  double t = __fma_rn(-r1, hfx, 3.0);
  double e = __dmul_rn(hxs, __ddiv_rn(__dsub_rn(r1, t), __fma_rn(-x, t, 6.0)));
  if (k == 0) return __dsub_rn(x, __fma_rn(x, e, -hxs));
  const double twopk = __hiloint2double(0x3ff00000 + (k << 20), 0);
  e = __fma_rn(x, __dsub_rn(e, c), -c);
  e = __dsub_rn(e, hxs);
  if (k == -1) return __fma_rn(0.5, __dsub_rn(x, e), -0.5);
  if (k == 1) {
    if (x < -0.25) return __dmul_rn(-2.0, __dsub_rn(e, __dadd_rn(x, 0.5)));
    return __fma_rn(2.0, __dsub_rn(x, e), 1.0);
  }
  double y;
  if (k <= -2 || k > 56) {
    y = __dsub_rn(1.0, __dsub_rn(e, x));
    y = __dmul_rn(y, twopk);
    return __dsub_rn(y, 1.0);
  }
  if (k < 20) {
    t = __hiloint2double(0x3ff00000 - (0x200000 >> k), 0);  // 1 - 2^-k
    y = __dsub_rn(t, __dsub_rn(e, x));
    y = __dmul_rn(y, twopk);
  } else {
    t = __hiloint2double((0x3ff - k) << 20, 0);  // 2^-k
    y = __dsub_rn(x, __dadd_rn(e, t));
    y = __dadd_rn(y, 1.0);
    y = __dmul_rn(y, twopk);
  }
  return y;
}

__device__ __forceinline__ double libm_tanh(double x) {
  const unsigned jx = (unsigned)__double2hiint(x);
  const unsigned ix = jx & 0x7fffffffu;
  if (ix >= 0x7ff00000u) return x != x ? x : ((jx >> 31) ? -1.0 : 1.0);  // NaN, +-inf
  double z;
  if (ix < 0x40360000u) {  // |x| < 22
    if (x == 0.0) return x;                                 // +-0
    if (ix < 0x3c800000u) return __dmul_rn(x, __dadd_rn(1.0, x));  // |x| < 2^-55
    const double ax = fabs(x);
    if (ix >= 0x3ff00000u) {  // |x| >= 1
      const double t = fw_expm1(__dmul_rn(2.0, ax));
      z = __dsub_rn(1.0, __ddiv_rn(2.0, __dadd_rn(t, 2.0)));
    } else {
      const double t = fw_expm1(__dmul_rn(-2.0, ax));
      z = __ddiv_rn(-t, __dadd_rn(t, 2.0));
    }
  } else {
    z = 1.0;  // |x| >= 22 (1 - tiny rounds to 1)
  }
  return (jx >> 31) ? -z : z;
}

}  // namespace fw
