/* Exhaustive check behind k_norm2's binary16 -> binary32 quotient
 * (gadi_kernels.cuh): for every pair of binary16 values 0 <= w <= m (m > 0
 * finite), Markstein's corrected product q1 = RN(q0 + RN(w - m q0) y) with
 * y = RN(1/m), q0 = RN(w y) equals RN32(w / m). Negative w is symmetric.
 *   gcc -O2 -mfma -fopenmp -ffp-contract=off tools/check_markstein.c -lm && ./a.out */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static float h2f(uint16_t h) {
  _Float16 x;
  memcpy(&x, &h, 2);
  return (float)x;
}
int main(void) {
  long bad = 0, tot = 0;
#pragma omp parallel for reduction(+ : bad, tot) schedule(dynamic, 64)
  for (int mi = 1; mi < 0x7c00; ++mi) {
    const float m = h2f((uint16_t)mi);
    const float y = (float)(1.0 / (double)m); /* RN(1/m): no double-rounding case for 11-bit m */
    for (int wi = 0; wi <= mi; ++wi) {
      const float w = h2f((uint16_t)wi);
      const float ref = (float)((double)w / (double)m);
      const float q0 = w * y;
      const float q1 = fmaf(fmaf(-q0, m, w), y, q0);
      ++tot;
      if (memcmp(&q1, &ref, 4)) ++bad;
    }
  }
  printf("pairs=%ld mismatches=%ld\n", tot, bad);
  return bad != 0;
}
