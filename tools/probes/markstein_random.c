// Host check of the Markstein-corrected division used by the Jacobi kernels.
// gcc -O2 -ffp-contract=off markstein_random.c -lm
// Empirical check of the Markstein correction: y = RN(1/d); q = RN(a*y);
// r = fma(-d, q, a); q' = fma(r, y, q) == RN(a/d) ?
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ull;
static inline uint64_t xr(void){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
static inline double bits(uint64_t u){ double d; memcpy(&d,&u,8); return d; }
int main(int argc, char** argv){
  double ds[] = {6.0, 4.0+2e-3, 26.0, 4.0, 3.0, 7.0, 12.0, 1.0/3.0, 0.1, 2.0/3.0, 6.002, 5.0, 11.0, 13.0, 4.004, 8.0+1e-3, -6.0, 1.5};
  long bad=0, tot=0;
  int nd = sizeof ds/sizeof ds[0];
  for (int k=0;k<nd+2000;k++){
    double d = k<nd ? ds[k] : bits((xr() & 0x800fffffffffffffull) | ((uint64_t)(1023 - 60 + xr()%120) << 52));
    double y = 1.0/d;
    for (long i=0;i<(k<nd?200000000L:2000000L);i++){
      uint64_t u = xr();
      // exponent within a safe range
      double a = bits((u & 0x800fffffffffffffull) | ((uint64_t)(1023 - 300 + (u>>52)%600) << 52));
      if (i & 1) a = bits(u & 0x800fffffffffffffull | ((uint64_t)(1023 + ((u>>52)&31) - 16) << 52)); // near 1
      double q = a*y;
      double r = fma(-d, q, a);
      double q2 = fma(r, y, q);
      double ref = a/d;
      tot++;
      if (memcmp(&q2,&ref,8)) { if (bad<10) printf("mismatch a=%a d=%a got %a ref %a\n",a,d,q2,ref); bad++; }
    }
  }
  printf("tested %ld bad %ld\n", tot, bad);
  return 0;
}
