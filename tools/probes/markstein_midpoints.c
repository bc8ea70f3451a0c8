// Host check of the Markstein-corrected division, midpoint-adjacent quotients.
// gcc -O2 -ffp-contract=off markstein_midpoints.c -lm
// Hard cases: a/d lands next to a rounding midpoint; plus all-ones-significand d.
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 1234567ull;
static inline uint64_t xr(void){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
static inline double bits(uint64_t u){ double d; memcpy(&d,&u,8); return d; }
static inline uint64_t ubits(double d){ uint64_t u; memcpy(&u,&d,8); return u; }
long bad=0, tot=0;
static void chk(double a, double d){
  double y=1.0/d, q=a*y, r=fma(-d,q,a), q2=fma(r,y,q), ref=a/d; tot++;
  if (memcmp(&q2,&ref,8)) { if (bad<10) printf("mismatch a=%a d=%a got %a ref %a\n",a,d,q2,ref); bad++; }
}
int main(){
  for (int k=0;k<4000;k++){
    double d;
    if (k%4==0) d = bits(((uint64_t)(1023 + (int)(xr()%40) - 20) << 52) | 0xfffffffffffffull); // all-ones significand
    else if (k%4==1) d = bits(((uint64_t)(1023 + (int)(xr()%40) - 20) << 52) | (0xfffffffffffffull - (xr()%64)));
    else d = bits(((uint64_t)(1023 + (int)(xr()%40) - 20) << 52) | (xr() & 0xfffffffffffffull));
    if (k < 8) d = (double[]){6.0,4.002,26.0,3.0,7.0,10.0,18.0,1.0/3.0}[k];
    for (int i=0;i<500000;i++){
      // q0 random, midpoint m = q0 + ulp/2; a near d*m (several neighbours)
      double q0 = bits(((uint64_t)(1023 + (int)(xr()%40) - 20) << 52) | (xr() & 0xfffffffffffffull));
      double up = nextafter(q0, INFINITY);
      long double m = ((long double)q0 + (long double)up) / 2;  // exact in 80-bit
      long double am = m * (long double)d;                        // ~ exact-ish
      double a = (double)am;
      chk(a, d); chk(nextafter(a, INFINITY), d); chk(nextafter(a, -INFINITY), d);
      // exact multiples: a = q0*d rounded
      chk(q0*d, d);
    }
  }
  printf("tested %ld bad %ld\n", tot, bad);
}
