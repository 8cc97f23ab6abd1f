#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
static float u2f(uint32_t u){float f; memcpy(&f,&u,4); return f;}
static uint32_t f2u(float f){uint32_t u; memcpy(&u,&f,4); return u;}
int main(){
  uint64_t bad=0, tot=0; uint64_t s=88172645463325252ull;
  for (uint32_t d=1; d<=(1u<<17); d = d<64? d+1 : d + 1 + (d>>6)) {
    float df=(float)d; float r = 1.0f/df;  // correctly rounded (SSE)
    for (int t=0;t<200000;t++){
      s^=s<<13; s^=s>>7; s^=s<<17;
      float x;
      int mode = t%4;
      if (mode==0) x = u2f((uint32_t)(s>>32));            // any bit pattern
      else if (mode==1) x = ((float)(int32_t)(s>>33))/ (float)(1u<<30); // [-1,1)
      else if (mode==2) x = u2f(((uint32_t)(s>>32) & 0x807FFFFFu) | (((uint32_t)((s>>20)%60)+100u)<<23)); // moderate exponents
      else x = (float)(s%100000) * 0.5f;
      if (!isfinite(x)) continue;
      float want = x/df;
      float q = x*r;
      float e = fmaf(-q, df, x);
      float q2 = fmaf(e, r, q);
      tot++;
      if (f2u(q2)!=f2u(want)) { if (isnormal(want) || want==0) { bad++; if (bad<10) printf("d=%u x=%a want=%a got=%a\n", d, x, want, q2);} }
    }
  }
  printf("tot=%llu bad(normal results)=%llu\n",(unsigned long long)tot,(unsigned long long)bad);
}
