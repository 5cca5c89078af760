// pipebench.cu -- measured integer-pipe throughput on this GPU (warp-instructions
// per SM per clock) for the instruction classes of the posit MAC.  Each thread
// runs 8 independent chains; the instruction is forced with inline PTX and
// checked in SASS.  Output: one JSON object.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
template <int OP>
__global__ void kern(unsigned* out, unsigned seed, long long* cyc) {
  unsigned r[CH];
  for (int i = 0; i < CH; i++) r[i] = seed * (threadIdx.x + 1) + i;
  unsigned b = seed ^ 0x1234567u, c = seed + 77u;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(b));
      if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 2) asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(r[i]) : "r"(c));
      if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 4) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 5) asm volatile("bfind.u32 %0, %0;" : "+r"(r[i]));
      if (OP == 6) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.b32 %0, %1, %2, p;}" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 7) { if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
                     else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(b), "r"(c)); }
      if (OP == 8) asm volatile("add.cc.u32 %0, %0, %1; addc.u32 %0, %0, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 9) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 10) { double d = __longlong_as_double(((long long)r[i] << 20) | 0x3FF0000000000000ll);
                      asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(d)); r[i] = (unsigned)__double_as_longlong(d); }
      if (OP == 11) asm volatile("add.u32 %0, %0, %1; add.u32 %0, %0, %2;" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 12) asm volatile("shr.u32 %0, %0, 3; add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(b));
      if (OP == 13) asm volatile("min.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(b));
      if (OP == 14) asm volatile("abs.s32 %0, %0;" : "+r"(r[i]));
      if (OP == 15) { unsigned lo, hi; asm volatile("mul.wide.u32 %0, %2, %3;" : "=l"(*(unsigned long long*)&lo) : "r"(0), "r"(r[i]), "r"(b)); }
      if (OP == 16) asm volatile("{.reg .u64 w; mul.wide.u32 w, %0, %1; cvt.u32.u64 %0, w;}" : "+r"(r[i]) : "r"(b));
      if (OP == 17) asm volatile("{.reg .u64 w; .reg .u32 l, h; mul.wide.u32 w, %0, %1; mov.b64 {l, h}, w; xor.b32 %0, l, h;}" : "+r"(r[i]) : "r"(b));
      if (OP == 18) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(r[i]) : "r"(b));
      if (OP == 19) asm volatile("shf.r.clamp.b32 %0, %0, %1, %0;" : "+r"(r[i]) : "r"(c));
      if (OP == 20) asm volatile("{.reg .f32 f; cvt.rn.f32.u32 f, %0; mov.b32 %0, f;}" : "+r"(r[i]));
      if (OP == 21) asm volatile("{.reg .u32 t; add.cc.u32 t, %0, %1; addc.u32 %0, %0, %2;}" : "+r"(r[i]) : "r"(b), "r"(c));
      if (OP == 22) asm volatile("{.reg .f64 d; mov.b64 d, {%0, %1}; fma.rn.f64 d, d, d, d; mov.b64 {%0, %1}, d;}" : "+r"(r[i]) : "r"(b));
      if (OP == 23) asm volatile("popc.b32 %0, %0;" : "+r"(r[i]));
      if (OP == 24) asm volatile("add.u32 %0, %0, 77;" : "+r"(r[i]));
      if (OP == 25) asm volatile("{.reg .u32 t; .reg .pred p; setp.ne.u32 p, %0, 0; selp.u32 t, 1, 0, p; or.b32 %0, %0, t;}" : "+r"(r[i]));
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
  for (int i = 0; i < CH; i++) acc ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
double run(const char* name, int per_instr, unsigned* out, long long* cyc, int nsm, bool last) {
  const int threads = 1024, blocks = nsm * 2;
  kern<OP><<<blocks, threads>>>(out, 3u, cyc);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  // warp-instructions per SM per clock: 2 CTAs/SM x 32 warps x ITERS x CH x per_instr / cycles
  double rate = 2.0 * 32 * ITERS * CH * per_instr / mx;
  printf("  \"%s\": %.3f%s\n", name, rate, last ? "" : ",");
  return rate;
}

// binary64 pipe: CH independent chains of real double registers per thread
template <int OP>
__global__ void kernd(unsigned* out, unsigned seed, long long* cyc) {
  double r[CH];
  unsigned q[CH];
  for (int i = 0; i < CH; i++) { r[i] = 1.0 + 1e-9 * (seed * (threadIdx.x + 1) + i); q[i] = seed * (threadIdx.x + 1) + i; }
  const double b = 1.0000001, c = -0.5e-7;
  const unsigned ib = seed ^ 0x1234567u, ic = seed + 77u;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) {
      if (OP == 0) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(c));
      if (OP == 1) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(r[i]) : "d"(b), "d"(c));
      if (OP == 2) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(b));
      if (OP == 3) asm volatile("add.rm.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(c));
      if (OP == 4) { asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(c));
                     asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(q[i]) : "r"(ib), "r"(ic)); }
      if (OP == 5) { asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(c));
                     asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(q[i]) : "r"(ib), "r"(ic)); }
      if (OP == 6) { asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(r[i]) : "d"(c));
                     asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(q[i]) : "r"(ib), "r"(ic));
                     asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(q[i]) : "r"(ib), "r"(ic)); }
    }
  }
  long long t1 = clock64();
  double acc = 0; unsigned u = 0;
  for (int i = 0; i < CH; i++) { acc += r[i]; u ^= q[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)__double2loint(acc) ^ u;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
double rund(const char* name, int per_instr, unsigned* out, long long* cyc, int nsm, bool last) {
  const int threads = 1024, blocks = nsm * 2;
  kernd<OP><<<blocks, threads>>>(out, 3u, cyc);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < blocks; i++) mx = h[i] > mx ? h[i] : mx;
  double rate = 2.0 * 32 * ITERS * CH * per_instr / mx;
  printf("  \"%s\": %.3f%s\n", name, rate, last ? "" : ",");
  return rate;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; long long* cyc;
  cudaMalloc(&out, sizeof(unsigned) * nsm * 2 * 1024); cudaMalloc(&cyc, sizeof(long long) * 4096);
  printf("{\n  \"units\": \"warp-instructions per SM per clock (issue limit 4)\",\n  \"sm_count\": %d,\n", nsm);
  run<0>("add.u32", 1, out, cyc, nsm, false);
  run<1>("lop3", 1, out, cyc, nsm, false);
  run<2>("shf", 1, out, cyc, nsm, false);
  run<3>("mad.lo (IMAD)", 1, out, cyc, nsm, false);
  run<4>("mad.hi (IMAD.HI)", 1, out, cyc, nsm, false);
  run<5>("bfind (FLO)", 1, out, cyc, nsm, false);
  run<6>("setp+selp (ISETP+SEL)", 2, out, cyc, nsm, false);
  run<7>("mad.lo/lop3 mix", 1, out, cyc, nsm, false);
  run<8>("add.cc+addc", 2, out, cyc, nsm, false);
  run<9>("fma.f32 (FFMA)", 1, out, cyc, nsm, false);
  run<11>("add+add 3-operand", 2, out, cyc, nsm, false);
  run<12>("shr+add (LEA.HI)", 2, out, cyc, nsm, false);
  run<13>("min.u32 (IMNMX)", 1, out, cyc, nsm, false);
  run<14>("abs (IABS)", 1, out, cyc, nsm, false);
  run<16>("mul.wide.u32 lo (IMAD.WIDE?)", 1, out, cyc, nsm, false);
  run<17>("mul.wide.u32 + xor (IMAD.WIDE + LOP3)", 2, out, cyc, nsm, false);
  run<18>("mad.hi.u32 with addend", 1, out, cyc, nsm, false);
  run<19>("shf.r.clamp funnel", 1, out, cyc, nsm, false);
  run<20>("cvt.rn.f32.u32 (I2F)", 1, out, cyc, nsm, false);
  run<21>("add.cc + addc pair", 2, out, cyc, nsm, false);
  run<22>("fma.rn.f64 (DFMA)", 1, out, cyc, nsm, false);
  run<23>("popc (POPC)", 1, out, cyc, nsm, false);
  run<24>("add.u32 imm (VIADD?)", 1, out, cyc, nsm, false);
  run<25>("setp+selp+or", 3, out, cyc, nsm, false);
  rund<0>("f64 add.rn (DADD)", 1, out, cyc, nsm, false);
  rund<1>("f64 fma.rn (DFMA)", 1, out, cyc, nsm, false);
  rund<2>("f64 mul.rn (DMUL)", 1, out, cyc, nsm, false);
  rund<3>("f64 add.rm (DADD.RM)", 1, out, cyc, nsm, false);
  rund<4>("DADD + LOP3 (1:1)", 2, out, cyc, nsm, false);
  rund<5>("DADD + IMAD (1:1)", 2, out, cyc, nsm, false);
  rund<6>("DADD + LOP3 + IMAD (1:1:1)", 3, out, cyc, nsm, true);
  printf("}\n");
  return 0;
}
