// softposit_style.cu -- CONTROL kernel for the Table tabrandom / tabprof
// analog: a Posit(32,2) add written the way the paper
// describes its GPU port of SoftPosit: decode by a
// sequential scan of the regime bits, encode by a loop that emits the regime,
// normalise by shifting one bit at a time.  Correctly rounded (RNE on the
// encoding), so it must produce the same bits as the product path's
// branch-free add (csrc/posit32.cuh); its cost depends on the operand
// magnitudes, which is what the paper measures on V100 (81-283 instructions
// per add, 91-95% branch efficiency).  Not part of the product library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared \
//        -o tools/libsoftposit_style.so tools/softposit_style.cu
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

// value = (-1)^neg * (1.frac) * 2^scale, frac with `fb` bits
__device__ void loop_decode(uint32_t x, uint32_t& neg, int& scale, uint64_t& sig, int& fb) {
  neg = x >> 31;
  if (neg) x = 0u - x;
  int pos = 30;
  const uint32_t r = (x >> pos) & 1u;
  int m = 0;
  while (pos >= 0 && ((x >> pos) & 1u) == r) {   // the regime run, one bit per iteration
    m++;
    pos--;
  }
  const int k = r ? m - 1 : -m;
  pos--;                                          // the terminating bit
  int e = 0;
  for (int i = 0; i < 2; i++) {                   // exponent bits (missing ones read as 0)
    e <<= 1;
    if (pos >= 0) {
      e |= (x >> pos) & 1u;
      pos--;
    }
  }
  fb = pos + 1 > 0 ? pos + 1 : 0;
  const uint32_t f = fb > 0 ? (x & ((1u << fb) - 1u)) : 0u;
  scale = 4 * k + e;
  sig = ((uint64_t)1 << fb) | f;
}

// round (-1)^neg * S * 2^(E - 62) (S leading one at bit 62, sticky in bit 0) to a pattern
__device__ uint32_t loop_encode(uint32_t neg, int E, uint64_t S) {
  if (E >= 120) return neg ? 0u - 0x7FFFFFFFu : 0x7FFFFFFFu;
  if (E < -120) return neg ? 0u - 1u : 1u;
  int k = E >> 2;
  const int e = E & 3;
  // emit the bit string regime || e || fraction into a 64-bit window, one bit at a time
  uint64_t w = 0;
  int n = 0;
  if (k >= 0) {
    for (int i = 0; i <= k; i++) { w = (w << 1) | 1u; n++; }
    w <<= 1; n++;
  } else {
    for (int i = 0; i < -k; i++) { w <<= 1; n++; }
    w = (w << 1) | 1u; n++;
  }
  w = (w << 2) | (uint64_t)e;
  n += 2;
  // fraction bits: S without its leading one, keep 63 - n bits plus a sticky
  const uint64_t frac = S << 2;                   // drop the leading one (bit 62 -> out), left-aligned
  const int keep = 64 - n;
  uint64_t bits = (w << keep) | (frac >> n);
  const uint32_t sticky = (frac << keep) != 0;
  uint32_t p = (uint32_t)(bits >> 33);
  const uint32_t guard = (uint32_t)(bits >> 32) & 1u;
  const uint32_t st = ((uint32_t)bits != 0u) | sticky;
  p += guard & (st | (p & 1u));
  if (p == 0u) p = 1u;
  return neg ? 0u - p : p;
}

__device__ uint32_t loop_add(uint32_t a, uint32_t b) {
  if (a == 0x80000000u || b == 0x80000000u) return 0x80000000u;
  if (a == 0u) return b;
  if (b == 0u) return a;
  uint32_t na, nb;
  int ea, eb, fa, fbb;
  uint64_t sa, sb;
  loop_decode(a, na, ea, sa, fa);
  loop_decode(b, nb, eb, sb, fbb);
  // significands with the leading one at bit 62
  sa <<= (62 - fa);
  sb <<= (62 - fbb);
  if (eb > ea || (eb == ea && sb > sa)) {
    uint32_t tn = na; na = nb; nb = tn;
    int te = ea; ea = eb; eb = te;
    uint64_t ts = sa; sa = sb; sb = ts;
  }
  int d = ea - eb;
  uint32_t sticky = 0;
  while (d > 0 && sb != 0) {                      // align one bit at a time
    sticky |= (uint32_t)(sb & 1u);
    sb >>= 1;
    d--;
  }
  if (d > 0) sb = 0;
  uint64_t s = (na == nb) ? sa + sb : sa - sb - (uint64_t)(sticky && na != nb);
  if (sticky && na != nb) sticky = 1;
  if (s == 0 && !sticky) return 0u;
  int E = ea;
  if (s >> 63) {                                   // carry: one right shift
    sticky |= (uint32_t)(s & 1u);
    s >>= 1;
    E++;
  }
  while (!(s >> 62)) {                             // normalise one bit at a time
    s <<= 1;
    E--;
  }
  return loop_encode(na, E, s | sticky);
}

__global__ void k_vec_add_loop(const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = loop_add(a[i], b[i]);
}

}  // namespace

extern "C" int softposit_style_add(const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t n, void* stream) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  k_vec_add_loop<<<(unsigned)(g < 1 ? 1 : g), 256, 0, (cudaStream_t)stream>>>(a, b, out, n);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -101;
}
