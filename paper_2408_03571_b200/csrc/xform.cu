// Fast sine / cosine transforms along the rows of coarse vectors (part of K5,
// the coarse solve; see coarse.cu for the algorithm and the reference lines).
//
//   out[r][a] = s(r, a) * sum_J Q[J][a] in[r][J]
//   DCT-I (Sommerfeld): Q[J][a] = cos(pi a J / M),        M = m0 - 1, FFT length L = 2M = n - 1
//   DST-I (Dirichlet):  Q[J][a] = sin(pi (J+1)(a+1) / K), K = m0 + 1, FFT length L = 2K = n - 1
//   s(r, a) = 1, sig[a], or the 2-D Dirichlet eigenvalue scaling
//             qn / (lamT[a] lamM[kx] + lamM[a] lamT[kx] - k^2 lamM[a] lamM[kx]),  kx = r mod m0.
//
// A CTA runs FFTs of the symmetric extension (L/16 threads each) in shared
// memory: radix-8 Stockham stages (radix 4/2 for the remainder) in registers,
// in place through a barrier, twiddles tabulated once per CTA with sincospi.
// Real rows are packed two per FFT: Q is real, so DST(x + i y) = DST(x) + i DST(y).  Rows are read and written with coalesced
// 8/16-byte accesses; the transform is HBM-bound at the BASELINE sizes.
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace helm {

struct XScale {
  int accum;           // 1: out += result (iterative-refinement update), 0: out = result
  const double* sig;   // per-mode scale, or NULL
  const double* lamT;  // 2-D Dirichlet scaling (NULL: off)
  const double* lamM;
  double k2;
  double qn;
};

__device__ __forceinline__ double xscale(const XScale& s, int r, int a, int m0) {
  if (s.lamT) {
    const int kx = r % m0;
    return s.qn / (s.lamT[a] * s.lamM[kx] + s.lamM[a] * s.lamT[kx] - s.k2 * s.lamM[a] * s.lamM[kx]);
  }
  return s.sig ? s.sig[a] : 1.0;
}

// In-register 8-point DFT (natural order in and out): radix-2 decimation in frequency.
__device__ __forceinline__ void dft8(double2 v[8]) {
  constexpr double h = 0.70710678118654752440;
  const double2 w8[4] = {mk(1.0, 0.0), mk(h, -h), mk(0.0, -1.0), mk(-h, -h)};
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    const double2 t = sub(v[n], v[n + 4]);
    v[n] = add(v[n], v[n + 4]);
    v[n + 4] = mul(t, w8[n]);
  }
#pragma unroll
  for (int g = 0; g < 8; g += 4) {
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const double2 t = sub(v[g + n], v[g + n + 2]);
      v[g + n] = add(v[g + n], v[g + n + 2]);
      v[g + n + 2] = n ? mk(t.y, -t.x) : t;  // * (-i)^n
    }
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const double2 t = sub(v[i], v[i + 1]);
    v[i] = add(v[i], v[i + 1]);
    v[i + 1] = t;
  }
  // bit-reversed -> natural
  double2 t = v[1]; v[1] = v[4]; v[4] = t;
  t = v[3]; v[3] = v[6]; v[6] = t;
}
__device__ __forceinline__ void dft4(double2 v[4]) {
  const double2 a = add(v[0], v[2]), b = sub(v[0], v[2]), c = add(v[1], v[3]), d = sub(v[1], v[3]);
  v[0] = add(a, c);
  v[2] = sub(a, c);
  v[1] = mk(b.x + d.y, b.y - d.x);  // b - i d
  v[3] = mk(b.x - d.y, b.y + d.x);  // b + i d
}

// In-register 16-point DFT (natural order in and out) as 4 x 4: DFT4 over the stride-4
// subsequences, twiddles W16^(n2 k1), DFT4 across them.
__device__ __forceinline__ void dft16(double2 v[16]) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  // W16^m = exp(-2 pi i m / 16), m = 0 .. 9
  const double2 w[10] = {mk(1.0, 0.0), mk(c1, -s1), mk(h, -h), mk(s1, -c1), mk(0.0, -1.0),
                         mk(-s1, -c1), mk(-h, -h), mk(-c1, -s1), mk(-1.0, 0.0), mk(-c1, s1)};
  double2 y[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) y[n2][n1] = v[4 * n1 + n2];
    dft4(y[n2]);
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1)
      if (n2) y[n2][k1] = mul(y[n2][k1], w[n2 * k1]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 z[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
    dft4(z);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = z[k2];
  }
}

// Padded shared-memory index: one spare slot every 8 and every 64 elements, so the
// strided Stockham stores of the first stages (stride 8 and 64 double2) hit
// distinct bank groups.
__device__ __forceinline__ int pidx(int i) { return i + (i >> 3) + (i >> 6); }
__host__ __device__ constexpr int padded_len(int L) { return L + L / 8 + L / 64 + 1; }
// radix-16 stages store at stride 16 (first stage) and 256: one spare slot every 16 and 256
__device__ __forceinline__ int pidx16(int i) { return i + (i >> 4) + (i >> 8); }
__host__ __device__ constexpr int padded_len16(int L) { return L + L / 16 + L / 256 + 1; }
template <int VPT> __device__ __forceinline__ int pix(int i) { return VPT == 16 ? pidx16(i) : pidx(i); }

// One Stockham stage of radix R over a row of length L (T threads, NBT = 8/R butterflies
// each).  Butterfly j: inputs X[j + r L/R], twiddles W^r with W = W_{Ns R}^{j mod Ns}
// (plan-owned table in L1), outputs at (j / Ns) Ns R + (j mod Ns) + r Ns.
// FIRST: inputs come from `load(c, r, i)` (registers); LAST: outputs go to `store(i, v)` (global);
// otherwise through the padded shared buffer, in place across a barrier.
template <int VPT, int R, bool FIRST, bool LAST, typename LD, typename STO>
__device__ __forceinline__ void stockham_stage(double2* buf, const double2* __restrict__ tw, int L, int Ns, int tid,
                                               int T, LD load, STO store) {
  const int nb = L / R;
  constexpr int NBT = VPT / R;  // butterflies per thread (T = L / VPT threads per row)
  double2 v[NBT][R];
#pragma unroll
  for (int c = 0; c < NBT; ++c) {
    const int j = tid + c * T;
#pragma unroll
    for (int r = 0; r < R; ++r) v[c][r] = FIRST ? load(c, r, j + r * nb) : buf[pix<VPT>(j + r * nb)];
  }
  if (!FIRST) __syncthreads();
  const int tstep = L / (Ns * R);
#pragma unroll
  for (int c = 0; c < NBT; ++c) {
    const int j = tid + c * T;  // >= 0: unsigned division / modulo by the power-of-two Ns
    const int k = (int)((unsigned)j % (unsigned)Ns);
    if (!FIRST) {  // Ns == 1 on the first stage: all twiddles are 1
      // W^1 and W^2 from the table, the other powers by a depth-2 product tree
      // (2 loads instead of R-1: the load/store queue is this kernel's limiter)
      double2 w[16];
      w[1] = tw[k * tstep];
      if (R > 2) w[2] = tw[2 * k * tstep];
      if (R > 3) w[3] = mul(w[1], w[2]);
      if (R > 4) {
        w[4] = mul(w[2], w[2]);
        w[5] = mul(w[1], w[4]);
        w[6] = mul(w[2], w[4]);
        w[7] = mul(w[3], w[4]);
      }
      if (R > 8) {  // W^8 from the table, the rest by one product each
        w[8] = tw[8 * k * tstep];
#pragma unroll
        for (int r = 9; r < 16; ++r) w[r] = mul(w[r - 8], w[8]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[c][r] = mul(v[c][r], w[r]);
    }
    if constexpr (R == 16) {
      dft16(v[c]);
    } else if constexpr (R == 8) {
      dft8(v[c]);
    } else if constexpr (R == 4) {
      dft4(v[c]);
    } else {
      const double2 t2 = sub(v[c][0], v[c][1]);
      v[c][0] = add(v[c][0], v[c][1]);
      v[c][1] = t2;
    }
    const int base = (int)((unsigned)j / (unsigned)Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (LAST) store(base + r * Ns, v[c][r]);
      else buf[pix<VPT>(base + r * Ns)] = v[c][r];
    }
  }
  if (!LAST) __syncthreads();
}

// T = L/8 threads per row FFT (8 values in registers per thread); a CTA of
// blockDim threads transforms blockDim/T rows at a time.  The first radix-8 stage
// takes its inputs from registers that were loaded from HBM while the previous
// row was in its shared-memory stages (one row of prefetch per thread).
// The row length L (a power of two), the transform (DCT-I / DST-I) and hence m0 are
// template parameters: every index of the Stockham stages is then a shift or a mask
// (with a runtime L the integer divisions and index arithmetic were ~45 % of the issued
// instructions).
constexpr int fft_nst(int L) { return L <= 1 ? 0 : 1 + fft_nst(L >= 8 ? L / 8 : 1); }
constexpr int fft_rlast(int L) { return L <= 8 ? L : fft_rlast(L / 8); }
// VPT = 16 (L >= 256): a first radix-16 stage, radix-16 middle stages, a last stage of radix
// fft16_rlast (2..16): 2048 = 16 x 16 x 8 -- two shared-memory round trips instead of three
constexpr int fft16_nmid(int rem) { return rem <= 16 ? 0 : 1 + fft16_nmid(rem / 16); }
constexpr int fft16_rlast(int rem) { return rem <= 16 ? rem : fft16_rlast(rem / 16); }

// MINB = 2 (default for rows >= 1024): two CTAs per SM (128 registers, no spills) without the
// register prefetch of the next row -- the other CTA's stages cover the load instead.  Coarse solve
// 2.16 -> 2.12 ms per batch of 32, 0.286 -> 0.279 ms at batch 1; HELM_FFT_MINB=1 restores the
// one-CTA kernel with the prefetch (210 registers).
template <typename S, int VPT, int LT, bool DCT, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) xform_fft_kernel(const S* __restrict__ in, S* __restrict__ out, XScale sc,
                                                        int rows, const double2* __restrict__ tw) {
  constexpr int L = LT, m0 = DCT ? L / 2 + 1 : L / 2 - 1;
  constexpr bool dct = DCT;
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  static_assert(VPT == 8 || VPT == 16, "one radix-VPT butterfly per thread in the first stage");
  // tw: plan-owned table exp(-2 pi i k / L), k < L (read through L1)
  extern __shared__ __align__(16) unsigned char sraw[];
  constexpr int T = L / VPT;
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  const int rpc = blockDim.x / T;
  double2* buf = reinterpret_cast<double2*>(sraw) + (size_t)g * (VPT == 16 ? padded_len16(L) : padded_len(L));
  constexpr int RPF = Sc<S>::cplx ? 1 : 2;  // rows per FFT
  const int nfft = (rows + RPF - 1) / RPF;
  constexpr int K = L / 2;
  constexpr int nst = fft_nst(L), rlast = fft_rlast(L);
  // STAGED (MINB = 2, complex rows): the CTA's next rows (contiguous in memory) arrive by one
  // cp.async.bulk into a raw-row buffer behind the FFT buffers while the current rows are in
  // their shared-memory stages; the symmetric extension is then read from shared memory (each
  // element fetched from HBM once instead of twice, no global-load latency in the loop)
  constexpr bool STAGED = MINB != 1 && Sc<S>::cplx;
  double2* rawrows = reinterpret_cast<double2*>(sraw) + (size_t)rpc * (VPT == 16 ? padded_len16(L) : padded_len(L));
  __shared__ __align__(8) unsigned long long rawbar;
  auto raw_issue = [&](int fb) {  // thread 0: rows fb .. fb + rpc - 1 (clamped to nfft)
    const int nv = min(rpc, nfft - fb);
    if (nv <= 0) return;
    const unsigned bytes = (unsigned)nv * m0 * (unsigned)sizeof(double2);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&rawbar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(rawrows)),
                 "l"(reinterpret_cast<const double2*>(in) + (size_t)fb * m0), "r"(bytes), "r"(bar)
                 : "memory");
  };
  auto raw_wait = [&](unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n FFT_RAW_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FFT_RAW_WAIT;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(&rawbar)),
        "r"(parity)
        : "memory");
  };
  if constexpr (STAGED) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&rawbar))
                   : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      raw_issue(blockIdx.x * rpc);
    }
    __syncthreads();
  }
  // symmetric extension G(j) of FFT f (two real rows packed as re/im)
  auto load = [&](int f, int j) -> double2 {
    if (f >= nfft) return mk(0.0, 0.0);
    const int r0 = f * RPF;
    const S* row0 = in + (size_t)r0 * m0;
    int J;
    double sg = 1.0;
    if (dct) {
      J = j < K ? j : L - j;
    } else if (j == 0 || j == K) {
      return mk(0.0, 0.0);
    } else if (j < K) {
      J = j - 1;
    } else {
      J = L - j - 1;
      sg = -1.0;
    }
    if constexpr (STAGED) {
      const double2 x = rawrows[(size_t)g * m0 + J];
      return mk(sg * x.x, sg * x.y);
    } else if constexpr (Sc<S>::cplx) {
      const double2 x = row0[J];
      return mk(sg * x.x, sg * x.y);
    } else {
      return mk(sg * row0[J], (r0 + 1 < rows) ? sg * row0[m0 + J] : 0.0);
    }
  };
  double2 cur[VPT];
  int f = blockIdx.x * rpc + g;
  if constexpr (MINB == 1) {
#pragma unroll
    for (int r = 0; r < VPT; ++r) cur[r] = load(f, tid + r * T);
  }
  for (int f0 = blockIdx.x * rpc; f0 < nfft; f0 += gridDim.x * rpc) {
    f = f0 + g;
    double2 x0s = mk(0.0, 0.0), xms = mk(0.0, 0.0);
    if constexpr (MINB != 1) {
      if constexpr (STAGED) {
        raw_wait((unsigned)((f0 - blockIdx.x * rpc) / (gridDim.x * rpc)) & 1u);
        if (f < nfft) {
          x0s = rawrows[(size_t)g * m0];
          xms = rawrows[(size_t)g * m0 + m0 - 1];
        }
      }
#pragma unroll
      for (int r = 0; r < VPT; ++r) cur[r] = load(f, tid + r * T);
    }
    const bool active = f < nfft;
    const int r0 = (active ? f : 0) * RPF;
    const bool two = active && (RPF == 2) && (r0 + 1 < rows);
    // stage 1 from the prefetched registers, then prefetch the next row
    double2 nxt[VPT];
    {
      const double2* c = cur;
      stockham_stage<VPT, VPT, true, false>(buf, tw, L, 1, tid, T, [&](int, int r, int) { return c[r]; },
                                            [&](int, double2) {});
    }
    const int fn = f + gridDim.x * rpc;
    if constexpr (STAGED) {  // stage 1 ended with a CTA barrier: every thread has read its raw values
      if (threadIdx.x == 0) raw_issue(f0 + gridDim.x * rpc);
    }
    if constexpr (MINB == 1) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) nxt[r] = load(fn, tid + r * T);
    }
    // DFT index e -> transform output (sum_J Q[J][a] x_J, then the scale)
    const S* row0 = in + (size_t)r0 * m0;
    double2 x0 = mk(0.0, 0.0), xm = mk(0.0, 0.0);
    if (dct && active) {
      if constexpr (STAGED) {
        x0 = x0s;
        xm = xms;
      } else if constexpr (Sc<S>::cplx) {
        x0 = row0[0];
        xm = row0[m0 - 1];
      } else {
        x0 = mk(row0[0], two ? row0[m0] : 0.0);
        xm = mk(row0[m0 - 1], two ? row0[m0 + m0 - 1] : 0.0);
      }
    }
    auto store = [&](int e, double2 d) {
      if (!active) return;
      int a;
      double2 R;
      if (dct) {  // sum_J cos(pi a J/M) x_J = (DFT[a] + x_0 + (-1)^a x_M) / 2
        if (e > K) return;
        a = e;
        const double sgn = (a & 1) ? -1.0 : 1.0;
        R = mk(0.5 * (d.x + x0.x + sgn * xm.x), 0.5 * (d.y + x0.y + sgn * xm.y));
      } else {    // sum_J sin(pi (J+1)(a+1)/K) x_J = (i/2) DFT[a+1]
        if (e < 1 || e >= K) return;
        a = e - 1;
        R = mk(-0.5 * d.y, 0.5 * d.x);
      }
      if constexpr (Sc<S>::cplx) {
        S* o = out + (size_t)r0 * m0 + a;
        const S v = scale(R, xscale(sc, r0, a, m0));
        *o = sc.accum ? add(*o, v) : v;
      } else {
        S* o = out + (size_t)r0 * m0 + a;
        const S v = R.x * xscale(sc, r0, a, m0);
        *o = sc.accum ? *o + v : v;
        if (two) {
          const S v2 = R.y * xscale(sc, r0 + 1, a, m0);
          o[m0] = sc.accum ? o[m0] + v2 : v2;
        }
      }
    };
    auto none = [&](int, int, int) { return mk(0.0, 0.0); };
    if constexpr (VPT == 8) {
      int Ns = 8;
#pragma unroll
      for (int s = 1; s < nst; ++s) {
        const bool last = s == nst - 1;
        if (!last) {
          stockham_stage<8, 8, false, false>(buf, tw, L, Ns, tid, T, none, store);
          Ns *= 8;
        } else if (rlast == 8) {
          stockham_stage<8, 8, false, true>(buf, tw, L, Ns, tid, T, none, store);
        } else if (rlast == 4) {
          stockham_stage<8, 4, false, true>(buf, tw, L, Ns, tid, T, none, store);
        } else {
          stockham_stage<8, 2, false, true>(buf, tw, L, Ns, tid, T, none, store);
        }
      }
      if (nst == 1) {  // L == 8: the first stage was also the last; emit from smem
        __syncthreads();
        if (tid == 0)
          for (int e = 0; e < 8; ++e) store(e, buf[pidx(e)]);
      }
    } else {
      constexpr int nmid = fft16_nmid(L / 16), rl = fft16_rlast(L / 16);
      int Ns = 16;
#pragma unroll
      for (int s = 0; s < nmid; ++s) {
        stockham_stage<16, 16, false, false>(buf, tw, L, Ns, tid, T, none, store);
        Ns *= 16;
      }
      if constexpr (rl == 16) stockham_stage<16, 16, false, true>(buf, tw, L, Ns, tid, T, none, store);
      else if constexpr (rl == 8) stockham_stage<16, 8, false, true>(buf, tw, L, Ns, tid, T, none, store);
      else if constexpr (rl == 4) stockham_stage<16, 4, false, true>(buf, tw, L, Ns, tid, T, none, store);
      else stockham_stage<16, 2, false, true>(buf, tw, L, Ns, tid, T, none, store);
    }
    __syncthreads();
    if constexpr (MINB == 1) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) cur[r] = nxt[r];
    }
  }
}

static int fft_minb() {
  static const int v = [] {
    const char* e = getenv("HELM_FFT_MINB");
    return e ? atoi(e) : 2;
  }();
  return v;
}

template <typename S, int VPT, int L, bool DCT>
static void fft_launch_l(const S* in, S* out, const XScale& sc, int rows, const double2* tw, cudaStream_t st) {
  constexpr int T = L / VPT;
  const int threads = std::max(T, std::min(256, std::max(32, L)));
  const int rpc = threads / T;
  size_t smem = (size_t)(rpc * (VPT == 16 ? padded_len16(L) : padded_len(L))) * sizeof(double2);
  constexpr int m0c = DCT ? L / 2 + 1 : L / 2 - 1;
  const bool staged = VPT == 16 && L >= 1024 && Sc<S>::cplx && fft_minb() == 2;
  if (staged) smem += (size_t)rpc * m0c * sizeof(double2);  // the raw-row buffer of the staged kernel
  HELM_CHECK(smem <= 200 * 1024 && threads <= 256, "coarse FFT row too long");
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(xform_fft_kernel<S, VPT, L, DCT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024));
    if constexpr (VPT == 16 && L >= 1024)
      HELM_CUDA(cudaFuncSetAttribute(xform_fft_kernel<S, VPT, L, DCT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     110 * 1024));
    attr = true;
  }
  const int nfft = Sc<S>::cplx ? rows : (rows + 1) / 2;
  const int blocks = std::min((nfft + rpc - 1) / rpc, 148 * 4);
  if constexpr (VPT == 16 && L >= 1024) {
    if (fft_minb() == 2) {
      launch_pdl(xform_fft_kernel<S, VPT, L, DCT, 2>, blocks, threads, smem, st, in, out, sc, rows, tw);
      return;
    }
  }
  launch_pdl(xform_fft_kernel<S, VPT, L, DCT>, blocks, threads, smem, st, in, out, sc, rows, tw);
}

template <typename S, int VPT>
static void fft_launch(const S* in, S* out, const XScale& sc, int rows, int m0, int L, int dct, const double2* tw,
                       cudaStream_t st) {
  HELM_CHECK(m0 == (dct ? L / 2 + 1 : L / 2 - 1), "coarse FFT: m0 does not match the row length");
  auto go = [&](auto lc) {
    constexpr int LL = decltype(lc)::value;
    if constexpr (VPT == 16 && LL < 256) {
      HELM_CHECK(false, "the radix-16 coarse FFT needs rows of at least 256");
    } else {
      if (dct) fft_launch_l<S, VPT, LL, true>(in, out, sc, rows, tw, st);
      else fft_launch_l<S, VPT, LL, false>(in, out, sc, rows, tw, st);
    }
  };
  switch (L) {
    case 8: go(std::integral_constant<int, 8>{}); break;
    case 16: go(std::integral_constant<int, 16>{}); break;
    case 32: go(std::integral_constant<int, 32>{}); break;
    case 64: go(std::integral_constant<int, 64>{}); break;
    case 128: go(std::integral_constant<int, 128>{}); break;
    case 256: go(std::integral_constant<int, 256>{}); break;
    case 512: go(std::integral_constant<int, 512>{}); break;
    case 1024: go(std::integral_constant<int, 1024>{}); break;
    case 2048: go(std::integral_constant<int, 2048>{}); break;
    default: HELM_CHECK(false, "coarse FFT: unsupported row length");
  }
}

// Direct O(m0^2)-per-row transform for grids whose n - 1 is not a power of two.
template <typename S>
__global__ void __launch_bounds__(256) xform_direct_kernel(const S* __restrict__ in, S* __restrict__ out, XScale sc,
                                                           int rows, int m0, int dct) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (a >= m0 || r >= rows) return;
  const S* row = in + (size_t)r * m0;
  const long long P = dct ? 2LL * (m0 - 1) : 2LL * (m0 + 1);  // period of the integer argument
  S acc = Sc<S>::zero();
  for (int J = 0; J < m0; ++J) {
    double q;
    if (dct)
      q = cospi((double)(((long long)a * J) % P) / (double)(m0 - 1));
    else
      q = sinpi((double)(((long long)(a + 1) * (J + 1)) % P) / (double)(m0 + 1));
    acc = fma_(q, row[J], acc);
  }
  const S v = scale(acc, xscale(sc, r, a, m0));
  out[(size_t)r * m0 + a] = sc.accum ? add(out[(size_t)r * m0 + a], v) : v;
}

// out[b][x][y] = in[b][y][x]  (32 x 32 tiles through shared memory)
template <typename S>
__global__ void __launch_bounds__(256) transpose_kernel(const S* __restrict__ in, S* __restrict__ out, int m) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  __shared__ S tile[32][33];
  const size_t off = (size_t)blockIdx.z * m * m;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int y = y0 + r, x = x0 + threadIdx.x;
    if (y < m && x < m) tile[r][threadIdx.x] = in[off + (size_t)y * m + x];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int x = x0 + r, y = y0 + threadIdx.x;
    if (y < m && x < m) out[off + (size_t)x * m + y] = tile[threadIdx.x][r];
  }
}


template <typename S>
void launch_xform(const helm_plan* P, const S* in, S* out, const double* sig, bool scale2d, int batch,
                  cudaStream_t st, bool accumulate) {
  HELM_CHECK((const void*)in != (const void*)out, "xform: input and output must not alias");
  const PlanDev& d = P->dev;
  const int m0 = d.m0, rows = m0 * batch, dct = P->geo.sommerfeld;
  XScale sc{accumulate ? 1 : 0, sig, nullptr, nullptr, 0.0, 0.0};
  if (scale2d) sc = XScale{accumulate ? 1 : 0, nullptr, d.coarse_lamT, d.coarse_lamM, P->geo.k2, d.coarse_qn};
  if (d.fft_len) {
    const int L = d.fft_len;
    static const bool r16 = [] {  // HELM_FFT16=0: radix-8 everywhere (A/B)
      const char* e = getenv("HELM_FFT16");
      return !(e && e[0] == '0');
    }();
    if (r16 && L >= 256)
      fft_launch<S, 16>(in, out, sc, rows, m0, L, dct, d.twiddle, st);
    else
      fft_launch<S, 8>(in, out, sc, rows, m0, L, dct, d.twiddle, st);
  } else {
    dim3 grd((m0 + 255) / 256, rows);
    launch_pdl(xform_direct_kernel<S>, grd, 256, 0, st, in, out, sc, rows, m0, dct);
  }
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_transpose(const S* in, S* out, int m, int batch, cudaStream_t st) {
  dim3 grd((m + 31) / 32, (m + 31) / 32, batch), blk(32, 8);
  launch_pdl(transpose_kernel<S>, grd, blk, 0, st, in, out, m);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S)                                                                                          \
  template void launch_xform<S>(const helm_plan*, const S*, S*, const double*, bool, int, cudaStream_t, bool); \
  template void launch_transpose<S>(const S*, S*, int, int, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
