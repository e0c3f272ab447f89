// learn.cu -- consumer-side steps that act on the rollout's trajectory tensors
// (first slice; oracle/learn.py states the definitions):
//   * fin_gae: generalised advantage estimation over [T][N] rewards / dones and [T+1][N]
//     values (reading R-GAE), float64 per env, t = T-1 .. 0, advantages and returns
//     stored f32; optional batch normalisation (population mean / std of the f64
//     advantages: per-thread Welford, Chan merges in a fixed order -- deterministic).
//     HBM bound: 4 + 4 + 1 B read, 8 B written per env-step.
//   * fin_kl_diversity: the Eq. 5 term: D[i][j] = mean over a batch of states
//     of KL(pi_j || pi_i) for M members' outputs [M][B][K] -- diagonal Gaussians with a
//     shared std (sum (mu_j - mu_i)^2 / (2 sigma^2)) or categorical softmax(Q).
#include "fin_internal.cuh"
#include "sm100.cuh"

namespace {

constexpr int kT = 128;

struct Wel {
  double n, mean, m2;
};
// per-thread shifted sums (shift = the thread's first value): no division per element;
// converted once to (n, mean, M2) for the Chan merges
struct Shift {
  double k, s1, s2, n;
};
__device__ __forceinline__ void sh_push(Shift& a, double x) {
  a.k = a.n == 0.0 ? x : a.k;
  const double d = x - a.k;
  a.s1 += d;
  a.s2 = fma(d, d, a.s2);
  a.n += 1.0;
}
__device__ __forceinline__ Wel sh_wel(const Shift& a) {
  Wel w = {a.n, 0.0, 0.0};
  if (a.n > 0.0) {
    w.mean = a.k + a.s1 / a.n;
    w.m2 = fmax(a.s2 - a.s1 * a.s1 / a.n, 0.0);
  }
  return w;
}
__device__ __forceinline__ Wel wel_merge(const Wel& a, const Wel& b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  Wel r;
  r.n = a.n + b.n;
  const double d = b.mean - a.mean;
  r.mean = a.mean + d * (b.n / r.n);
  r.m2 = a.m2 + b.m2 + d * d * (a.n * b.n / r.n);
  return r;
}

// one thread per env, reverse time; the next U rows (earlier t) are loaded ahead
__global__ void __launch_bounds__(kT) k_gae(const float* __restrict__ rew, const float* __restrict__ val,
                                            const uint8_t* __restrict__ done, int T, int N, double gamma,
                                            double lam, float* __restrict__ adv, float* __restrict__ ret,
                                            Wel* __restrict__ part) {
  constexpr int U = 8;
  const int i = blockIdx.x * kT + threadIdx.x;
  Shift acc = {0.0, 0.0, 0.0, 0.0};
  if (i < N) {
    const double gl = gamma * lam;
    double a = 0.0;
    double vnext = (double)__ldg(val + (size_t)T * N + i);
    for (int t1 = T; t1 > 0; t1 -= U) {
      float rb[U], vb[U];
      uint8_t db[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t1 - 1 - u;
        rb[u] = t >= 0 ? __ldg(rew + (size_t)t * N + i) : 0.f;
        vb[u] = t >= 0 ? __ldg(val + (size_t)t * N + i) : 0.f;
        db[u] = t >= 0 ? __ldg(done + (size_t)t * N + i) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t1 - 1 - u;
        if (t >= 0) {
          const double keep = db[u] ? 0.0 : 1.0;
          const double v = (double)vb[u];
          const double delta = fsub64(fadd64((double)rb[u], fmul64(fmul64(gamma, vnext), keep)), v);
          a = fadd64(delta, fmul64(fmul64(gl, keep), a));
          adv[(size_t)t * N + i] = (float)a;
          ret[(size_t)t * N + i] = (float)fadd64(a, v);
          if (part) sh_push(acc, a);
          vnext = v;
        }
      }
    }
  }
  if (!part) return;
  // block merge in a fixed order (thread 0 folds warp results in warp order)
  __shared__ Wel ws[kT / 32];
  Wel w = sh_wel(acc);
  for (int off = 16; off > 0; off >>= 1) {
    Wel o;
    o.n = __shfl_down_sync(0xffffffffu, w.n, off);
    o.mean = __shfl_down_sync(0xffffffffu, w.mean, off);
    o.m2 = __shfl_down_sync(0xffffffffu, w.m2, off);
    w = wel_merge(w, o);
  }
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    Wel b = ws[0];
    for (int k = 1; k < kT / 32; ++k) b = wel_merge(b, ws[k]);
    part[blockIdx.x] = b;
  }
}

// TMA-staged variant (N % 16 == 0, 16-B aligned tensors): a producer warp streams, per
// 128-env block and in reverse time, chunks of R rows of reward (512 B per row), value
// (512 B) and done (128 B) into an S-slot shared-memory ring (1-D bulk copies completing
// on the slot's mbarrier); the consumer threads run the same recurrence out of shared
// memory.  (The register-prefetch kernel above keeps 8 rows per thread in flight: ~28% of
// HBM at 65,536 envs, where only 3.5 blocks of 128 envs sit on each SM.)
constexpr int kGS = 3, kGR = 8;
struct GaeSmem {
  float r[kGS][kGR][kT];
  float v[kGS][kGR][kT];
  uint8_t d[kGS][kGR][kT];
  uint64_t full[kGS], empty[kGS];
};
__global__ void __launch_bounds__(kT + 32) k_gae_tma(const float* __restrict__ rew, const float* __restrict__ val,
                                                    const uint8_t* __restrict__ done, int T, int N, double gamma,
                                                    double lam, float* __restrict__ adv, float* __restrict__ ret,
                                                    Wel* __restrict__ part) {
  __shared__ GaeSmem sm;
  __shared__ Wel ws[kT / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * kT;
  const int nb = min(kT, N - i0);                  // multiple of 16
  const int nch = (T + kGR - 1) / kGR;             // chunk c covers t = T-1-c*R down to ...
  if (tid == 0) {
    for (int q = 0; q < kGS; ++q) {
      sm100::mbar_init(&sm.full[q], 1);
      sm100::mbar_init(&sm.empty[q], kT / 32);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();
  Shift acc = {0.0, 0.0, 0.0, 0.0};
  if (warp == kT / 32) {
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int slot = c % kGS;
        if (c >= kGS) sm100::mbar_wait(&sm.empty[slot], (uint32_t)(c / kGS - 1) & 1u);
        const int rows = min(kGR, T - c * kGR);
        sm100::mbar_arrive_expect_tx(&sm.full[slot], (uint32_t)(rows * nb * 9));
        for (int r = 0; r < rows; ++r) {
          const size_t t = (size_t)(T - 1 - c * kGR - r);
          sm100::bulk_g2s(sm.r[slot][r], rew + t * N + i0, (uint32_t)nb * 4, &sm.full[slot]);
          sm100::bulk_g2s(sm.v[slot][r], val + t * N + i0, (uint32_t)nb * 4, &sm.full[slot]);
          sm100::bulk_g2s(sm.d[slot][r], done + t * N + i0, (uint32_t)nb, &sm.full[slot]);
        }
      }
    }
  } else {
    const bool live = tid < nb;
    const int i = i0 + tid;
    const double gl = gamma * lam;
    double a = 0.0;
    double vnext = live ? (double)__ldg(val + (size_t)T * N + i) : 0.0;
    for (int c = 0; c < nch; ++c) {
      const int slot = c % kGS;
      sm100::mbar_wait(&sm.full[slot], (uint32_t)(c / kGS) & 1u);
      const int rows = min(kGR, T - c * kGR);
      if (live) {
#pragma unroll
        for (int r = 0; r < kGR; ++r) {
          if (r < rows) {
            const int t = T - 1 - c * kGR - r;
            const double keep = sm.d[slot][r][tid] ? 0.0 : 1.0;
            const double v = (double)sm.v[slot][r][tid];
            const double delta = fsub64(fadd64((double)sm.r[slot][r][tid], fmul64(fmul64(gamma, vnext), keep)), v);
            a = fadd64(delta, fmul64(fmul64(gl, keep), a));
            adv[(size_t)t * N + i] = (float)a;
            ret[(size_t)t * N + i] = (float)fadd64(a, v);
            if (part) sh_push(acc, a);
            vnext = v;
          }
        }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&sm.empty[slot]);
    }
  }
  if (!part) return;
  Wel w = sh_wel(acc);
  for (int off = 16; off > 0; off >>= 1) {
    Wel o;
    o.n = __shfl_down_sync(0xffffffffu, w.n, off);
    o.mean = __shfl_down_sync(0xffffffffu, w.mean, off);
    o.m2 = __shfl_down_sync(0xffffffffu, w.m2, off);
    w = wel_merge(w, o);
  }
  if (lane == 0 && warp < kT / 32) ws[warp] = w;
  __syncthreads();
  if (tid == 0) {
    Wel b = ws[0];
    for (int k = 1; k < kT / 32; ++k) b = wel_merge(b, ws[k]);
    part[blockIdx.x] = b;
  }
}

// one block: thread k folds partials k, k + 256, ... in order, then a fixed tree
__global__ void k_gae_stats(const Wel* __restrict__ part, int nb, double* stats) {
  __shared__ Wel red[256];
  Wel w = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nb; b += 256) w = wel_merge(w, part[b]);
  red[threadIdx.x] = w;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] = wel_merge(red[threadIdx.x], red[threadIdx.x + h]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    stats[0] = red[0].mean;
    stats[1] = red[0].n > 0.0 ? sqrt(red[0].m2 / red[0].n) : 0.0;
  }
}

__global__ void k_gae_normalise(float* __restrict__ adv, size_t n, const double* __restrict__ stats) {
  const double m = stats[0], sd = stats[1];
  const double inv = sd > 0.0 ? 1.0 / sd : 1.0;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x)
    adv[k] = (float)((adv[k] - m) * inv);
}

// partial sums of KL(pi_j(.|s_b) || pi_i(.|s_b)) over the states of chunk blockIdx.y
// (kKlChunk states), one block per (pair, chunk); k_kl_final sums the chunks in order
constexpr int kKlChunk = 2048;
__global__ void k_kl(const float* __restrict__ out, int M, int B, int K, int kind, double sigma,
                     double* __restrict__ P) {
  const int i = blockIdx.x / M, j = blockIdx.x % M;
  const int b0 = blockIdx.y * kKlChunk, b1 = min(B, b0 + kKlChunk);
  double s = 0.0;
  if (i != j) {
    for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
      const float* oj = out + ((size_t)j * B + b) * K;
      const float* oi = out + ((size_t)i * B + b) * K;
      double kl = 0.0;
      if (kind == 0) {
        for (int k = 0; k < K; ++k) {
          const double d = (double)oj[k] - (double)oi[k];
          kl += d * d;
        }
        kl /= 2.0 * sigma * sigma;
      } else {   // categorical over softmax of the outputs, in log space
        double mj = -1e300, mi = -1e300;
        for (int k = 0; k < K; ++k) { mj = fmax(mj, (double)oj[k]); mi = fmax(mi, (double)oi[k]); }
        double zj = 0.0, zi = 0.0;
        for (int k = 0; k < K; ++k) { zj += exp((double)oj[k] - mj); zi += exp((double)oi[k] - mi); }
        const double lzj = log(zj) + mj, lzi = log(zi) + mi;
        for (int k = 0; k < K; ++k) {
          const double lj = (double)oj[k] - lzj, li = (double)oi[k] - lzi;
          kl += exp(lj) * (lj - li);
        }
      }
      s += kl;
    }
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {   // fixed tree: deterministic
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) P[(size_t)blockIdx.x * gridDim.y + blockIdx.y] = red[0];
}

__global__ void k_kl_final(const double* __restrict__ P, int pairs, int nch, int M, int B, double* __restrict__ D) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= pairs) return;
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s += P[(size_t)q * nch + c];
  D[q] = (q / M == q % M) ? 0.0 : s / (double)B;
}

}  // namespace

namespace fin {

cudaError_t launch_gae(const float* rew, const float* val, const uint8_t* done, int T, int N, double gamma,
                       double lam, int normalise, float* adv, float* ret, cudaStream_t s) {
  const int nb = (N + kT - 1) / kT;
  Wel* part = nullptr;
  double* stats = nullptr;
  cudaError_t e = cudaSuccess;
  if (normalise) {
    e = cudaMallocAsync(&part, sizeof(Wel) * nb, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&stats, 2 * sizeof(double), s);
    if (e != cudaSuccess) return e;
  }
  const bool tma = N % 16 == 0 && ((uintptr_t)rew & 15) == 0 && ((uintptr_t)val & 15) == 0 &&
                   ((uintptr_t)done & 15) == 0 && !getenv("FIN_GAE_NOTMA");
  if (tma) k_gae_tma<<<nb, kT + 32, 0, s>>>(rew, val, done, T, N, gamma, lam, adv, ret, part);
  else k_gae<<<nb, kT, 0, s>>>(rew, val, done, T, N, gamma, lam, adv, ret, part);
  if (normalise) {
    k_gae_stats<<<1, 256, 0, s>>>(part, nb, stats);
    const size_t n = (size_t)T * N;
    int grid = (int)((n + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    k_gae_normalise<<<grid, 256, 0, s>>>(adv, n, stats);
    cudaFreeAsync(part, s);
    cudaFreeAsync(stats, s);
  }
  return cudaGetLastError();
}

cudaError_t launch_kl_diversity(const float* out, int M, int B, int K, int kind, double sigma, double* D,
                                cudaStream_t s) {
  const int nch = (B + kKlChunk - 1) / kKlChunk;
  double* P = nullptr;
  cudaError_t e = cudaMallocAsync(&P, sizeof(double) * (size_t)M * M * nch, s);
  if (e != cudaSuccess) return e;
  k_kl<<<dim3(M * M, nch), 256, 0, s>>>(out, M, B, K, kind, sigma, P);
  k_kl_final<<<(M * M + 127) / 128, 128, 0, s>>>(P, M * M, nch, M, B, D);
  cudaFreeAsync(P, s);
  return cudaGetLastError();
}

}  // namespace fin
