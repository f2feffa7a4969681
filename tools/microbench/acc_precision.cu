// Micro-experiment: how does the tcgen05 f32 accumulator round, and how much
// error do multi-term tf32 / bf16 splits of f32 GEMMs carry at ResNet-18's
// K (up to 4608) with and without K-chunked promotion into RN registers?
//
// One CTA, 128 threads, D[128][64] = sum_k A[m][k] * B[n][k] over a list of
// split "products" (plane_a, plane_b, accumulator). Operands staged in shared
// memory in the SWIZZLE_NONE K-major core-matrix layout (8 rows x 16 B).
// Accumulator 0 ("main") is folded into f32 registers (__fadd_rn) every
// `chunk` K elements and restarted; accumulator 1 ("small") runs the whole K.
//
// Output: probe rows (rounding mode) and error statistics vs f64 exact and
// vs the reference's sequential f32 sum (R/src/texpr.cpp:205-232).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include "sm100_ptx.cuh"
using namespace tec_sm100;

constexpr int M = 128, N = 64;

__device__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

struct Prod { int a, b, acc; };
struct Job {
  int kind;      // 0 tf32, 1 bf16
  int K, chunk;  // chunk in K elements (multiple of the K block), 0 = never
  int nprod;
  Prod prod[9];
  int planes;
};

// Element (row, k) of a plane with `rows` rows, es-byte elements, at
// (k / epc) * rows * 16 + row * 16 + (k % epc) * es, epc = 16 / es.
template <typename T>
__global__ void accprec(const T* __restrict__ A, const T* __restrict__ B, Job job, float* out) {
  constexpr int es = sizeof(T);
  constexpr int epc = 16 / es;
  constexpr int KB = 64;  // K elements per smem block
  constexpr int kstep = es == 4 ? 8 : 16;
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int P = job.planes;
  uint8_t* sA = sm;                          // P planes of M x KB
  uint8_t* sB = sm + P * M * KB * es;        // P planes of N x KB
  uint64_t* bar = (uint64_t*)(sB + P * N * KB * es);
  uint32_t* slot = (uint32_t*)(bar + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<128>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  constexpr uint32_t idesc = es == 4 ? make_idesc<MmaKind::kTF32>(M, N) : make_idesc<MmaKind::kF16>(M, N);
  float sum[N];
  for (int j = 0; j < N; ++j) sum[j] = 0.f;
  bool started[2] = {false, false};
  uint32_t phase = 0;
  int since = 0;
  for (int k0 = 0; k0 < job.K; k0 += KB) {
    for (int p = 0; p < P; ++p) {
      for (int i = threadIdx.x; i < M * KB; i += blockDim.x) {
        int r = i / KB, k = i % KB;
        *(T*)(sA + p * M * KB * es + (k / epc) * M * 16 + r * 16 + (k % epc) * es) =
            A[((size_t)p * M + r) * job.K + k0 + k];
      }
      for (int i = threadIdx.x; i < N * KB; i += blockDim.x) {
        int r = i / KB, k = i % KB;
        *(T*)(sB + p * N * KB * es + (k / epc) * N * 16 + r * 16 + (k % epc) * es) =
            B[((size_t)p * N + r) * job.K + k0 + k];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
      for (int kk = 0; kk < KB; kk += kstep) {
        for (int q = 0; q < job.nprod; ++q) {
          const Prod pr = job.prod[q];
          const uint32_t a = smem_u32(sA + pr.a * M * KB * es) + (kk / epc) * M * 16;
          const uint32_t b = smem_u32(sB + pr.b * N * KB * es) + (kk / epc) * N * 16;
          const uint64_t ad = desc_none(a, M * 16, 128);
          const uint64_t bd = desc_none(b, N * 16, 128);
          if (es == 4) tc_mma<MmaKind::kTF32>(tmem + pr.acc * N, ad, bd, idesc, started[pr.acc]);
          else tc_mma<MmaKind::kF16>(tmem + pr.acc * N, ad, bd, idesc, started[pr.acc]);
          started[pr.acc] = true;
        }
      }
      tc_commit(&bar[0]);
    }
    mbar_wait(&bar[0], phase);
    phase ^= 1;
    tc_fence_after();
    since += KB;
    const bool last = k0 + KB >= job.K;
    if ((job.chunk > 0 && since >= job.chunk) || last) {
      // fold accumulator 0 into the RN register sum, restart it
      uint32_t v[32];
      for (int c = 0; c < N; c += 32) {
        tmem_ld32(tmem + ((warp * 32) << 16) + c, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) sum[c + j] = __fadd_rn(sum[c + j], __uint_as_float(v[j]));
      }
      since = 0;
      started[0] = false;
    }
    tc_fence_before();
    __syncthreads();
  }
  // small accumulator (if used) added last
  bool used1 = false;
  for (int q = 0; q < job.nprod; ++q) used1 |= job.prod[q].acc == 1;
  if (used1) {
    uint32_t v[32];
    for (int c = 0; c < N; c += 32) {
      tmem_ld32(tmem + ((warp * 32) << 16) + N + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) sum[c + j] = __fadd_rn(sum[c + j], __uint_as_float(v[j]));
    }
  }
  for (int j = 0; j < N; ++j) out[(warp * 32 + lane) * N + j] = sum[j];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= ~0x1FFFu; memcpy(&x, &u, 4); return x; }
static float tf32_rn(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  u += 0xFFFu + ((u >> 13) & 1u); u &= ~0x1FFFu; memcpy(&x, &u, 4); return x;
}
static __nv_bfloat16 bf(float x) { return __float2bfloat16_rn(x); }
static float fb(__nv_bfloat16 x) { return __bfloat162float(x); }

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

template <typename T>
static std::vector<float> run(const std::vector<T>& A, const std::vector<T>& B, Job job) {
  T *dA, *dB; float* dO;
  CK(cudaMalloc(&dA, A.size() * sizeof(T)));
  CK(cudaMalloc(&dB, B.size() * sizeof(T)));
  CK(cudaMalloc(&dO, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * sizeof(T), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * sizeof(T), cudaMemcpyHostToDevice));
  const int smem = 1024 + job.planes * (M + N) * 64 * sizeof(T) + 64;
  CK(cudaFuncSetAttribute(accprec<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  accprec<T><<<1, 128, smem>>>(dA, dB, job, dO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> o(M * N);
  CK(cudaMemcpy(o.data(), dO, M * N * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA); cudaFree(dB); cudaFree(dO);
  return o;
}

int main() {
  // ------------------------------------------------------------ probes
  {
    const int K = 64;
    std::vector<float> A(M * K, 0.f), B(N * K, 0.f);
    for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) B[n * K + k] = 1.f;
    auto set = [&](int r, int k, double v) { A[r * K + k] = (float)v; };
    set(0, 0, 1 + std::ldexp(1, -11) + std::ldexp(1, -13));   // operand: RN -> 1+2^-10, trunc -> 1
    set(1, 0, 1); set(1, 8, 0.75 * std::ldexp(1, -23));       // across MMAs: RN 1+2^-23, RZ/RD 1
    set(2, 0, 1); set(2, 8, -0.25 * std::ldexp(1, -24));      // RN 1, RZ/RD 1-2^-24
    set(3, 0, -1); set(3, 8, 0.25 * std::ldexp(1, -24));      // RN -1, RZ -(1-2^-24), RD -1
    set(4, 0, 1); set(4, 1, 0.75 * std::ldexp(1, -23));       // inside one MMA
    set(5, 0, 1); set(5, 1, std::ldexp(1, -24)); set(5, 2, std::ldexp(1, -24)); set(5, 3, std::ldexp(1, -24));
    set(6, 0, 1); set(6, 1, -0.25 * std::ldexp(1, -24));      // inside one MMA, RN 1
    set(7, 0, -1); set(7, 1, 0.25 * std::ldexp(1, -24));      // inside one MMA
    set(8, 0, std::ldexp(1, 20)); set(8, 8, 1); set(8, 9, 0.5);  // big acc + small: 2^20+1.5 exact
    Job j{}; j.kind = 0; j.K = K; j.chunk = 0; j.nprod = 1; j.prod[0] = {0, 0, 0}; j.planes = 1;
    auto o = run<float>(A, B, j);
    printf("tf32 probes (row: value, delta from 1 in units of 2^-24):\n");
    for (int r = 0; r < 9; ++r) printf("  row %d: %.10g  (%+.3f)\n", r, o[r * N], (std::fabs((double)o[r * N]) - (r == 8 ? std::ldexp(1, 20) : 1.0)) / std::ldexp(1, -24));
    std::vector<__nv_bfloat16> Ab(M * K), Bb(N * K);
    for (int i = 0; i < M * K; ++i) Ab[i] = bf(A[i]);
    for (int i = 0; i < N * K; ++i) Bb[i] = bf(B[i]);
    j.kind = 1;
    auto ob = run<__nv_bfloat16>(Ab, Bb, j);
    printf("bf16 probes (rows 1-8):\n");
    for (int r = 1; r < 9; ++r) printf("  row %d: %.10g  (%+.3f)\n", r, ob[r * N], (std::fabs((double)ob[r * N]) - (r == 8 ? std::ldexp(1, 20) : 1.0)) / std::ldexp(1, -24));
  }
  // ------------------------------------------------------------ statistics
  const int K = 4608;
  std::mt19937_64 g(0);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> x(M * K), w(N * K);
  for (auto& v : x) v = U(g);
  for (auto& v : w) v = U(g);
  std::vector<double> ex(M * N);
  std::vector<float> seq(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double e = 0; float f = 0;
      for (int k = 0; k < K; ++k) {
        e += (double)x[m * K + k] * w[n * K + k];
        volatile float pr = x[m * K + k] * w[n * K + k];
        f = f + pr;
      }
      ex[m * N + n] = e; seq[m * N + n] = f;
    }
  auto stats = [&](const char* name, const std::vector<float>& o) {
    double se = 0, se2 = 0, mx = 0, mr = 0, mrs = 0;
    int bad = 0;
    for (int i = 0; i < M * N; ++i) {
      const double e = o[i] - ex[i];
      se += e; se2 += e * e; mx = std::max(mx, std::fabs(e));
      const double t = std::max({std::fabs((double)o[i]), std::fabs(ex[i]), 1.0});
      mr = std::max(mr, std::fabs(e) / t);
      const double d = std::fabs((double)o[i] - seq[i]);
      const double ts = std::max({std::fabs((double)o[i]), std::fabs((double)seq[i]), 1.0});
      mrs = std::max(mrs, d / ts);
      bad += d / ts > 1e-4;
    }
    printf("%-44s vs exact: mean %+.2e std %.2e max %.2e | vs ref: max_rel %.2e bad %d\n", name,
           se / (M * N), std::sqrt(se2 / (M * N)), mx, mrs, bad);
  };
  stats("reference sequential f32", seq);
  // tf32 planes: 0 = raw x, 1 = RN hi, 2 = lo of raw (x - trunc(x)), 3 = lo of RN
  auto planes_tf32 = [&](const std::vector<float>& v, int rows) {
    std::vector<float> o(4 * rows * K);
    for (int i = 0; i < rows * K; ++i) {
      o[i] = v[i];
      o[rows * K + i] = tf32_rn(v[i]);
      o[2 * rows * K + i] = v[i] - tf32_trunc(v[i]);
      o[3 * rows * K + i] = v[i] - tf32_rn(v[i]);
    }
    return o;
  };
  auto At = planes_tf32(x, M), Bt = planes_tf32(w, N);
  struct Cfg { const char* name; int nprod; Prod p[9]; int chunk; };
  std::vector<Cfg> tc = {
      {"tf32 1x raw", 1, {{0, 0, 0}}, 0},
      {"tf32 1x RN", 1, {{1, 1, 0}}, 0},
      {"tf32x3 raw-hi, 1 acc", 3, {{0, 0, 0}, {0, 2, 0}, {2, 0, 0}}, 0},
      {"tf32x3 RN-hi, 1 acc", 3, {{1, 1, 0}, {1, 3, 0}, {3, 1, 0}}, 0},
      {"tf32x3 raw-hi, chunk 512", 3, {{0, 0, 0}, {0, 2, 0}, {2, 0, 0}}, 512},
      {"tf32x3 raw-hi, chunk 128", 3, {{0, 0, 0}, {0, 2, 0}, {2, 0, 0}}, 128},
      {"tf32x3 raw-hi, chunk 64", 3, {{0, 0, 0}, {0, 2, 0}, {2, 0, 0}}, 64},
      {"tf32x3 raw-hi, small acc, chunk 1024", 3, {{0, 0, 0}, {0, 2, 1}, {2, 0, 1}}, 1024},
      {"tf32x3 raw-hi, small acc, chunk 512", 3, {{0, 0, 0}, {0, 2, 1}, {2, 0, 1}}, 512},
      {"tf32x3 raw-hi, small acc, chunk 256", 3, {{0, 0, 0}, {0, 2, 1}, {2, 0, 1}}, 256},
      {"tf32x3 raw-hi, small acc, chunk 128", 3, {{0, 0, 0}, {0, 2, 1}, {2, 0, 1}}, 128},
      {"tf32x3 RN-hi, small acc, chunk 128", 3, {{1, 1, 0}, {1, 3, 1}, {3, 1, 1}}, 128},
      {"tf32x3 raw-hi, small acc, chunk 64", 3, {{0, 0, 0}, {0, 2, 1}, {2, 0, 1}}, 64},
  };
  for (auto& c : tc) {
    Job j{}; j.kind = 0; j.K = K; j.chunk = c.chunk; j.nprod = c.nprod; j.planes = 4;
    for (int i = 0; i < c.nprod; ++i) j.prod[i] = c.p[i];
    stats(c.name, run<float>(At, Bt, j));
  }
  // bf16 planes: 0 hi, 1 mid, 2 lo
  auto planes_bf = [&](const std::vector<float>& v, int rows) {
    std::vector<__nv_bfloat16> o(3 * rows * K);
    for (int i = 0; i < rows * K; ++i) {
      const __nv_bfloat16 h = bf(v[i]);
      const float r1 = v[i] - fb(h);
      const __nv_bfloat16 m = bf(r1);
      const float r2 = r1 - fb(m);
      o[i] = h; o[rows * K + i] = m; o[2 * rows * K + i] = bf(r2);
    }
    return o;
  };
  auto Ab = planes_bf(x, M), Bb = planes_bf(w, N);
  std::vector<Cfg> bc = {
      {"bf16x3 (hh,hm,mh), 1 acc", 3, {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}}, 0},
      {"bf16x6, 1 acc", 6, {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}, {0, 2, 0}, {2, 0, 0}, {1, 1, 0}}, 0},
      {"bf16x6, chunk 128", 6, {{0, 0, 0}, {0, 1, 0}, {1, 0, 0}, {0, 2, 0}, {2, 0, 0}, {1, 1, 0}}, 128},
      {"bf16x6, small acc, chunk 1024", 6, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}, {1, 1, 1}}, 1024},
      {"bf16x6, small acc, chunk 256", 6, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}, {1, 1, 1}}, 256},
      {"bf16x6, small acc, chunk 128", 6, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}, {1, 1, 1}}, 128},
      {"bf16x6, small acc, chunk 64", 6, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}, {1, 1, 1}}, 64},
      {"bf16x5 (no mm), small acc, chunk 256", 5, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {0, 2, 1}, {2, 0, 1}}, 256},
      {"bf16x4 (no hl, lh), small acc, chunk 256", 4, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}, {1, 1, 1}}, 256},
      {"bf16x3 (hh,hm,mh), small acc, chunk 256", 3, {{0, 0, 0}, {0, 1, 1}, {1, 0, 1}}, 256},
  };
  for (auto& c : bc) {
    Job j{}; j.kind = 1; j.K = K; j.chunk = c.chunk; j.nprod = c.nprod; j.planes = 3;
    for (int i = 0; i < c.nprod; ++i) j.prod[i] = c.p[i];
    stats(c.name, run<__nv_bfloat16>(Ab, Bb, j));
  }
  return 0;
}
