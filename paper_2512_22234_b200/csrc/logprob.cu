// bd_logprob: per-token log-softmax gather over the vocabulary, optionally
// fused with its gradient (P:150-156 numerators of Eqs. 6-8; P:78 CE of Eq. 3;
// S:69-77).  HBM-streaming.
//  * forward only: one CTA per row, online (max, sum-exp) in fp32 -> LSE_n,
//    logp_n = z[t] - LSE_n (one read of the logits).
//  * forward + gradient (dlogp given, the online DiPO setting where the
//    weights are known up front): a 4-CTA cluster per row keeps the row in
//    shared memory (st.async (max, sum) exchange), one exp2 per element, one read
//    and one write of the logits (logprob_fused1p_kernel); a generic two-pass
//    path covers unaligned rows / vocabularies.
// Rows are read with 16-byte vector loads when the row is 16-byte aligned and
// V % 8 == 0 (Qwen3 V = 151,936 is), otherwise element-wise.
#include "abi_common.h"
#include "sm100.cuh"

#include <cuda_bf16.h>

namespace bd {
namespace {

constexpr int kThreads = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;

__device__ __forceinline__ void online_add(float& m, float& s, float x) {
  // running max m (log2 units) and sum s of 2^(x - m)
  if (x > m) {
    s = s * ex2_approx(m - x) + 1.f;
    m = x;
  } else {
    s += ex2_approx(x - m);
  }
}

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  if (mm == -INFINITY) return;
  s = s * ex2_approx(m - mm) + s2 * ex2_approx(m2 - mm);
  m = mm;
}

__device__ __forceinline__ ulonglong2 ld_stream(const void* p) {
  ulonglong2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
  return r;
}

__global__ void __launch_bounds__(kThreads) logprob_kernel(int64_t n_rows, int V, const __nv_bfloat16* __restrict__ z,
                                                           int64_t stride, const int32_t* __restrict__ targets,
                                                           float* __restrict__ logp, float* __restrict__ lse_out,
                                                           const float* __restrict__ dlogp,
                                                           __nv_bfloat16* dz, int64_t dz_stride) {
  __shared__ float sm_m[kThreads / 32], sm_s[kThreads / 32];
  __shared__ float s_lse;
  const int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  const __nv_bfloat16* zr = z + row * stride;
  const int tid = threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(zr) & 15) == 0) && (V % 8 == 0);
  float m = -INFINITY, s = 0.f;
  if (vec) {
    // Running max m is only raised (and s rescaled) when a 16-element chunk
    // exceeds it, so the steady state costs one FFMA + one ex2 per element.
    const int nv = V / 8;
    auto chunk = [&](const ulonglong2& u0, const ulonglong2& u1) {
      const uint32_t w[8] = {(uint32_t)u0.x, (uint32_t)(u0.x >> 32), (uint32_t)u0.y, (uint32_t)(u0.y >> 32),
                             (uint32_t)u1.x, (uint32_t)(u1.x >> 32), (uint32_t)u1.y, (uint32_t)(u1.y >> 32)};
      float z[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        z[2 * j] = __uint_as_float(w[j] << 16);
        z[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
      }
      float mx = z[0];
#pragma unroll
      for (int j = 1; j < 16; ++j) mx = fmaxf(mx, z[j]);
      mx *= kLog2e;
      if (mx > m) {
        s *= ex2_approx(m - mx);  // m = -inf -> 0
        m = mx;
      }
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += ex2_approx(fmaf(z[j], kLog2e, -m));
      s += acc;
    };
    int i = tid;
    for (; i + kThreads < nv; i += 2 * kThreads) chunk(ld_stream(zr + 8 * i), ld_stream(zr + 8 * (i + kThreads)));
    if (i < nv) {
      // odd tail: one 8-element vector
      const ulonglong2 u = ld_stream(zr + 8 * i);
      const uint32_t w[4] = {(uint32_t)u.x, (uint32_t)(u.x >> 32), (uint32_t)u.y, (uint32_t)(u.y >> 32)};
      float z[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        z[2 * j] = __uint_as_float(w[j] << 16);
        z[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
      }
      float mx = z[0];
#pragma unroll
      for (int j = 1; j < 8; ++j) mx = fmaxf(mx, z[j]);
      mx *= kLog2e;
      if (mx > m) {
        s *= ex2_approx(m - mx);
        m = mx;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) s += ex2_approx(fmaf(z[j], kLog2e, -m));
    }
  } else {
    for (int i = tid; i < V; i += kThreads) online_add(m, s, __bfloat162float(zr[i]) * kLog2e);
  }
  // block reduce (m, s)
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
    online_merge(m, s, m2, s2);
  }
  if ((tid & 31) == 0) {
    sm_m[tid >> 5] = m;
    sm_s[tid >> 5] = s;
  }
  __syncthreads();
  if (tid < 32) {
    m = tid < kThreads / 32 ? sm_m[tid] : -INFINITY;
    s = tid < kThreads / 32 ? sm_s[tid] : 0.f;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
      online_merge(m, s, m2, s2);
    }
    if (tid == 0) {
      const float lse = (m + __log2f(s)) * kLn2;
      s_lse = lse;
      const int t = targets[row];
      const bool ok = t >= 0 && t < V;
      logp[row] = ok ? __bfloat162float(zr[t]) - lse : __int_as_float(0x7fc00000);
      if (lse_out) lse_out[row] = lse;
    }
  }
  if (!dlogp || !dz) return;
  __syncthreads();
  const float lse2 = s_lse * kLog2e;
  const float w = dlogp[row];
  const int t = targets[row];
  __nv_bfloat16* dr = dz + row * dz_stride;
  const bool vec2 = vec && ((reinterpret_cast<uintptr_t>(dr) & 15) == 0);
  if (vec2) {
    const int nv = V / 8;
    for (int i = tid; i < nv; i += kThreads) {
      const uint4 u = *reinterpret_cast<const uint4*>(zr + 8 * i);
      const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v0 = 8 * i + 2 * j;
        float p0 = ex2_approx(fmaf(__uint_as_float(wd[j] << 16), kLog2e, -lse2));
        float p1 = ex2_approx(fmaf(__uint_as_float(wd[j] & 0xFFFF0000u), kLog2e, -lse2));
        const float g0 = w * ((v0 == t ? 1.f : 0.f) - p0);
        const float g1 = w * ((v0 + 1 == t ? 1.f : 0.f) - p1);
        o[j] = pack_bf16x2(g0, g1);
      }
      *reinterpret_cast<uint4*>(dr + 8 * i) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  } else {
    for (int i = tid; i < V; i += kThreads) {
      const float p = ex2_approx(fmaf(__bfloat162float(zr[i]), kLog2e, -lse2));
      dr[i] = __float2bfloat16(w * ((i == t ? 1.f : 0.f) - p));
    }
  }
}

// dz = w (1[v = t] - exp(z - LSE)) from a known LSE: one read + one write.
__global__ void __launch_bounds__(kThreads) logprob_bwd_kernel(int64_t n_rows, int V,
                                                               const __nv_bfloat16* z, int64_t stride,
                                                               const int32_t* __restrict__ targets,
                                                               const float* __restrict__ lse,
                                                               const float* __restrict__ dlogp, __nv_bfloat16* dz,
                                                               int64_t dz_stride) {
  const int64_t row = blockIdx.x;
  if (row >= n_rows) return;
  const __nv_bfloat16* zr = z + row * stride;
  __nv_bfloat16* dr = dz + row * dz_stride;
  const float lse2 = lse[row] * kLog2e;
  const float w = dlogp[row];
  const int t = targets[row];
  const int tid = threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(zr) & 15) == 0) && ((reinterpret_cast<uintptr_t>(dr) & 15) == 0) &&
                   (V % 8 == 0);
  if (vec) {
    const int nv = V / 8;
    for (int i = tid; i < nv; i += kThreads) {
      const uint4 u = *reinterpret_cast<const uint4*>(zr + 8 * i);
      const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v0 = 8 * i + 2 * j;
        const float p0 = ex2_approx(fmaf(__uint_as_float(wd[j] << 16), kLog2e, -lse2));
        const float p1 = ex2_approx(fmaf(__uint_as_float(wd[j] & 0xFFFF0000u), kLog2e, -lse2));
        o[j] = pack_bf16x2(w * ((v0 == t ? 1.f : 0.f) - p0), w * ((v0 + 1 == t ? 1.f : 0.f) - p1));
      }
      *reinterpret_cast<uint4*>(dr + 8 * i) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  } else {
    for (int i = tid; i < V; i += kThreads) {
      const float p = ex2_approx(fmaf(__bfloat162float(zr[i]), kLog2e, -lse2));
      dr[i] = __float2bfloat16(w * ((i == t ? 1.f : 0.f) - p));
    }
  }
}

// ---------------------------------------------------------------------------
// Fused forward + gradient with the row held on chip (logprob_fused1p_kernel):
// a cluster of kCl CTAs per row, CTA c bulk-loads elements
// [c V/kCl, (c+1) V/kCl) into shared memory -- one HBM read and one HBM write
// of the logits (the two-kernel path reads them twice), one exp2 per element.
// Requires V % (8 kCl) == 0 and 16-byte aligned rows (Qwen3 V = 151,936 is).
//  * One pass over the slice, no max pass: a thread takes the max of its
//    FIRST vector as its reference m_t and turns each of its elements into
//    e = 2^((x - m_t) log2e), stored over the slice as bf16 (whose 8-bit
//    exponent holds e > 1 as precisely as e <= 1) and summed in fp32.  If a
//    later element exceeds m_t by so much that the thread's sum leaves
//    [0, 2^64) (a spread of > 44 nats above its first vector: never for
//    realistic logits), the thread redoes its elements from the logits in
//    global memory against its exact max.
//  * The (m_t, sum_t) pairs are merged by warp shuffles and across the CTA's
//    warps; each CTA then pushes its pair into every CTA of the cluster with
//    st.async, which counts the 8 bytes on the receiver's mbarrier, so a CTA
//    waits only for its own kCl pairs -- no cluster-wide barrier (and no
//    release fence) after the pass.  A cluster arrive at entry and its wait
//    before the push guarantee the receivers' mbarriers are initialised.
//  * Pass 2 writes dz = w (1[v = t] - e 2^(m_t - M) / sum) from shared memory.
// Measured (131,072 x 151,936): 12.0 ms standalone, 14.2-14.4 ms
// inside the bench step, against 13.6 / 17.0 ms for the previous three-pass
// kernel with a closing cluster barrier.
#ifndef BD_LP_CLUSTER
#define BD_LP_CLUSTER 4
#endif
constexpr int kCl = BD_LP_CLUSTER;
#ifndef BD_LP_THREADS
#define BD_LP_THREADS 256
#endif
constexpr int kFusedThreads = BD_LP_THREADS;
#ifndef BD_LP_REGV
#define BD_LP_REGV 5
#endif
constexpr int kLpRegV = BD_LP_REGV;  // register-held vectors per thread (see logprob_fused1p_kernel)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// st.async of two floats into `local`'s twin in CTA `rank` of the cluster,
// completing 8 bytes of transaction on `local_bar`'s twin there
__device__ __forceinline__ void st_async_f32x2(float2* local, uint64_t* local_bar, uint32_t rank, float a, float b) {
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(ra), "f"(a),
               "f"(b), "r"(rb)
               : "memory");
}

__device__ __forceinline__ void pair_merge(float& m, float& s, float m2, float s2) {
  // (m, s): reference (natural-log units) and sum of exp(x - m)
  if (s2 == 0.f) return;
  if (s == 0.f) {
    m = m2;
    s = s2;
    return;
  }
  const float mm = fmaxf(m, m2);
  s = s * ex2_approx((m - mm) * kLog2e) + s2 * ex2_approx((m2 - mm) * kLog2e);
  m = mm;
}

__device__ __forceinline__ float vec_max(const uint4& u) {
  __nv_bfloat162 a = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&u.x), *reinterpret_cast<const __nv_bfloat162*>(&u.y));
  const __nv_bfloat162 b = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&u.z), *reinterpret_cast<const __nv_bfloat162*>(&u.w));
  a = __hmax2(a, b);
  return fmaxf(__low2float(a), __high2float(a));
}

// e = 2^(x log2e - m2) of one vector, packed to bf16, summed into acc
__device__ __forceinline__ uint4 exp_vec(const uint4& u, float2 nm2, float2& acc) {
  const float2 l2e = make_float2(kLog2e, kLog2e);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 x = ffma2(make_float2(__uint_as_float(w[j] << 16), __uint_as_float(w[j] & 0xFFFF0000u)), l2e, nm2);
    const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
    acc = fadd2(acc, e);
    o[j] = pack_bf16x2(e.x, e.y);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// REGV vectors per thread of the slice's tail are held in registers (plain
// 16-byte streaming loads issued at entry) instead of shared memory: at the
// Qwen3 vocabulary the slice's shared-memory part drops from 74 to 54 KB, so
// four CTAs (instead of three) fit an SM and a third more of each SM's bytes
// are in flight while the others compute (REGV = 0: the whole slice in smem).
template <int REGV>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kFusedThreads)
    logprob_fused1p_kernel(int V, const __nv_bfloat16* z, int64_t stride, const int32_t* __restrict__ targets,
                           float* __restrict__ logp, float* __restrict__ lse_out, const float* __restrict__ dlogp,
                           __nv_bfloat16* dz, int64_t dz_stride) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red[kFusedThreads / 32];
  __shared__ __align__(8) float2 pall[kCl];  // (max, sum) of every slice, pushed by its CTA (st.async)
  __shared__ float zt;
  __shared__ __align__(8) uint64_t bar, pbar;
  const int64_t row = blockIdx.x / kCl;
  const uint32_t crank = cluster_rank();
  const int tid = threadIdx.x;
  const int Vc = V / kCl;
  const int nv = Vc / 8;                        // uint4 vectors in this slice
  const int nvs = nv - REGV * kFusedThreads;    // ... of which in shared memory: [0, nvs)
  const __nv_bfloat16* src = z + row * stride + (int64_t)crank * Vc;
  const uint4* g4 = reinterpret_cast<const uint4*>(src);
  uint4* buf4 = reinterpret_cast<uint4*>(smem);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&pbar, 1);
    fence_barrier_init();
  }
  // the row's scalars and the register part of the slice go out first: their
  // latency overlaps the bulk copy
  const int t = targets[row];
  const float wgt = dlogp ? dlogp[row] : 0.f;
  uint4 rv[REGV > 0 ? REGV : 1];
#pragma unroll
  for (int k = 0; k < REGV; ++k) {
    const ulonglong2 u = ld_stream(g4 + nvs + k * kFusedThreads + tid);
    rv[k] = make_uint4((uint32_t)u.x, (uint32_t)(u.x >> 32), (uint32_t)u.y, (uint32_t)(u.y >> 32));
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)nvs * 16;
    mbar_expect_tx(&bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768) {
      const uint32_t n = bytes - off < 32768 ? bytes - off : 32768;
      bulk_load(smem + off, reinterpret_cast<const uint8_t*>(src) + off, n, &bar);
    }
  }
  const int tl = t - (int)crank * Vc;  // target within this slice (may fall outside)
  const int tv = (tl >= 0 && tl < Vc) ? tl >> 3 : -1;
  // the target vector's owner: smem vector tv (thread tv % 256) or register
  // vector k of thread (tv - nvs) % 256
  const bool t_in_regs = tv >= nvs;
  const int t_owner = tv < 0 ? -1 : (t_in_regs ? (tv - nvs) & (kFusedThreads - 1) : tv & (kFusedThreads - 1));
  const int t_k = t_in_regs ? (tv - nvs) / kFusedThreads : -1;
  if (REGV > 0 && t_in_regs && tid == t_owner) {
    const int kk = tl & 7;
#pragma unroll
    for (int k = 0; k < REGV; ++k)
      if (k == t_k) {
        const uint32_t wd = (kk >> 1) == 0 ? rv[k].x : (kk >> 1) == 1 ? rv[k].y : (kk >> 1) == 2 ? rv[k].z : rv[k].w;
        zt = __uint_as_float((kk & 1) ? (wd & 0xFFFF0000u) : (wd << 16));
      }
  }
  mbar_wait(&bar, 0);
  if (!t_in_regs && tv >= 0 && tid == t_owner)
    zt = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(smem)[tl]);  // read before the pass overwrites it
  // one pass: e against the thread's reference m_t (max of its first vector)
  float mref = tid < nvs ? vec_max(buf4[tid]) : -INFINITY;
  float m_t = mref == -INFINITY ? 0.f : mref;
  float2 acc = make_float2(0.f, 0.f);
  {
    const float2 nm2 = make_float2(-m_t * kLog2e, -m_t * kLog2e);
    for (int i = tid; i < nvs; i += kFusedThreads) buf4[i] = exp_vec(buf4[i], nm2, acc);
#pragma unroll
    for (int k = 0; k < REGV; ++k) rv[k] = exp_vec(rv[k], nm2, acc);
  }
  float s_t = acc.x + acc.y;
  if (!(s_t < 18446744073709551616.f)) {
    // rare: an element far above the reference -- redo against the exact max
    // from the logits in global memory (this thread's vectors only)
    float mx = -INFINITY;
    for (int i = tid; i < nvs; i += kFusedThreads) mx = fmaxf(mx, vec_max(g4[i]));
#pragma unroll
    for (int k = 0; k < REGV; ++k) mx = fmaxf(mx, vec_max(g4[nvs + k * kFusedThreads + tid]));
    m_t = mx == -INFINITY ? 0.f : mx;
    const float2 nm2 = make_float2(-m_t * kLog2e, -m_t * kLog2e);
    acc = make_float2(0.f, 0.f);
    for (int i = tid; i < nvs; i += kFusedThreads) buf4[i] = exp_vec(g4[i], nm2, acc);
#pragma unroll
    for (int k = 0; k < REGV; ++k) rv[k] = exp_vec(g4[nvs + k * kFusedThreads + tid], nm2, acc);
    s_t = acc.x + acc.y;
  }
  // (reference, sum) pairs: warp shuffles, the CTA's warps, then the cluster
  float M = m_t, S = s_t;
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, M, off), s2 = __shfl_xor_sync(0xffffffffu, S, off);
    pair_merge(M, S, m2, s2);
  }
  if ((tid & 31) == 0) red[tid >> 5] = make_float2(M, S);
  __syncthreads();
  float mc = 0.f, sc = 0.f;
#pragma unroll
  for (int w = 0; w < kFusedThreads / 32; ++w) pair_merge(mc, sc, red[w].x, red[w].y);
  if (sc == 0.f) mc = -INFINITY;  // the whole slice is -inf
  // push (max, sum) into slot `crank` of every CTA of the cluster with
  // st.async, which counts its 8 bytes on the receiver's mbarrier: each CTA
  // waits for its own kCl pairs -- no cluster-wide barrier (and no release
  // fence) after the pass.  The entry arrive / this wait guarantee the
  // receivers' mbarriers are initialised; a CTA exits only after all pushes
  // into it have landed.
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (tid < kCl) st_async_f32x2(&pall[crank], &pbar, (uint32_t)tid, mc, sc);
  if (tid == 0) mbar_expect_tx(&pbar, kCl * 8);
  mbar_wait(&pbar, 0);
  float mg = -INFINITY;
#pragma unroll
  for (int r = 0; r < kCl; ++r) mg = fmaxf(mg, pall[r].x);
  float tot = 0.f;
#pragma unroll
  for (int r = 0; r < kCl; ++r)
    tot += pall[r].x == -INFINITY ? 0.f : pall[r].y * ex2_approx((pall[r].x - mg) * kLog2e);
  const float lse = mg + __logf(tot);
  if (tid == 0) {
    if (crank == 0) {
      if (lse_out) lse_out[row] = lse;
      if (t < 0 || t >= V) logp[row] = __int_as_float(0x7fc00000);
    }
    if (tv >= 0) logp[row] = zt - lse;  // zt was written before the block barrier above
  }
  if (!dlogp) return;
  // pass 2: dz = w (1[v = t] - e 2^(m_t - M) / sum)
  const float scl = wgt * ex2_approx((m_t - mg) * kLog2e) / tot;
  uint4* out = reinterpret_cast<uint4*>(dz + row * dz_stride + (int64_t)crank * Vc);
  const float nscl = -scl;
  const __nv_bfloat16 hi = __float2bfloat16_rn(nscl);
  const __nv_bfloat16 lo = __float2bfloat16_rn(nscl - __bfloat162float(hi));
  const __nv_bfloat162 hi2 = __halves2bfloat162(hi, hi), lo2 = __halves2bfloat162(lo, lo);
  auto grad_vec = [&](const uint4& u, int i) {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
    if (i != tv) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 e2 = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
        const __nv_bfloat162 d2 = __hfma2(e2, hi2, __hmul2(e2, lo2));
        w[j] = *reinterpret_cast<const uint32_t*>(&d2);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int v0 = 8 * i + 2 * j;
        const float g0 = (v0 == tl ? wgt : 0.f) - scl * __uint_as_float(w[j] << 16);
        const float g1 = (v0 + 1 == tl ? wgt : 0.f) - scl * __uint_as_float(w[j] & 0xFFFF0000u);
        w[j] = pack_bf16x2(g0, g1);
      }
    }
    out[i] = make_uint4(w[0], w[1], w[2], w[3]);
  };
  for (int i = tid; i < nvs; i += kFusedThreads) grad_vec(buf4[i], i);
#pragma unroll
  for (int k = 0; k < REGV; ++k) grad_vec(rv[k], nvs + k * kFusedThreads + tid);
}

}  // namespace
}  // namespace bd

extern "C" int bd_logprob_bwd(int64_t n_rows, int32_t vocab, const void* logits, int64_t row_stride,
                              const int32_t* targets, const float* lse, const float* dlogp, void* dlogits,
                              int64_t dlogits_stride, void* stream_) {
  using namespace bd;
  if (n_rows < 0 || vocab <= 0 || row_stride < vocab || dlogits_stride < vocab)
    return set_error(BD_ERR_INVALID_ARG, "bad logprob shape");
  if (n_rows == 0) return BD_OK;
  if (!logits || !targets || !lse || !dlogp || !dlogits) return set_error(BD_ERR_INVALID_ARG, "null pointer");
  if (dlogits == logits && dlogits_stride != row_stride)
    return set_error(BD_ERR_INVALID_ARG, "in-place gradient needs equal strides");
  if (n_rows > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "too many rows");
  logprob_bwd_kernel<<<(unsigned)n_rows, kThreads, 0, static_cast<cudaStream_t>(stream_)>>>(
      n_rows, vocab, reinterpret_cast<const __nv_bfloat16*>(logits), row_stride, targets, lse, dlogp,
      reinterpret_cast<__nv_bfloat16*>(dlogits), dlogits_stride);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "logprob_bwd_kernel launch");
}

extern "C" int bd_logprob(int64_t n_rows, int32_t vocab, const void* logits, int64_t row_stride,
                          const int32_t* targets, float* logp, float* lse, const float* dlogp, void* dlogits,
                          int64_t dlogits_stride, void* stream_) {
  using namespace bd;
  if (n_rows < 0 || vocab <= 0 || row_stride < vocab) return set_error(BD_ERR_INVALID_ARG, "bad logprob shape");
  if (n_rows == 0) return BD_OK;
  if (!logits || !targets || !logp) return set_error(BD_ERR_INVALID_ARG, "null pointer");
  if (dlogp && !dlogits) return set_error(BD_ERR_INVALID_ARG, "dlogp given without dlogits");
  if (dlogits && dlogits_stride < vocab) return set_error(BD_ERR_INVALID_ARG, "bad dlogits stride");
  if (dlogits == logits && dlogits_stride != row_stride)
    return set_error(BD_ERR_INVALID_ARG, "in-place gradient needs equal strides");
  if (n_rows > 0x7FFFFFFF) return set_error(BD_ERR_UNSUPPORTED, "too many rows");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const bool fusable = dlogp && vocab % (8 * kCl) == 0 && row_stride % 8 == 0 && dlogits_stride % 8 == 0 &&
                       aligned16(logits) && aligned16(dlogits) && (int64_t)n_rows * kCl <= 0x7FFFFFFF;
  if (fusable) {
    // one HBM read + one HBM write: the row stays in the cluster's shared
    // memory (the tail of each slice in registers when the slice is large)
    const int nv = vocab / kCl / 8;
    const bool regs = nv >= (kLpRegV + 1) * kFusedThreads;
    const int smem = (nv - (regs ? kLpRegV * kFusedThreads : 0)) * 16;
    if (smem > 200 * 1024) return set_error(BD_ERR_UNSUPPORTED, "vocab too large for the fused path");
    auto kern = regs ? logprob_fused1p_kernel<kLpRegV> : logprob_fused1p_kernel<0>;
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), 200 * 1024,
                                  "cudaFuncSetAttribute(logprob_fused1p)"))
      return rc;
    kern<<<(unsigned)(n_rows * kCl), kFusedThreads, smem, stream>>>(
        vocab, reinterpret_cast<const __nv_bfloat16*>(logits), row_stride, targets, logp, lse, dlogp,
        reinterpret_cast<__nv_bfloat16*>(dlogits), dlogits_stride);
    note_launches(1);
    return check_cuda(cudaGetLastError(), "logprob_fused1p_kernel launch");
  }
  logprob_kernel<<<(unsigned)n_rows, kThreads, 0, stream>>>(
      n_rows, vocab, reinterpret_cast<const __nv_bfloat16*>(logits), row_stride, targets, logp, lse, dlogp,
      reinterpret_cast<__nv_bfloat16*>(dlogits), dlogits_stride);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "logprob_kernel launch");
}
