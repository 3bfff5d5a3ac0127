// dual_sm100.cuh -- K3 + K4 in ONE pass over dY.
//
// Cases 1 and 2 of the reference's packed_backward (lorapack.py:224-225) both stream the
// upstream gradient dY_i [T_i][k]:
//   Case 2 (K4):  dH_i   = alpha_i dY_i B_i^T     -- a reduction over k   ([T_i][r_i])
//   Case 1 (K3):  dB_i^T = Hs_i^T dY_i            -- a reduction over T_i ([k][r_i])
// Run separately they read dY twice.  Here a CTA owns a UNIT = up to kDualRC 128-row
// m-tiles of one adapter x one column chunk of k, and walks the chunk in 128-column steps.
// Every dY stage [128 rows][128 cols] (two SW128 boxes) lands in shared memory once and
// feeds two tcgen05 MMAs with the same bytes:
//   * K-major A of  D_h[j] (128 tokens x 64)  += dY_j     * L_i[128 k x 64]     (shrink)
//   * MN-major A of D_b    (128 k    x 64)    += dY_j^T   * Hs_j[128 tok x 64]  (segment red.)
// D_h[j] (one per m-tile) accumulates over the chunk's steps; D_b accumulates over the
// unit's m-tiles for one step and is drained per step (double-buffered).  What crosses
// units goes through fp32 partials in a caller-owned workspace and a deterministic fix-up
// (fixed summation order, no atomics):
//   dB partial [unit][kc][rpad16_i]  -> sum over the adapter's row chunks  -> grad region
//   dH partial [c][T][64] (nc > 1)   -> sum over column chunks, * alpha    -> bf16 dH
// With kDualRC = 4 and two column chunks (C3: 128 units) the partials cost ~1/3 of the dY
// bytes they replace.
//
// Roles (192 threads, 1 CTA/SM): warp 0 TMA producer, warp 1 MMA issuer (one lane) and
// Hs tail masking, warps 2..5 epilogue (TMEM lane quarter = warp % 4).
#pragma once
#include "sm100.cuh"
#include "pdl.cuh"

namespace plora {

#ifndef PLORA_DUAL_RANK_N
// MMA N = the adapter's rpad16 instead of 64 (build-time knob): parity-green, but no faster
// at C3 (K = 4096: 92.1 vs 90.2 us isolated, profiles/r2_dual_kernels.log) -- the kernel is
// paced by the tensor pipe's per-MMA cost at K = 16 x N = 64, not by B-operand bytes
#define PLORA_DUAL_RANK_N 0
#endif

constexpr int kDualRC = 4;                 // m-tiles per unit
constexpr int kDualStages = 4;             // dY ring: [128 rows][128 cols] bf16 = 32 KB per stage
constexpr int kDualMaxUnits = 2560;
constexpr int kDualMaxAdapters = 256;
constexpr int kDualMaxTargets = 3;         // targets of one launch (q/k/v or gate/up share the pack)
constexpr int kDualYBytes = 32768;
constexpr int kDualLBytes = 16384;         // L_i slice [128 k][64 r]
constexpr int kDualHBytes = 16384;         // Hs tile [128 tokens][64 r]
constexpr int kDualSmemBytes = kDualStages * kDualYBytes + 2 * kDualLBytes + kDualRC * kDualHBytes +
                               1024 /*align*/ + 256 /*barriers*/;

// Host-built unit list (kernel parameter space).  unit[u] = g0 | (rc - 1) << 20 | c << 22 |
// target << 25: first m-tile index g0 in the pack's 128-row tile list, rc consecutive m-tiles
// of one adapter, column chunk c (< 8) of target `target` (one launch serves up to 3 targets
// of a layer that share the pack).  boff[u] = float offset / 16 of the unit's dB partials.
struct DualTarget {
  int32_t k;         // dY width (h_out of the target)
  int32_t kc;        // column-chunk width (multiple of 128)
  int32_t nc;        // column chunks
  int32_t pad;
};
struct DualSched {
  int32_t n_units;
  int32_t n_targets;
  int32_t pad[2];
  DualTarget tg[kDualMaxTargets];
  uint32_t unit[kDualMaxUnits];
  uint32_t boff[kDualMaxUnits];
};

struct __align__(64) DualArgs {
  CUtensorMap tmY[kDualMaxTargets];   // dY [T][k], box {64 cols, 128 rows}
  CUtensorMap tmL[kDualMaxTargets];   // Bt_sh [n][k][64], box {64, 64, 1}
  CUtensorMap tmH[kDualMaxTargets];   // Hs [T][64], box {64, 128 rows}
  const int32_t* mtiles;    // [n_mtiles][4] {m0, m_len, adapter, 0}
  const float* alpha;
  const int32_t* rpad_off;
  __nv_bfloat16* dH[kDualMaxTargets];   // [T][64] bf16 (written directly when nc == 1)
  float* part_b;                        // dB partials (all targets)
  float* part_h[kDualMaxTargets];       // [nc][T][64] fp32 dH partials (nc > 1)
  int64_t T;
};

__device__ __forceinline__ void dual_decode(uint32_t u, int& g0, int& rc, int& c, int& tg) {
  g0 = static_cast<int>(u & 0xFFFFFu);
  rc = static_cast<int>((u >> 20) & 3u) + 1;
  c = static_cast<int>((u >> 22) & 7u);
  tg = static_cast<int>(u >> 25);
}

__global__ void __launch_bounds__(192, 1)
    plora_dual_kernel(const __grid_constant__ DualArgs args, const __grid_constant__ DualSched sched) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sY = smem;
  uint8_t* sL = sY + kDualStages * kDualYBytes;
  uint8_t* sH = sL + 2 * kDualLBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sH + kDualRC * kDualHBytes);
  uint64_t* empty = full + kDualStages;
  uint64_t* lfull = empty + kDualStages;
  uint64_t* lempty = lfull + 2;
  uint64_t* bfull = lempty + 2;
  uint64_t* bempty = bfull + 2;
  uint64_t* hfull = bempty + 2;
  uint64_t* hempty = hfull + 1;
  uint64_t* dhfull = hempty + 1;
  uint64_t* dhempty = dhfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dhempty + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int t = 0; t < sched.n_targets; ++t) {
      tma_prefetch(&args.tmY[t]);
      tma_prefetch(&args.tmL[t]);
      tma_prefetch(&args.tmH[t]);
    }
    for (int s = 0; s < kDualStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&lfull[s], 1);
      mbar_init(&lempty[s], 1);
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 4);
    }
    mbar_init(hfull, 1);
    mbar_init(hempty, 1);
    mbar_init(dhfull, 1);
    mbar_init(dhempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0, ls = 0;
      uint32_t ph = 0, lph = 0, hph = 0;
      for (int ui = blockIdx.x; ui < sched.n_units; ui += gridDim.x) {
        int g0, rc, c, tg;
        dual_decode(sched.unit[ui], g0, rc, c, tg);
        const int k = sched.tg[tg].k, kc = sched.tg[tg].kc;
        const int4* mt = reinterpret_cast<const int4*>(args.mtiles) + g0;
        const int a = mt[0].z;
        const int col0 = c * kc;
        const int nsteps = (min(kc, k - col0)) / 128;
        for (int s = 0; s < nsteps; ++s) {
          const int kcol = col0 + s * 128;
          mbar_wait(&lempty[ls], lph ^ 1);
          mbar_expect_tx(&lfull[ls], kDualLBytes);
          tma_load_3d(sL + ls * kDualLBytes, &args.tmL[tg], &lfull[ls], 0, kcol, a);
          tma_load_3d(sL + ls * kDualLBytes + 8192, &args.tmL[tg], &lfull[ls], 0, kcol + 64, a);
          if (++ls == 2) { ls = 0; lph ^= 1; }
          for (int j = 0; j < rc; ++j) {
            const int m0 = mt[j].x;
            mbar_wait(&empty[st], ph ^ 1);
            mbar_expect_tx(&full[st], kDualYBytes);
            tma_load_2d(sY + st * kDualYBytes, &args.tmY[tg], &full[st], kcol, m0);
            tma_load_2d(sY + st * kDualYBytes + 16384, &args.tmY[tg], &full[st], kcol + 64, m0);
            if (++st == kDualStages) { st = 0; ph ^= 1; }
          }
          if (s == 0) {
            // the unit's Hs tiles, after its first step's dY loads are in flight (the
            // buffer frees when the previous unit's last MMA retires)
            mbar_wait(hempty, hph ^ 1);
            hph ^= 1;
            mbar_expect_tx(hfull, rc * kDualHBytes);
            for (int j = 0; j < rc; ++j) tma_load_2d(sH + j * kDualHBytes, &args.tmH[tg], hfull, 0, mt[j].x);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int st = 0, ls = 0, bb = 0;
    uint32_t ph = 0, lph = 0, hph = 0, bph = 0, dph = 0;
    for (int ui = blockIdx.x; ui < sched.n_units; ui += gridDim.x) {
      int g0, rc, c, tg;
      dual_decode(sched.unit[ui], g0, rc, c, tg);
      const int k = sched.tg[tg].k, kc = sched.tg[tg].kc;
      const int4* mt = reinterpret_cast<const int4*>(args.mtiles) + g0;
      const int col0 = c * kc;
      const int nsteps = (min(kc, k - col0)) / 128;
#if PLORA_DUAL_RANK_N
      // N = the adapter's rpad16 (16..64): fewer B-operand bytes read from shared memory
      // per MMA -- the kernel is bound by shared-memory bandwidth (each staged dY byte is
      // read by two MMAs); columns past rpad16 of D_h stay stale and are not stored
      const uint32_t nr = static_cast<uint32_t>(args.rpad_off[mt[0].z + 1] - args.rpad_off[mt[0].z]);
#else
      const uint32_t nr = 64;
#endif
      const uint32_t idesc_shrink = idesc_bf16(128, nr, false, true);
      const uint32_t idesc_red = idesc_bf16(128, nr, true, true);
      mbar_wait(&dhempty[0], dph ^ 1);   // D_h of the previous unit drained
      dph ^= 1;
      tc_fence_after();
      for (int s = 0; s < nsteps; ++s) {
        if (s == 0) {
          mbar_wait(hfull, hph);
          hph ^= 1;
          // tokens past a segment's end (a partial last m-tile) belong to the next adapter:
          // zero their Hs rows so the segment reduction ignores them (the shrink rows they
          // produce are not stored)
          bool masked = false;
          for (int j = 0; j < rc; ++j) {
            const int ml = mt[j].y;
            if (ml < 128) {
              uint4* base = reinterpret_cast<uint4*>(sH + j * kDualHBytes + ml * 128);
              for (int i = lane; i < (128 - ml) * 8; i += 32) base[i] = make_uint4(0, 0, 0, 0);
              masked = true;
            }
          }
          if (masked) fence_proxy_async_smem();
          __syncwarp();
          tc_fence_after();
        }
        mbar_wait(&bempty[bb], bph ^ 1);
        mbar_wait(&lfull[ls], lph);
        tc_fence_after();
        for (int j = 0; j < rc; ++j) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t y0 = smem_u32(sY + st * kDualYBytes);
            const uint32_t l0 = smem_u32(sL + ls * kDualLBytes);
            const uint32_t h0 = smem_u32(sH + j * kDualHBytes);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {   // shrink: K = 128 dY columns (two SW128 K atoms)
              const uint64_t ad = smem_desc_sw128(y0 + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
              const uint64_t bd = smem_desc_sw128(l0 + ks * 2048, 8192, 1024);
              umma_bf16(tmem + 64 * j, ad, bd, idesc_shrink, (s > 0 || ks > 0) ? 1u : 0u);
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {   // segment reduction: K = 128 tokens, M = the 128 columns
              const uint64_t ad = smem_desc_sw128(y0 + ks * 2048, 16384, 1024);
              const uint64_t bd = smem_desc_sw128(h0 + ks * 2048, 8192, 1024);
              umma_bf16(tmem + 256 + 64 * bb, ad, bd, idesc_red, (j > 0 || ks > 0) ? 1u : 0u);
            }
            umma_commit(&empty[st]);
          }
          __syncwarp();
          if (++st == kDualStages) { st = 0; ph ^= 1; }
        }
        if (lane == 0) {
          umma_commit(&lempty[ls]);
          umma_commit(&bfull[bb]);
        }
        __syncwarp();
        if (++ls == 2) { ls = 0; lph ^= 1; }
        if (++bb == 2) { bb = 0; bph ^= 1; }
      }
      if (lane == 0) {
        umma_commit(hempty);
        umma_commit(dhfull);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int bb = 0;
    uint32_t bph = 0, dph = 0;
    for (int ui = blockIdx.x; ui < sched.n_units; ui += gridDim.x) {
      int g0, rc, c, tg;
      dual_decode(sched.unit[ui], g0, rc, c, tg);
      const int k = sched.tg[tg].k, kc = sched.tg[tg].kc, nc = sched.tg[tg].nc;
      const int4* mt = reinterpret_cast<const int4*>(args.mtiles) + g0;
      const int a = mt[0].z;
      const int rp = args.rpad_off[a + 1] - args.rpad_off[a];   // rpad16 of this adapter (<= 64)
      const int col0 = c * kc;
      const int nsteps = (min(kc, k - col0)) / 128;
      float* pb = args.part_b + static_cast<size_t>(sched.boff[ui]) * 16;
      for (int s = 0; s < nsteps; ++s) {
        mbar_wait(&bfull[bb], bph);
        tc_fence_after();
        float* dst = pb + static_cast<size_t>(s * 128 + row) * rp;   // dB^T partial row (k column)
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (h * 32 < rp) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + 256 + 64 * bb + h * 32 + lane_off, r);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (h * 32 + q * 4 < rp)
                *reinterpret_cast<float4*>(dst + h * 32 + q * 4) =
                    make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bempty[bb]);
        if (++bb == 2) { bb = 0; bph ^= 1; }
      }
      mbar_wait(dhfull, dph);
      dph ^= 1;
      tc_fence_after();
      const float alpha = args.alpha[a];
      for (int j = 0; j < rc; ++j) {
        const int4 m = mt[j];
        const bool ok = row < m.y;
        const int64_t t = static_cast<int64_t>(m.x) + row;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          uint32_t r[32];
          if (h * 32 < rp) {
            tmem_ld_32x32b_x32(tmem + 64 * j + h * 32 + lane_off, r);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (h * 32 + q >= rp) r[q] = 0u;   // past rpad16: not computed (N = rpad16)
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) r[q] = 0u;
          }
          if (!ok) continue;
          if (nc == 1) {   // complete: alpha-scaled bf16 dH (zero past the rank: L is zero-padded)
            __nv_bfloat16* o = args.dH[tg] + t * 64 + h * 32;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 w;
              w.x = pack_bf16x2(alpha * __uint_as_float(r[8 * q + 0]), alpha * __uint_as_float(r[8 * q + 1]));
              w.y = pack_bf16x2(alpha * __uint_as_float(r[8 * q + 2]), alpha * __uint_as_float(r[8 * q + 3]));
              w.z = pack_bf16x2(alpha * __uint_as_float(r[8 * q + 4]), alpha * __uint_as_float(r[8 * q + 5]));
              w.w = pack_bf16x2(alpha * __uint_as_float(r[8 * q + 6]), alpha * __uint_as_float(r[8 * q + 7]));
              reinterpret_cast<uint4*>(o)[q] = w;
            }
          } else if (h * 32 < rp) {
            float* o = args.part_h[tg] + (static_cast<int64_t>(c) * args.T + t) * 64 + h * 32;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (h * 32 + q * 4 < rp)
                *reinterpret_cast<float4*>(o + q * 4) =
                    make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dhempty);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Fix-up of the fused pass (deterministic: fixed summation order), every target of the
// launch in one grid:
//   blocks [bB[t], bB[t+1]): the dB^T grad region of target t, one float4 per thread:
//     G_t[k rpad_off[a] + kr rp_a + col] = sum_{q < nq_a} Pb[unit(t, a, q, kr / kc)][kr % kc][col]
//   blocks [bH[t], bH[t+1]) (nc_t > 1): one per m-tile, dH_t[t][:] = bf16(alpha_a sum_c Ph_t[c][t][:]).
struct DualFix {
  int32_t n;          // adapters
  int32_t n_targets;
  int32_t bB[kDualMaxTargets + 1];
  int32_t bH[kDualMaxTargets + 1];
  int32_t ubase[kDualMaxTargets][kDualMaxAdapters + 1];   // first unit of (target, adapter): units ordered t, a, q, c
};
struct DualOut {
  float* G[kDualMaxTargets];
  __nv_bfloat16* dH[kDualMaxTargets];
  const float* part_h[kDualMaxTargets];
};

__global__ void __launch_bounds__(256) plora_dual_fix_kernel(const __grid_constant__ DualFix f,
                                                             const __grid_constant__ DualSched sched,
                                                             const __grid_constant__ DualOut out,
                                                             const float* __restrict__ part_b,
                                                             const int32_t* __restrict__ rpad_off,
                                                             const float* __restrict__ alpha,
                                                             const int32_t* __restrict__ mtiles, int64_t T) {
  pdl_wait();
  pdl_trigger();
  const int b = static_cast<int>(blockIdx.x);
  if (b < f.bB[f.n_targets]) {
    int tg = 0;
    while (b >= f.bB[tg + 1]) ++tg;
    const DualTarget& tt = sched.tg[tg];
    const int64_t e = (static_cast<int64_t>(b - f.bB[tg]) * blockDim.x + threadIdx.x) * 4;   // element of G_t
    const int64_t k = tt.k;
    if (e >= k * rpad_off[f.n]) return;
    int lo = 0, hi = f.n - 1;   // adapter a: k * rpad_off[a] <= e < k * rpad_off[a + 1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (k * rpad_off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const int a = lo;
    const int rp = rpad_off[a + 1] - rpad_off[a];
    const int64_t o = e - k * rpad_off[a];
    const int kr = static_cast<int>(o / rp);
    const int col = static_cast<int>(o - static_cast<int64_t>(kr) * rp);
    const int c = kr / tt.kc;
    const int kk = kr - c * tt.kc;
    const int u0 = f.ubase[tg][a];
    const int nq = (f.ubase[tg][a + 1] - u0) / tt.nc;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < nq; ++q) {
      const int u = u0 + q * tt.nc + c;
      const float4 v = __ldcs(reinterpret_cast<const float4*>(part_b + static_cast<size_t>(sched.boff[u]) * 16 +
                                                              static_cast<int64_t>(kk) * rp + col));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    *reinterpret_cast<float4*>(out.G[tg] + e) = acc;
    return;
  }
  // dH: one block per (target, 128-row m-tile); thread -> (row, 8 columns)
  int tg = 0;
  while (b >= f.bH[tg + 1]) ++tg;
  const int nc = sched.tg[tg].nc;
  const int4 m = reinterpret_cast<const int4*>(mtiles)[b - f.bH[tg]];
  const int a = m.z;
  const int rp = rpad_off[a + 1] - rpad_off[a];
  const float al = alpha[a];
  const float* ph = out.part_h[tg];
  __nv_bfloat16* dH = out.dH[tg];
  for (int i = threadIdx.x; i < m.y * 8; i += blockDim.x) {
    const int r = i >> 3, c8 = (i & 7) * 8;
    const int64_t t = static_cast<int64_t>(m.x) + r;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
    if (c8 < rp) {
      for (int c = 0; c < nc; ++c) {
        const float4* p = reinterpret_cast<const float4*>(ph + (static_cast<int64_t>(c) * T + t) * 64 + c8);
        const float4 x = __ldcs(p), y = __ldcs(p + 1);
        v[0] += x.x; v[1] += x.y; v[2] += x.z; v[3] += x.w;
        v[4] += y.x; v[5] += y.y; v[6] += y.z; v[7] += y.w;
      }
    }
    uint4 w;
    w.x = pack_bf16x2(al * v[0], al * v[1]);
    w.y = pack_bf16x2(al * v[2], al * v[3]);
    w.z = pack_bf16x2(al * v[4], al * v[5]);
    w.w = pack_bf16x2(al * v[6], al * v[7]);
    *reinterpret_cast<uint4*>(dH + t * 64 + c8) = w;
  }
}

}  // namespace plora
