// swiglu_sm100.cuh -- the SwiGLU backward and the down projection's dA (K5) in ONE pass.
//
// The MLP backward needs, per layer (reference lorapack.py:226, Case 3, for the down target):
//   dg = d_act * u * s (1 + g (1 - s)),  du = d_act * g * s,  s = sigmoid(g)     (SwiGLU bwd)
//   dA_down_i = act_i^T dH_down_i,        act = silu(g) * u                      (K5)
// Unfused, the SwiGLU backward writes act (T x ffn bf16) and the segment reduction reads it
// back.  Here a CTA owns a segment-reduction tile (adapter i, 128 ffn columns) and walks
// the adapter's tokens in 64-token k-blocks: TMA brings d_act, g, u ([64 tok][128 col],
// SW128 boxes) and dH_down ([64 tok][64 r]) into one stage; four transform warps turn the
// staged tiles into dg / du (written over the d_act / u tiles and TMA-stored to global,
// in place of g / u) and act (written over the g tile -- in exactly the swizzled MN-major
// layout the tensor core reads as the A operand); the MMA warp accumulates
// act^T dH over the tokens in TMEM; the same warps drain the fp32 dA tile at the end.
// act never leaves the SM.  Elementwise arithmetic is that of swiglu_bwd_kernel (same
// fp32 formulas on the bf16 inputs, bf16 rounding) and the MMA order that of the segment
// reduction, so dg, du and dA are bit-identical to the two-kernel path.
//
// Roles (1 CTA/SM): warp 0 TMA producer, warp 1 MMA issuer, 16 transform warps (the first
// four also drain the accumulator).  Tiles come from the same host LPT schedule as K3/K5
// (SegSched), or round-robin when the pack has no host row offsets (sched.n_ctas == 0).
#pragma once
#include "gemm_sm100.cuh"

namespace plora {

constexpr int kSwStages = 3;
constexpr int kSwXWarps = 16;                  // transform warps (the elementwise math needs the issue slots)
constexpr int kSwThreads = 64 + 32 * kSwXWarps;
constexpr int kSwTile = 16384;                 // [64 tok][128 col] bf16 = two SW128 boxes
constexpr int kSwQ = 8192;                     // dH_down [64 tok][64 r]
constexpr int kSwStageBytes = 3 * kSwTile + kSwQ;   // d_act, g, u, dH: 56 KB
constexpr int kSwSmemBytes = kSwStages * kSwStageBytes + 1024 + 256;

struct __align__(64) SwArgs {
  CUtensorMap tmD;   // d_act [T][ffn]      box {64, 64}
  CUtensorMap tmG;   // g     [T][ffn]      box {64, 64}
  CUtensorMap tmU;   // u     [T][ffn]
  CUtensorMap tmQ;   // dH_down [T][64]     box {64, 64}
  CUtensorMap tmDG;  // dg out (may alias g)
  CUtensorMap tmDU;  // du out (may alias u)
  __nv_bfloat16* dg;
  __nv_bfloat16* du;
  const int64_t* row_off;
  const int32_t* rpad_off;
  float* out;        // dA region of the down target (f32, adapter-major)
  int64_t ffn;
  int32_t M;         // = ffn (SEGRED rows)
  int32_t mt_per;    // ceil(ffn / 128)
  int32_t n_groups;  // n_adapters * mt_per
};

// Swizzled 16-byte chunk j (8 columns) of row r in a [64][64-col] SW128 box.
__device__ __forceinline__ uint32_t sw_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

__device__ __forceinline__ void sw_unpack(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 sw_pack(const float (&f)[8]) {
  uint4 v;
  v.x = pack_bf16x2(f[0], f[1]);
  v.y = pack_bf16x2(f[2], f[3]);
  v.z = pack_bf16x2(f[4], f[5]);
  v.w = pack_bf16x2(f[6], f[7]);
  return v;
}

// Tile idx of the segment-reduction grid (as decode_tile<64, MODE_SEGRED>): adapter
// idx / mt_per, ffn columns m0.. (128), tokens k0 .. k0 + k_len (the adapter's segment).
__device__ __forceinline__ TileInfo sw_decode(const SwArgs& a, int idx) {
  TileInfo t;
  t.adapter = idx / a.mt_per;
  t.m0 = (idx - t.adapter * a.mt_per) * kBM;
  t.m_len = min(kBM, a.M - t.m0);
  const int64_t r0 = a.row_off[t.adapter];
  t.k0 = static_cast<int>(r0);
  t.k_len = static_cast<int>(a.row_off[t.adapter + 1] - r0);
  t.n_main = (t.k_len + kBK - 1) / kBK;
  t.n0 = 0;
  t.n_lora = 0;
  t.rank = 0;
  return t;
}

// Named barrier of the transform warps (warps 2 .. 2 + kSwXWarps - 1).
__device__ __forceinline__ void sw_bar() { asm volatile("bar.sync 2, %0;" ::"n"(32 * kSwXWarps) : "memory"); }

__global__ void __launch_bounds__(kSwThreads, 1)
    plora_swiglu_segred_kernel(const __grid_constant__ SwArgs args, const __grid_constant__ SegSched sched) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSwStages * kSwStageBytes);
  uint64_t* xform = full + kSwStages;
  uint64_t* empty = xform + kSwStages;
  uint64_t* tfull = empty + kSwStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&args.tmD);
    tma_prefetch(&args.tmG);
    tma_prefetch(&args.tmU);
    tma_prefetch(&args.tmQ);
    for (int s = 0; s < kSwStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&xform[s], 1);
      mbar_init(&empty[s], 2);   // the MMA's commit + the transform warps (their TMA stores have read smem)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (TileIter it(sched.n_ctas ? &sched : nullptr, args.n_groups); it.valid(); it.next()) {
        const TileInfo t = sw_decode(args, it.tile());
        for (int b = 0; b < t.n_main; ++b) {
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t* s0 = smem + st * kSwStageBytes;
          const int kc = t.k0 + b * kBK;
          mbar_expect_tx(&full[st], kSwStageBytes);
          tma_load_2d(s0, &args.tmD, &full[st], t.m0, kc);
          tma_load_2d(s0 + 8192, &args.tmD, &full[st], t.m0 + 64, kc);
          tma_load_2d(s0 + kSwTile, &args.tmG, &full[st], t.m0, kc);
          tma_load_2d(s0 + kSwTile + 8192, &args.tmG, &full[st], t.m0 + 64, kc);
          tma_load_2d(s0 + 2 * kSwTile, &args.tmU, &full[st], t.m0, kc);
          tma_load_2d(s0 + 2 * kSwTile + 8192, &args.tmU, &full[st], t.m0 + 64, kc);
          tma_load_2d(s0 + 3 * kSwTile, &args.tmQ, &full[st], 0, kc);
          if (++st == kSwStages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer: dA += act^T dH
    constexpr uint32_t idesc = idesc_bf16(kBM, 64, true, true);
    int st = 0, acc = 0;
    uint32_t ph = 0, acc_phase = 0;
    for (TileIter it(sched.n_ctas ? &sched : nullptr, args.n_groups); it.valid(); it.next()) {
      const TileInfo t = sw_decode(args, it.tile());
      if (t.n_main == 0) continue;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * 64;
      for (int b = 0; b < t.n_main; ++b) {
        mbar_wait(&xform[st], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem + st * kSwStageBytes + kSwTile);       // act (over g)
          const uint32_t b0 = smem_u32(smem + st * kSwStageBytes + 3 * kSwTile);   // dH
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            umma_bf16(d_tmem, smem_desc_sw128(a0 + ks * 2048, 8192, 1024), smem_desc_sw128(b0 + ks * 2048, 8192, 1024),
                      idesc, (b > 0 || ks > 0) ? 1u : 0u);
          umma_commit(&empty[st]);
        }
        __syncwarp();
        if (++st == kSwStages) { st = 0; ph ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ transform (warps 2..17) + epilogue (2..5)
    const int tid = threadIdx.x - 64;   // 0 .. 32 * kSwXWarps - 1
    const bool epi = warp < 6;          // warps 2..5 drain the accumulator (one per TMEM lane quarter)
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    int st = 0, acc = 0, pend = -1;     // pend: stage whose TMA stores are still reading smem
    uint32_t ph = 0, acc_phase = 0;
    for (TileIter it(sched.n_ctas ? &sched : nullptr, args.n_groups); it.valid(); it.next()) {
      const TileInfo t = sw_decode(args, it.tile());
      const int ld = args.rpad_off[t.adapter + 1] - args.rpad_off[t.adapter];
      for (int b = 0; b < t.n_main; ++b) {
        const int valid = min(kBK, t.k_len - b * kBK);   // token rows of this segment in the k-block
        const int kc = t.k0 + b * kBK;
        mbar_wait(&full[st], ph);
        uint8_t* s0 = smem + st * kSwStageBytes;
        // 1024 16-byte chunks per tensor tile: chunk i -> box i/512, row (i%512)/8, column chunk i%8
#pragma unroll
        for (int k = 0; k < 1024 / (32 * kSwXWarps); ++k) {
          const int i = tid + 32 * kSwXWarps * k;
          const int box = i >> 9, r = (i >> 3) & 63, j = i & 7;
          const uint32_t off = box * 8192 + sw_off(r, j);
          float af[8], gf[8], uf[8], og[8], ou[8], oa[8];
          sw_unpack(*reinterpret_cast<const uint4*>(s0 + off), af);
          sw_unpack(*reinterpret_cast<const uint4*>(s0 + kSwTile + off), gf);
          sw_unpack(*reinterpret_cast<const uint4*>(s0 + 2 * kSwTile + off), uf);
#pragma unroll
          for (int e = 0; e < 8; ++e) swiglu_bwd_elem(af[e], gf[e], uf[e], og[e], ou[e], oa[e]);
          const bool in_seg = r < valid;
          *reinterpret_cast<uint4*>(s0 + kSwTile + off) = in_seg ? sw_pack(oa) : make_uint4(0, 0, 0, 0);
          const uint4 vg = sw_pack(og), vu = sw_pack(ou);
          if (valid == kBK) {   // full k-block: dg / du leave through TMA stores of the staged tiles
            *reinterpret_cast<uint4*>(s0 + off) = vg;
            *reinterpret_cast<uint4*>(s0 + 2 * kSwTile + off) = vu;
          } else if (in_seg) {  // last k-block of a segment: direct stores of its own rows only
            const int64_t col = static_cast<int64_t>(t.m0) + box * 64 + j * 8;
            if (col < args.ffn) {
              const int64_t o = static_cast<int64_t>(kc + r) * args.ffn + col;
              *reinterpret_cast<uint4*>(args.dg + o) = vg;
              *reinterpret_cast<uint4*>(args.du + o) = vu;
            }
          }
        }
        fence_proxy_async_smem();
        sw_bar();
        if (tid == 0) {
          mbar_arrive(&xform[st]);   // act is in place: the MMA may read the stage
          if (valid == kBK) {
            tma_store_2d(&args.tmDG, s0, t.m0, kc);
            tma_store_2d(&args.tmDG, s0 + 8192, t.m0 + 64, kc);
            tma_store_2d(&args.tmDU, s0 + 2 * kSwTile, t.m0, kc);
            tma_store_2d(&args.tmDU, s0 + 2 * kSwTile + 8192, t.m0 + 64, kc);
          }
          bulk_commit();
          // the previous stage's stores have read their smem: release it (second arrival)
          if (pend >= 0) {
            bulk_wait_read<1>();
            mbar_arrive(&empty[pend]);
          }
        }
        pend = st;
        if (++st == kSwStages) { st = 0; ph ^= 1; }
      }
      // epilogue of the tile: fp32 dA rows (TMEM lane = ffn column within the tile)
      if (!epi) continue;
      const int64_t goff = static_cast<int64_t>(args.M) * args.rpad_off[t.adapter] + static_cast<int64_t>(t.m0 + row) * ld;
      const bool row_ok = row < t.m_len;
      float* grow = args.out + goff;
      if (t.n_main == 0) {
        if (row_ok)
          for (int c = 0; c < ld; c += 4) *reinterpret_cast<float4*>(grow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * 64 + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        float v[32];
        tmem_chunk(tb, c, v);
        if (row_ok) {
#pragma unroll
          for (int q = 0; q < 32; q += 4)
            if (c * 32 + q < ld)
              *reinterpret_cast<float4*>(grow + c * 32 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (tid == 0) {
      bulk_wait<0>();
      if (pend >= 0) mbar_arrive(&empty[pend]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem_base);
  }
}

}  // namespace plora
