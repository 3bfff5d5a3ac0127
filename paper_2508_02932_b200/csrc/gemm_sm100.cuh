// gemm_sm100.cuh -- the packed-LoRA tensor-core engine for sm_100a.
//
// One persistent, warp-specialised tcgen05 kernel template covers every
// contraction on the packed-LoRA hot path (reference lorapack.py:183-231):
//
//   MODE_GEMM   Y[T][N]  = X[T][K] op(W)  (+ Hs_i[T][r] B_i^T  as extra K-steps)  (+ residual)
//               K1 base projection with K2b fused LoRA expand (forward), and
//               K6 dX = dY W^T + dH_i A_i^T (backward).  Tiles: 128 token rows of ONE
//               adapter (segment-index tile list) x BN output columns.
//   MODE_SHRINK H[T][64nb] = alpha_i X_i[T][K] L_i[K][64nb]
//               K2a (Hs = alpha X A) and K4 (dH = alpha dY B^T): per-tile adapter operand.
//   MODE_SEGRED G_i[M][rpad16_i] = sum_{t in segment i} P[t][M]^T Q[t][64nb]
//               K3 (dB_i^T = Hs_i^T dY_i) and K5 (dA_i = X_i^T dH_i): token-segment
//               reductions written as fp32 straight into the adapter-major grad region
//               (deterministic: one CTA owns each output tile, no atomics).
//
// Roles (192 threads, 1 CTA/SM): warp 0 = TMA producer, warp 1 = TMEM owner + UMMA
// issuer (one lane), warps 2..5 = epilogue (TMEM -> registers -> global).
// Pipelines: smem ring (full/empty mbarriers, TMA complete_tx / tcgen05.commit) and a
// double-buffered TMEM accumulator (tmem_full/tmem_empty).  All operands are staged by
// TMA with 128-byte swizzle; UMMA reads them through shared-memory descriptors.
#pragma once
#include "sm100.cuh"
#include "pdl.cuh"
#include "swiglu_math.cuh"

namespace plora {

#ifndef PLORA_EPI_SUSPEND_NS
#define PLORA_EPI_SUSPEND_NS 0   // epilogue accumulator wait: 0 = poll, else try_wait suspend hint (ns)
#endif
#if PLORA_EPI_SUSPEND_NS > 0
#define PLORA_EPI_WAIT(bar, par) mbar_wait_suspend(bar, par, PLORA_EPI_SUSPEND_NS)
#else
#define PLORA_EPI_WAIT(bar, par) mbar_wait(bar, par)
#endif


enum GemmMode : int { MODE_GEMM = 0, MODE_SHRINK = 1, MODE_SEGRED = 2 };

struct __align__(64) GemmArgs {
  CUtensorMap tmA;  // main A operand
  CUtensorMap tmB;  // main B operand
  CUtensorMap tmH;  // LoRA-block A operand: Hs or dH, K-major [T][64nb]
  CUtensorMap tmL;  // LoRA-block B operand: 3D [n][N][64nb], K-major
  CUtensorMap tmY;  // output [M][N] bf16, 32x32 boxes, SWIZZLE_64B (pair-kernel TMA store epilogue)
  const int32_t* mtiles;    // GEMM/SHRINK tile list [n_groups][4]; nullptr = uniform 128-row tiles
  const int64_t* row_off;   // SEGRED: token segment offsets [n+1]
  const int32_t* ranks;     // GEMM with LoRA: r_i
  const int32_t* rpad_off;  // SEGRED: grad layout prefix sums of rpad16
  const float* alpha;       // SHRINK: alpha_i
  void* out;
  const __nv_bfloat16* residual;  // GEMM: optional, same layout as out
  int64_t ldo;
  int32_t M;         // rows (uniform GEMM) or SEGRED output rows (Mdim)
  int32_t N;         // valid output columns
  int32_t K;         // reduction length (GEMM/SHRINK)
  int32_t n_groups;  // row groups
  int32_t n_ntiles;  // column tiles
  int32_t mt_per;    // SEGRED: ceil(M/128)
  int32_t has_lora;
  int32_t nb;        // 64-column rank blocks
  int32_t accumulate;  // pair kernel: Y += result (TMA reduce-add) instead of Y = result
  // Multi-target SHRINK / SEGRED (n_multi > 1, rank <= 64): targets j = 0..n_multi-1 share
  // the A operand (the same X), each with its own 64-column B operand (tmB, tmB2, tmB3)
  // and output (out, out2, out3); BN = 64 * n_multi and column chunk c belongs to target c/2.
  int32_t n_multi;
  CUtensorMap tmB2;
  CUtensorMap tmB3;
  void* out2;
  void* out3;
  const __nv_bfloat16* bias;   // GEMM: optional per-column bias added to the bf16 result
  // Stream-K partition of SHRINK / SEGRED (sk != 0; see SkIter): fp32 partials of split
  // tiles in sk_part (2 slots of 128 x BN per CTA), arrival counters in sk_cnt (one per
  // CTA, zero between launches: the last arriving piece resets its counter).
  int32_t sk;
  int32_t* sk_cnt;
  float* sk_part;
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 192;
constexpr int kBand = 16;  // row groups per raster band (L2 reuse of the B operand)

#ifndef PLORA_G64_STAGES
#define PLORA_G64_STAGES 8    // 1-CTA kernel stages at BN = 64 / 128 / 192 (build-time knobs)
#endif
#ifndef PLORA_G128_STAGES
#define PLORA_G128_STAGES 6
#endif
#ifndef PLORA_G192_STAGES
#define PLORA_G192_STAGES 5
#endif

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;              // 16 KB
  static constexpr int kBBytes = BN * kBK * 2;               // BN x 64 bf16
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (BN == 256) ? 4 : (BN == 192 ? PLORA_G192_STAGES : (BN == 128 ? PLORA_G128_STAGES :
                                                                                     PLORA_G64_STAGES));
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 :
                                   (2 * BN <= 256 ? 256 : 512)));   // power of two >= 2 accumulators
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct TileInfo {
  int m0, m_len, adapter, k0, k_len, n0, n_main, n_lora, rank;
};

// Static longest-processing-time-first schedule for the segment reductions (K3/K5):
// their tiles cost ~T_i (the adapter's token count), which varies 4x across a pack,
// so round-robin tile assignment leaves some SMs with 1.5x the mean work.  The host
// computes the LPT assignment (plora_abi.cu) and passes it in kernel parameter space:
// CTA b runs tiles[off[b] .. off[b+1]).
constexpr int kSchedMaxCtas = 160;
constexpr int kSchedMaxTiles = 6144;
struct SegSched {
  int32_t n_ctas;
  uint16_t off[kSchedMaxCtas + 1];
  uint16_t tiles[kSchedMaxTiles];
};

// The persistent tile loop shared by the three warp roles.
struct TileIter {
  int j, end, step;
  const uint16_t* list;
  __device__ __forceinline__ TileIter(const SegSched* sched, int total) {
    if (sched != nullptr) {
      j = sched->off[blockIdx.x];
      end = sched->off[blockIdx.x + 1];
      step = 1;
      list = sched->tiles;
    } else {
      j = blockIdx.x;
      end = total;
      step = gridDim.x;
      list = nullptr;
    }
  }
  __device__ __forceinline__ bool valid() const { return j < end; }
  __device__ __forceinline__ int tile() const { return list ? static_cast<int>(list[j]) : j; }
  __device__ __forceinline__ void next() { j += step; }
};

// Stream-K partition of the skinny LoRA contractions (K2a/K4 shrink, K3/K5 segment
// reductions).  Their tiles are few and long (a 128-row shrink tile streams all of h; a
// segment-reduction tile streams its adapter's whole token segment): at T = 4096 per GPU
// the shrink has 32 tiles for 148 SMs, at T = 32768 it has 1.8 waves.  Instead of whole
// tiles, CTA c of G takes the linear k-block range [c W / G, (c+1) W / G) of the tile
// sequence (W = total k-blocks), so every SM streams the same number of bytes.  A tile cut
// by CTA boundaries is computed as pieces; every piece stores its fp32 partial in its
// CTA's slot, and the LAST piece to finish (arrival counter) sums all pieces in piece
// order -- deterministic for a given pack, no waiting, no atomics on the data.
//   SHRINK: every tile has ceil(K / 64) k-blocks.  SEGRED: the tiles of adapter a have
//   max(1, ceil(T_a / 64)) (an empty segment costs one unit and writes zeros).
struct SkUnit {
  int tile, kb0, kb1, piece, np, c0;
  bool first;   // the CTA's first unit (partial slot 0) -- else slot 1
};

template <int MODE>
struct SkIter {
  const GemmArgs& a;
  int64_t W, x, xend, cstart;
  int G, c, per, nkb;
  int ad, len;       // SEGRED: current adapter and its tile length
  int64_t ap;        // SEGRED: linear start of adapter `ad`'s tiles
  int64_t tend;
  SkUnit u;

  __device__ __forceinline__ int seglen(int i) const {
    const int64_t t = a.row_off[i + 1] - a.row_off[i];
    return t > 0 ? static_cast<int>((t + kBK - 1) / kBK) : 1;
  }
  __device__ __forceinline__ int cta_of(int64_t pos) const { return static_cast<int>(((pos + 1) * G - 1) / W); }

  __device__ __forceinline__ explicit SkIter(const GemmArgs& args) : a(args) {}
  __device__ __forceinline__ void init() {
    G = gridDim.x;
    c = blockIdx.x;
    per = a.n_ntiles * (MODE == MODE_SEGRED ? a.mt_per : 1);
    nkb = (a.K + kBK - 1) / kBK;
    if (MODE == MODE_SEGRED) {
      W = 0;
      const int n = a.n_groups / a.mt_per;
      for (int i = 0; i < n; ++i) W += static_cast<int64_t>(per) * seglen(i);
      ad = 0;
      ap = 0;
      len = n > 0 ? seglen(0) : 1;
    } else {
      W = static_cast<int64_t>(a.n_groups) * a.n_ntiles * nkb;
    }
    cstart = x = W * c / G;
    xend = W * (c + 1) / G;
    if (x < xend) load();
  }
  __device__ __forceinline__ void load() {
    int64_t tstart;
    if (MODE == MODE_SEGRED) {
      while (x >= ap + static_cast<int64_t>(per) * len) {
        ap += static_cast<int64_t>(per) * len;
        ++ad;
        len = seglen(ad);
      }
      const int j = static_cast<int>((x - ap) / len);
      u.tile = ad * per + j;
      tstart = ap + static_cast<int64_t>(j) * len;
      tend = tstart + len;
    } else {
      u.tile = static_cast<int>(x / nkb);
      tstart = static_cast<int64_t>(u.tile) * nkb;
      tend = tstart + nkb;
    }
    u.kb0 = static_cast<int>(x - tstart);
    u.kb1 = static_cast<int>((tend < xend ? tend : xend) - tstart);
    u.c0 = cta_of(tstart);
    u.np = cta_of(tend - 1) - u.c0 + 1;
    u.piece = c - u.c0;
    u.first = x == cstart;
    pstart0 = W * u.c0 / G == tstart;
  }
  bool pstart0;   // piece 0 is its CTA's first unit (partial slot 0)
  __device__ __forceinline__ bool valid() const { return x < xend; }
  __device__ __forceinline__ void next() {
    x = tend < xend ? tend : xend;
    if (x < xend) load();
  }
  // partial slot of piece p of the current unit's tile
  __device__ __forceinline__ int slot(int p) const { return 2 * (u.c0 + p) + ((p == 0 && !pstart0) ? 1 : 0); }
};

// The persistent unit loop of the 1-CTA kernel's three warp roles: whole tiles
// (round-robin or a host LPT list) or stream-K pieces.
// SK is a compile-time choice (the launcher instantiates the stream-K kernel only when the
// pack carries a workspace and the launch is short of SMs), so whole-tile launches run
// without the stream-K bookkeeping in their registers.
template <int MODE, bool SK>
struct UnitLoop {
  TileIter ti;
  SkIter<MODE> si;
  static constexpr bool sk = SK && MODE != MODE_GEMM;
  __device__ __forceinline__ UnitLoop(const GemmArgs& a, const SegSched* sched, int total)
      : ti(sched, total), si(a) {
    if (sk) si.init();
  }
  __device__ __forceinline__ bool valid() const { return sk ? si.valid() : ti.valid(); }
  __device__ __forceinline__ int tile() const { return sk ? si.u.tile : ti.tile(); }
  __device__ __forceinline__ int kb0() const { return sk ? si.u.kb0 : 0; }
  __device__ __forceinline__ int kb1(int nblk) const { return sk ? min(si.u.kb1, nblk) : nblk; }
  __device__ __forceinline__ bool split() const { return sk && si.u.np > 1; }
  __device__ __forceinline__ void next() {
    if (sk) si.next();
    else    ti.next();
  }
};

template <int BN, int MODE>
__device__ __forceinline__ TileInfo decode_tile(const GemmArgs& a, int idx) {
  TileInfo t;
  int g, nt;
  if (MODE == MODE_SEGRED) {
    g = idx / a.n_ntiles;
    nt = idx - g * a.n_ntiles;
    t.adapter = g / a.mt_per;
    t.m0 = (g - t.adapter * a.mt_per) * kBM;
    t.m_len = min(kBM, a.M - t.m0);
    const int64_t r0 = a.row_off[t.adapter];
    t.k0 = static_cast<int>(r0);
    t.k_len = static_cast<int>(a.row_off[t.adapter + 1] - r0);
    t.n_lora = 0;
    t.rank = 0;
  } else {
    const int per_band = kBand * a.n_ntiles;
    const int band = idx / per_band;
    const int rem = idx - band * per_band;
    const int g0 = band * kBand;
    const int bsz = min(kBand, a.n_groups - g0);
    nt = rem / bsz;
    g = g0 + (rem - nt * bsz);
    if (a.mtiles != nullptr) {
      const int4 mt = reinterpret_cast<const int4*>(a.mtiles)[g];
      t.m0 = mt.x;
      t.m_len = mt.y;
      t.adapter = mt.z;
    } else {
      t.m0 = g * kBM;
      t.m_len = min(kBM, a.M - t.m0);
      t.adapter = 0;
    }
    t.k0 = 0;
    t.k_len = a.K;
    if (MODE == MODE_GEMM && a.has_lora) {
      t.rank = a.ranks[t.adapter];
      t.n_lora = min((t.rank + 63) / 64, a.nb);
    } else {
      t.rank = 0;
      t.n_lora = 0;
    }
  }
  t.n0 = nt * BN;
  t.n_main = (t.k_len + kBK - 1) / kBK;
  return t;
}

// Chunk c (32 fp32 columns) of this thread's TMEM accumulator row.
__device__ __forceinline__ void tmem_chunk(uint32_t tb, int c, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(tb + c * 32, r);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Named barrier of the 4 epilogue warps (warps 2..5) of the 1-CTA kernel.
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Stream-K piece of a split tile: store the fp32 partial in this CTA's slot (layout
// [chunk][quarter][float4 q][lane]: coalesced 512-byte rows), then count the arrival.
// Returns true on the piece that arrived last -- it owns the fix-up and the output.
template <int BN, int MODE>
__device__ __forceinline__ bool sk_arrive(const GemmArgs& a, const SkIter<MODE>& si, uint32_t tb, int quarter,
                                          int lane, int* flag) {
  float4* mine = reinterpret_cast<float4*>(a.sk_part) +
                 static_cast<size_t>(2 * si.c + (si.u.first ? 0 : 1)) * (BN * 32);
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    float v[32];
    tmem_chunk(tb, c, v);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      __stcg(mine + ((c * 4 + quarter) * 8 + q) * 32 + lane, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
  }
  __threadfence();
  epi_bar();
  if (threadIdx.x == 64) {
    const int old = atomicAdd(&a.sk_cnt[si.u.c0], 1);
    const int last = old == si.u.np - 1;
    if (last) a.sk_cnt[si.u.c0] = 0;   // ready for the next launch (stream-ordered)
    *reinterpret_cast<volatile int*>(flag) = last;
  }
  epi_bar();
  const bool last = *reinterpret_cast<volatile int*>(flag) != 0;
  if (last) __threadfence();
  return last;
}

// Chunk c of a split tile: the pieces' partials summed in piece order (this piece's own
// from TMEM), so the result does not depend on which piece arrived last.
template <int BN, int MODE>
__device__ __forceinline__ void sk_gather(const GemmArgs& a, const SkIter<MODE>& si, uint32_t tb, int c, int quarter,
                                          int lane, float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = 0.f;
  for (int p = 0; p < si.u.np; ++p) {
    if (p == si.u.piece) {
      float w[32];
      tmem_chunk(tb, c, w);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += w[j];
    } else {
      const float4* src = reinterpret_cast<const float4*>(a.sk_part) + static_cast<size_t>(si.slot(p)) * (BN * 32) +
                          ((c * 4 + quarter) * 8) * 32 + lane;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = __ldcg(src + q * 32);
        v[4 * q] += f.x;
        v[4 * q + 1] += f.y;
        v[4 * q + 2] += f.z;
        v[4 * q + 3] += f.w;
      }
    }
  }
}

template <int BN, int MODE, bool B_MN, bool SK>
__device__ __forceinline__ void gemm_body(const GemmArgs& args, const SegSched* sched) {
  using Cfg = GemmCfg<BN>;
  constexpr bool A_MN = (MODE == MODE_SEGRED);
  constexpr bool MAIN_B_MN = (MODE == MODE_GEMM) ? B_MN : true;
  constexpr int S = Cfg::kStages;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int total = args.n_groups * args.n_ntiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&args.tmA);
    tma_prefetch(&args.tmB);
    if (MODE == MODE_GEMM && args.has_lora) {
      tma_prefetch(&args.tmH);
      tma_prefetch(&args.tmL);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();   // the next kernel may launch and run its prologue under this one's tail
  pdl_wait();      // ... and this one touches global memory only after the previous grid completed

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (UnitLoop<MODE, SK> it(args, sched, total); it.valid(); it.next()) {
        const TileInfo t = decode_tile<BN, MODE>(args, it.tile());
        const int b1 = it.kb1(t.n_main + t.n_lora);
        for (int b = it.kb0(); b < b1; ++b) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sA = smem + stage * Cfg::kStageBytes;
          uint8_t* sB = sA + Cfg::kABytes;
          mbar_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          if (b < t.n_main) {
            const int kc = t.k0 + b * kBK;
            if (A_MN) {
              tma_load_2d(sA, &args.tmA, &full_bar[stage], t.m0, kc);
              tma_load_2d(sA + 8192, &args.tmA, &full_bar[stage], t.m0 + 64, kc);
            } else {
              tma_load_2d(sA, &args.tmA, &full_bar[stage], kc, t.m0);
            }
            if (MODE != MODE_GEMM && args.n_multi > 1) {   // one 64-column B chunk per target
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) {
                const CUtensorMap* mj = j == 0 ? &args.tmB : (j == 1 ? &args.tmB2 : &args.tmB3);
                if (MODE == MODE_SHRINK) tma_load_3d(sB + j * 8192, mj, &full_bar[stage], 0, kc, t.adapter);
                else                     tma_load_2d(sB + j * 8192, mj, &full_bar[stage], 0, kc);
              }
            } else if (MODE == MODE_SHRINK) {
              tma_load_3d(sB, &args.tmB, &full_bar[stage], t.n0, kc, t.adapter);
            } else if (MAIN_B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sB + j * 8192, &args.tmB, &full_bar[stage], t.n0 + 64 * j, kc);
            } else {
              tma_load_2d(sB, &args.tmB, &full_bar[stage], kc, t.n0);
            }
          } else {
            const int lb = b - t.n_main;
            tma_load_2d(sA, &args.tmH, &full_bar[stage], lb * 64, t.m0);
            tma_load_3d(sB, &args.tmL, &full_bar[stage], lb * 64, t.n0, t.adapter);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer
    constexpr uint32_t idesc_main = idesc_bf16(kBM, BN, A_MN, MAIN_B_MN);
    constexpr uint32_t idesc_lora = idesc_bf16(kBM, BN, false, false);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (UnitLoop<MODE, SK> it(args, sched, total); it.valid(); it.next()) {
      const TileInfo t = decode_tile<BN, MODE>(args, it.tile());
      const int kb_lo = it.kb0();
      const int kb_hi = it.kb1(t.n_main + t.n_lora);
      if (kb_hi <= kb_lo) continue;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int b = kb_lo; b < kb_hi; ++b) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        uint8_t* sA = smem + stage * Cfg::kStageBytes;
        uint8_t* sB = sA + Cfg::kABytes;
        const bool lora = b >= t.n_main;
        if (MODE == MODE_SEGRED) {
          // Token rows past the segment end belong to the next adapter: zero them in
          // both operands before the tensor core reads the stage.
          const int valid = t.k_len - b * kBK;
          if (valid < kBK) {
            const int nrows = kBK - valid;
            const int per = nrows * 8;  // 16-byte chunks per sub-tile
            for (int i = lane; i < (2 + BN / 64) * per; i += 32) {
              const int sub = i / per;
              const int rem = i - sub * per;
              uint8_t* base = (sub < 2) ? (sA + sub * 8192) : sB + (sub - 2) * 8192;
              reinterpret_cast<uint4*>(base + (valid + rem / 8) * 128)[rem % 8] = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncwarp();
          }
        }
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sA);
          const uint32_t b0 = smem_u32(sB);
          int ksteps = 4;
          if (lora) ksteps = min(4, (t.rank - (b - t.n_main) * 64 + 15) / 16);
          for (int ks = 0; ks < ksteps; ++ks) {
            uint64_t ad, bd;
            if (!lora && A_MN) ad = smem_desc_sw128(a0 + ks * 2048, 8192, 1024);
            else               ad = smem_desc_sw128(a0 + ks * 32, 16, 1024);
            if (!lora && MAIN_B_MN) bd = smem_desc_sw128(b0 + ks * 2048, 8192, 1024);
            else                    bd = smem_desc_sw128(b0 + ks * 32, 16, 1024);
            umma_bf16(d_tmem, ad, bd, lora ? idesc_lora : idesc_main, (b > kb_lo || ks > 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int* sk_flag = reinterpret_cast<int*>(tmem_slot + 1);
    for (UnitLoop<MODE, SK> it(args, sched, total); it.valid(); it.next()) {
      const TileInfo t = decode_tile<BN, MODE>(args, it.tile());
      const bool empty = it.kb1(t.n_main + t.n_lora) <= it.kb0();
      if (MODE == MODE_SEGRED) {
        const int ld = args.rpad_off[t.adapter + 1] - args.rpad_off[t.adapter];
        const int64_t goff = static_cast<int64_t>(args.M) * args.rpad_off[t.adapter] +
                             static_cast<int64_t>(t.m0 + row) * ld;
        const bool multi = args.n_multi > 1;
        const bool row_ok = row < t.m_len;
        if (empty) {
          if (row_ok) {
            for (int j = 0; j < (multi ? args.n_multi : 1); ++j) {
              float* grow = reinterpret_cast<float*>(j == 0 ? args.out : (j == 1 ? args.out2 : args.out3)) + goff;
              const int c_lo = multi ? 0 : t.n0;
              const int c_hi = multi ? min(64, ld) : min(t.n0 + BN, ld);
              for (int c = c_lo; c < c_hi; c += 4)
                *reinterpret_cast<float4*>(grow + c) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          continue;
        }
        PLORA_EPI_WAIT(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t tb = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
        const bool split = it.split();
        if (!split || sk_arrive<BN>(args, it.si, tb, quarter, lane, sk_flag)) {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            if (split) sk_gather<BN>(args, it.si, tb, c, quarter, lane, v);
            else       tmem_chunk(tb, c, v);
            const int tg = multi ? (c >> 1) : 0;
            float* grow = reinterpret_cast<float*>(tg == 0 ? args.out : (tg == 1 ? args.out2 : args.out3)) + goff;
            const int col0 = multi ? (c & 1) * 32 : t.n0 + c * 32;
            if (row_ok) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                if (col0 + j < ld)
                  *reinterpret_cast<float4*>(grow + col0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            }
          }
        }
      } else {
        if (empty) continue;
        PLORA_EPI_WAIT(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t tb = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
        const float scale = (MODE == MODE_SHRINK) ? args.alpha[t.adapter] : 1.0f;
        const bool row_ok = row < t.m_len;
        const int64_t orow = static_cast<int64_t>(t.m0 + row) * args.ldo;
        const bool multi = MODE == MODE_SHRINK && args.n_multi > 1;
        const __nv_bfloat16* res = (MODE == MODE_GEMM && args.residual) ? args.residual + orow : nullptr;
        const bool split = it.split();
        if (!split || sk_arrive<BN>(args, it.si, tb, quarter, lane, sk_flag)) {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            if (split) sk_gather<BN>(args, it.si, tb, c, quarter, lane, v);
            else       tmem_chunk(tb, c, v);
            const int tg = multi ? (c >> 1) : 0;
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(tg == 0 ? args.out : (tg == 1 ? args.out2 : args.out3)) +
                               orow;
            const int col0 = multi ? (c & 1) * 32 : t.n0 + c * 32;
            if (row_ok && col0 < args.N) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= scale;
              if (MODE == MODE_GEMM && args.bias != nullptr) {   // round(round(y) + b): as a bf16 bias add
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col0 + j < args.N)
                    v[j] = __bfloat162float(__float2bfloat16_rn(v[j])) + __bfloat162float(args.bias[col0 + j]);
              }
              if (col0 + 32 <= args.N) {
                if (res) {
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const uint4 rv = *reinterpret_cast<const uint4*>(res + col0 + q * 8);
                    const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                      const float2 f = __bfloat1622float2(rh[h]);
                      v[q * 8 + 2 * h] += f.x;
                      v[q * 8 + 2 * h + 1] += f.y;
                    }
                  }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint4 w;
                  w.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
                  w.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
                  w.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
                  w.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
                  *reinterpret_cast<uint4*>(o + col0 + q * 8) = w;
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  if (col0 + j < args.N) {
                    float x = v[j];
                    if (res) x += __bfloat162float(res[col0 + j]);
                    o[col0 + j] = __float2bfloat16_rn(x);
                  }
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

template <int BN, int MODE, bool B_MN, bool SK = false>
__global__ void __launch_bounds__(kThreads, 1) plora_gemm_kernel(const __grid_constant__ GemmArgs args) {
  gemm_body<BN, MODE, B_MN, SK>(args, nullptr);
}

// Segment reduction with a host-computed LPT tile schedule (see SegSched).
template <int BN>
__global__ void __launch_bounds__(kThreads, 1) plora_segred_lpt_kernel(const __grid_constant__ GemmArgs args,
                                                                        const __grid_constant__ SegSched sched) {
  gemm_body<BN, MODE_SEGRED, true, false>(args, &sched);
}

// ============================================================================
// CTA-pair variant of MODE_GEMM (K1 + K2b forward, K6 dX): a cluster of 2 CTAs on
// one TPC computes a 256 x (256*NB) tile with tcgen05.mma.cta_group::2 (M = 256).
// Each CTA stages its own 128 rows of A and its half of every 256-column chunk of B
// per K-block (16 KB + NB x 16 KB per stage).  NB = 2 (256 x 512 tiles) moves 25%
// fewer operand bytes per FLOP than NB = 1 -- L2->SMEM bandwidth (~10 TB/s measured)
// is what bounds this kernel -- at the price of a single (not double-buffered)
// 512-column TMEM accumulator.  The leader (rank 0) owns the full barriers (TMA
// bytes of both CTAs land on it), issues the UMMAs and multicasts commits to both
// CTAs' empty / tmem_full barriers; both CTAs' epilogues drain their own 128 TMEM
// lanes and arrive on the leader's tmem_empty barrier.  Pair tiles never straddle
// adapters (meta builder), so the fused LoRA K-steps use one adapter's B_i.
#ifndef PLORA_PAIR_STAGES
#define PLORA_PAIR_STAGES 3   // NB = 2 mainloop stages (build-time knob for experiments)
#endif
#ifndef PLORA_PAIR_NB1_STAGES
#define PLORA_PAIR_NB1_STAGES 6   // NB = 1 (256 x 256, K <= 1024) mainloop stages
#endif
#ifndef PLORA_PAIR_BUFS
#define PLORA_PAIR_BUFS 4     // NB = 2 epilogue staging buffers per warp
#endif
#ifndef PLORA_STORE_EVICT_FIRST
#define PLORA_STORE_EVICT_FIRST 0   // pair-epilogue TMA stores with an L2 evict_first policy (experiment knob)
#endif
#ifndef PLORA_PAIR_MAXNREG
#define PLORA_PAIR_MAXNREG 0     // > 0: __maxnreg__ instead of launch_bounds(320, 1) (= 168 regs); 184 / 192 / 200
                                 // compile with fewer SwiGLU-epilogue spills but fail to launch ("too many resources")
#endif
#if PLORA_PAIR_MAXNREG > 0
#define PLORA_PAIR_BOUNDS __maxnreg__(PLORA_PAIR_MAXNREG)
#else
#define PLORA_PAIR_BOUNDS __launch_bounds__(PairCfg<NB>::kThreads, 1)
#endif
#ifndef PLORA_SWIGLU_DIRECT
#define PLORA_SWIGLU_DIRECT 2       // SwiGLU epilogue: gate/up chunk pairs stored before the accumulator release
#endif
#ifndef PLORA_PAIR_KDIRECT
#define PLORA_PAIR_KDIRECT 4  // NB = 2 chunks stored before the accumulator release (rest parked)
#endif

template <int NB, int EPI_ = 0>
struct PairCfg {
  static constexpr int kBN = 256 * NB;                      // output columns per pair tile
  static constexpr int kABytes = kBM * kBK * 2;             // 16 KB (own 128 rows)
  static constexpr int kBBytes = NB * 128 * kBK * 2;        // own half of each 256-col chunk
  static constexpr int kStageBytes = kABytes + kBBytes;
  // NB = 2: 3 mainloop stages (3 k-blocks = 3 x 1024 MMA cycles of lookahead) and 4 epilogue
  // staging buffers per warp, 4 chunks stored before the accumulator release (4 parked: no
  // spills).  Same-box A/B against 4 stages / 2 buffers / 3 direct: GEMM time equal at locked
  // clocks, step +1.9% (stages) and +0.5% (kDirect) with the SM clock higher under the power
  // cap; 2 stages starve the MMA (-14%) (profiles/r1s3_stages_ab.log).
  static constexpr int kStages = NB == 1 ? PLORA_PAIR_NB1_STAGES : PLORA_PAIR_STAGES;
  static constexpr int kStgBufs = NB == 1 ? 2 : PLORA_PAIR_BUFS;
  static constexpr int kAccStages = NB == 1 ? 2 : 1;
  static constexpr int kTmemCols = 512;
  static constexpr int kEpiWarps = 8;                       // 2 per TMEM lane quarter
  static constexpr int kThreads = 64 + 32 * kEpiWarps;      // producer + MMA + epilogue
  static constexpr int kStgBytes = kEpiWarps * kStgBufs * 2048;   // per warp: kStgBufs x [32 rows x 32 bf16], SW64
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*barriers*/ + kStgBytes + 1024 /*align*/;
  static constexpr int kBand = 8;                           // pair tiles per raster band
};

// Segmented pair GEMM: up to 3 problems sharing one accumulator schedule.
//  * N-segments (n_seg > 1, k_seg == 1): targets that share the input X (q/k/v, gate/up)
//    -- one launch, the output tiles of every target enumerated together; target s has
//    its own weight, LoRA operands and output.
//  * K-segments (k_seg > 1, n_seg == 1): input gradients of those targets, which sum
//    into ONE dX = sum_s dY_s W_s + dH_s A_s^T -- one accumulator over the concatenated
//    K range (fp32 in TMEM, no bf16 read-modify-write between targets).
// Segment 0 uses g.tmA/tmB/tmH/tmL/tmY; segments 1, 2 the arrays below.
struct __align__(64) PairArgs {
  GemmArgs g;
  CUtensorMap tmA2[2];
  CUtensorMap tmB2[2];
  CUtensorMap tmH2[2];
  CUtensorMap tmL2[2];
  CUtensorMap tmY2[2];
  int32_t n_seg;
  int32_t k_seg;
  int32_t seg_nt_end[3];   // N-segments: cumulative n-tile counts
  int32_t seg_N[3];        // N-segments: valid output columns
  int32_t seg_kb_end[3];   // K-segments: cumulative main K-block counts
  int32_t band;            // tile raster: > 0 M-band row groups, < 0 N-band column tiles, 0 = kBand rows
  int32_t paired;          // gate/up + SwiGLU: chunk c of every 256-column tile is segment c (see EPI_SWIGLU)
  void* seg_out[3];        // N-segments: output base (masked direct stores)
  int64_t seg_ldo[3];
  const void* seg_bias[3]; // N-segments: optional bf16 bias [N] added in the epilogue
};

// Epilogue variants of the pair kernel.
//  EPI_STORE  : bf16 result (+ reduce-add) through TMA.
//  EPI_SWIGLU : "paired" gate/up tiles -- TMEM columns [0,256) hold gate, [256,512) up for
//               the same 256 ffn columns; the epilogue stores g, u (segments 0, 1) and
//               act = silu(g) u (segment 2's map) computed from the bf16-rounded g, u,
//               bit-identical to swiglu_fwd_kernel.
enum PairEpi : int { EPI_STORE = 0, EPI_SWIGLU = 2 };

__device__ __forceinline__ const CUtensorMap* seg_map(const CUtensorMap* m0, const CUtensorMap* rest, int s) {
  return s == 0 ? m0 : rest + (s - 1);
}

struct PairTile {
  int m0, m_len, adapter, n0, n_main, n_lora, rank, seg, nlps;
};

template <int NB>
__device__ __forceinline__ PairTile decode_pair_tile(const PairArgs& p, int idx) {
  const GemmArgs& a = p.g;
  PairTile t;
  int g, nt;
  if (p.band >= 0) {   // M-bands: `band` row groups, all column tiles, row group fastest
    const int bw = p.band > 0 ? p.band : PairCfg<NB>::kBand;
    const int per_band = bw * a.n_ntiles;
    const int band = idx / per_band;
    const int rem = idx - band * per_band;
    const int g0 = band * bw;
    const int bsz = min(bw, a.n_groups - g0);
    nt = rem / bsz;
    g = g0 + (rem - nt * bsz);
  } else {             // N-bands: -band column tiles, all row groups, column tile fastest
    const int bw = -p.band;
    const int per_band = bw * a.n_groups;
    const int band = idx / per_band;
    const int rem = idx - band * per_band;
    const int n0b = band * bw;
    const int bsz = min(bw, a.n_ntiles - n0b);
    g = rem / bsz;
    nt = n0b + (rem - g * bsz);
  }
  if (a.mtiles != nullptr) {
    const int4 mt = reinterpret_cast<const int4*>(a.mtiles)[g];
    t.m0 = mt.x;
    t.m_len = mt.y;
    t.adapter = mt.z;
  } else {
    t.m0 = g * 256;
    t.m_len = min(256, a.M - t.m0);
    t.adapter = 0;
  }
  int sg = 0;
  if (p.paired) {
    t.seg = 0;
    t.n0 = nt * 256;
  } else {
    while (sg + 1 < p.n_seg && nt >= p.seg_nt_end[sg]) ++sg;
    t.seg = sg;
    t.n0 = (nt - (sg ? p.seg_nt_end[sg - 1] : 0)) * PairCfg<NB>::kBN;
  }
  t.n_main = p.seg_kb_end[p.k_seg - 1];
  if (a.has_lora) {
    t.rank = a.ranks[t.adapter];
    t.nlps = min((t.rank + 63) / 64, a.nb);
    t.n_lora = t.nlps * (p.paired ? 2 : p.k_seg);
  } else {
    t.rank = 0;
    t.nlps = 0;
    t.n_lora = 0;
  }
  return t;
}

__device__ __forceinline__ uint32_t peer_masked(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }

// Pair-kernel epilogue: one 32 x 32 bf16 chunk out of registers -- staged through the
// warp's two 2 KB smem buffers (64-byte swizzle) into a TMA store / reduce-add for full
// 32-row warps, masked direct stores otherwise.
struct PairOut {
  const CUtensorMap* tm;
  __nv_bfloat16* out;
  int64_t ldo;
  int N;
  int accumulate;
  const __nv_bfloat16* bias;   // optional per-column bias (q/k/v of Qwen2), added to the bf16 result
};

// Word q (columns col0 + 2q, +1) of a bf16-packed chunk, plus the optional bias with the
// rounding of adding a bf16 bias to the bf16 output: round(float(y) + float(b)).
__device__ __forceinline__ uint32_t chunk_word(const PairOut& po, int col0, const uint32_t (&v)[16], int q) {
  if (po.bias == nullptr) return v[q];
  const int c = col0 + 2 * q;
  const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[q]));
  const float b0 = c < po.N ? __bfloat162float(po.bias[c]) : 0.f;
  const float b1 = c + 1 < po.N ? __bfloat162float(po.bias[c + 1]) : 0.f;
  return pack_bf16x2(y.x + b0, y.y + b1);
}

template <int NBUF = 2>
__device__ __forceinline__ void pair_emit_chunk(const PairOut& po, uint8_t* stg, int& issued, int lane, int col0,
                                                int m0, int m_len, const uint32_t (&v)[16]) {
  if (col0 >= po.N) return;
  if (m_len == 32) {
    uint8_t* buf = stg + (issued % NBUF) * 2048;
    if (issued >= NBUF) {
      if (lane == 0) bulk_wait_read<NBUF - 1>();   // the store that last used this buffer has read it
      __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(buf + lane * 64 + 16 * (q ^ ((lane >> 1) & 3))) =
          make_uint4(chunk_word(po, col0, v, 4 * q), chunk_word(po, col0, v, 4 * q + 1),
                     chunk_word(po, col0, v, 4 * q + 2), chunk_word(po, col0, v, 4 * q + 3));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (po.accumulate) tma_reduce_add_2d(po.tm, buf, col0, m0);
#if PLORA_STORE_EVICT_FIRST
      else               tma_store_2d_hint(po.tm, buf, col0, m0, l2_policy_evict_first());
#else
      else               tma_store_2d(po.tm, buf, col0, m0);
#endif
      bulk_commit();
    }
    ++issued;
  } else if (lane < m_len) {
    __nv_bfloat16* o = po.out + static_cast<int64_t>(m0 + lane) * po.ldo;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int cc = col0 + 2 * q;
      if (cc < po.N) {
        const uint32_t w = chunk_word(po, col0, v, q);
        float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
        if (po.accumulate) {
          const float2 old = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + cc));
          f.x += old.x;
          f.y += old.y;
        }
        *reinterpret_cast<__nv_bfloat162*>(o + cc) = __floats2bfloat162_rn(f.x, f.y);
      }
    }
  }
}

// EPI_SWIGLU: one gate chunk and the matching up chunk (bf16-packed) -> stores g, u and
// act = silu(g) u from the bf16-rounded values (the arithmetic of swiglu_fwd_kernel).
template <int NBUF>
__device__ __forceinline__ void pair_emit_swiglu(const PairOut& pg, const PairOut& pu, const PairOut& pa, uint8_t* stg,
                                                 int& issued, int lane, int col0, int m0, int m_len,
                                                 const uint32_t (&vg)[16], const uint32_t (&vu)[16]) {
  uint32_t va[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vg[q]));
    const float2 u = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vu[q]));
    va[q] = pack_bf16x2(swiglu_act(g.x, u.x), swiglu_act(g.y, u.y));
  }
  pair_emit_chunk<NBUF>(pg, stg, issued, lane, col0, m0, m_len, vg);
  pair_emit_chunk<NBUF>(pu, stg, issued, lane, col0, m0, m_len, vu);
  pair_emit_chunk<NBUF>(pa, stg, issued, lane, col0, m0, m_len, va);
}

template <bool B_MN, int NB, int EPI>
__global__ void __cluster_dims__(2, 1, 1) PLORA_PAIR_BOUNDS
    plora_gemm_pair_kernel(const __grid_constant__ PairArgs p) {
  using Cfg = PairCfg<NB, EPI>;
  const GemmArgs& args = p.g;
  constexpr int S = Cfg::kStages;
  constexpr int AS = Cfg::kAccStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  const int total = args.n_groups * args.n_ntiles;

  const int nseg = p.n_seg > p.k_seg ? p.n_seg : p.k_seg;
  if (warp == 0 && lane == 0) {
    for (int sg = 0; sg < nseg; ++sg) {
      if (sg == 0 || p.k_seg > 1) tma_prefetch(seg_map(&args.tmA, p.tmA2, sg));
      tma_prefetch(seg_map(&args.tmB, p.tmB2, sg));
      if (args.has_lora) {
        tma_prefetch(seg_map(&args.tmH, p.tmH2, sg));
        tma_prefetch(seg_map(&args.tmL, p.tmL2, sg));
      }
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);   // leader: one arrive.expect_tx per phase (both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);  // one multicast commit per phase
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * Cfg::kEpiWarps);  // epilogue warps of both CTAs (leader's copy)
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int half = static_cast<int>(rank) * 128;
      for (int idx = cluster; idx < total; idx += n_clusters) {
        const PairTile t = decode_pair_tile<NB>(p, idx);
        const int nblk = t.n_main + t.n_lora;
        for (int b = 0; b < nblk; ++b) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sA = smem + stage * Cfg::kStageBytes;
          uint8_t* sB = sA + Cfg::kABytes;
          const bool paired_lora = EPI == EPI_SWIGLU && b >= t.n_main;   // A + one B chunk
          if (leader) mbar_expect_tx(&full_bar[stage], paired_lora ? 2 * (Cfg::kABytes + 16384) : 2 * Cfg::kStageBytes);
          const uint32_t fb = peer_masked(&full_bar[stage]);
          if (b < t.n_main) {
            int ks = 0;   // K-segment of this K-block
            while (ks + 1 < p.k_seg && b >= p.seg_kb_end[ks]) ++ks;
            const int kc = (b - (ks ? p.seg_kb_end[ks - 1] : 0)) * kBK;
            const CUtensorMap* mA = seg_map(&args.tmA, p.tmA2, ks);
            tma_load_2d_pair(sA, mA, fb, kc, t.m0 + half);
#pragma unroll
            for (int c = 0; c < NB; ++c) {
              // paired: chunk c is segment c (gate / up) at the same columns
              const CUtensorMap* mB = seg_map(&args.tmB, p.tmB2, EPI == EPI_SWIGLU ? c : (p.k_seg > 1 ? ks : t.seg));
              const int n = (EPI == EPI_SWIGLU ? t.n0 : t.n0 + 256 * c) + half;
              if (B_MN) {
                tma_load_2d_pair(sB + c * 16384, mB, fb, n, kc);
                tma_load_2d_pair(sB + c * 16384 + 8192, mB, fb, n + 64, kc);
              } else {
                tma_load_2d_pair(sB + c * 16384, mB, fb, kc, n);
              }
            }
          } else {
            const int lb = b - t.n_main;
            const bool per_seg = p.k_seg > 1 || EPI == EPI_SWIGLU;
            const int ls = per_seg ? lb / t.nlps : t.seg;   // LoRA operands of this segment
            const int lbs = per_seg ? lb - ls * t.nlps : lb;
            tma_load_2d_pair(sA, seg_map(&args.tmH, p.tmH2, ls), fb, lbs * 64, t.m0 + half);
            if (EPI == EPI_SWIGLU) {   // only chunk ls (gate or up) takes this LoRA block
              tma_load_3d_pair(sB + ls * 16384, seg_map(&args.tmL, p.tmL2, ls), fb, lbs * 64, t.n0 + half, t.adapter);
            } else {
#pragma unroll
              for (int c = 0; c < NB; ++c)
                tma_load_3d_pair(sB + c * 16384, seg_map(&args.tmL, p.tmL2, ls), fb, lbs * 64, t.n0 + 256 * c + half,
                                 t.adapter);
            }
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ UMMA issuer (leader only)
    if (leader) {
      constexpr uint32_t idesc_main = idesc_bf16(256, 256, false, B_MN);
      constexpr uint32_t idesc_lora = idesc_bf16(256, 256, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int idx = cluster; idx < total; idx += n_clusters) {
        const PairTile t = decode_pair_tile<NB>(p, idx);
        const int nblk = t.n_main + t.n_lora;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * Cfg::kBN;
        for (int b = 0; b < nblk; ++b) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            uint8_t* sA = smem + stage * Cfg::kStageBytes;
            uint8_t* sB = sA + Cfg::kABytes;
            const uint32_t a0 = smem_u32(sA);
            const uint32_t b0 = smem_u32(sB);
            const bool lora = b >= t.n_main;
            const bool per_seg = p.k_seg > 1 || EPI == EPI_SWIGLU;
            const int lbs = lora ? (per_seg ? (b - t.n_main) % t.nlps : b - t.n_main) : 0;
            const int lchunk = (EPI == EPI_SWIGLU && lora) ? (b - t.n_main) / t.nlps : -1;
            const int ksteps = lora ? min(4, (t.rank - lbs * 64 + 15) / 16) : 4;
            for (int ks = 0; ks < ksteps; ++ks) {
              const uint64_t ad = smem_desc_sw128(a0 + ks * 32, 16, 1024);
#pragma unroll
              for (int c = 0; c < NB; ++c) {
                if (lchunk >= 0 && c != lchunk) continue;
                uint64_t bd;
                if (!lora && B_MN) bd = smem_desc_sw128(b0 + c * 16384 + ks * 2048, 8192, 1024);
                else               bd = smem_desc_sw128(b0 + c * 16384 + ks * 32, 16, 1024);
                umma_bf16_pair(d_tmem + 256 * c, ad, bd, lora ? idesc_lora : idesc_main,
                               (b > 0 || ks > 0) ? 1u : 0u);
              }
            }
            umma_commit_pair_mc(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit_pair_mc(&tfull_bar[acc], 0x3);
        __syncwarp();
        if (++acc == AS) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    // 8 warps: warp w drains TMEM lane quarter w%4, column half (w-2)/4, as 32-column
    // chunks.  The first kDirect chunks go TMEM -> registers -> bf16 -> per-warp smem
    // staging (two 2 KB buffers, 64-byte swizzle, bank-conflict free) -> TMA bulk tensor
    // store (or TMA reduce-add when accumulating into Y); the remaining chunks are parked
    // in registers (bf16-packed) so the accumulator is released after one TMEM pass and
    // the next tile's mainloop overlaps the rest of the stores.  Warps whose 32 rows are
    // only partly inside the tile (unaligned segments) use masked direct stores.
    const int ew = warp - 2;
    const int quarter = warp & 3;         // tcgen05.ld lane-quarter rule: warp w reads lanes 32*(w%4)..
    const int chalf = ew >> 2;
    constexpr int kChunks = Cfg::kBN / 32 / 2;   // chunks per warp
    // chunks stored before the accumulator is released: all of them when the accumulator is
    // double-buffered (NB = 1), otherwise park the rest in registers
    constexpr int kDirect = Cfg::kAccStages > 1 ? kChunks : PLORA_PAIR_KDIRECT;
    constexpr int kParked = kChunks - kDirect;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    uint8_t* stg = smem + S * Cfg::kStageBytes + 1024 + ew * (Cfg::kStgBufs * 2048);   // 1024-B aligned
    int acc = 0;
    uint32_t acc_phase = 0;
    int issued = 0;
    if constexpr (EPI == EPI_SWIGLU) {
      // paired gate/up tile: warp (quarter, chalf) owns gate chunks chalf*4+i (TMEM cols
      // 0..255) and the matching up chunks 8+chalf*4+i; per pair it stores g, u and act.
      constexpr int kPairs = 4, kDirectPairs = PLORA_SWIGLU_DIRECT;
      for (int idx = cluster; idx < total; idx += n_clusters) {
        const PairTile t = decode_pair_tile<NB>(p, idx);
        const int m0 = t.m0 + static_cast<int>(rank) * 128 + quarter * 32;
        const int m_len = min(32, t.m_len - static_cast<int>(rank) * 128 - quarter * 32);
        PLORA_EPI_WAIT(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t tb = tmem_base + acc * Cfg::kBN + (static_cast<uint32_t>(quarter * 32) << 16);
        const bool store = m_len > 0;
        PairOut pg, pu, pa;
        pg.tm = &args.tmY;
        pu.tm = &p.tmY2[0];
        pa.tm = &p.tmY2[1];
        pg.out = static_cast<__nv_bfloat16*>(p.seg_out[0]);
        pu.out = static_cast<__nv_bfloat16*>(p.seg_out[1]);
        pa.out = static_cast<__nv_bfloat16*>(p.seg_out[2]);
        pg.ldo = pu.ldo = pa.ldo = p.seg_ldo[0];
        pg.N = pu.N = pa.N = p.seg_N[0];
        pg.accumulate = pu.accumulate = pa.accumulate = 0;
        pg.bias = pu.bias = pa.bias = nullptr;
        uint32_t kg[kPairs - kDirectPairs][16], ku[kPairs - kDirectPairs][16];
#pragma unroll
        for (int i = 0; i < kPairs; ++i) {
          uint32_t r[32], vg[16], vu[16];
          tmem_ld_32x32b_x32(tb + (chalf * 4 + i) * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) vg[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
          tmem_ld_32x32b_x32(tb + (8 + chalf * 4 + i) * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) vu[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
          if (i < kDirectPairs) {
            if (store) pair_emit_swiglu<Cfg::kStgBufs>(pg, pu, pa, stg, issued, lane, t.n0 + (chalf * 4 + i) * 32, m0, m_len, vg, vu);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              kg[i - kDirectPairs][q] = vg[q];
              ku[i - kDirectPairs][q] = vu[q];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);   // accumulator free: next mainloop
        if (++acc == AS) { acc = 0; acc_phase ^= 1; }
        if (!store) continue;
#pragma unroll
        for (int i = kDirectPairs; i < kPairs; ++i)
          pair_emit_swiglu<Cfg::kStgBufs>(pg, pu, pa, stg, issued, lane, t.n0 + (chalf * 4 + i) * 32, m0, m_len,
                           kg[i - kDirectPairs], ku[i - kDirectPairs]);
      }
    } else
    for (int idx = cluster; idx < total; idx += n_clusters) {
      const PairTile t = decode_pair_tile<NB>(p, idx);
      const int m0 = t.m0 + static_cast<int>(rank) * 128 + quarter * 32;   // this warp's 32 rows
      const int m_len = min(32, t.m_len - static_cast<int>(rank) * 128 - quarter * 32);
      PLORA_EPI_WAIT(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * Cfg::kBN + (static_cast<uint32_t>(quarter * 32) << 16);
      const int c0 = chalf * kChunks;
      const bool store = m_len > 0;
      PairOut po;
      po.tm = seg_map(&args.tmY, p.tmY2, t.seg);
      po.out = static_cast<__nv_bfloat16*>(p.seg_out[t.seg]);
      po.ldo = p.seg_ldo[t.seg];
      po.N = p.seg_N[t.seg];
      po.accumulate = args.accumulate;
      po.bias = static_cast<const __nv_bfloat16*>(p.seg_bias[t.seg]);
      uint32_t pk[kParked > 0 ? kParked : 1][16];
      {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tb + c0 * 32, r);
#pragma unroll
        for (int j = 0; j < kChunks; ++j) {
          tmem_ld_wait();
          if (j < kDirect) {
            uint32_t v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            if (j + 1 < kChunks) tmem_ld_32x32b_x32(tb + (c0 + j + 1) * 32, r);   // overlaps the store below
            if (store) pair_emit_chunk<Cfg::kStgBufs>(po, stg, issued, lane, t.n0 + (c0 + j) * 32, m0, m_len, v);
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              pk[j - kDirect][q] = pack_bf16x2(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            if (j + 1 < kChunks) tmem_ld_32x32b_x32(tb + (c0 + j + 1) * 32, r);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);   // accumulator free: next mainloop
      if (++acc == AS) { acc = 0; acc_phase ^= 1; }
      if (!store) continue;
#pragma unroll
      for (int j = kDirect; j < kChunks; ++j)
        pair_emit_chunk<Cfg::kStgBufs>(po, stg, issued, lane, t.n0 + (c0 + j) * 32, m0, m_len, pk[j - kDirect]);
    }
    if (lane == 0) bulk_wait<0>();   // all TMA stores complete before the CTA retires
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
  }
}

}  // namespace plora
