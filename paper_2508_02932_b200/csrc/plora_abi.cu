// plora_abi.cu -- extern "C" entry points of libplora (declared in include/plora.h).
//
// Host responsibilities: validate arguments, encode TMA tensor maps for the
// caller-owned device buffers, pick the tile shape and launch the sm_100a
// kernels on the caller's stream.  No device allocation happens here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <queue>
#include <atomic>
#include <unordered_map>
#include <vector>
#include <string>

#include "../../include/plora.h"
#include "gemm_sm100.cuh"
#include "dual_sm100.cuh"
#include "swiglu_sm100.cuh"

namespace plora {

static thread_local std::string g_last_error;

static int fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
static int fail(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return 1;
}

int set_error(const std::string& msg) {
  g_last_error = msg;
  return 1;
}

#define PLORA_CUDA(expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) return fail("%s: %s", #expr, cudaGetErrorString(_e));      \
  } while (0)

// ------------------------------------------------------------------ driver entry
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2D bf16 tensor [outer][inner] with row pitch `pitch_elems`, 128B-swizzled boxes.
#ifndef PLORA_LOAD_L2_PROMOTION
#define PLORA_LOAD_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B   // operand loads (build-time knob)
#endif

// Tensor-map cache: a CUtensorMap is a pure function of (kind, base, extents, pitch, box),
// and the caching allocators behind the callers hand the same buffers back step after
// step, so each map is encoded once per process (per-launch host work matters when
// tokens per GPU shrink under the planner split).  Bounded; thread-safe.
struct MapKey {
  uint64_t v[7];
  bool operator==(const MapKey& o) const { return memcmp(v, o.v, sizeof(v)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t x : k.v) h = (h ^ x) * 1099511628211ull;
    return static_cast<size_t>(h);
  }
};
static std::mutex g_map_mu;
static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

template <typename F>
static int cached_map(CUtensorMap* m, const MapKey& key, F&& encode) {
  {
    std::lock_guard<std::mutex> lock(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *m = it->second;
      return 0;
    }
  }
  int rc = encode(m);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(g_map_mu);
  if (g_maps.size() >= 8192) g_maps.clear();
  g_maps.emplace(key, *m);
  return 0;
}

static int make_map_2d_enc(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer);

static int make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer) {
  const MapKey key{{1, reinterpret_cast<uint64_t>(base), inner, outer, pitch_elems, box_inner,
                    static_cast<uint64_t>(box_outer)}};
  return cached_map(m, key, [&](CUtensorMap* mm) {
    return make_map_2d_enc(mm, base, inner, outer, pitch_elems, box_inner, box_outer);
  });
}

static int make_map_2d_enc(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                           uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (reinterpret_cast<uintptr_t>(base) % 16) return fail("tensor base not 16-byte aligned");
  if ((pitch_elems * 2) % 16) return fail("row pitch %llu elems not a multiple of 16 bytes",
                                          (unsigned long long)pitch_elems);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   PLORA_LOAD_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail("cuTensorMapEncodeTiled(2d inner=%llu outer=%llu box=%u,%u) failed: %d",
                (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer, (int)r);
  return 0;
}

// 2D bf16 output tensor for the TMA-store epilogue: 32x32 boxes, 64-byte swizzle.
static int make_map_out_enc(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems);

static int make_map_out(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems) {
  const MapKey key{{2, reinterpret_cast<uint64_t>(base), cols, rows, pitch_elems, 32, 32}};
  return cached_map(m, key, [&](CUtensorMap* mm) { return make_map_out_enc(mm, base, cols, rows, pitch_elems); });
}

static int make_map_out_enc(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (reinterpret_cast<uintptr_t>(base) % 16 || (pitch_elems * 2) % 16)
    return fail("output base/pitch not 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled(out) failed: %d", (int)r);
  return 0;
}

// 3D bf16 tensor [n][mid][inner] (dense), box {box_inner, box_mid, 1}.
static int make_map_3d_enc(CUtensorMap* m, const void* base, uint64_t inner, uint64_t mid, uint64_t n,
                           uint32_t box_inner, uint32_t box_mid);

static int make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t mid, uint64_t n,
                       uint32_t box_inner, uint32_t box_mid) {
  const MapKey key{{3, reinterpret_cast<uint64_t>(base), inner, mid, n, box_inner, box_mid}};
  return cached_map(m, key, [&](CUtensorMap* mm) { return make_map_3d_enc(mm, base, inner, mid, n, box_inner, box_mid); });
}

static int make_map_3d_enc(CUtensorMap* m, const void* base, uint64_t inner, uint64_t mid, uint64_t n,
                           uint32_t box_inner, uint32_t box_mid) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail("cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  if (reinterpret_cast<uintptr_t>(base) % 16) return fail("tensor base not 16-byte aligned");
  cuuint64_t dims[3] = {inner, mid, n};
  cuuint64_t strides[2] = {inner * 2, inner * mid * 2};
  cuuint32_t box[3] = {box_inner, box_mid, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   PLORA_LOAD_L2_PROMOTION, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled(3d) failed: %d", (int)r);
  return 0;
}

// Opt a kernel into its dynamic shared memory size on the current device (the attribute
// is per device; the per-instantiation bit mask makes it once per device and thread-safe).
template <typename K>
static int ensure_smem(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  PLORA_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    PLORA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.fetch_or(bit, std::memory_order_release);
  }
  return 0;
}

static int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

template <int BN, int MODE, bool B_MN, bool SK>
static int launch_as(const GemmArgs& args, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = plora_gemm_kernel<BN, MODE, B_MN, SK>;
  static std::atomic<uint64_t> configured{0};   // per instantiation, bit per device
  if (ensure_smem(kern, Cfg::kSmemBytes, configured)) return 1;
  const int total = args.n_groups * args.n_ntiles;
  if (total <= 0) return 0;
  const int grid = SK ? args.sk : (total < num_sms() ? total : num_sms());
  PLORA_CUDA(launch_pdl(kern, dim3(grid), dim3(kThreads), Cfg::kSmemBytes, stream, args));
  PLORA_CUDA(cudaGetLastError());
  return 0;
}

// The stream-K instantiation exists for the skinny LoRA modes only (setup_sk sets args.sk).
template <int BN, int MODE, bool B_MN>
static int launch(const GemmArgs& args, cudaStream_t stream) {
  if constexpr (MODE != MODE_GEMM) {
    if (args.sk) return launch_as<BN, MODE, B_MN, true>(args, stream);
  }
  return launch_as<BN, MODE, B_MN, false>(args, stream);
}

static int pick_bn(int64_t N) { return N >= 256 ? 256 : (N > 64 ? 128 : 64); }

// Tile-shape policy of the base GEMMs.  Build-time constants (-D overrides for
// experiments, tools/build_variant.sh); the values are the measured optima of round 1
// (DESIGN.md section 6).
#ifndef PLORA_PAIR_NB1_MAXK
#define PLORA_PAIR_NB1_MAXK 1024   // K at or below which 256x256 double-buffered pair tiles are used
#endif
#ifndef PLORA_PAIR512_MIN_N
#define PLORA_PAIR512_MIN_N 2048   // N at which the 256x512 pair tile is used
#endif
#ifndef PLORA_PAIR_BAND
#define PLORA_PAIR_BAND (-8)       // pair-GEMM raster: N-bands of 8 column tiles
#endif
#ifndef PLORA_GROUP_MIN_N
#define PLORA_GROUP_MIN_N 64       // narrowest segment of a grouped (multi-target) pair launch
#endif

template <bool B_MN, int NB, int EPI = EPI_STORE>
static int launch_pair(const PairArgs& args, cudaStream_t stream) {
  auto kern = plora_gemm_pair_kernel<B_MN, NB, EPI>;
  static std::atomic<uint64_t> configured{0};   // per instantiation, bit per device
  if (ensure_smem(kern, PairCfg<NB, EPI>::kSmemBytes, configured)) return 1;
  const int total = args.g.n_groups * args.g.n_ntiles;
  if (total <= 0) return 0;
  const int max_clusters = num_sms() / 2;
  const int clusters = total < max_clusters ? total : max_clusters;
  PLORA_CUDA(launch_pdl(kern, dim3(clusters * 2), dim3(PairCfg<NB, EPI>::kThreads), PairCfg<NB, EPI>::kSmemBytes,
                        stream, args));
  PLORA_CUDA(cudaGetLastError());
  return 0;
}

// 256x256 tiles at K <= 1024: C4 TP shards (o: K = 640, q/k/v dX: K = 896), ~1% per layer.
static constexpr int g_pair_nb1_max_k = PLORA_PAIR_NB1_MAXK;
static constexpr int g_pair_nb_min_n = PLORA_PAIR512_MIN_N;
// Tile raster of the pair GEMM: N-bands of 8 column tiles (4096 output columns at
// NB = 2), row groups stepping inside a band, so every A row block is consumed by 8
// concurrently running clusters.  Measured on the C3 step (same box, alternating runs):
// DRAM reads per GEMM -27%, SM clock under the power cap +45 MHz, +2.6% tokens/s vs
// 8-row-group M-bands (the previous raster, PLORA_PAIR_BAND >= 0).
static constexpr int g_pair_band = PLORA_PAIR_BAND;
#ifndef PLORA_SWIGLU_BAND
#define PLORA_SWIGLU_BAND PLORA_PAIR_BAND   // raster of the gate/up + SwiGLU launch (experiment knob)
#endif

// One segment of a (segmented) pair GEMM; see PairArgs in gemm_sm100.cuh.
struct PairSeg {
  const void* A;   // [M][K] (K-segments: per segment; N-segments: segment 0's is shared)
  int64_t K;
  const void* W;   // w_kmajor ? [N][K] : [K][N]
  int64_t N;
  const void* H;   // LoRA A operand [M][64nb] (may be NULL: no LoRA)
  const void* L;   // LoRA B operand [n][N][64nb]
  void* Y;         // [M][ldy] (K-segments: segment 0's is the shared output)
  int64_t ldy;
  const void* bias = nullptr;   // optional bf16 [N] added to the bf16 result (N-segments)
};

// CTA-pair GEMM over 1..3 N-segments (shared A) or K-segments (shared output).
static int run_pair_segments(cudaStream_t st, const plora_pack_t* pack, int64_t M, int n_seg, int k_seg,
                             const PairSeg* sg, int w_kmajor, const void* residual, void* swiglu_act = nullptr) {
  if (n_seg < 1 || k_seg < 1 || n_seg > 3 || k_seg > 3 || (n_seg > 1 && k_seg > 1))
    return fail("pair gemm: 1..3 N-segments or 1..3 K-segments");
  const int nseg = n_seg > k_seg ? n_seg : k_seg;
  int64_t Nmin = sg[0].N;
  for (int s = 1; s < n_seg; ++s) Nmin = sg[s].N < Nmin ? sg[s].N : Nmin;
  int64_t Ntot = 0;
  for (int s = 0; s < n_seg; ++s) Ntot += sg[s].N;
  const bool paired = swiglu_act != nullptr;   // gate/up + SwiGLU (EPI_SWIGLU): segments 0, 1 share columns
  if (paired && (n_seg != 2 || sg[0].N != sg[1].N || !w_kmajor || residual))
    return fail("gate/up SwiGLU GEMM: two equal-width nn.Linear-layout segments");
  int64_t Ktot = 0;
  for (int s = 0; s < (k_seg > 1 ? k_seg : 1); ++s) Ktot += sg[s].K;
  // 256 x 512 tiles (single accumulator) unless the output is narrow or the K loop is so
  // short that the epilogue bubble outweighs the operand-traffic saving (then 256 x 256
  // tiles with a double-buffered accumulator)
  const int NB = paired ? 2 : (((n_seg > 1 ? Ntot : Nmin) >= g_pair_nb_min_n && Ktot > g_pair_nb1_max_k) ? 2 : 1);
  const int tile_n = 256 * NB;
  PairArgs pa;
  memset(&pa, 0, sizeof(pa));
  GemmArgs& a = pa.g;
  CUtensorMap* mA[3] = {&a.tmA, &pa.tmA2[0], &pa.tmA2[1]};
  CUtensorMap* mB[3] = {&a.tmB, &pa.tmB2[0], &pa.tmB2[1]};
  CUtensorMap* mH[3] = {&a.tmH, &pa.tmH2[0], &pa.tmH2[1]};
  CUtensorMap* mL[3] = {&a.tmL, &pa.tmL2[0], &pa.tmL2[1]};
  CUtensorMap* mY[3] = {&a.tmY, &pa.tmY2[0], &pa.tmY2[1]};
  const bool lora = pack != nullptr && sg[0].H != nullptr && sg[0].L != nullptr;
  const int64_t R64 = pack ? 64LL * pack->nb : 64;
  int rc;
  int nt = 0, kb = 0;
  for (int s = 0; s < nseg; ++s) {
    const PairSeg& g = sg[s];
    const int64_t K = (k_seg > 1) ? g.K : sg[0].K;
    const int64_t N = (n_seg > 1) ? g.N : sg[0].N;
    if (K <= 0 || K % 8 || N % 8) return fail("pair gemm: K and N must be positive multiples of 8");
    if (s == 0 || k_seg > 1)
      if ((rc = make_map_2d(mA[s], g.A, K, M, K, 64, kBM))) return rc;
    if (w_kmajor) rc = make_map_2d(mB[s], g.W, K, N, K, 64, 128);
    else          rc = make_map_2d(mB[s], g.W, N, K, N, 64, 64);
    if (rc) return rc;
    if (lora) {
      if (!g.H || !g.L) return fail("pair gemm: every segment needs its LoRA operands");
      if ((rc = make_map_2d(mH[s], g.H, R64, M, R64, 64, kBM))) return rc;
      if ((rc = make_map_3d(mL[s], g.L, R64, N, pack->n_adapters, 64, 128))) return rc;
    }
    if (s == 0 || n_seg > 1) {
      if (!g.Y || g.ldy % 8 || reinterpret_cast<uintptr_t>(g.Y) % 16)
        return fail("pair gemm: output must be 16-byte aligned with ldy a multiple of 8");
      if ((rc = make_map_out(mY[s], g.Y, N, M, g.ldy))) return rc;
      pa.seg_out[s] = g.Y;
      pa.seg_ldo[s] = g.ldy;
      pa.seg_bias[s] = g.bias;
      pa.seg_N[s] = static_cast<int>(N);
      if (!paired || s == 0) nt += static_cast<int>((N + (paired ? 256 : tile_n) - 1) / (paired ? 256 : tile_n));
      pa.seg_nt_end[s] = nt;
    }
    if (s == 0 || k_seg > 1) {
      kb += static_cast<int>((K + kBK - 1) / kBK);
      pa.seg_kb_end[s] = kb;
    }
  }
  pa.n_seg = n_seg;
  pa.k_seg = k_seg;
  if (paired) {   // act output: segment 2's output slot
    if (reinterpret_cast<uintptr_t>(swiglu_act) % 16) return fail("gate/up SwiGLU GEMM: act must be 16-byte aligned");
    if ((rc = make_map_out(mY[2], swiglu_act, sg[0].N, M, sg[0].ldy))) return rc;
    pa.seg_out[2] = swiglu_act;
    pa.seg_ldo[2] = sg[0].ldy;
    pa.seg_N[2] = static_cast<int>(sg[0].N);
    pa.paired = 1;
  }
  if (lora) {
    a.ranks = pack->d_ranks;
    a.nb = pack->nb;
    a.has_lora = 1;
  }
  a.mtiles = pack ? pack->d_ptiles : nullptr;
  a.n_groups = pack ? pack->n_ptiles : static_cast<int>((M + 255) / 256);
  a.M = static_cast<int>(M);
  a.n_ntiles = nt;
  // Y = result + residual is computed as Y <- residual (skipped when in place), then a
  // TMA reduce-add of the result (bf16 add in L2).
  if (residual) {
    if (n_seg > 1) return fail("pair gemm: residual needs a single output");
    if (residual != sg[0].Y)
      PLORA_CUDA(cudaMemcpy2DAsync(sg[0].Y, sg[0].ldy * 2, residual, sg[0].ldy * 2, sg[0].N * 2, M,
                                   cudaMemcpyDeviceToDevice, st));
    a.accumulate = 1;
  }
  pa.band = paired ? PLORA_SWIGLU_BAND : g_pair_band;
  if (paired) return launch_pair<false, 2, EPI_SWIGLU>(pa, st);
  if (NB == 2) return w_kmajor ? launch_pair<false, 2>(pa, st) : launch_pair<true, 2>(pa, st);
  return w_kmajor ? launch_pair<false, 1>(pa, st) : launch_pair<true, 1>(pa, st);
}

// CTA-pair GEMM (N >= 256), one problem.
static int run_gemm_pair(cudaStream_t st, const plora_pack_t* pack, int64_t M, int64_t N, int64_t K,
                         const void* A, const void* W, int w_kmajor, const void* H, const void* L,
                         void* Y, int64_t ldy, const void* residual, const void* bias = nullptr) {
  PairSeg sg{A, K, W, N, H, L, Y, ldy, bias};
  return run_pair_segments(st, pack, M, 1, 1, &sg, w_kmajor, residual);
}

// Base GEMM (+ fused LoRA expand).  A: [M][K] K-major.  W: see w_kmajor.
static int run_gemm(cudaStream_t st, const plora_pack_t* pack, int64_t M, int64_t N, int64_t K,
                    const void* A, const void* W, int w_kmajor, const void* H, const void* L,
                    void* Y, int64_t ldy, const void* residual, const void* bias = nullptr) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) return fail("gemm: K must be positive");
  if (K % 8 || N % 8 || ldy % 8) return fail("gemm: K, N and ldy must be multiples of 8");
  if (reinterpret_cast<uintptr_t>(Y) % 16 || (residual && reinterpret_cast<uintptr_t>(residual) % 16))
    return fail("gemm: output/residual must be 16-byte aligned");
  if (N >= 256 && (pack == nullptr || pack->d_ptiles != nullptr || pack->n_ptiles == 0))
    return run_gemm_pair(st, pack, M, N, K, A, W, w_kmajor, H, L, Y, ldy, residual, bias);
  const int BN = pick_bn(N);
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc = make_map_2d(&a.tmA, A, K, M, K, 64, kBM);
  if (rc) return rc;
  if (w_kmajor) rc = make_map_2d(&a.tmB, W, K, N, K, 64, BN);
  else          rc = make_map_2d(&a.tmB, W, N, K, N, 64, 64);
  if (rc) return rc;
  const bool lora = pack != nullptr && H != nullptr && L != nullptr;
  if (lora) {
    const int64_t R64 = 64LL * pack->nb;
    if ((rc = make_map_2d(&a.tmH, H, R64, M, R64, 64, kBM))) return rc;
    if ((rc = make_map_3d(&a.tmL, L, R64, N, pack->n_adapters, 64, BN))) return rc;
    a.ranks = pack->d_ranks;
    a.nb = pack->nb;
    a.has_lora = 1;
  }
  a.mtiles = pack ? pack->d_mtiles : nullptr;
  a.n_groups = pack ? pack->n_mtiles : static_cast<int>((M + kBM - 1) / kBM);
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(N);
  a.K = static_cast<int>(K);
  a.n_ntiles = static_cast<int>((N + BN - 1) / BN);
  a.out = Y;
  a.ldo = ldy;
  a.residual = static_cast<const __nv_bfloat16*>(residual);
  a.bias = static_cast<const __nv_bfloat16*>(bias);
  if (BN == 256) return w_kmajor ? launch<256, MODE_GEMM, false>(a, st) : launch<256, MODE_GEMM, true>(a, st);
  if (BN == 128) return w_kmajor ? launch<128, MODE_GEMM, false>(a, st) : launch<128, MODE_GEMM, true>(a, st);
  return w_kmajor ? launch<64, MODE_GEMM, false>(a, st) : launch<64, MODE_GEMM, true>(a, st);
}

// Stream-K partition of a shrink / segment reduction (SkIter in gemm_sm100.cuh) when the
// pack carries a workspace: W = total k-blocks (0 = unknown on the host), BN = the
// launch's accumulator width.  G = min(#SMs, W) CTAs, each with two partial slots.
static int64_t sk_need_bytes(int G, int BN) { return 1024 + 2LL * G * kBM * BN * 4; }

// At least kSkMinKb k-blocks per CTA: below that the fixed per-CTA cost (prologue,
// pipeline fill, partial write-back) outweighs the extra SMs.
static constexpr int64_t kSkMinKb = 8;

#ifndef PLORA_SK_MAX_WAVES
#define PLORA_SK_MAX_WAVES 1   // stream-K below this many whole-tile waves (build-time knob)
#endif

static bool setup_sk(GemmArgs& a, const plora_pack_t* pack, int BN, int64_t W) {
  // Whole tiles when they fill every SM at least once: at C3 (T = 32768, 1.7 waves) the
  // stream-K split times the same in isolation and lost 1.3% of the step in a same-box
  // A/B (profiles/r2_streamk_gate_ab.log); below one wave (planner-split ranks, T <= 16384)
  // it is 1.4-2.4x faster (profiles/r2_split_kernels_streamk.log).
  if (pack->d_ws == nullptr ||
      a.n_groups * static_cast<int64_t>(a.n_ntiles) >= static_cast<int64_t>(PLORA_SK_MAX_WAVES) * num_sms())
    return false;
  int G = num_sms();
  if (W > 0 && W / kSkMinKb < G) G = static_cast<int>(W / kSkMinKb > 0 ? W / kSkMinKb : 1);
  if (G > 256 || pack->ws_bytes < sk_need_bytes(G, BN)) return false;
  a.sk = G;
  a.sk_cnt = static_cast<int32_t*>(pack->d_ws);
  a.sk_part = reinterpret_cast<float*>(static_cast<char*>(pack->d_ws) + 1024);
  return true;
}

// SEGRED stream-K work: per * sum_a max(1, ceil(T_a / 64)) k-blocks (0 without host offsets).
static int64_t segred_work(const plora_pack_t* pack, int per) {
  if (pack->h_row_off == nullptr) return 0;
  int64_t W = 0;
  for (int i = 0; i < pack->n_adapters; ++i) {
    const int64_t t = pack->h_row_off[i + 1] - pack->h_row_off[i];
    W += per * (t > 0 ? (t + kBK - 1) / kBK : 1);
  }
  return W;
}

// Shrink: out[T][64nb] = alpha_i * P[T][K] * L_i[K][64nb]  (L stored [n][K][64nb]).
static int run_shrink(cudaStream_t st, const plora_pack_t* pack, int64_t K, const void* P,
                      const void* L, void* out) {
  const int64_t T = pack->total_tokens;
  if (T <= 0 || pack->n_mtiles == 0) return 0;
  if (K % 8) return fail("shrink: K must be a multiple of 8");
  const int64_t R64 = 64LL * pack->nb;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_map_2d(&a.tmA, P, K, T, K, 64, kBM))) return rc;
  if ((rc = make_map_3d(&a.tmB, L, R64, K, pack->n_adapters, 64, 64))) return rc;
  a.mtiles = pack->d_mtiles;
  a.alpha = pack->d_alpha;
  a.n_groups = pack->n_mtiles;
  a.n_ntiles = pack->nb;
  a.M = static_cast<int>(T);
  a.N = static_cast<int>(R64);
  a.K = static_cast<int>(K);
  a.out = out;
  a.ldo = R64;
  setup_sk(a, pack, 64, static_cast<int64_t>(a.n_groups) * a.n_ntiles * ((K + kBK - 1) / kBK));
  return launch<64, MODE_SHRINK, true>(a, st);
}

// LPT schedule for the segment reductions: tile (adapter a, m-tile, n-tile) costs
// ceil(T_a / 64) K-blocks + a fixed epilogue/fill overhead; tiles are taken in
// decreasing cost and each goes to the least-loaded CTA (list scheduling in LPT order,
// within 4/3 of optimal).  Schedules are cached per (row offsets, tile grid, SM count).
static bool segred_schedule(const plora_pack_t* pack, int mt_per, int n_ntiles, SegSched* dst) {
  const int n = pack->n_adapters;
  const int per = mt_per * n_ntiles;
  const int64_t total = static_cast<int64_t>(n) * per;
  const int sms = num_sms();
  if (total <= 0 || total > kSchedMaxTiles || sms > kSchedMaxCtas) return false;
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i <= n; ++i) h = (h ^ static_cast<uint64_t>(pack->h_row_off[i])) * 1099511628211ull;
  h = (h ^ static_cast<uint64_t>(n)) * 1099511628211ull;
  const uint64_t key = h ^ (static_cast<uint64_t>(mt_per) << 40) ^ (static_cast<uint64_t>(n_ntiles) << 52) ^
                       static_cast<uint64_t>(sms);
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::unique_ptr<SegSched>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    memcpy(dst, it->second.get(), sizeof(SegSched));   // copied under the lock: entries may be evicted
    return true;
  }
  const int ctas = static_cast<int>(total < sms ? total : sms);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  auto cost = [&](int a) { return (pack->h_row_off[a + 1] - pack->h_row_off[a] + 63) / 64 + 3; };
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost(x) > cost(y); });
  std::vector<std::vector<uint16_t>> lists(ctas);
  using Slot = std::pair<int64_t, int>;   // (load, cta)
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int c = 0; c < ctas; ++c) heap.push({0, c});
  for (int a : order) {
    const int64_t w = cost(a);
    for (int t = 0; t < per; ++t) {
      Slot s = heap.top();
      heap.pop();
      lists[s.second].push_back(static_cast<uint16_t>(a * per + t));
      heap.push({s.first + w, s.second});
    }
  }
  auto sched = std::make_unique<SegSched>();
  memset(sched.get(), 0, sizeof(SegSched));
  sched->n_ctas = ctas;
  int pos = 0;
  for (int c = 0; c < ctas; ++c) {
    sched->off[c] = static_cast<uint16_t>(pos);
    for (uint16_t t : lists[c]) sched->tiles[pos++] = t;
  }
  sched->off[ctas] = static_cast<uint16_t>(pos);
  memcpy(dst, sched.get(), sizeof(SegSched));
  if (cache.size() >= 256) cache.clear();
  cache.emplace(key, std::move(sched));
  return true;
}

template <int BN>
static int launch_segred_lpt(const GemmArgs& args, const SegSched& sched, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = plora_segred_lpt_kernel<BN>;
  static std::atomic<uint64_t> configured{0};   // per instantiation, bit per device
  if (ensure_smem(kern, Cfg::kSmemBytes, configured)) return 1;
  PLORA_CUDA(launch_pdl(kern, dim3(sched.n_ctas), dim3(kThreads), Cfg::kSmemBytes, stream, args, sched));
  PLORA_CUDA(cudaGetLastError());
  return 0;
}

// Segment reduction: G_i[Mdim][rpad16_i] = P_i^T Q_i over the tokens of segment i.
//   P: [T][Mdim] bf16, Q: [T][64nb] bf16, G: f32 adapter-major region.
static int run_segred(cudaStream_t st, const plora_pack_t* pack, int64_t Mdim, const void* P,
                      const void* Q, float* G) {
  const int64_t T = pack->total_tokens;
  if (Mdim % 8) return fail("segment reduction: Mdim must be a multiple of 8");
  const int64_t R64 = 64LL * pack->nb;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  // TMA needs a non-empty tensor; with T == 0 every tile is empty and only writes zeros.
  const int64_t Tm = T > 0 ? T : 1;
  if ((rc = make_map_2d(&a.tmA, P, Mdim, Tm, Mdim, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmB, Q, R64, Tm, R64, 64, 64))) return rc;
  a.row_off = pack->d_row_off;
  a.rpad_off = pack->d_rpad_off;
  a.mt_per = static_cast<int>((Mdim + kBM - 1) / kBM);
  a.n_groups = pack->n_adapters * a.mt_per;
  a.n_ntiles = pack->nb;
  a.M = static_cast<int>(Mdim);
  a.N = static_cast<int>(R64);
  a.out = G;
  // Stream-K only for a segment reduction too small to fill a quarter of the SMs with whole
  // tiles (one adapter at T = 4096: 32 tiles); otherwise the LPT schedule, whose CTAs read
  // the same token rows at the same time (each tile is a 256-byte column stripe of them) --
  // the stream-K pieces start at staggered rows and lose DRAM locality (same-box A/B at
  // C3: 47.1 vs 42.6 ms/step, tools/split_projection.py --whole-lora).
  const bool sk = static_cast<int64_t>(a.n_groups) * a.n_ntiles * 4 <= num_sms() &&
                  setup_sk(a, pack, 64, segred_work(pack, a.mt_per * a.n_ntiles));
  if (!sk && pack->h_row_off != nullptr) {
    SegSched sched;
    if (segred_schedule(pack, a.mt_per, a.n_ntiles, &sched)) return launch_segred_lpt<64>(a, sched, st);
  }
  return launch<64, MODE_SEGRED, true>(a, st);
}

// Multi-target shrink: out_j[T][64] = alpha_i * P[T][K] * L_j,i[K][64] for n_multi targets
// that share P (q/k/v or gate/up): P is read once.  Requires nb == 1 (ranks <= 64).
static int run_shrink_multi(cudaStream_t st, const plora_pack_t* pack, int64_t K, const void* P, int n_multi,
                            const void* const* L, void* const* out) {
  const int64_t T = pack->total_tokens;
  if (T <= 0 || pack->n_mtiles == 0) return 0;
  if (K % 8) return fail("shrink: K must be a multiple of 8");
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_map_2d(&a.tmA, P, K, T, K, 64, kBM))) return rc;
  CUtensorMap* maps[3] = {&a.tmB, &a.tmB2, &a.tmB3};
  for (int j = 0; j < n_multi; ++j)
    if ((rc = make_map_3d(maps[j], L[j], 64, K, pack->n_adapters, 64, 64))) return rc;
  a.mtiles = pack->d_mtiles;
  a.alpha = pack->d_alpha;
  a.n_groups = pack->n_mtiles;
  a.n_ntiles = 1;
  a.M = static_cast<int>(T);
  a.N = 64;
  a.K = static_cast<int>(K);
  a.out = out[0];
  a.out2 = n_multi > 1 ? out[1] : nullptr;
  a.out3 = n_multi > 2 ? out[2] : nullptr;
  a.ldo = 64;
  a.n_multi = n_multi;
  setup_sk(a, pack, 64 * n_multi, static_cast<int64_t>(a.n_groups) * ((K + kBK - 1) / kBK));
  return n_multi == 3 ? launch<192, MODE_SHRINK, true>(a, st) : launch<128, MODE_SHRINK, true>(a, st);
}

// Multi-target segment reduction: G_j,i[Mdim][rpad16_i] = P_i^T Q_j,i for n_multi targets
// sharing P (the layer input X of q/k/v or gate/up).  Requires nb == 1.
static int run_segred_multi(cudaStream_t st, const plora_pack_t* pack, int64_t Mdim, const void* P, int n_multi,
                            const void* const* Q, float* const* G) {
  const int64_t T = pack->total_tokens;
  if (Mdim % 8) return fail("segment reduction: Mdim must be a multiple of 8");
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  const int64_t Tm = T > 0 ? T : 1;
  if ((rc = make_map_2d(&a.tmA, P, Mdim, Tm, Mdim, 64, 64))) return rc;
  CUtensorMap* maps[3] = {&a.tmB, &a.tmB2, &a.tmB3};
  for (int j = 0; j < n_multi; ++j)
    if ((rc = make_map_2d(maps[j], Q[j], 64, Tm, 64, 64, 64))) return rc;
  a.row_off = pack->d_row_off;
  a.rpad_off = pack->d_rpad_off;
  a.mt_per = static_cast<int>((Mdim + kBM - 1) / kBM);
  a.n_groups = pack->n_adapters * a.mt_per;
  a.n_ntiles = 1;
  a.M = static_cast<int>(Mdim);
  a.N = 64;
  a.out = G[0];
  a.out2 = n_multi > 1 ? G[1] : nullptr;
  a.out3 = n_multi > 2 ? G[2] : nullptr;
  a.n_multi = n_multi;
  if (pack->h_row_off != nullptr) {   // whole tiles (LPT): see run_segred
    SegSched sched;
    if (segred_schedule(pack, a.mt_per, a.n_ntiles, &sched))
      return n_multi == 3 ? launch_segred_lpt<192>(a, sched, st) : launch_segred_lpt<128>(a, sched, st);
  }
  return n_multi == 3 ? launch<192, MODE_SEGRED, true>(a, st) : launch<128, MODE_SEGRED, true>(a, st);
}

}  // namespace plora

using namespace plora;

// ---------------------------------------------------------------- SwiGLU backward + K5 of down (swiglu_sm100.cuh)
static int run_swiglu_segred(cudaStream_t st, const plora_pack_t* pack, int64_t ffn, const void* d_act,
                             const void* g, const void* u, const void* dH, void* dg, void* du, float* G) {
  const int64_t T = pack->total_tokens;
  const int64_t Tm = T > 0 ? T : 1;
  SwArgs a;
  memset(&a, 0, sizeof(a));
  int rc;
  if ((rc = make_map_2d(&a.tmD, d_act, ffn, Tm, ffn, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmG, g, ffn, Tm, ffn, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmU, u, ffn, Tm, ffn, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmQ, dH, 64, Tm, 64, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmDG, dg, ffn, Tm, ffn, 64, 64))) return rc;
  if ((rc = make_map_2d(&a.tmDU, du, ffn, Tm, ffn, 64, 64))) return rc;
  a.dg = static_cast<__nv_bfloat16*>(dg);
  a.du = static_cast<__nv_bfloat16*>(du);
  a.row_off = pack->d_row_off;
  a.rpad_off = pack->d_rpad_off;
  a.out = G;
  a.ffn = ffn;
  a.M = static_cast<int>(ffn);
  a.mt_per = static_cast<int>((ffn + kBM - 1) / kBM);
  a.n_groups = pack->n_adapters * a.mt_per;
  // LPT tile schedule when the host row offsets are known and the tile count fits the
  // schedule; otherwise round-robin tiles (sched.n_ctas = 0)
  auto sched = std::make_unique<SegSched>();
  int grid;
  if (pack->h_row_off != nullptr && segred_schedule(pack, a.mt_per, 1, sched.get())) {
    grid = sched->n_ctas;
  } else {
    memset(sched.get(), 0, sizeof(SegSched));
    grid = a.n_groups < num_sms() ? a.n_groups : num_sms();
  }
  if (grid <= 0) return 0;
  static std::atomic<uint64_t> configured{0};
  if (ensure_smem(plora_swiglu_segred_kernel, kSwSmemBytes, configured)) return 1;
  PLORA_CUDA(launch_pdl(plora_swiglu_segred_kernel, dim3(grid), dim3(kSwThreads), kSwSmemBytes, st, a, *sched));
  return 0;
}

// ---------------------------------------------------------------- fused K3 + K4 (dual_sm100.cuh)
// Plan of the one-dY-pass kernel for (pack, k): units of rcs (1, 2 or 4) 128-row m-tiles of
// one adapter x nc (1..8) column chunks of k.  The (rcs, nc) pair is chosen with a small
// time model -- waves of units streaming dY at a per-SM rate, plus the fp32 partials'
// round trip and the fix-up -- and compared against the two separate passes (two
// launches' fixed cost + dY twice); the separate K4 / K3 kernels win for packs too small
// to amortise the partials.  Nor is a pack eligible with rank blocks > 1 or k % 128 != 0.
// Returns the workspace bytes (partials) or -1 when the separate kernels are used.
#ifndef PLORA_DUAL_SM_GBS
#define PLORA_DUAL_SM_GBS 40.0        // dY streaming rate of one CTA of the fused kernel (GB/s)
#endif
#ifndef PLORA_DUAL_HBM_GBS
#define PLORA_DUAL_HBM_GBS 5000.0     // achieved HBM rate of the LoRA kernels (GB/s)
#endif
#ifndef PLORA_DUAL_LAUNCH_US
#define PLORA_DUAL_LAUNCH_US 12.0     // fixed cost of one LoRA launch (fill, tail, launch gap)
#endif
#ifndef PLORA_DUAL_UNIT_US
#define PLORA_DUAL_UNIT_US 2.0        // per-unit cost of the fused kernel (Hs load, D_h drain)
#endif
struct DualPlan {
  DualSched sched;
  DualFix fix;
  int64_t part_b_floats;
  int64_t part_h_off[kDualMaxTargets];   // float offsets (after the dB partials) of each target's dH partials
  int64_t part_h_floats;
};

// The (rows per chunk, column chunks) options of one target: units, cost of one unit and
// fp32 partial bytes under the time model.
struct DualOpt {
  int rcs, nc;
  int64_t units;
  double unit_us, part_bytes;
};

static int dual_options(const plora_pack_t* pack, int64_t k, const int32_t* h_rpad_off, DualOpt* opt) {
  const int n = pack->n_adapters;
  const int64_t T = pack->total_tokens;
  int64_t sum_rp = 0, tiles_all = 0;
  for (int a = 0; a < n; ++a) {
    const int64_t tiles = (pack->h_row_off[a + 1] - pack->h_row_off[a] + kBM - 1) / kBM;
    sum_rp += (h_rpad_off[a + 1] - h_rpad_off[a]) * tiles;   // partials scale with rpad16 per m-tile
    tiles_all += tiles;
  }
  if (tiles_all == 0) return 0;
  const double avg_rp = static_cast<double>(sum_rp) / tiles_all;
  int no = 0;
  for (int rcs : {4, 2, 1}) {
    int64_t chunks = 0;
    for (int a = 0; a < n; ++a) {
      const int64_t tiles = (pack->h_row_off[a + 1] - pack->h_row_off[a] + kBM - 1) / kBM;
      chunks += (tiles + rcs - 1) / rcs;
    }
    for (int nc = 1; nc <= 8 && k / 128 >= nc; nc *= 2) {
      const int64_t units = chunks * nc;
      if (units > kDualMaxUnits) break;
      const int64_t kc = ((k + nc - 1) / nc + 127) / 128 * 128;
      DualOpt& o = opt[no++];
      o.rcs = rcs;
      o.nc = nc;
      o.units = units;
      o.unit_us = rcs * 128.0 * kc * 2 / (PLORA_DUAL_SM_GBS * 1e3) + PLORA_DUAL_UNIT_US;
      o.part_bytes = 4.0 * avg_rp * (static_cast<double>(chunks) * k + (nc > 1 ? nc * static_cast<double>(T) : 0.0));
    }
  }
  return no;
}

// Best options of the n_t targets of ONE launch, chosen jointly: the kernel hands unit u
// to CTA u mod grid with the targets' units in sequence, so the main-loop time is the
// heaviest CTA's sum of unit costs over all targets (a per-target choice would size each
// target for the whole machine and the launch would run ~2 waves).  Compared against the
// separate K4 + K3 passes of every target; false = those are expected to be faster.
static bool dual_choose(const plora_pack_t* pack, int n_t, const int64_t* ks, const int32_t* h_rpad_off,
                        int* rcs_out, int* nc_out) {
  constexpr int kMaxOpt = 12;
  DualOpt opt[kDualMaxTargets][kMaxOpt];
  int no[kDualMaxTargets];
  const int sms = num_sms();
  const int64_t T = pack->total_tokens;
  double sep_us = 0;
  for (int t = 0; t < n_t; ++t) {
    no[t] = dual_options(pack, ks[t], h_rpad_off, opt[t]);
    if (no[t] == 0) return false;
    sep_us += 2.0 * PLORA_DUAL_LAUNCH_US + 4.0 * T * ks[t] / (PLORA_DUAL_HBM_GBS * 1e3);
  }
  double best_us = sep_us;
  bool found = false;
  int idx[kDualMaxTargets] = {0, 0, 0};
  for (;;) {
    int64_t units = 0;
    double work = 0, part = 0, cmax = 0;
    for (int t = 0; t < n_t; ++t) {
      const DualOpt& o = opt[t][idx[t]];
      units += o.units;
      work += o.units * o.unit_us;
      part += o.part_bytes;
      cmax = o.unit_us > cmax ? o.unit_us : cmax;
    }
    const double fixed = 2.0 * part / (PLORA_DUAL_HBM_GBS * 1e3) + PLORA_DUAL_LAUNCH_US;
    const int64_t grid = units < sms ? units : sms;
    const double lower = (work / grid > cmax ? work / grid : cmax) + fixed;
    if (units <= kDualMaxUnits && lower < best_us) {
      double tmain = 0;   // heaviest CTA: units [s, s + U_t) of target t, unit u on CTA u % grid
      for (int64_t i = 0; i < grid; ++i) {
        double load = 0;
        int64_t s = 0;
        for (int t = 0; t < n_t; ++t) {
          const int64_t U = opt[t][idx[t]].units;
          const int64_t cnt = (s + U - 1 - i >= 0 ? (s + U - 1 - i) / grid + 1 : 0) - (s - 1 - i >= 0 ? (s - 1 - i) / grid + 1 : 0);
          load += cnt * opt[t][idx[t]].unit_us;
          s += U;
        }
        tmain = load > tmain ? load : tmain;
      }
      const double us = tmain + fixed;
      if (us < best_us) {
        best_us = us;
        found = true;
        for (int t = 0; t < n_t; ++t) {
          rcs_out[t] = opt[t][idx[t]].rcs;
          nc_out[t] = opt[t][idx[t]].nc;
        }
      }
    }
    int t = 0;   // next combination
    while (t < n_t && ++idx[t] == no[t]) idx[t++] = 0;
    if (t == n_t) break;
  }
  return found;
}

// Plan of one fused launch over n_t targets of the pack (dY widths ks[t]) -- the targets'
// (rows per chunk, column chunks) are chosen jointly by dual_choose; the units of all
// targets go into one unit list.  Returns the workspace bytes, or -1 when the separate
// kernels are expected to be faster or the pack is not eligible (rank blocks > 1, k % 128 != 0,
// unit list or adapter table too large): then every target runs separately.
static int64_t dual_plan(const plora_pack_t* pack, int n_t, const int64_t* ks, const int32_t* h_rpad_off,
                         DualPlan* plan) {
  const int n = pack->n_adapters;
  if (!pack->h_row_off || !h_rpad_off || pack->nb != 1 || n > kDualMaxAdapters || n_t < 1 || n_t > kDualMaxTargets)
    return -1;
  for (int a = 0; a < n; ++a) {
    const int rp = h_rpad_off[a + 1] - h_rpad_off[a];
    if (rp <= 0 || rp > 64) return -1;
  }
  DualSched& sc = plan->sched;
  DualFix& f = plan->fix;
  sc.n_targets = f.n_targets = n_t;
  f.n = n;
  int u = 0;
  int64_t boff = 0;   // floats
  int rcs_t[kDualMaxTargets], nc_t[kDualMaxTargets];
  for (int t = 0; t < n_t; ++t)
    if (ks[t] <= 0 || ks[t] % 128 || ks[t] > (1 << 24)) return -1;
  if (!dual_choose(pack, n_t, ks, h_rpad_off, rcs_t, nc_t)) return -1;
  for (int t = 0; t < n_t; ++t) {
    const int64_t k = ks[t];
    int nc = nc_t[t];
    const int kc = static_cast<int>(((k + nc - 1) / nc + 127) / 128 * 128);
    nc = static_cast<int>((k + kc - 1) / kc);
    sc.tg[t].k = static_cast<int>(k);
    sc.tg[t].kc = kc;
    sc.tg[t].nc = nc;
  }
  for (int t = 0; t < n_t; ++t) {
    const int rcs = rcs_t[t], nc = sc.tg[t].nc, kc = sc.tg[t].kc;
    int64_t g = 0;
    for (int a = 0; a < n; ++a) {
      f.ubase[t][a] = u;
      const int64_t tiles = (pack->h_row_off[a + 1] - pack->h_row_off[a] + kBM - 1) / kBM;
      const int rp = h_rpad_off[a + 1] - h_rpad_off[a];
      for (int64_t q = 0; q < tiles; q += rcs) {
        const int rc = static_cast<int>(tiles - q < rcs ? tiles - q : rcs);
        if (g + q >= (1 << 20) || u + nc > kDualMaxUnits) return -1;
        for (int c = 0; c < nc; ++c) {
          sc.unit[u] = static_cast<uint32_t>(g + q) | static_cast<uint32_t>(rc - 1) << 20 |
                       static_cast<uint32_t>(c) << 22 | static_cast<uint32_t>(t) << 25;
          sc.boff[u] = static_cast<uint32_t>(boff / 16);
          boff += static_cast<int64_t>(kc) * rp;   // a multiple of 16 floats
          ++u;
        }
      }
      g += tiles;
    }
    f.ubase[t][n] = u;
  }
  sc.n_units = u;
  plan->part_b_floats = boff;
  int64_t ph = 0;
  for (int t = 0; t < n_t; ++t) {
    plan->part_h_off[t] = boff + ph;
    if (sc.tg[t].nc > 1) ph += static_cast<int64_t>(sc.tg[t].nc) * pack->total_tokens * 64;
  }
  plan->part_h_floats = ph;
  return (plan->part_b_floats + plan->part_h_floats) * 4 + 256;
}

static int run_dual(cudaStream_t st, const plora_pack_t* pack, const DualPlan& plan, const void* const* dY,
                    const void* const* Bt_sh, const void* const* Hs, void* const* dH, float* const* gradB, void* ws) {
  const int64_t T = pack->total_tokens;
  const int n_t = plan.sched.n_targets;
  auto a = std::make_unique<DualArgs>();
  memset(a.get(), 0, sizeof(DualArgs));
  DualOut out;
  memset(&out, 0, sizeof(out));
  int rc;
  float* part_b = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  for (int t = 0; t < n_t; ++t) {
    const int64_t k = plan.sched.tg[t].k;
    if ((rc = make_map_2d(&a->tmY[t], dY[t], k, T, k, 64, kBM))) return rc;
    if ((rc = make_map_3d(&a->tmL[t], Bt_sh[t], 64, k, pack->n_adapters, 64, 64))) return rc;
    if ((rc = make_map_2d(&a->tmH[t], Hs[t], 64, T, 64, 64, kBM))) return rc;
    a->dH[t] = static_cast<__nv_bfloat16*>(dH[t]);
    a->part_h[t] = part_b + plan.part_h_off[t];
    out.G[t] = gradB[t];
    out.dH[t] = static_cast<__nv_bfloat16*>(dH[t]);
    out.part_h[t] = a->part_h[t];
  }
  a->mtiles = pack->d_mtiles;
  a->alpha = pack->d_alpha;
  a->rpad_off = pack->d_rpad_off;
  a->part_b = part_b;
  a->T = T;
  static std::atomic<uint64_t> configured{0};
  if (ensure_smem(plora_dual_kernel, kDualSmemBytes, configured)) return 1;
  const int grid = plan.sched.n_units < num_sms() ? plan.sched.n_units : num_sms();
  PLORA_CUDA(launch_pdl(plora_dual_kernel, dim3(grid), dim3(192), kDualSmemBytes, st, *a, plan.sched));
  auto f = std::make_unique<DualFix>(plan.fix);
  int blocks = 0;
  for (int t = 0; t < n_t; ++t) {   // dB blocks of every target, then the dH blocks
    f->bB[t] = blocks;
    if (gradB[t]) blocks += static_cast<int>(((plan.sched.tg[t].k * pack->rpad16_total + 3) / 4 + 255) / 256);
  }
  f->bB[n_t] = blocks;
  for (int t = n_t + 1; t <= kDualMaxTargets; ++t) f->bB[t] = blocks;
  for (int t = 0; t < n_t; ++t) {
    f->bH[t] = blocks;
    if (plan.sched.tg[t].nc > 1) blocks += pack->n_mtiles;
  }
  for (int t = n_t; t <= kDualMaxTargets; ++t) f->bH[t] = blocks;
  if (blocks > 0) {
    PLORA_CUDA(launch_pdl(plora_dual_fix_kernel, dim3(blocks), dim3(256), 0, st, *f, plan.sched, out,
                          static_cast<const float*>(part_b), pack->d_rpad_off, pack->d_alpha, pack->d_mtiles, T));
  }
  return 0;
}

extern "C" {

int plora_abi_version(void) { return PLORA_ABI_VERSION; }

int64_t plora_lora_workspace_bytes(void) { return sk_need_bytes(num_sms(), 192); }

const char* plora_last_error(void) { return g_last_error.c_str(); }

int plora_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail("no CUDA device: %s", cudaGetErrorString(e));
  cudaDeviceProp p;
  PLORA_CUDA(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10 || p.minor != 0)
    return fail("libplora is built for sm_100a; device %d is sm_%d%d", dev, p.major, p.minor);
  return 0;
}

int plora_gemm_bf16(void* stream, int64_t M, int64_t N, int64_t K, const void* A, const void* W,
                    int32_t w_kmajor, void* Y, int64_t ldy, const void* residual) {
  return run_gemm(static_cast<cudaStream_t>(stream), nullptr, M, N, K, A, W, w_kmajor, nullptr,
                  nullptr, Y, ldy, residual);
}

static int check_pack(const plora_pack_t* p) {
  if (!p) return fail("pack is NULL");
  if (p->n_adapters <= 0) return fail("pack has no adapters");
  if (p->nb <= 0) return fail("pack rank blocks must be positive");
  if (!p->d_mtiles && p->n_mtiles) return fail("pack tile list missing");
  if (!p->d_row_off || !p->d_ranks || !p->d_rpad_off || !p->d_alpha)
    return fail("pack device arrays missing");
  return 0;
}

int plora_linear_fwd(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int64_t k,
                     const void* W, int32_t w_kmajor, const void* A_sh, const void* Bt_sh,
                     void* Hs_out, void* Y, int64_t ldy, const void* residual) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // K2a: Hs = alpha_i X_i A_i
  if ((rc = run_shrink(st, pack, d, X, A_sh, Hs_out))) return rc;
  // K1 + K2b: Y = X op(W) + Hs_i B_i (+ residual)
  return run_gemm(st, pack, pack->total_tokens, k, d, X, W, w_kmajor, Hs_out, Bt_sh, Y, ldy,
                  residual);
}

int plora_lora_shrink(void* stream, const plora_pack_t* pack, int64_t K, const void* P,
                      const void* L_sh, void* out) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  return run_shrink(static_cast<cudaStream_t>(stream), pack, K, P, L_sh, out);
}

int plora_lora_segred(void* stream, const plora_pack_t* pack, int64_t Mdim, const void* P,
                      const void* Q, float* G) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (!G) return fail("segred: output region is NULL");
  return run_segred(static_cast<cudaStream_t>(stream), pack, Mdim, P, Q, G);
}

int plora_lora_shrink_multi(void* stream, const plora_pack_t* pack, int64_t K, const void* P, int32_t n_multi,
                            const void* const* L_sh, void* const* outs) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (n_multi < 1 || n_multi > 3) return fail("shrink_multi: n_multi must be 1..3");
  if (pack->nb != 1 || n_multi == 1) {   // ranks > 64: one launch per target
    for (int j = 0; j < n_multi; ++j)
      if ((rc = run_shrink(static_cast<cudaStream_t>(stream), pack, K, P, L_sh[j], outs[j]))) return rc;
    return 0;
  }
  return run_shrink_multi(static_cast<cudaStream_t>(stream), pack, K, P, n_multi, L_sh, outs);
}

int plora_swiglu_bwd_segred(void* stream, const plora_pack_t* pack, int64_t ffn, const void* d_act, const void* g,
                            const void* u, const void* dH, void* dg, void* du, float* gradA) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (!d_act || !g || !u || !dH || !dg || !du || !gradA) return fail("swiglu_bwd_segred: NULL operand");
  if (ffn % 8) return fail("swiglu_bwd_segred: ffn must be a multiple of 8");
  if (pack->nb != 1) return fail("swiglu_bwd_segred: rank blocks > 1 (use plora_swiglu_bwd + plora_lora_segred)");
  return run_swiglu_segred(static_cast<cudaStream_t>(stream), pack, ffn, d_act, g, u, dH, dg, du, gradA);
}

int64_t plora_lora_dual_workspace_bytes(const plora_pack_t* pack, int32_t n_targets, const int64_t* ks,
                                        const int32_t* h_rpad_off) {
  if (check_pack(pack) || !ks) return -1;
  auto plan = std::make_unique<DualPlan>();
  const int64_t b = dual_plan(pack, n_targets, ks, h_rpad_off, plan.get());
  return b < 0 ? 0 : b;
}

int plora_lora_dual(void* stream, const plora_pack_t* pack, int32_t n_targets, const int64_t* ks,
                    const int32_t* h_rpad_off, const void* const* dY, const void* const* Bt_sh, const void* const* Hs,
                    void* const* dH, float* const* gradB, void* ws, int64_t ws_bytes) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (n_targets < 1 || n_targets > kDualMaxTargets) return fail("lora_dual: 1..3 targets");
  if (!ks || !dY || !Bt_sh || !Hs || !dH || !gradB) return fail("lora_dual: NULL operand array");
  for (int t = 0; t < n_targets; ++t)
    if (!dY[t] || !Bt_sh[t] || !dH[t] || (gradB[t] && !Hs[t])) return fail("lora_dual: NULL operand");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (pack->total_tokens > 0 && pack->n_mtiles > 0) {
    auto plan = std::make_unique<DualPlan>();
    const int64_t need = dual_plan(pack, n_targets, ks, h_rpad_off, plan.get());
    if (need >= 0 && ws != nullptr && ws_bytes >= need)
      return run_dual(st, pack, *plan, dY, Bt_sh, Hs, dH, gradB, ws);
  }
  // not eligible (or no workspace): the separate K4 / K3 kernels per target, same results up
  // to fp32 association
  for (int t = 0; t < n_targets; ++t) {
    if ((rc = run_shrink(st, pack, ks[t], dY[t], Bt_sh[t], dH[t]))) return rc;
    if (gradB[t] && (rc = run_segred(st, pack, ks[t], dY[t], Hs[t], gradB[t]))) return rc;
  }
  return 0;
}

int plora_lora_segred_multi(void* stream, const plora_pack_t* pack, int64_t Mdim, const void* P, int32_t n_multi,
                            const void* const* Q, float* const* G) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (n_multi < 1 || n_multi > 3) return fail("segred_multi: n_multi must be 1..3");
  for (int j = 0; j < n_multi; ++j)
    if (!G[j]) return fail("segred_multi: output region is NULL");
  if (pack->nb != 1 || n_multi == 1) {
    for (int j = 0; j < n_multi; ++j)
      if ((rc = run_segred(static_cast<cudaStream_t>(stream), pack, Mdim, P, Q[j], G[j]))) return rc;
    return 0;
  }
  return run_segred_multi(static_cast<cudaStream_t>(stream), pack, Mdim, P, n_multi, Q, G);
}

int plora_linear_expand(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int64_t k,
                        const void* W, int32_t w_kmajor, const void* Bt_sh, const void* Hs, void* Y,
                        int64_t ldy, const void* residual) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  return run_gemm(static_cast<cudaStream_t>(stream), pack, pack->total_tokens, k, d, X, W, w_kmajor,
                  Hs, Bt_sh, Y, ldy, residual);
}

// narrowest grouped segment (narrower: separate launches); narrow TP-shard k/v (N = 128)
// ride the grouped launch: ~1% per C4 layer
static constexpr int g_group_min_n = PLORA_GROUP_MIN_N;

static bool group_pair_ok(const plora_pack_t* pack, int n, const int64_t* N) {
  if (pack->d_ptiles == nullptr && pack->n_ptiles != 0) return false;
  int64_t widest = 0;
  for (int j = 0; j < n; ++j) {
    if (N[j] < g_group_min_n) return false;
    widest = N[j] > widest ? N[j] : widest;
  }
  return widest >= 256;
}

int plora_linear_expand_group(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int32_t n,
                              const int64_t* k_out, const void* const* W, int32_t w_kmajor,
                              const void* const* Bt_sh, const void* const* Hs, void* const* Y,
                              const void* const* bias) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (n < 1 || n > 3) return fail("expand_group: 1..3 targets");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t T = pack->total_tokens;
  if (T <= 0) return 0;
  if (!group_pair_ok(pack, n, k_out)) {   // narrow targets: one launch per target
    for (int j = 0; j < n; ++j)
      if ((rc = run_gemm(st, pack, T, k_out[j], d, X, W[j], w_kmajor, Hs[j], Bt_sh[j], Y[j], k_out[j], nullptr,
                         bias ? bias[j] : nullptr)))
        return rc;
    return 0;
  }
  PairSeg sg[3];
  for (int j = 0; j < n; ++j)
    sg[j] = PairSeg{X, d, W[j], k_out[j], Hs[j], Bt_sh[j], Y[j], k_out[j], bias ? bias[j] : nullptr};
  return run_pair_segments(st, pack, T, n, 1, sg, w_kmajor, nullptr);
}

int plora_linear_gate_up_swiglu(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int64_t ffn,
                                const void* W_gate, const void* W_up, const void* Bt_gate, const void* Bt_up,
                                const void* Hs_gate, const void* Hs_up, void* g, void* u, void* act) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (!g || !u || !act) return fail("gate_up_swiglu: g, u and act are required");
  const int64_t T = pack->total_tokens;
  if (T <= 0) return 0;
  if ((pack->d_ptiles == nullptr && pack->n_ptiles != 0) || ffn < 256)
    return fail("gate_up_swiglu: needs the CTA-pair GEMM and ffn >= 256");
  PairSeg sg[2] = {PairSeg{X, d, W_gate, ffn, Hs_gate, Bt_gate, g, ffn}, PairSeg{X, d, W_up, ffn, Hs_up, Bt_up, u, ffn}};
  return run_pair_segments(static_cast<cudaStream_t>(stream), pack, T, 2, 1, sg, 1, nullptr, act);
}

int plora_linear_dx_group(void* stream, const plora_pack_t* pack, int32_t n, const void* const* dY,
                          const int64_t* k_out, const void* const* W, int32_t w_kmajor, const void* const* A_sh,
                          const void* const* dH, int64_t d, void* dX, int64_t lddx, const void* dX_residual) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  if (n < 1 || n > 3) return fail("dx_group: 1..3 targets");
  if (!dX) return fail("dx_group: dX is NULL");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t T = pack->total_tokens;
  if (T <= 0) return 0;
  const int64_t dd[3] = {d, d, d};
  if (!group_pair_ok(pack, 1, dd)) {
    for (int j = 0; j < n; ++j)
      if ((rc = run_gemm(st, pack, T, d, k_out[j], dY[j], W[j], !w_kmajor, dH[j], A_sh[j], dX, lddx,
                         j == 0 ? dX_residual : dX)))
        return rc;
    return 0;
  }
  PairSeg sg[3];
  for (int j = 0; j < n; ++j) sg[j] = PairSeg{dY[j], k_out[j], W[j], d, dH[j], A_sh[j], dX, lddx};
  return run_pair_segments(st, pack, T, 1, n, sg, !w_kmajor, dX_residual);
}

int plora_linear_bwd(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int64_t k,
                     const void* W, int32_t w_kmajor, const void* A_sh, const void* Bt_sh,
                     const void* Hs, const void* dY, void* dH_ws, void* dX, int64_t lddx,
                     const void* dX_residual, float* gradA, float* gradB) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // Case 2 (K4): dH = alpha_i dY_i B_i^T   (B^T stored [n][k][64nb] = L[K=k][N=r])
  if ((rc = run_shrink(st, pack, k, dY, Bt_sh, dH_ws))) return rc;
  // Case 1 (K3): dB_i^T[k][r] = Hs_i^T dY_i  ->  sum_t dY[t][k] Hs[t][r]
  if (gradB && (rc = run_segred(st, pack, k, dY, Hs, gradB))) return rc;
  // Case 3 (K5): dA_i[d][r] = X_i^T dH_i
  if (gradA && (rc = run_segred(st, pack, d, X, dH_ws, gradA))) return rc;
  // Case 4 (K6): dX = dY op(W)^T + dH_i A_i^T.  op(W)^T as a B operand [N=d][K=k]:
  //   nn.Linear W [k][d] is MN-major for this product; reference W [d][k] is K-major.
  if (dX)
    return run_gemm(st, pack, pack->total_tokens, d, k, dY, W, w_kmajor ? 0 : 1, dH_ws, A_sh, dX,
                    lddx, dX_residual);
  return 0;
}

}  // extern "C"
