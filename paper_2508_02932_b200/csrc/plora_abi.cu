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
#include <mutex>
#include <string>

#include "../../include/plora.h"
#include "gemm_sm100.cuh"

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
static int make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
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
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail("cuTensorMapEncodeTiled(2d inner=%llu outer=%llu box=%u,%u) failed: %d",
                (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer, (int)r);
  return 0;
}

// 2D bf16 output tensor for the TMA-store epilogue: 32x32 boxes, 64-byte swizzle.
static int make_map_out(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_elems) {
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
static int make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t mid, uint64_t n,
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
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail("cuTensorMapEncodeTiled(3d) failed: %d", (int)r);
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

template <int BN, int MODE, bool B_MN>
static int launch(const GemmArgs& args, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = plora_gemm_kernel<BN, MODE, B_MN>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    PLORA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes));
    configured = true;
  }
  const int total = args.n_groups * args.n_ntiles;
  if (total <= 0) return 0;
  const int grid = total < num_sms() ? total : num_sms();
  kern<<<grid, kThreads, Cfg::kSmemBytes, stream>>>(args);
  PLORA_CUDA(cudaGetLastError());
  return 0;
}

static int pick_bn(int64_t N) { return N >= 256 ? 256 : (N > 64 ? 128 : 64); }

static int g_debug_flags = [] {
  const char* e = getenv("PLORA_DEBUG_FLAGS");
  return e ? atoi(e) : 0;
}();

static bool g_pair_enabled = [] {
  const char* e = getenv("PLORA_GEMM_PAIR");
  return !(e && e[0] == '0');
}();

template <bool B_MN, int NB>
static int launch_pair(const GemmArgs& args, cudaStream_t stream) {
  auto kern = plora_gemm_pair_kernel<B_MN, NB>;
  static bool configured = false;
  if (!configured) {
    PLORA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<NB>::kSmemBytes));
    configured = true;
  }
  const int total = args.n_groups * args.n_ntiles;
  if (total <= 0) return 0;
  const int max_clusters = num_sms() / 2;
  const int clusters = total < max_clusters ? total : max_clusters;
  kern<<<clusters * 2, PairCfg<NB>::kThreads, PairCfg<NB>::kSmemBytes, stream>>>(args);
  PLORA_CUDA(cudaGetLastError());
  return 0;
}

static int g_pair_nb_min_n = [] {   // N at which the 256x512 pair tile is used
  const char* e = getenv("PLORA_PAIR512_MIN_N");
  return e ? atoi(e) : 2048;
}();

// CTA-pair GEMM (N >= 256): 256 x 256 tiles with tcgen05 cta_group::2.
static int run_gemm_pair(cudaStream_t st, const plora_pack_t* pack, int64_t M, int64_t N, int64_t K,
                         const void* A, const void* W, int w_kmajor, const void* H, const void* L,
                         void* Y, int64_t ldy, const void* residual) {
  const int NB = N >= g_pair_nb_min_n ? 2 : 1;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int rc = make_map_2d(&a.tmA, A, K, M, K, 64, kBM);
  if (rc) return rc;
  if (w_kmajor) rc = make_map_2d(&a.tmB, W, K, N, K, 64, 128);
  else          rc = make_map_2d(&a.tmB, W, N, K, N, 64, 64);
  if (rc) return rc;
  const bool lora = pack != nullptr && H != nullptr && L != nullptr;
  if (lora) {
    const int64_t R64 = 64LL * pack->nb;
    if ((rc = make_map_2d(&a.tmH, H, R64, M, R64, 64, kBM))) return rc;
    if ((rc = make_map_3d(&a.tmL, L, R64, N, pack->n_adapters, 64, 128))) return rc;
    a.ranks = pack->d_ranks;
    a.nb = pack->nb;
    a.has_lora = 1;
  }
  a.mtiles = pack ? pack->d_ptiles : nullptr;
  a.n_groups = pack ? pack->n_ptiles : static_cast<int>((M + 255) / 256);
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(N);
  a.K = static_cast<int>(K);
  a.n_ntiles = static_cast<int>((N + 256 * NB - 1) / (256 * NB));
  a.out = Y;
  a.ldo = ldy;
  if ((rc = make_map_out(&a.tmY, Y, N, M, ldy))) return rc;
  // Y = result + residual is computed as Y <- residual (skipped when in place), then a
  // TMA reduce-add of the result (bf16 add in L2).
  if (residual) {
    if (residual != Y)
      PLORA_CUDA(cudaMemcpy2DAsync(Y, ldy * 2, residual, ldy * 2, N * 2, M, cudaMemcpyDeviceToDevice, st));
    a.accumulate = 1;
  }
  a.debug = g_debug_flags;
  if (NB == 2) return w_kmajor ? launch_pair<false, 2>(a, st) : launch_pair<true, 2>(a, st);
  return w_kmajor ? launch_pair<false, 1>(a, st) : launch_pair<true, 1>(a, st);
}

// Base GEMM (+ fused LoRA expand).  A: [M][K] K-major.  W: see w_kmajor.
static int run_gemm(cudaStream_t st, const plora_pack_t* pack, int64_t M, int64_t N, int64_t K,
                    const void* A, const void* W, int w_kmajor, const void* H, const void* L,
                    void* Y, int64_t ldy, const void* residual) {
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0) return fail("gemm: K must be positive");
  if (K % 8 || N % 8 || ldy % 8) return fail("gemm: K, N and ldy must be multiples of 8");
  if (reinterpret_cast<uintptr_t>(Y) % 16 || (residual && reinterpret_cast<uintptr_t>(residual) % 16))
    return fail("gemm: output/residual must be 16-byte aligned");
  if (g_pair_enabled && N >= 256 && (pack == nullptr || pack->d_ptiles != nullptr || pack->n_ptiles == 0))
    return run_gemm_pair(st, pack, M, N, K, A, W, w_kmajor, H, L, Y, ldy, residual);
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
  if (BN == 256) return w_kmajor ? launch<256, MODE_GEMM, false>(a, st) : launch<256, MODE_GEMM, true>(a, st);
  if (BN == 128) return w_kmajor ? launch<128, MODE_GEMM, false>(a, st) : launch<128, MODE_GEMM, true>(a, st);
  return w_kmajor ? launch<64, MODE_GEMM, false>(a, st) : launch<64, MODE_GEMM, true>(a, st);
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
  return launch<64, MODE_SHRINK, true>(a, st);
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
  return launch<64, MODE_SEGRED, true>(a, st);
}

}  // namespace plora

using namespace plora;

extern "C" {

int plora_abi_version(void) { return PLORA_ABI_VERSION; }

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

int plora_linear_expand(void* stream, const plora_pack_t* pack, const void* X, int64_t d, int64_t k,
                        const void* W, int32_t w_kmajor, const void* Bt_sh, const void* Hs, void* Y,
                        int64_t ldy, const void* residual) {
  int rc;
  if ((rc = check_pack(pack))) return rc;
  return run_gemm(static_cast<cudaStream_t>(stream), pack, pack->total_tokens, k, d, X, W, w_kmajor,
                  Hs, Bt_sh, Y, ldy, residual);
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
