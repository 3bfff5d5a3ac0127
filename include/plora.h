/*
 * plora.h -- C-ABI of libplora, the B200 (sm_100a) packed multi-LoRA hot path.
 *
 * This is the drop-in boundary for the reference's packed-LoRA operator API
 * (`lorasweep.lorapack`, reference pkg/src/lorasweep/lorapack.py:31-42,128-231).
 * The reference has no FFI of its own (it is pure Python/numpy); its "plugin
 * interface" is the set of Python functions re-exported at
 * pkg/src/lorasweep/__init__.py:78-89.  The Python host mirror
 * `paper_2508_02932_b200.lorapack` keeps those names and binds the entry points
 * below with ctypes (see INTEGRATION.md for the binding a maintainer would add
 * to lorasweep itself).
 *
 * Conventions
 *   - Every function returns int status: 0 = ok, non-zero = error; the message
 *     is available from plora_last_error() (thread-local).  Nothing throws
 *     across the ABI.
 *   - All tensor arguments are CALLER-OWNED device buffers (plain pointers);
 *     no entry point allocates device memory.  Work is enqueued on the
 *     caller's stream (cudaStream_t passed as void*), stream-ordered and
 *     re-entrant.
 *   - Element types: "bf16" = IEEE bfloat16 (uint16 storage), "f32" = float.
 *   - Shapes are row-major; "[T][d]" means T rows of d contiguous elements.
 *
 * Device layouts
 *   rank blocks : every adapter's rank is zero-padded to rpad64 = 64*nb columns
 *                 in the bf16 compute shadows (nb = ceil(max_rank/64)), and to
 *                 rpad16_i = roundup(r_i,16) in fp32 master/grad/moment buffers.
 *   A_sh  bf16 [n][d][rpad64]  -- adapter down-projection A_i (d x r_i), rank-minor
 *   Bt_sh bf16 [n][k][rpad64]  -- adapter up-projection  B_i^T (k x r_i), rank-minor
 *   Hs    bf16 [T][rpad64]     -- alpha_i * X_i A_i  (saved from forward)
 *   dH    bf16 [T][rpad64]     -- alpha_i * dY_i B_i^T
 *   gradA f32  region [sum_i d*rpad16_i]: adapter i block [d][rpad16_i] at d*rpad_off[i]
 *   gradB f32  region [sum_i k*rpad16_i]: adapter i block [k][rpad16_i] at k*rpad_off[i]
 */
#ifndef PLORA_H_
#define PLORA_H_

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define PLORA_API __attribute__((visibility("default")))
#else
#define PLORA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PLORA_ABI_VERSION 9

/* Device-resident description of one pack (segment index + adapter table).
 * Built by plora_meta_build on the host, copied to device by the caller. */
typedef struct plora_pack {
  int32_t n_adapters;
  int32_t n_mtiles;        /* entries in d_mtiles */
  int64_t total_tokens;    /* T = row_offsets[n] */
  int32_t nb;              /* 64-column rank blocks per adapter in the shadows */
  int32_t rpad16_total;    /* sum_i rpad16_i */
  const int32_t* d_mtiles; /* [n_mtiles][4] = {m0, m_len (1..128), adapter, 0} */
  const int64_t* d_row_off;/* [n+1] token row offsets (reference row_offsets) */
  const int32_t* d_ranks;  /* [n]   r_i */
  const int32_t* d_rpad_off;/*[n+1] prefix sums of rpad16_i */
  const float*   d_alpha;  /* [n]   raw alpha_i (no alpha/r) */
  int32_t n_ptiles;        /* entries in d_ptiles */
  int32_t pad_;
  const int32_t* d_ptiles; /* [n_ptiles][4] = {m0, m_len (1..256), adapter, 0}: CTA-pair tiles */
  const int64_t* h_row_off;/* [n+1] HOST copy of the row offsets (may be NULL): lets the
                              segment reductions balance their tiles across SMs (LPT) */
  void* d_ws;              /* device workspace of the shrink / segment-reduction kernels
                              (may be NULL): plora_lora_workspace_bytes() bytes, ZERO-filled
                              once by the caller; the kernels leave it zeroed.  With it, K2a/K4
                              and K3/K5 split their long tiles across all SMs (stream-K) --
                              without it they run whole tiles (fewer SMs busy at small T).
                              Launches sharing one workspace must be stream-ordered. */
  int64_t ws_bytes;        /* size of d_ws */
} plora_pack_t;

/* Library / error plumbing. */
PLORA_API int plora_abi_version(void);
/* Bytes of the pack workspace (plora_pack_t.d_ws) on the current device. */
PLORA_API int64_t plora_lora_workspace_bytes(void);
PLORA_API const char* plora_last_error(void);
PLORA_API int plora_device_check(void);   /* 0 iff an sm_100 device is current */

/* K8: segment-index / adapter-metadata builder (host, bit-exact with
 * lorapack.pack_adapters rank/row offsets, reference lorapack.py:146-150).
 *   ranks[n] >= 1, tokens[n] >= 0.
 *   Outputs (caller-allocated host arrays):
 *     rank_off[n+1], row_off[n+1], rpad_off[n+1]
 *     mtiles[max_mtiles][4]  (tile list: every tile lies inside one segment)
 *     ptiles[max_mtiles][4]  (256-row CTA-pair tiles, same rule; may be NULL)
 *     token_adapter[T]       (may be NULL)
 *   *n_mtiles receives the tile count; if it exceeds max_mtiles nothing is
 *   written to mtiles and status 2 is returned. */
PLORA_API int plora_meta_build(int32_t n, const int64_t* ranks, const int64_t* tokens,
                     int64_t* rank_off, int64_t* row_off, int32_t* rpad_off,
                     int32_t* mtiles, int32_t max_mtiles, int32_t* n_mtiles,
                     int32_t* ptiles, int32_t* n_ptiles, int32_t* token_adapter);

/* Upper bound on the tile count for plora_meta_build. */
PLORA_API int32_t plora_meta_max_mtiles(int32_t n, const int64_t* tokens);

/* K1 (+K2b): Y[T][N] = A[T][K] * op(W) (+ LoRA expand) (+ residual), bf16 out,
 * fp32 accumulation in TMEM.  Plain library GEMM entry used by the model for
 * frozen projections without adapters (lm_head) and by tests.
 *   w_kmajor = 1: W stored [N][K] (nn.Linear layout, y = x W^T)
 *   w_kmajor = 0: W stored [K][N] (reference layout,  y = x W)
 *   pack may be NULL (then M = T rows, single group, no LoRA). */
PLORA_API int plora_gemm_bf16(void* stream, int64_t M, int64_t N, int64_t K,
                    const void* A, const void* W, int32_t w_kmajor,
                    void* Y, int64_t ldy, const void* residual);

/* Packed LoRA linear, forward (reference packed_forward, lorapack.py:183-199):
 *   Hs = alpha_i * X_i A_i                         (K2a shrink, tcgen05)
 *   Y  = X op(W) + Hs_i B_i (+ residual)           (K1 GEMM, K2b as extra K-steps)
 * X bf16 [T][d]; W bf16 [k][d] (w_kmajor=1) or [d][k] (w_kmajor=0);
 * A_sh, Bt_sh as above; Hs_out bf16 [T][rpad64]; Y bf16 [T][ldy].
 * residual (may be NULL; may equal Y for in-place accumulation): Y = result + residual. */
PLORA_API int plora_linear_fwd(void* stream, const plora_pack_t* pack,
                     const void* X, int64_t d, int64_t k,
                     const void* W, int32_t w_kmajor,
                     const void* A_sh, const void* Bt_sh,
                     void* Hs_out, void* Y, int64_t ldy, const void* residual);

/* K2a / K4 alone: out[T][rpad64] = alpha_i * P_i[T_i][K] * L_i[K][rpad64],
 * L stored [n][K][rpad64] (A_sh for the forward shrink, Bt_sh for dH). */
PLORA_API int plora_lora_shrink(void* stream, const plora_pack_t* pack, int64_t K,
                     const void* P, const void* L_sh, void* out);

/* K3 / K5 alone: G_i[Mdim][rpad16_i] = P_i^T Q_i over segment i's tokens, fp32,
 * written into the adapter-major region G (P bf16 [T][Mdim], Q bf16 [T][rpad64]). */
PLORA_API int plora_lora_segred(void* stream, const plora_pack_t* pack, int64_t Mdim,
                     const void* P, const void* Q, float* G);

/* SwiGLU backward + K5 of the down projection in ONE pass (reference lorapack.py:226 for the
 * down target, whose input is act = silu(g) * u):
 *   dg = d_act * u * s (1 + g (1 - s)), du = d_act * g * s   (bf16 [T][ffn]; may alias g / u)
 *   gradA region (down) = dA_i = act_i^T dH_i per segment    (f32, as plora_lora_segred with P = act)
 * act is formed in shared memory and never written; results bit-identical to plora_swiglu_bwd
 * followed by plora_lora_segred.  d_act, g, u bf16 [T][ffn]; dH bf16 [T][64].  Needs nb == 1
 * and the pack's host row offsets (tile schedule). */
PLORA_API int plora_swiglu_bwd_segred(void* stream, const plora_pack_t* pack, int64_t ffn, const void* d_act,
                    const void* g, const void* u, const void* dH, void* dg, void* du, float* gradA);

/* K4 + K3 in ONE pass over dY (reference lorapack.py:224-225, Cases 2 and 1), for 1..3
 * targets of the pack in one launch (q/k/v or gate/up of a layer):
 *   dH[t][T][64]   = alpha_i * dY[t]_i B[t]_i^T       (bf16, as plora_lora_shrink with L = Bt_sh[t])
 *   gradB[t]       = dB_i^T = Hs[t]_i^T dY[t]_i        (f32 region, as plora_lora_segred; may be NULL)
 * dY[t] bf16 [T][ks[t]], Bt_sh[t] bf16 [n][ks[t]][64], Hs[t] bf16 [T][64].  Every dY tile is
 * read once and feeds both tensor-core contractions; cross-tile sums go through fp32 partials
 * in the caller-owned workspace ws (plora_lora_dual_workspace_bytes; no zero-fill needed) and a
 * deterministic fix-up.  h_rpad_off = HOST copy of the rpad16 prefix sums [n+1]; the pack must
 * carry h_row_off.  Packs whose targets a time model expects to run faster as separate
 * passes (or nb > 1, k % 128 != 0, too small a workspace) run the separate K4 / K3 kernels. */
PLORA_API int64_t plora_lora_dual_workspace_bytes(const plora_pack_t* pack, int32_t n_targets, const int64_t* ks,
                    const int32_t* h_rpad_off);
PLORA_API int plora_lora_dual(void* stream, const plora_pack_t* pack, int32_t n_targets, const int64_t* ks,
                    const int32_t* h_rpad_off, const void* const* dY, const void* const* Bt_sh,
                    const void* const* Hs, void* const* dH, float* const* gradB, void* ws, int64_t ws_bytes);

/* Multi-target K2a / K5 for n_multi (1..3) targets that share their input P (the
 * normed layer input of q/k/v, or of gate/up): P is read ONCE for all targets.
 *   shrink_multi : outs[j][T][rpad64] = alpha_i * P_i L_sh[j]_i
 *   segred_multi : G[j] (f32 region) = P_i^T Q[j]_i per segment
 * L_sh / outs / Q / G are host arrays of n_multi device pointers.  With ranks > 64
 * (nb > 1) they fall back to one launch per target. */
PLORA_API int plora_lora_shrink_multi(void* stream, const plora_pack_t* pack, int64_t K,
                     const void* P, int32_t n_multi, const void* const* L_sh, void* const* outs);
PLORA_API int plora_lora_segred_multi(void* stream, const plora_pack_t* pack, int64_t Mdim,
                     const void* P, int32_t n_multi, const void* const* Q, float* const* G);

/* K1 + K2b only: Y = X op(W) + Hs_i B_i (+ residual) with a caller-provided Hs
 * (e.g. saved from an earlier shrink, or perturbed by a gradient checker). */
PLORA_API int plora_linear_expand(void* stream, const plora_pack_t* pack,
                     const void* X, int64_t d, int64_t k,
                     const void* W, int32_t w_kmajor, const void* Bt_sh,
                     const void* Hs, void* Y, int64_t ldy, const void* residual);

/* Grouped K1 + K2b for n (1..3) targets sharing the input X (q/k/v, gate/up): ONE
 * launch enumerates every target's output tiles (N-segments of the pair GEMM);
 * Y[j] bf16 [T][k_out[j]] = X op(W[j]) + Hs[j]_i Bt_sh[j]_i^T.  W / Bt_sh / Hs / Y are
 * host arrays of n device pointers. */
PLORA_API int plora_linear_expand_group(void* stream, const plora_pack_t* pack,
                     const void* X, int64_t d, int32_t n, const int64_t* k_out,
                     const void* const* W, int32_t w_kmajor, const void* const* Bt_sh,
                     const void* const* Hs, void* const* Y,
                     const void* const* bias /* may be NULL; bias[j] bf16 [k_out[j]] or NULL */);
/* y[r][c] += bias[c] (bf16, rows x n, row pitch ldy): a standalone broadcast row bias. */
PLORA_API int plora_add_row_bias(void* stream, int64_t rows, int64_t n, void* y, int64_t ldy, const void* bias);

/* gate/up projections fused with the SwiGLU forward: one pair-GEMM launch whose tiles
 * hold 256 gate and the same 256 up columns, so the epilogue writes
 *   g = X W_gate^T + Hs_gate,i Bt_gate,i^T,  u = (same for up),  act = silu(g) u
 * (act from the bf16-rounded g, u: bit-identical to plora_swiglu_fwd).  W_* nn.Linear
 * layout [ffn][d]; g / u / act bf16 [T][ffn]. */
PLORA_API int plora_linear_gate_up_swiglu(void* stream, const plora_pack_t* pack, const void* X,
                     int64_t d, int64_t ffn, const void* W_gate, const void* W_up,
                     const void* Bt_gate, const void* Bt_up, const void* Hs_gate, const void* Hs_up,
                     void* g, void* u, void* act);

/* Grouped K6 for those targets: dX [T][lddx] = sum_j dY[j] op(W[j])^T + dH[j]_i A_sh[j]_i^T
 * (+ dX_residual), one accumulator over the concatenated K range (K-segments). */
PLORA_API int plora_linear_dx_group(void* stream, const plora_pack_t* pack, int32_t n,
                     const void* const* dY, const int64_t* k_out, const void* const* W,
                     int32_t w_kmajor, const void* const* A_sh, const void* const* dH,
                     int64_t d, void* dX, int64_t lddx, const void* dX_residual);

/* Packed LoRA linear, backward (reference packed_backward, lorapack.py:202-231):
 *   dH  = alpha_i dY_i B_i^T                       (Case 2, K4 shrink)
 *   dB_i^T = Hs_i^T dY_i  -> gradB (f32)           (Case 1, K3 segment reduction)
 *   dA_i   = X_i^T dH_i   -> gradA (f32)           (Case 3, K5 segment reduction)
 *   dX  = dY op(W)^T + dH_i A_i^T                  (Case 4, K6 GEMM + extra K-steps)
 * dX may be NULL (first layer: input gradient not needed).  dX_residual (may be
 * NULL, same layout as dX) is added in the dX epilogue, so the input gradients of
 * several linears that share an input (q/k/v, gate/up) accumulate without a pass.
 * gradA / gradB are the adapter-major f32 regions described above (written,
 * not accumulated). dH_ws is a bf16 [T][rpad64] workspace. */
PLORA_API int plora_linear_bwd(void* stream, const plora_pack_t* pack,
                     const void* X, int64_t d, int64_t k,
                     const void* W, int32_t w_kmajor,
                     const void* A_sh, const void* Bt_sh,
                     const void* Hs, const void* dY, void* dH_ws,
                     void* dX, int64_t lddx, const void* dX_residual,
                     float* gradA, float* gradB);

/* K7: fused per-adapter AdamW (torch.optim.AdamW semantics, decoupled decay)
 * over fp32 master weights with bf16 shadow write-back.  One call updates
 * every (layer, target, A|B) region of every adapter.
 *   chunks: device array [n_chunks][4] int64 =
 *     {master element offset, shadow element offset, n_rows | rpad16 << 32,
 *      adapter | shadow_ld << 32}
 *   hp: device array [n][4] f32 = {lr, weight_decay, step, unused}
 *   step: optimizer step count (>= 1) used for bias correction of every adapter, or
 *     0: each adapter's own count hp[i].z (>= 1, kept on the device by the caller --
 *     a launch sequence that CUDA graphs can replay, and adapters that joined a
 *     packed job at different times). */
PLORA_API int plora_adamw(void* stream, int64_t n_chunks, const int64_t* chunks,
                float* param, const float* grad, float* exp_avg, float* exp_avg_sq,
                void* shadow, const float* hp, float beta1, float beta2, float eps,
                int64_t step);

/* ---- fused HBM-bound helpers of the decoder step (off the LoRA hot path) ---- */

/* y = x * rstd * w with rstd = rsqrt(mean(x^2) + eps) (use_given_rstd = 0 computes
 * and stores rstd[rows]; 1 recomputes y from a saved rstd).  bf16 [rows][d], d <= 8192. */
PLORA_API int plora_rmsnorm_fwd(void* stream, int64_t rows, int64_t d, const void* x, const void* w,
                                float eps, void* y, float* rstd, int32_t use_given_rstd);
/* Fused residual add + RMSNorm: sum = a + b (bf16), y = rmsnorm(sum) * w, rstd[rows]. */
PLORA_API int plora_add_rmsnorm_fwd(void* stream, int64_t rows, int64_t d, const void* a, const void* b,
                                    const void* w, float eps, void* sum, void* y, float* rstd);
/* dx = rstd * (g - xhat * mean(g * xhat)) (+ residual), g = dy * w. */
PLORA_API int plora_rmsnorm_bwd(void* stream, int64_t rows, int64_t d, const void* dy, const void* x,
                                const float* rstd, const void* w, const void* residual, void* dx);
/* a = silu(g) * u ;  (dg, du) from da. n elements, multiple of 8.  The backward may
 * also re-emit a (act may be NULL) in the same pass, so the down-projection's
 * dA = a^T dH needs no separate recompute of the activation; dg / du may alias g / u. */
PLORA_API int plora_swiglu_fwd(void* stream, int64_t n, const void* g, const void* u, void* a);
PLORA_API int plora_swiglu_bwd(void* stream, int64_t n, const void* da, const void* g, const void* u,
                               void* dg, void* du, void* act);
/* out[t][h][:] = rope(in[b][h][p][:]) (t = b*s + p; element strides sb, sp, sh), half
 * rotation with cos/sin [s][hd/2] f32; inverse = 1 rotates by -theta (backward);
 * rotate = 0 performs only the layout change.  out is contiguous [T][H][hd]. */
PLORA_API int plora_rope(void* stream, const void* in, void* out, const float* cosv, const float* sinv,
                         int64_t T, int32_t s, int32_t H, int32_t hd, int64_t sb, int64_t sp, int64_t sh,
                         int32_t rotate, int32_t inverse);
/* Weighted cross entropy over bf16 logits [rows][V] (overwritten with the gradient
 * weight_t * (softmax_t - onehot_t)); tok_loss[t] = weight_t * CE_t. */
PLORA_API int plora_cross_entropy(void* stream, int64_t rows, int64_t V, void* logits,
                                  const int64_t* labels, const float* weight, float* tok_loss);

/* Vocabulary-parallel cross entropy (tensor-parallel lm_head, config C4): logits
 * [rows][V] hold vocabulary slice [v0, v0+V) of each row.
 *   plora_ce_stats : stats[rows][3] = (max_v x, sum_v exp(x - max), x[label] if
 *                    label in the slice else 0); the caller all-reduces these across
 *                    the tensor-parallel group to get lse = M + log(S').
 *   plora_ce_apply : overwrites the slice with weight_t * (exp(x - lse_t) - onehot). */
PLORA_API int plora_ce_stats(void* stream, int64_t rows, int64_t V, const void* logits,
                             const int64_t* labels, int64_t v0, float* stats);
PLORA_API int plora_ce_apply(void* stream, int64_t rows, int64_t V, void* logits,
                             const int64_t* labels, int64_t v0, const float* lse, const float* weight);

/* Tensor-parallel collectives of one packed job (config C4: the base is Megatron-sharded
 * over NVLink; the LoRA-aware all-reduce placement is described in DESIGN.md section 7).
 * NCCL is resolved at run time (dlopen of libnccl.so.2, reusing a copy already loaded in
 * the process).  Rank 0 creates the id, the host distributes it to the group's ranks
 * (any out-of-band channel), every rank calls plora_tp_comm_init.  All-reduce is in
 * place on the caller's stream. */
#define PLORA_TP_ID_BYTES 128
#define PLORA_TP_BF16 0
#define PLORA_TP_F32 1
#define PLORA_TP_SUM 0
#define PLORA_TP_MAX 1
PLORA_API int plora_tp_get_unique_id(char* id_out /* PLORA_TP_ID_BYTES */);
PLORA_API int plora_tp_comm_init(void** comm, const char* id, int32_t nranks, int32_t rank);
PLORA_API int plora_tp_comm_destroy(void* comm);
PLORA_API int plora_tp_allreduce(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t op);
/* Sequence-parallel pieces: recv[nranks * count] = concat of every rank's send[count];
 * recv[recv_count] = sum over ranks of send[rank * recv_count ...]; buf on root = sum. */
PLORA_API int plora_tp_allgather(void* stream, void* comm, const void* send, void* recv, int64_t count,
                                 int32_t dtype);
PLORA_API int plora_tp_reducescatter(void* stream, void* comm, const void* send, void* recv, int64_t recv_count,
                                     int32_t dtype);
PLORA_API int plora_tp_reduce(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t root);
/* buf on every rank = buf on root (in place). */
PLORA_API int plora_tp_broadcast(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t root);

#ifdef __cplusplus
}
#endif

#endif /* PLORA_H_ */
