// meta.cpp -- K8: the segment-index / adapter-metadata builder (host C++).
//
// Restates the offset bookkeeping of the reference's pack_adapters
// (pkg/src/lorasweep/lorapack.py:146-150: rank_offsets / row_offsets are exact
// integer prefix sums) and adds what the sm_100a kernels need on top:
//   * rpad_off  -- prefix sums of roundup(r_i, 16): the adapter-major layout of
//                  fp32 master weights, gradients and Adam moments;
//   * mtiles    -- the grouped-GEMM tile list {m0, m_len, adapter, 0}: 128-row
//                  tiles that never straddle two adapters' token segments, so a
//                  tile's fused LoRA expand uses exactly one adapter's B_i;
//   * ptiles    -- the same rule at 256 rows: tiles of the CTA-pair (cta_group::2) GEMM;
//   * token_adapter -- per-token adapter id (np.repeat(arange(n), diff(row_off))).
// Empty segments (T_i = 0) are legal (reference lorapack.py:90-91) and produce
// no tiles; rank 0 is rejected exactly like AdapterWeights/PackedAdapters do
// (strictly increasing rank offsets, lorapack.py:88-89).
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/plora.h"

namespace plora {
int set_error(const std::string& msg);
}

extern "C" int32_t plora_meta_max_mtiles(int32_t n, const int64_t* tokens) {
  if (n <= 0 || !tokens) return 0;
  int64_t total = 0;
  for (int32_t i = 0; i < n; ++i) total += tokens[i] > 0 ? (tokens[i] + 127) / 128 : 0;
  return total > INT32_MAX ? INT32_MAX : static_cast<int32_t>(total);
}

extern "C" int plora_meta_build(int32_t n, const int64_t* ranks, const int64_t* tokens,
                                int64_t* rank_off, int64_t* row_off, int32_t* rpad_off,
                                int32_t* mtiles, int32_t max_mtiles, int32_t* n_mtiles,
                                int32_t* ptiles, int32_t* n_ptiles, int32_t* token_adapter) {
  if (n <= 0) return plora::set_error("nothing to pack");
  if (!ranks || !tokens || !rank_off || !row_off || !rpad_off || !n_mtiles)
    return plora::set_error("plora_meta_build: NULL argument");
  rank_off[0] = 0;
  row_off[0] = 0;
  rpad_off[0] = 0;
  int64_t tiles = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (ranks[i] < 1) return plora::set_error("rank offsets must be strictly increasing");
    if (tokens[i] < 0) return plora::set_error("row offsets must be non-decreasing");
    rank_off[i + 1] = rank_off[i] + ranks[i];
    row_off[i + 1] = row_off[i] + tokens[i];
    const int64_t rp = (ranks[i] + 15) / 16 * 16;
    if (rpad_off[i] + rp > INT32_MAX) return plora::set_error("packed rank too large");
    rpad_off[i + 1] = static_cast<int32_t>(rpad_off[i] + rp);
    tiles += (tokens[i] + 127) / 128;
  }
  if (row_off[n] > INT32_MAX) return plora::set_error("packed token count exceeds 2^31");
  *n_mtiles = static_cast<int32_t>(tiles);
  if (tiles > max_mtiles) {
    plora::set_error("tile list larger than max_mtiles");
    return 2;
  }
  if (mtiles) {
    int64_t t = 0;
    for (int32_t i = 0; i < n; ++i) {
      for (int64_t m = row_off[i]; m < row_off[i + 1]; m += 128) {
        const int64_t len = row_off[i + 1] - m < 128 ? row_off[i + 1] - m : 128;
        mtiles[4 * t + 0] = static_cast<int32_t>(m);
        mtiles[4 * t + 1] = static_cast<int32_t>(len);
        mtiles[4 * t + 2] = i;
        mtiles[4 * t + 3] = 0;
        ++t;
      }
    }
  }
  int64_t pt = 0;
  for (int32_t i = 0; i < n; ++i) {
    for (int64_t m = row_off[i]; m < row_off[i + 1]; m += 256) {
      if (ptiles) {
        const int64_t len = row_off[i + 1] - m < 256 ? row_off[i + 1] - m : 256;
        ptiles[4 * pt + 0] = static_cast<int32_t>(m);
        ptiles[4 * pt + 1] = static_cast<int32_t>(len);
        ptiles[4 * pt + 2] = i;
        ptiles[4 * pt + 3] = 0;
      }
      ++pt;
    }
  }
  if (n_ptiles) *n_ptiles = static_cast<int32_t>(pt);
  if (token_adapter) {
    for (int32_t i = 0; i < n; ++i)
      for (int64_t r = row_off[i]; r < row_off[i + 1]; ++r) token_adapter[r] = i;
  }
  return 0;
}
