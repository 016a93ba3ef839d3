// Host-side inspector (offline; Sec. 2.3 P:71 "it can be done offline
// at compile time as the sparse weight matrix is fully known").
//
// Steps:
//  a1  CSR ingest + validation
//  a2  row grouping + nnz-balanced row panels: the paper's block-level
//      strategy (b) "assign different number of elements in M to different
//      thread blocks to balance the number of nonzero values" (Fig. 2b).
//      B200 variant: fixed panel height (Mp row slots), variable membership:
//      rows sorted by nnz (desc, stable by id) are LPT-binned into panels, so
//      no accumulator registers are wasted (the drawback named in P:165).
//      Inside a panel the rows are LPT-binned again across the warps (thread
//      groups).
//  a3  split-K groups: each row's nonzeros of a chunk are cut into G_k
//      contiguous k-ascending pieces, "each thread group except the last one
//      processes the same number of non-zeros" (Fig. 3b); the cut is
//      computed on device from the slot offsets, identically for every call.
//  a4  K-chunking + packing: per (panel, chunk) one 16-byte aligned block
//      (see plan.h) staged into shared memory beside its X tile.
//  a5  tile-parameter selection (heuristic; the paper's autotuned parameters
//      M_blocks, N_blocks, Gy).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>

#include "plan.h"
#include "../../include/sparsert.h"

namespace srt {

uint16_t f32_to_f16_rn(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ax = x & 0x7fffffffu;
  if (ax >= 0x7f800000u) {  // inf / nan
    return (uint16_t)(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u : 0u));
  }
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);  // >= 65520 -> inf
  if (ax < 0x33000000u) return (uint16_t)sign;               // < 2^-25 -> 0
  int32_t e = (int32_t)(ax >> 23) - 127;
  uint32_t m = (ax & 0x7fffffu) | 0x800000u;  // 24-bit significand
  int32_t shift;
  uint32_t base;
  if (e < -14) {  // subnormal half: value = m * 2^(e-23); half unit = 2^-24
    shift = -e - 14 + 13;  // bits to drop
    base = 0;
  } else {
    shift = 13;
    base = (uint32_t)(e + 15) << 10;
    m &= 0x7fffffu;
  }
  uint32_t q = m >> shift;
  const uint32_t rem = m & ((1u << shift) - 1u);
  const uint32_t half = 1u << (shift - 1);
  if (rem > half || (rem == half && (q & 1u))) q += 1;
  return (uint16_t)(sign | (base + q));  // carry into exponent is correct IEEE behaviour
}

float f16_to_f32(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ffu;
  float f;
  if (e == 0) {
    f = std::ldexp((float)m, -24);
  } else if (e == 31) {
    f = m ? NAN : INFINITY;
  } else {
    f = std::ldexp((float)(m | 0x400u), (int)e - 25);
  }
  uint32_t x;
  std::memcpy(&x, &f, 4);
  x |= sign;
  std::memcpy(&f, &x, 4);
  return f;
}

static uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
  const uint8_t* p = (const uint8_t*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

static int pow2_ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

static int64_t align16(int64_t v) { return (v + 15) & ~int64_t(15); }

// fp32 -> nearest TF32 value (10 explicit mantissa bits, round to nearest even), kept in an
// fp32 container with the low 13 bits zero (finite inputs; the 3xTF32 split W = hi + lo)
static float tf32_rn(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0xfffu + ((u >> 13) & 1u);
  u &= 0xffffe000u;
  std::memcpy(&f, &u, 4);
  return f;
}

namespace {
struct Entry {
  int32_t k;
  float w;
  uint16_t wh;
};
}  // namespace

int build_plan(Plan& p, int32_t M, int32_t K, int64_t nnz, const int32_t* row_ptr,
               const int32_t* col_idx, const float* values, int32_t dtype,
               const BuildOpts& o, std::string& err) {
  const auto t0 = std::chrono::steady_clock::now();
  char buf[256];
  if (M < 1 || K < 1 || nnz < 0) {
    err = "M and K must be >= 1 and nnz >= 0";
    return SPARSE_EINVAL;
  }
  if (dtype != SPARSE_F32 && dtype != SPARSE_F16 && dtype != SPARSE_BF16) {
    err = "dtype must be SPARSE_F32, SPARSE_F16 or SPARSE_BF16";
    return SPARSE_EINVAL;
  }
  if (dtype == SPARSE_BF16 && (o.executor == 1 || o.tm)) {
    err = "bf16 plans: no JIT executor / TMEM X source";
    return SPARSE_EUNSUPPORTED;
  }
  if (o.kind != SPARSE_SPMM && o.kind != SPARSE_CONV3X3) {
    err = "kind must be SPARSE_SPMM or SPARSE_CONV3X3";
    return SPARSE_EINVAL;
  }
  if (!row_ptr || (nnz > 0 && (!col_idx || !values))) {
    err = "null CSR array";
    return SPARSE_EINVAL;
  }
  if (K > 65535) {
    err = "K > 65535 is not supported";
    return SPARSE_EUNSUPPORTED;
  }
  if (nnz > (int64_t)INT32_MAX) {
    err = "nnz exceeds int32 range";
    return SPARSE_EUNSUPPORTED;
  }
  if (o.kind == SPARSE_CONV3X3) {
    if (o.c_in < 1 || o.h < 1 || o.w < 1) {
      err = "conv plan needs c_in, h, w >= 1";
      return SPARSE_EINVAL;
    }
    if ((int64_t)K != 9 * (int64_t)o.c_in) {
      snprintf(buf, sizeof buf, "conv plan: K (%d) != 9*c_in (%d)", K, 9 * o.c_in);
      err = buf;
      return SPARSE_EUNSUPPORTED;
    }
  }

  // ---------------- a1: validation ----------------
  if (row_ptr[0] != 0) {
    err = "row 0: row_ptr[0] != 0";
    return SPARSE_EMATRIX;
  }
  for (int32_t m = 0; m < M; ++m) {
    if (row_ptr[m + 1] < row_ptr[m]) {
      snprintf(buf, sizeof buf, "row %d: row_ptr not monotone (%d > %d)", m, row_ptr[m],
               row_ptr[m + 1]);
      err = buf;
      return SPARSE_EMATRIX;
    }
  }
  if ((int64_t)row_ptr[M] != nnz) {
    snprintf(buf, sizeof buf, "row %d: row_ptr[M] (%d) != nnz (%lld)", M, row_ptr[M],
             (long long)nnz);
    err = buf;
    return SPARSE_EMATRIX;
  }
  std::vector<std::vector<Entry>> rows(M);
  int64_t kept = 0;
  for (int32_t m = 0; m < M; ++m) {
    int32_t prev = -1;
    for (int32_t e = row_ptr[m]; e < row_ptr[m + 1]; ++e) {
      const int32_t k = col_idx[e];
      const float v = values[e];
      if (k < 0 || k >= K) {
        snprintf(buf, sizeof buf, "row %d: col_idx %d out of [0,%d) at %d", m, k, K,
                 e - row_ptr[m]);
        err = buf;
        return SPARSE_EMATRIX;
      }
      if (k <= prev) {
        snprintf(buf, sizeof buf, "row %d: col_idx not strictly increasing at %d", m,
                 e - row_ptr[m]);
        err = buf;
        return SPARSE_EMATRIX;
      }
      prev = k;
      if (!std::isfinite(v)) {
        snprintf(buf, sizeof buf, "row %d: non-finite value at %d", m, e - row_ptr[m]);
        err = buf;
        return SPARSE_EMATRIX;
      }
      uint16_t wh = 0;
      float wv = v;
      if (dtype == SPARSE_F16) {
        wh = f32_to_f16_rn(v);
        if ((wh & 0x7c00u) == 0x7c00u) {
          snprintf(buf, sizeof buf, "row %d: value %g overflows fp16 at %d", m, (double)v,
                   e - row_ptr[m]);
          err = buf;
          return SPARSE_EMATRIX;
        }
        wv = f16_to_f32(wh);
      } else if (dtype == SPARSE_BF16) {
        uint32_t u;
        std::memcpy(&u, &v, 4);
        u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even (v finite)
        wh = (uint16_t)(u >> 16);
        if ((wh & 0x7f80u) == 0x7f80u) {
          snprintf(buf, sizeof buf, "row %d: value %g overflows bf16 at %d", m, (double)v,
                   e - row_ptr[m]);
          err = buf;
          return SPARSE_EMATRIX;
        }
        const uint32_t b = (uint32_t)wh << 16;
        std::memcpy(&wv, &b, 4);
      }
      if (wv == 0.0f) {
        if (o.drop_zeros) continue;
        snprintf(buf, sizeof buf, "row %d: explicit zero%s at %d", m,
                 v != 0.0f ? " (after fp16 rounding)" : "", e - row_ptr[m]);
        err = buf;
        return SPARSE_EMATRIX;
      }
      rows[m].push_back(Entry{k, wv, wh});
      ++kept;
    }
  }

  // ---------------- tensor-core sub-blocks (NEXT #1): fp16 SpMM plans only ----------------
  // Aligned 16 x 16 tiles of W holding >= tc_min_pct % nonzeros are dense enough to be a
  // real dense contraction: their nonzeros leave the CUDA-core rows and are packed as dense
  // fp16 tiles in mma.m16n8k16 A-fragment order (lane l = 4 g + t holds rows g, g + 8 and
  // columns 2t, 2t + 1, 2t + 8, 2t + 9).
  std::vector<int32_t> tc_rb, tc_tile_begin, tc_cb, ws_row;
  std::vector<uint16_t> tc_a;
  int64_t tc_nnz = 0;
  // (not with the JIT executor, which bakes every nonzero into its code)
  const int tc_pct = (dtype == SPARSE_F16 && o.kind == SPARSE_SPMM && o.executor != 1 && o.executor != 3 && o.executor != 4 && !o.ps) ? o.tc_min_pct : 0;
  if (tc_pct < 0 || tc_pct > 100) {
    err = "tc_min_density must be in [0, 100] (percent)";
    return SPARSE_EINVAL;
  }
  const int64_t nrb = (M + 15) / 16, ncb = (K + 15) / 16;
  if (tc_pct > 0 && nrb * ncb <= (int64_t)1 << 26) {
    const int thr = std::max(1, (tc_pct * 256 + 99) / 100);
    std::vector<uint16_t> cnt((size_t)(nrb * ncb), 0);
    for (int32_t m = 0; m < M; ++m)
      for (const Entry& en : rows[m]) cnt[(size_t)((m / 16) * ncb + en.k / 16)]++;
    ws_row.assign(M, -1);
    for (int64_t rb = 0; rb < nrb; ++rb) {
      bool any = false;
      for (int64_t cb = 0; cb < ncb; ++cb) {
        if (cnt[(size_t)(rb * ncb + cb)] < thr) continue;
        if (!any) {
          tc_rb.push_back((int32_t)rb);
          tc_tile_begin.push_back((int32_t)tc_cb.size());
          any = true;
        }
        tc_cb.push_back((int32_t)cb);
        tc_a.resize(tc_a.size() + 256, 0);
      }
    }
    tc_tile_begin.push_back((int32_t)tc_cb.size());
    if (!tc_cb.empty()) {
      // dense tile index of (rb, cb), -1 if not dense
      std::vector<int32_t> tile_of((size_t)(nrb * ncb), -1);
      for (size_t i = 0; i + 1 < tc_tile_begin.size(); ++i)
        for (int32_t t = tc_tile_begin[i]; t < tc_tile_begin[i + 1]; ++t)
          tile_of[(size_t)(tc_rb[i] * ncb + tc_cb[t])] = t;
      for (size_t i = 0; i < tc_rb.size(); ++i)
        for (int r = 0; r < 16 && tc_rb[i] * 16 + r < M; ++r) ws_row[tc_rb[i] * 16 + r] = (int32_t)(i * 16 + r);
      for (int32_t m = 0; m < M; ++m) {
        std::vector<Entry> keep;
        keep.reserve(rows[m].size());
        for (const Entry& en : rows[m]) {
          const int32_t t = tile_of[(size_t)((m / 16) * ncb + en.k / 16)];
          if (t < 0) {
            keep.push_back(en);
            continue;
          }
          const int r = m % 16, c = en.k % 16;
          const int g = r % 8, hi_r = r / 8, tq = (c % 8) / 2, hi_c = c / 8, lo = c % 2;
          const int lane = 4 * g + tq;
          const int slot = hi_c * 4 + hi_r * 2 + lo;  // a0..a7
          tc_a[(size_t)t * 256 + lane * 8 + slot] = en.wh;
          ++tc_nnz;
        }
        rows[m].swap(keep);
      }
    }
  }

  p = Plan();
  p.M = M;
  p.K = K;
  p.dtype = dtype;
  p.kind = o.kind;
  p.nnz = kept;
  p.tc_min_pct = tc_pct;
  p.tc_nrb = (int32_t)tc_rb.size();
  p.tc_ntiles = (int64_t)tc_cb.size();
  p.tc_nnz = tc_nnz;
  if (p.tc_ntiles > 0) {
    p.tc_rb.swap(tc_rb);
    p.tc_tile_begin.swap(tc_tile_begin);
    p.tc_cb.swap(tc_cb);
    p.tc_a.swap(tc_a);
    p.ws_row.swap(ws_row);
  }
  p.n_hint = o.n_hint;
  const bool f16 = dtype != SPARSE_F32;  // 16-bit storage (fp16 or bf16)
  const int S = f16 ? 2 : 4;
  p.entry_bytes = f16 ? 4 : 8;

  // ---------------- a5: tile parameters ----------------
  const int kTargetCtas = 2 * 148;  // >= 2 waves on 148 SMs
  p.entry_align = 16 / p.entry_bytes;
  if (o.kind == SPARSE_SPMM) {
    p.C = f16 ? 8 : 4;  // 16 bytes of X per lane -> one 128-bit shared load
    int gk = 1;
    if (o.split_k) {
      gk = o.split_k;
    } else if (o.n_hint > 0 && !o.ps) {  // (the parameter-plan kernel has no split-K groups)
      int L = pow2_ceil((int)((o.n_hint + p.C - 1) / p.C));
      L = std::max(4, std::min(32, L));
      gk = 32 / L;
    }
    if (gk != 1 && gk != 2 && gk != 4 && gk != 8) {
      err = "split_k must be 1, 2, 4 or 8";
      return SPARSE_EUNSUPPORTED;
    }
    p.gk = gk;
    p.n_tile = (32 / gk) * p.C;
    if (o.tm != 0 && o.tm != 1) {
      err = "x_source must be 0 (shared memory) or 1 (tensor memory)";
      return SPARSE_EINVAL;
    }
    if (o.tm && (gk != 1 || o.k_chunk > 56)) {
      err = "x_source = 1 (tensor memory) needs split_k = 1 and k_chunk <= 56";
      return SPARSE_EUNSUPPORTED;
    }
    if (o.k_chunk) {
      if (o.k_chunk % 8 || o.k_chunk < 8 || o.k_chunk > 256) {
        err = "k_chunk must be a multiple of 8 in [8, 256]";
        return SPARSE_EUNSUPPORTED;
      }
      p.kc = o.k_chunk;
    } else {
      // 128 rows per stage (fewer, larger chunks measured fastest on B200);
      // tensor memory: 56 (two 256-column buffers of kc rows + a zero row each)
      p.kc = o.tm ? 56 : 128;
      if (K <= p.kc) p.kc = (K + 7) / 8 * 8;
    }
    p.nchunks = (K + p.kc - 1) / p.kc;
    // kc X rows plus one zero row (target of the neutral padding entries), 128-byte aligned
    p.x_stage_bytes = (int)(((int64_t)(p.kc + 1) * p.n_tile * S + 127) & ~int64_t(127));
  } else {
    // implicit im2col conv: padded-position tiles
    p.c_in = o.c_in;
    p.h = o.h;
    p.w = o.w;
    p.gk = 1;
    const int wp = o.w + 2;
    p.conv_wp = wp;
    const int kMaxPos = 256;  // 32 lanes x up to 8 positions
    if (o.h * wp <= kMaxPos) {
      p.conv_rb = o.h;
      int ipt = std::max(1, kMaxPos / (o.h * wp));
      if (o.n_hint > 0) ipt = (int)std::min<int64_t>(ipt, o.n_hint);
      p.conv_ipt = ipt;
    } else {
      int rb = 0;
      for (int d = 1; d <= o.h; ++d)
        if (o.h % d == 0 && d * wp <= kMaxPos) rb = d;
      if (rb == 0) {
        snprintf(buf, sizeof buf, "conv: image width %d too large (W+2 > %d)", o.w, kMaxPos);
        err = buf;
        return SPARSE_EUNSUPPORTED;
      }
      p.conv_rb = rb;
      p.conv_ipt = 1;
    }
    p.n_tile = p.conv_ipt * p.conv_rb * wp;
    {
      const int cp = (p.n_tile + 31) / 32;  // positions per lane, instantiated as 2, 4, 7 or 8
      p.C = cp <= 2 ? 2 : cp <= 4 ? 4 : cp <= 7 ? 7 : 8;
    }
    p.conv_simg = (p.conv_rb + 2) * wp;
    p.conv_sci = p.conv_ipt * p.conv_simg;
    p.conv_guard = wp + 1;
    int cc = o.k_chunk;
    if (cc) {
      if (cc < 1 || cc > 64) {
        err = "conv k_chunk (channels per stage) must be in [1, 64]";
        return SPARSE_EUNSUPPORTED;
      }
    } else {
      cc = std::max(1, std::min(o.c_in, (f16 ? 8192 : 4096) / p.conv_sci));
      cc = std::min(cc, 64);
    }
    if ((int64_t)cc * p.conv_sci + 2 * p.conv_guard > 32000)
      cc = std::max(1, (32000 - 2 * p.conv_guard) / p.conv_sci);
    p.cc = cc;
    p.kc = 9 * cc;
    p.nchunks = (o.c_in + cc - 1) / cc;
    p.conv_stage_elems = cc * p.conv_sci + 2 * p.conv_guard;
    p.x_stage_bytes = (int)align16((int64_t)p.conv_stage_elems * S);
    // Vectorised variant (conv3x3_vec_kernel) when a padded row fits twice in a warp's
    // positions: lane owns C consecutive output positions (16 bytes), rows padded to wp
    // (a multiple of C), and the staged input is kept as three copies shifted by dx - 1 so
    // every tap is one aligned 128-bit shared load; entries use the SpMM unit format.
    {
      const int Cv = f16 ? 8 : 4, NTv = 32 * Cv;
      const int wpv = (o.w + 2 + Cv - 1) / Cv * Cv;
      if (o.conv_vec && 2 * wpv <= NTv) {
        const int threads = 32 * (o.warps ? o.warps : 16);
        p.conv_vec = 1;
        p.C = Cv;
        p.n_tile = NTv;
        p.conv_wp = wpv;
        p.conv_rb = std::min(o.h, NTv / wpv);
        p.conv_ipt = 1;
        p.conv_guard = 8;
        p.conv_sci = (p.conv_guard + (p.conv_rb + 2) * wpv + 8 + 7) / 8 * 8;  // per channel
        const int per_ch = 3 * p.conv_sci * S;
        int ccv = o.k_chunk ? o.k_chunk : std::max(1, std::min(o.c_in, (48 * 1024) / per_ch));
        // register-staged fill: at most 8 input elements per thread and chunk
        ccv = std::max(1, std::min(ccv, 8 * threads / ((p.conv_rb + 2) * o.w)));
        ccv = std::min(ccv, 64);
        p.cc = ccv;
        p.kc = 9 * ccv;
        p.nchunks = (o.c_in + ccv - 1) / ccv;
        p.conv_cs = ccv * p.conv_sci;  // elements per shifted copy
        p.conv_stage_elems = 3 * p.conv_cs + NTv + 16;  // + zero block
        p.x_stage_bytes = (int)align16((int64_t)p.conv_stage_elems * S);
        // interleaved kernel (conv3x3_il_kernel): 4 positions per lane, 128 per tile; il_g images
        // interleaved per row so that a tap shift (dy - 1) P keeps a lane's vector aligned
        // (P % 4 == 0); the tile's span starts 16-byte aligned, up to 16 / S - 4 elements early
        int ilg = 0;
        for (int gg = 1; gg <= 8 && !ilg; ++gg)  // (and whole 16-byte group blocks in the copies)
          if ((gg * o.w) % 4 == 0 && ((int64_t)(o.h + 2) * gg * o.w * S) % 16 == 0) ilg = gg;
        int illc = 0;
        if (ilg) {
          const int P = ilg * o.w, HP = o.h * P;
          const int nb = (127 + HP - 1) / HP;  // group boundaries inside a 128-position tile
          illc = P + 127 + nb * 2 * P + P + 4 + (16 / S - 4);
          illc = (illc + 15) / 16 * 16;
        }
        if (o.conv_vec == 4 && (!ilg || illc > 256)) {
          err = "interleaved conv (conv_kernel 4): image too wide for one 256-element TMA span";
          return SPARSE_EUNSUPPORTED;
        }
        if (o.conv_vec == 4) {
          p.conv_vec = 4;
          p.C = 4;
          p.n_tile = 128;
          p.conv_rb = 0;
          p.conv_ipt = 0;
          p.conv_wp = ilg * o.w;
          p.conv_guard = 0;
          p.il_g = ilg;
          p.il_lc = illc;
          const int per_ch = 3 * illc * S;
          int cci = o.k_chunk ? o.k_chunk : std::max(1, std::min(o.c_in, (64 * 1024) / per_ch));
          cci = std::min(cci, 64);
          p.cc = cci;
          p.kc = 9 * cci;
          p.nchunks = (o.c_in + cci - 1) / cci;
          p.conv_cs = (int)(((int64_t)cci * illc * S + 127) / 128 * 128 / S);  // 128-byte aligned copies
          p.conv_sci = illc;
          p.conv_stage_elems = 3 * p.conv_cs + illc;  // + the zero block
          p.x_stage_bytes = (int)(((int64_t)p.conv_stage_elems * S + 127) & ~int64_t(127));
        } else if (o.conv_vec == 2 && wpv <= 64) {  // (pad_conv_input holds a padded row in registers)
          // TMA-fed variant (conv3x3_tma_kernel): each shifted copy is one 4-D TMA box
          // {wp, rb + 2, 1 image, cc channels} of the width-padded input (no guard), at a
          // 128-byte aligned offset; no register staging, so up to 64 channels per chunk
          p.conv_vec = 2;
          p.conv_guard = 0;
          p.conv_sci = (p.conv_rb + 2) * wpv;
          const int per_ch3 = 3 * p.conv_sci * S;
          int cct = o.k_chunk ? o.k_chunk : std::max(1, std::min(o.c_in, (64 * 1024) / per_ch3));
          cct = std::min(cct, 64);
          p.cc = cct;
          p.kc = 9 * cct;
          p.nchunks = (o.c_in + cct - 1) / cct;
          p.conv_cs = (int)((int64_t)cct * p.conv_sci * S + 127) / 128 * 128 / S;
          p.conv_stage_elems = 3 * p.conv_cs + NTv + 16;
          p.x_stage_bytes = (int)(((int64_t)p.conv_stage_elems * S + 127) & ~int64_t(127));
        }
      }
    }
  }
  if (dtype == SPARSE_BF16 && o.kind == SPARSE_CONV3X3 && p.conv_vec != 2 && p.conv_vec != 4) {
    err = "bf16 conv plans need the TMA-fed or packed conv kernel (conv_kernel 0, 2 or 4)";
    return SPARSE_EUNSUPPORTED;
  }
  p.warps = o.warps ? o.warps : (o.kind == SPARSE_SPMM || p.conv_vec ? 16 : 8);
  if (p.warps < 1 || p.warps > kMaxWarps) {
    err = "warps must be in [1, 16]";
    return SPARSE_EUNSUPPORTED;
  }
  {
    int64_t ntiles;
    if (o.kind == SPARSE_SPMM) {
      const int64_t nh = o.n_hint > 0 ? o.n_hint : 4096;
      ntiles = (nh + p.n_tile - 1) / p.n_tile;
    } else {
      const int64_t nb = o.n_hint > 0 ? o.n_hint : 64;
      ntiles = p.conv_vec == 4 ? (nb * o.h * o.w + p.n_tile - 1) / p.n_tile
                               : ((nb + p.conv_ipt - 1) / p.conv_ipt) * (o.h / p.conv_rb);
    }
    // accumulators per thread: R * C fp32 registers; keep <= 64
    // R = 4 rows per warp x 8 warps: Mp = 32 rows; measured best on B200 for both dtypes
    // (R = 8 halves occupancy through registers, scripts/sweep.py)
    // SpMM executors are persistent: one wave of 148 CTAs is the target
    const int rmax = 4;
    const int max_ks = o.kind == SPARSE_SPMM ? std::min(4, p.nchunks) : 1;
    const int64_t target = o.kind == SPARSE_SPMM ? 148 : kTargetCtas;
    int bestR = 1, bestKs = 1;
    bool found = false;
    for (int R = rmax; R >= 1 && !found; R /= 2) {
      const int64_t panels = (M + (int64_t)p.warps * R - 1) / ((int64_t)p.warps * R);
      for (int ks = 1; ks <= max_ks; ks *= 2) {
        if (panels * ntiles * ks >= target) {
          bestR = R;
          bestKs = ks;
          found = true;
          break;
        }
      }
    }
    if (!found) {  // not enough work for two waves: maximise CTAs
      bestR = 1;
      bestKs = 1;
      while (bestKs * 2 <= max_ks) bestKs *= 2;
    }
    p.R = o.rows_per_warp ? o.rows_per_warp : bestR;
    p.ks = o.k_split ? o.k_split : (o.rows_per_warp || o.ps ? 1 : bestKs);
  }
  if (p.R != 1 && p.R != 2 && p.R != 4 && p.R != 8 && p.R != 16) {
    err = "rows_per_warp must be 1, 2, 4, 8 or 16";
    return SPARSE_EUNSUPPORTED;
  }
  if (p.conv_vec && p.R > 8) {
    err = "rows_per_warp must be <= 8 for the vectorised conv kernels";
    return SPARSE_EUNSUPPORTED;
  }
  if (p.R * p.C > 128) {
    err = "rows_per_warp too large for this dtype (accumulator registers)";
    return SPARSE_EUNSUPPORTED;
  }
  if (o.executor == 4) {
    // tcgen05 block executor: k_split = K slices per tile, partial sums reduced in slice order by
    // a second kernel (small-N layers: few tiles for 148 SMs); the CUDA-core part keeps 1
    p.tcg_ks = o.k_split ? o.k_split : 1;
    p.ks = 1;
    if (p.tcg_ks != 1 && p.tcg_ks != 2 && p.tcg_ks != 4 && p.tcg_ks != 8 && p.tcg_ks != 16) {
      err = "k_split must be 1, 2, 4, 8 or 16 for the tcgen05 block executor";
      return SPARSE_EUNSUPPORTED;
    }
    if (p.tcg_ks > 1 && o.kind != SPARSE_SPMM) {
      err = "k_split is only supported for SpMM plans";
      return SPARSE_EUNSUPPORTED;
    }
  }
  if (p.ks != 1 && p.ks != 2 && p.ks != 4 && p.ks != 8) {
    err = "k_split must be 1, 2, 4 or 8";
    return SPARSE_EUNSUPPORTED;
  }
  if (p.ks > 1 && o.kind != SPARSE_SPMM) {
    err = "k_split is only supported for SpMM plans";
    return SPARSE_EUNSUPPORTED;
  }
  if (p.ks > p.nchunks) p.ks = 1 << (31 - __builtin_clz((unsigned)p.nchunks));
  p.cm = o.cm ? o.cm : 1;
  if (p.cm != 1 && p.cm != 2 && p.cm != 4 && p.cm != 8) {
    err = "x_multicast must be 1, 2, 4 or 8";
    return SPARSE_EUNSUPPORTED;
  }
  if (o.executor == 4) {
    // the tcgen05 block executor's own cluster (row blocks sharing each X tile); the CUDA-core
    // part of the plan (conv plans keep one) does not multicast
    if (p.cm > 4) {
      err = "x_multicast must be 1, 2 or 4 for the tcgen05 block executor";
      return SPARSE_EUNSUPPORTED;
    }
    if (o.pair && p.cm > 2) {
      err = "cta_pair = 1 needs x_multicast 0, 1 or 2 (the CTA pair is the cluster)";
      return SPARSE_EUNSUPPORTED;
    }
    p.tcg_pair = o.pair ? 1 : 0;
    p.tcg_cs = o.pair ? 2 : p.cm;
    p.cm = 1;
  } else if (o.pair) {
    err = "cta_pair = 1 needs the tcgen05 block executor (executor 4 / conv_kernel 5)";
    return SPARSE_EUNSUPPORTED;
  }
  if (p.cm > 1 && (o.kind != SPARSE_SPMM || p.ks > 1)) {
    err = "x_multicast > 1 needs an SpMM plan with k_split = 1";
    return SPARSE_EUNSUPPORTED;
  }
  p.tm = o.kind == SPARSE_SPMM ? o.tm : 0;
  if (p.tm && (p.ks > 1 || p.cm > 1 || p.R > 8 || p.warps % 4)) {
    err = "x_source = 1 (tensor memory) needs k_split = 1, x_multicast = 1, rows_per_warp <= 8 "
          "and warps a multiple of 4";
    return SPARSE_EUNSUPPORTED;
  }
  p.Mp = p.warps * p.R;
  p.npanels = (M + p.Mp - 1) / p.Mp;
  // a multicast cluster takes cm consecutive panels: pad with empty panels (no rows)
  p.npanels = (p.npanels + p.cm - 1) / p.cm * p.cm;

  // ---------------- a2: row grouping + LPT panels ----------------
  std::vector<int32_t> order(M);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return rows[a].size() > rows[b].size();
  });
  // min-heap over (panel nnz, panel id) among panels with free slots
  using PI = std::pair<int64_t, int32_t>;
  std::priority_queue<PI, std::vector<PI>, std::greater<PI>> heap;
  for (int32_t q = 0; q < p.npanels; ++q) heap.push({0, q});
  std::vector<std::vector<int32_t>> panel_rows(p.npanels);
  std::vector<int64_t> panel_nnz(p.npanels, 0);
  p.row_order = o.row_order;
  if (o.row_order == 1) {
    // ablation ("without load balancing"): panel q takes rows q*Mp .. q*Mp+Mp-1 and
    // warp w of it the slots w*R .. w*R+R-1, in natural row order
    for (int32_t m = 0; m < M; ++m) {
      panel_rows[m / p.Mp].push_back(m);
      panel_nnz[m / p.Mp] += (int64_t)rows[m].size();
    }
  } else {
    for (int32_t m : order) {
      PI top = heap.top();
      heap.pop();
      const int32_t q = top.second;
      panel_rows[q].push_back(m);
      panel_nnz[q] += (int64_t)rows[m].size();
      if ((int)panel_rows[q].size() < p.Mp) heap.push({panel_nnz[q], q});
    }
  }
  p.max_panel_nnz = *std::max_element(panel_nnz.begin(), panel_nnz.end());
  p.min_panel_nnz = *std::min_element(panel_nnz.begin(), panel_nnz.end());

  // within a panel: LPT across warps (R slots each)
  p.row_id.assign((size_t)p.npanels * p.Mp, -1);
  for (int32_t q = 0; o.row_order == 1 && q < p.npanels; ++q)
    for (size_t i = 0; i < panel_rows[q].size(); ++i) p.row_id[(size_t)q * p.Mp + i] = panel_rows[q][i];
  for (int32_t q = 0; o.row_order != 1 && q < p.npanels; ++q) {
    std::vector<int64_t> wl(p.warps, 0);
    std::vector<int> wfill(p.warps, 0);
    for (int32_t m : panel_rows[q]) {  // already in descending nnz order
      int best = -1;
      for (int wi = 0; wi < p.warps; ++wi) {
        if (wfill[wi] >= p.R) continue;
        if (best < 0 || wl[wi] < wl[best]) best = wi;
      }
      p.row_id[(size_t)q * p.Mp + best * p.R + wfill[best]] = m;
      wfill[best]++;
      wl[best] += (int64_t)rows[m].size();
    }
  }

  // ---------------- a4: chunking + packing ----------------
  // (block layouts in plan.h)
  const int A = p.entry_align;
  const bool units = o.kind == SPARSE_SPMM || p.conv_vec;  // SpMM unit format (plan.h)
  const int G = o.kind == SPARSE_SPMM ? p.gk : 1;
  const int hdr = (int)align16((int64_t)p.Mp * G * 4);
  p.hdr_bytes = hdr;
  p.blk_off.assign((size_t)p.npanels * p.nchunks + 1, 0);
  p.blob.clear();
  p.blob.reserve((size_t)(kept * p.entry_bytes +
                          (int64_t)p.npanels * p.nchunks * (hdr + 16 + p.Mp * G * 16)));
  std::vector<int32_t> cursor(M, 0);
  std::vector<uint32_t> shdr((size_t)p.Mp * G);
  std::vector<uint8_t> ents;
  // element offset of K row kl inside the staged tile (SpMM: X row kl; vectorised conv: tap
  // (ci, dy, dx) = shifted copy dx, channel plane ci, row dy; kl == kc: the zero row/block)
  auto elem_off = [&](int32_t kl) -> int64_t {
    if (o.kind == SPARSE_SPMM) return (int64_t)kl * p.n_tile;
    if (p.conv_vec == 4) {  // interleaved: copy dx, channel ci, tap row dy (biased by one pitch)
      if (kl == p.kc) return 3 * (int64_t)p.conv_cs + p.conv_wp;
      const int ci = kl / 9, t = kl % 9, dy = t / 3, dx = t % 3;
      return (int64_t)dx * p.conv_cs + (int64_t)ci * p.il_lc + (int64_t)dy * p.conv_wp;
    }
    if (kl == p.kc) return 3 * (int64_t)p.conv_cs;
    const int ci = kl / 9, t = kl % 9, dy = t / 3, dx = t % 3;
    return (int64_t)dx * p.conv_cs + (int64_t)ci * p.conv_sci + (int64_t)dy * p.conv_wp;
  };
  auto put_spmm = [&](int32_t kl, float w, uint16_t wh) {
    uint8_t rec[8];
    if (f16) {
      const uint16_t o16 = (uint16_t)(elem_off(kl) * 2 / (p.conv_vec == 4 ? 8 : 16));
      std::memcpy(rec, &o16, 2);
      std::memcpy(rec + 2, &wh, 2);
    } else {
      const uint32_t o32 = (uint32_t)(elem_off(kl) * 4);
      std::memcpy(rec, &o32, 4);
      std::memcpy(rec + 4, &w, 4);
    }
    ents.insert(ents.end(), rec, rec + p.entry_bytes);
  };
  int64_t maxblk = 0;
  for (int32_t q = 0; q < p.npanels; ++q) {
    for (int32_t m : panel_rows[q]) cursor[m] = 0;
    for (int32_t c = 0; c < p.nchunks; ++c) {
      const int32_t k0 = c * p.kc, k1 = std::min(K, k0 + p.kc);
      ents.clear();
      int32_t cnt = 0;  // entries (conv) / units (SpMM) so far
      for (int s = 0; s < p.Mp; ++s) {
        const int32_t m = p.row_id[(size_t)q * p.Mp + s];
        int32_t e0 = 0, e1 = 0;  // this row's entries in [k0, k1): rows[m][e0, e1)
        if (m >= 0) {
          int32_t& cur = cursor[m];
          e0 = cur;
          while (cur < (int32_t)rows[m].size() && rows[m][cur].k < k1) ++cur;
          e1 = cur;
        }
        if (units) {
          // G contiguous k-ascending pieces, all but the last of `per` entries
          const int32_t n = e1 - e0;
          int32_t per = (n + G - 1) / G;
          per = (per + A - 1) / A * A;
          for (int g = 0; g < G; ++g) {
            const int32_t lo = std::min(g * per, n), hi = std::min(lo + per, n);
            const int32_t units = (hi - lo + A - 1) / A;
            for (int32_t e = e0 + lo; e < e0 + hi; ++e)
              put_spmm(rows[m][e].k - k0, rows[m][e].w, rows[m][e].wh);
            for (int32_t e = hi - lo; e < units * A; ++e)  // neutral: -0 * (zero row)
              put_spmm(p.kc, -0.0f, (uint16_t)0x8000u);
            if (cnt > 65535 || units > 65535) {
              err = "internal: block unit count overflow (lower k_chunk)";
              return SPARSE_EUNSUPPORTED;
            }
            shdr[(size_t)s * G + g] = (uint32_t)cnt | ((uint32_t)units << 16);
            cnt += units;
          }
        } else {
          while (cnt % A) {  // align the slot's first entry
            ents.insert(ents.end(), (size_t)p.entry_bytes, (uint8_t)0);
            ++cnt;
          }
          const int32_t start = cnt;
          for (int32_t e = e0; e < e1; ++e) {
            const Entry& en = rows[m][e];
            const int32_t kl = en.k - k0;
            const int ci = kl / 9, t = kl % 9, dy = t / 3, dx = t % 3;
            const int32_t off = ci * p.conv_sci + (dy - 1) * p.conv_wp + (dx - 1);
            uint8_t rec[8];
            if (f16) {
              const int16_t o16 = (int16_t)off;
              std::memcpy(rec, &o16, 2);
              std::memcpy(rec + 2, &en.wh, 2);
            } else {
              std::memcpy(rec, &off, 4);
              std::memcpy(rec + 4, &en.w, 4);
            }
            ents.insert(ents.end(), rec, rec + p.entry_bytes);
            ++cnt;
          }
          if (cnt > 65535) {
            err = "internal: block entry count overflow (lower k_chunk)";
            return SPARSE_EUNSUPPORTED;
          }
          shdr[s] = (uint32_t)start | ((uint32_t)(cnt - start) << 16);
        }
      }
      const size_t st = p.blob.size();
      p.blk_off[(size_t)q * p.nchunks + c] = (int64_t)st;
      p.blob.resize(st + hdr, 0);
      std::memcpy(p.blob.data() + st, shdr.data(), (size_t)p.Mp * G * 4);
      p.blob.insert(p.blob.end(), ents.begin(), ents.end());
      p.blob.resize((size_t)align16((int64_t)p.blob.size()), 0);
      maxblk = std::max<int64_t>(maxblk, (int64_t)(p.blob.size() - st));
    }
  }
  p.blk_off[(size_t)p.npanels * p.nchunks] = (int64_t)p.blob.size();
  if (p.blob.empty()) p.blob.resize(16, 0);
  p.max_blk_bytes = (int32_t)maxblk;
  if (o.kind == SPARSE_SPMM) {
    // fixed block stride: block bi lives at bi * max_blk_bytes, so the executor computes a
    // chunk's plan address without a dependent global load on its pipeline refill path
    const int64_t nb = (int64_t)p.npanels * p.nchunks;
    std::vector<uint8_t> fixed((size_t)std::max<int64_t>(16, nb * maxblk), 0);
    for (int64_t bi = 0; bi < nb; ++bi)
      std::memcpy(fixed.data() + bi * maxblk, p.blob.data() + p.blk_off[bi],
                  (size_t)(p.blk_off[bi + 1] - p.blk_off[bi]));
    for (int64_t bi = 0; bi <= nb; ++bi) p.blk_off[bi] = bi * maxblk;
    p.blob.swap(fixed);
  }

  // pipeline depth and shared memory
  int stage_bytes = p.x_stage_bytes + p.max_blk_bytes;
  if (o.kind == SPARSE_SPMM) {
    stage_bytes = (stage_bytes + 127) & ~127;  // TMA destinations 128-byte aligned
    // k_split == 1: persistent CTAs, the ring runs across tiles; k_split > 1: one tile
    // per CTA, no point in more stages than chunks
    const int per_chunks = (p.nchunks + p.ks - 1) / p.ks;
    // default depth (stages = 0, or -1 from the tuner): as many stages as fit in ~200 KB
    // (one CTA per SM, the deepest X pipeline); stages = -2 (tuner): ~100 KB, two CTAs per
    // SM.  At least 2 (1 if a single stage needs more than half of the budget), at most 8.
    int stages = o.stages;
    if (stages <= 0) {
      const int budget = (stages == -2 ? 100 : 200) * 1024;
      stages = std::max(1, std::min(kMaxStages, budget / stage_bytes));
      if (stages == 1 && 2 * stage_bytes + 128 <= 227 * 1024) stages = 2;
    }
    if (p.ks > 1) stages = std::min(stages, per_chunks);
    stages = std::max(1, stages);
    p.stages = stages;
    p.red_bytes = p.ks > 1 ? p.Mp * p.n_tile * 4 : 0;
    if (p.tm) p.stages = std::max(p.stages, std::min(3, 227 * 1024 / stage_bytes));
    p.smem_bytes = std::max(p.stages * stage_bytes, p.red_bytes) + 256;  // + mbarriers etc.
    // tensor memory plans allocate all 512 TMEM columns: one CTA per SM (> half the smem)
    if (p.tm) p.smem_bytes = std::max(p.smem_bytes, 116 * 1024);
  } else if (p.conv_vec == 4) {
    // interleaved conv: stage = three copies + zero block | plan block (128-byte aligned)
    p.il_blk_at = p.x_stage_bytes;
    stage_bytes = (p.x_stage_bytes + p.max_blk_bytes + 127) & ~127;
    p.il_stage_bytes = stage_bytes;
    p.stages = o.stages > 0 ? o.stages : std::max(2, std::min(kMaxStages, 200 * 1024 / stage_bytes));
    p.red_bytes = 0;
    p.smem_bytes = p.stages * stage_bytes + 256;
  } else if (p.conv_vec == 2) {
    // TMA-fed conv: mbarrier ring as deep as ~200 KB allows (persistent CTAs)
    stage_bytes = (stage_bytes + 127) & ~127;
    p.stages = o.stages > 0 ? o.stages : std::max(2, std::min(kMaxStages, 200 * 1024 / stage_bytes));
    p.red_bytes = 0;
    p.smem_bytes = p.stages * stage_bytes + 256;
  } else {
    p.stages = 2;
    p.red_bytes = 0;
    p.smem_bytes = p.stages * stage_bytes;
  }
  if (p.smem_bytes > 227 * 1024) {
    snprintf(buf, sizeof buf, "plan needs %d bytes of shared memory (> 227 KB); lower k_chunk",
             p.smem_bytes);
    err = buf;
    return SPARSE_EUNSUPPORTED;
  }
  p.plan_bytes = (int64_t)p.blob.size() + (int64_t)p.row_id.size() * 4 +
                 (int64_t)p.blk_off.size() * 8 + (int64_t)p.tc_a.size() * 2 +
                 (int64_t)(p.tc_cb.size() + p.tc_rb.size() + p.tc_tile_begin.size() + p.ws_row.size()) * 4;

  p.ps = o.ps;
  if (o.ps != 0 && o.ps != 1) {
    err = "plan_source must be 0 (staged with X) or 1 (kernel parameters)";
    return SPARSE_EINVAL;
  }
  if (o.ps == 1) {
    // plan in kernel parameters (spmm_param_kernel): the plain persistent plan-driven SpMM only
    if (o.kind != SPARSE_SPMM || (o.executor != 0 && o.executor != 2) || p.ks != 1 || p.cm != 1 || p.tm ||
        p.gk != 1 || p.tc_ntiles > 0 || p.R > 8) {
      err = "plan_source = 1 needs a plan-driven SpMM plan with split_k = k_split = x_multicast = 1, "
            "x_source = 0, no tensor-core sub-blocks and rows_per_warp <= 8";
      return SPARSE_EUNSUPPORTED;
    }
    if ((int64_t)p.blob.size() > 30 * 1024) {
      snprintf(buf, sizeof buf, "plan_source = 1: plan blob of %lld bytes exceeds the 30 KB parameter space",
               (long long)p.blob.size());
      err = buf;
      return SPARSE_EUNSUPPORTED;
    }
  }

  if (o.executor == 1) {
    if (o.kind != SPARSE_SPMM) {
      err = "executor = JIT is only supported for SpMM plans";
      return SPARSE_EUNSUPPORTED;
    }
    std::vector<std::vector<RowEntry>> re(M);
    for (int32_t m = 0; m < M; ++m) {
      re[m].reserve(rows[m].size());
      for (const Entry& en : rows[m]) re[m].push_back(RowEntry{en.k, en.w});
    }
    const int rc = jit_generate(p, re, o, err);
    if (rc != SPARSE_OK) return rc;
  } else if (o.executor == 4) {
    // ---- tcgen05 block executor (SURVEY NEXT #1 on Blackwell's 5th-generation tensor cores).
    // W is cut into 128-row x BK-column blocks (BK = 64 for 16-bit data, 32 for fp32); every
    // block holding at least one nonzero is stored dense (zeros included) in the tcgen05
    // K-major, 128-byte-swizzled shared memory layout (8-row atoms of 1 KB, 16-byte chunk c of
    // row r at c ^ (r % 8)), so the executor copies it verbatim into shared memory and
    // multiplies it with tcgen05.mma (M = 128 rows, N = 256 columns, fp32 accumulate in TMEM).
    // fp32 plans run as 3xTF32: W = W_hi + W_lo with both halves exact TF32 values (RN), the
    // block stores [W_hi | W_lo] (2 x 16 KB), and the executor sums W_hi X_hi + W_lo X_hi +
    // W_hi X_lo (X split the same way on the device) - relative error ~2^-22 per product.
    // All-zero blocks are skipped.  "Dense enough" is decided by measurement: the tuner times
    // this executor against the CUDA-core ones; at 90 % uniform sparsity a 128 x 64
    // block holds ~820 nonzeros and the tensor cores' ~30x throughput advantage outweighs the
    // ~10x zero work.  A group of tcg_cs consecutive row blocks (one thread-block cluster,
    // sharing each X tile by multicast) walks the union of its row blocks' nonzero k-blocks
    // (a row block lacking one gets a zero block).  Metadata: tcp_step_off = [ngroups + 1]
    // prefix of union entries, then their k-block indices; tcp_steps = the blocks, entry-major
    // then rank (entry j of the group list, rank r at (j * tcg_cs + r)).
    const bool conv = o.kind == SPARSE_CONV3X3;
    const bool f32 = dtype == SPARSE_F32;
    const int BM = 128, BK = f32 ? 32 : 64, S = f32 ? 4 : 2;
    const int CS = p.tcg_cs;
    p.tcg_bk = BK;
    // conv: implicit im2col over the interleaved dx-shifted copies (kernel 3b layout); the K
    // axis is cut into k-blocks = (BK input channels, tap), so the B tile of a k-block is one
    // 2-D slab of copy dx shifted by (dy - 1) pitches (fp32: slabs of the X_hi and the X_lo
    // copies, which the pre-pass writes split).  Order: channel block, then dx, then dy - the
    // three dy slabs of one copy overlap in all but 2 pitches, so consecutive k-blocks hit in
    // L2 and each copy is read from HBM about once per tile (tap-major order re-read it 3x)
    int32_t ncb = 0;
    if (conv) {
      ncb = (o.c_in + BK - 1) / BK;
      int gg = 1;
      while ((gg * o.w) % 8) ++gg;  // pitch a multiple of 8 elements: 16-byte TMA box starts
      p.tcg_g = gg;
      p.tcg_ncb = ncb;
    }
    // k-block of column k: SpMM k / BK; conv (ci, tap = 3 dy + dx) -> (ci / BK) 9 + 3 dx + dy,
    // column ci % BK
    auto kblock = [&](int32_t k) {
      return conv ? ((k / 9) / BK) * 9 + ((k % 9) % 3) * 3 + (k % 9) / 3 : k / BK;
    };
    auto kcol = [&](int32_t k) { return conv ? (k / 9) % BK : k % BK; };
    const int32_t nrb = (M + BM - 1) / BM, nkb = conv ? 9 * ncb : (K + BK - 1) / BK;
    const int32_t ngroups = (nrb + CS - 1) / CS;
    p.tcp_npanels = nrb;
    p.tcp_nchunks = nkb;
    p.tcg_ngroups = ngroups;
    std::vector<int32_t> pref(1, 0), kbs;
    std::vector<char> nzb((size_t)ngroups * CS * nkb, 0);
    for (int32_t m = 0; m < M; ++m)
      for (const Entry& en : rows[m]) nzb[(size_t)(m / BM) * nkb + kblock(en.k)] = 1;
    std::vector<int64_t> slot((size_t)ngroups * CS * nkb, -1);  // (row block, k-block) -> block
    for (int32_t g = 0; g < ngroups; ++g) {
      for (int32_t kb = 0; kb < nkb; ++kb) {
        bool any = false;
        for (int r = 0; r < CS; ++r) any = any || nzb[(size_t)(g * CS + r) * nkb + kb];
        if (!any) continue;
        for (int r = 0; r < CS; ++r) slot[(size_t)(g * CS + r) * nkb + kb] = (int64_t)kbs.size() * CS + r;
        kbs.push_back(kb);
      }
      pref.push_back((int32_t)kbs.size());
    }
    p.tcp_step_off = pref;
    p.tcp_step_off.insert(p.tcp_step_off.end(), kbs.begin(), kbs.end());
    const size_t half = (size_t)BM * BK * S, blk = f32 ? 2 * half : half;
    p.tcp_steps.assign(kbs.size() * CS * blk, 0);
    // byte offset of (row r, column c) inside a 128 x BK block (128-byte rows, SW128)
    auto sw = [&](int r, int c) {
      const int b = c * S;
      return (size_t)(r / 8) * 1024 + (size_t)(r % 8) * 128 + (size_t)(((b / 16) ^ (r % 8)) * 16) + (size_t)(b % 16);
    };
    for (int32_t m = 0; m < M; ++m) {
      const int r = m % BM;
      for (const Entry& en : rows[m]) {
        const int64_t bi = slot[(size_t)(m / BM) * nkb + kblock(en.k)];
        const size_t off = (size_t)bi * blk + sw(r, kcol(en.k));
        if (f32) {
          const float hi = tf32_rn(en.w), lo = tf32_rn(en.w - hi);
          std::memcpy(&p.tcp_steps[off], &hi, 4);
          std::memcpy(&p.tcp_steps[off + half], &lo, 4);
        } else {
          std::memcpy(&p.tcp_steps[off], &en.wh, 2);
        }
      }
    }
    p.tcp_nsteps = (int64_t)kbs.size();
    p.executor = 4;
    if (!conv) p.n_tile = 256;
    // stage = the W block(s) + a 256-column X tile (fp32: X_hi and X_lo): 48 KB / 96 KB; a CTA
    // of a pair stages half of the X tile: 32 KB / 64 KB
    const int st_bytes = p.tcg_pair ? (f32 ? 64 * 1024 : 32 * 1024) : (f32 ? 96 * 1024 : 48 * 1024);
    p.stages = p.tcg_pair ? (f32 ? 3 : 6) : (f32 ? 2 : 4);
    // + align, barriers, conv table, block lists, the epilogue warps' store staging (16 KB)
    p.smem_bytes = p.stages * st_bytes + 1024 + 2048 + 8192 + 16384;
    p.plan_bytes += (int64_t)p.tcp_steps.size() + (int64_t)p.tcp_step_off.size() * 4;
  } else if (o.executor == 3) {
    // ---- condensed-panel tensor-core executor (fp16 SpMM) ----
    // Panels of 16 consecutive rows; per K chunk of kTcpKc rows the union U of the panel's
    // nonzero columns is the dense contraction: W[16 x U] (zeros where a row lacks a column)
    // times the gathered X rows U.  U is laid out in k16 steps of two 8-row halves; rows of a
    // half have distinct k mod 8 (the staged X chunk is 128-byte swizzled, so ldmatrix rows
    // with distinct k mod 8 hit distinct banks), padded with zero-weight rows (SRT_TCP_STRICT;
    // measured faster than filling halves with conflicting rows: BERT fp16 303 -> 279 us).
    if (o.kind != SPARSE_SPMM || dtype == SPARSE_F32) {
      err = "executor = 3 (tensor-core condensed panels) needs an fp16 or bf16 SpMM plan";
      return SPARSE_EUNSUPPORTED;
    }
    const int KC = kTcpKc;
    p.tcp_npanels = (M + 15) / 16;
    p.tcp_nchunks = (K + KC - 1) / KC;
    const int32_t ngroups = (p.tcp_npanels + kTcpPanels - 1) / kTcpPanels;
    // steps stored group-major, then chunk, then panel: the steps of one CTA's kTcpPanels
    // panels for one chunk are contiguous (one bulk copy into the chunk's pipeline stage)
    p.tcp_step_off.assign((size_t)ngroups * p.tcp_nchunks * (kTcpPanels + 1), 0);
    p.tcp_steps.clear();
    p.tcp_max_blk = 0;
    std::vector<uint16_t> wd((size_t)16 * KC);
    std::vector<int32_t> cursor_all((size_t)p.tcp_npanels * 16, 0);
    int64_t nsteps = 0;
    for (int32_t G = 0; G < ngroups; ++G)
    for (int32_t c = 0; c < p.tcp_nchunks; ++c) {
      const int64_t blk0 = (int64_t)p.tcp_steps.size();
      for (int32_t pi = 0; pi < kTcpPanels; ++pi) {
        const int32_t q = G * kTcpPanels + pi;
        p.tcp_step_off[((size_t)G * p.tcp_nchunks + c) * (kTcpPanels + 1) + pi] = (int32_t)p.tcp_steps.size();
        if (q >= p.tcp_npanels) continue;
        int32_t* cur = cursor_all.data() + (size_t)q * 16;
      {
        const int32_t k0 = c * KC, k1 = std::min(K, k0 + KC);
        std::fill(wd.begin(), wd.end(), (uint16_t)0);
        bool used[256] = {false};
        for (int i = 0; i < 16; ++i) {
          const int32_t m = 16 * q + i;
          if (m >= M) continue;
          int32_t& e = cur[i];
          while (e < (int32_t)rows[m].size() && rows[m][e].k < k1) {
            const int kl = rows[m][e].k - k0;
            wd[(size_t)i * KC + kl] = rows[m][e].wh;
            used[kl] = true;
            ++e;
          }
        }
        std::vector<int> bucket[8];
        int nu = 0;
        for (int kl = 0; kl < k1 - k0; ++kl)
          if (used[kl]) {
            bucket[kl & 7].push_back(kl);
            ++nu;
          }
        // halves of 8 rows: distinct residues first (largest buckets first), then fill
        std::vector<std::array<int, 8>> halves;
        int left = nu;
        while (left > 0) {
          std::array<int, 8> hf;
          hf.fill(-1);
          bool taken[8] = {false};
          int order[8] = {0, 1, 2, 3, 4, 5, 6, 7};
          std::sort(order, order + 8, [&](int a, int b) { return bucket[a].size() > bucket[b].size(); });
          int n = 0;
          for (int t = 0; t < 8 && left > 0; ++t) {
            const int r = order[t];
            if (bucket[r].empty()) continue;
            hf[n++] = bucket[r].back();
            bucket[r].pop_back();
            taken[r] = true;
            --left;
          }
          for (int t = 0; t < 8 && n < 8 && left > 0 && !SRT_TCP_STRICT; ++t) {  // conflicting fill
            const int r = order[t];
            while (!bucket[r].empty() && n < 8) {
              hf[n++] = bucket[r].back();
              bucket[r].pop_back();
              --left;
            }
          }
          for (int r = 0; r < 8 && n < 8; ++r)  // zero-weight pads on free residues
            if (!taken[r] && r < k1 - k0) {
              hf[n++] = 256 + r;  // 256 + k_local marks a zero-weight pad slot
              taken[r] = true;
            }
          for (; n < 8; ++n) hf[n] = 256;
          halves.push_back(hf);
        }
        if (halves.size() % 2) {
          std::array<int, 8> pad;
          for (int r = 0; r < 8; ++r) pad[r] = 256 + (r < k1 - k0 ? r : 0);
          halves.push_back(pad);
        }
        // steps: A fragment (lane l = 4 g + t: W[g][2t, 2t+1], W[g+8][2t, 2t+1],
        // W[g][2t+8, 2t+9], W[g+8][2t+8, 2t+9] of the step's 16 slots) + 16 slot rows
        for (size_t hs = 0; hs < halves.size(); hs += 2) {
          int slot[16];
          for (int j = 0; j < 8; ++j) {
            slot[j] = halves[hs][j];
            slot[8 + j] = halves[hs + 1][j];
          }
          // a pad slot reads some staged row (maybe also a real slot elsewhere): weight 0
          bool real[16];
          for (int j = 0; j < 16; ++j) {
            real[j] = slot[j] < 256;
            slot[j] &= 255;
          }
          auto wv = [&](int i, int j) -> uint16_t { return real[j] ? wd[(size_t)i * KC + slot[j]] : (uint16_t)0; };
          uint16_t fr[32][8];  // A fragment, lane l = 4 g + t
          for (int l = 0; l < 32; ++l) {
            const int g = l / 4, t = l % 4;
            uint16_t* f = fr[l];
            f[0] = wv(g, 2 * t);
            f[1] = wv(g, 2 * t + 1);
            f[2] = wv(g + 8, 2 * t);
            f[3] = wv(g + 8, 2 * t + 1);
            f[4] = wv(g, 2 * t + 8);
            f[5] = wv(g, 2 * t + 9);
            f[6] = wv(g + 8, 2 * t + 8);
            f[7] = wv(g + 8, 2 * t + 9);
          }
          const size_t off = p.tcp_steps.size();
          if (SRT_TCP_PACK) {
            // packed step: [0, 16) slot rows | [16, 48) per-lane mask of nonzero fragment
            // halves | [48, 80) per-lane count of values before the lane | [80, 82) record
            // bytes | [96, ...) the nonzero halves, lane-major (~12 % of the 256)
            std::vector<uint16_t> vals;
            uint8_t hdr[96] = {0};
            for (int l = 0; l < 32; ++l) {
              uint8_t m = 0;
              hdr[48 + l] = (uint8_t)vals.size();
              for (int i = 0; i < 8; ++i)
                if (fr[l][i]) {
                  m |= (uint8_t)(1u << i);
                  vals.push_back(fr[l][i]);
                }
              hdr[16 + l] = m;
            }
            for (int j = 0; j < 16; ++j) hdr[j] = (uint8_t)slot[j];
            const uint16_t rec = (uint16_t)(96 + ((vals.size() * 2 + 15) & ~(size_t)15));
            std::memcpy(hdr + 80, &rec, 2);
            p.tcp_steps.resize(off + rec, 0);
            std::memcpy(p.tcp_steps.data() + off, hdr, 96);
            if (!vals.empty()) std::memcpy(p.tcp_steps.data() + off + 96, vals.data(), vals.size() * 2);
          } else {
            p.tcp_steps.resize(off + kTcpStepBytes, 0);
            std::memcpy(p.tcp_steps.data() + off, fr, 512);
            uint8_t* idx = p.tcp_steps.data() + off + 512;
            for (int j = 0; j < 16; ++j) idx[j] = (uint8_t)slot[j];
          }
          ++nsteps;
        }
      }
      }
      p.tcp_step_off[((size_t)G * p.tcp_nchunks + c) * (kTcpPanels + 1) + kTcpPanels] = (int32_t)p.tcp_steps.size();
      p.tcp_max_blk = std::max<int32_t>(p.tcp_max_blk, (int32_t)(p.tcp_steps.size() - blk0));
    }
    p.tcp_nsteps = nsteps;
    p.executor = 3;
    p.plan_bytes += (int64_t)p.tcp_steps.size() + (int64_t)p.tcp_step_off.size() * 4;
  } else if (o.executor != 0) {
    err = "executor must be 0 (plan-driven), 1 (JIT), 2 (auto), 3 (tensor-core condensed panels) or 4 (tcgen05 blocks)";
    return SPARSE_EINVAL;
  }

  uint64_t h = 1469598103934665603ull;
  const int32_t cfg[] = {p.M,  p.K,      p.dtype,   p.kind,    p.c_in,   p.h,
                         p.w,  p.warps,  p.R,       p.gk,      p.C,      p.n_tile,
                         p.kc, p.nchunks, p.npanels, p.conv_rb, p.conv_ipt, p.ks, p.cm, p.tm,
                         p.conv_vec, p.row_order, p.executor, p.jit_mp, p.jit_warps, p.stages,
                         p.tc_min_pct, p.ps, p.tcg_cs, p.tcg_bk, p.tcg_pair, p.tcg_ks};
  h = fnv1a(h, cfg, sizeof cfg);
  h = fnv1a(h, p.row_id.data(), p.row_id.size() * 4);
  h = fnv1a(h, p.blk_off.data(), p.blk_off.size() * 8);
  h = fnv1a(h, p.blob.data(), p.blob.size());
  h = fnv1a(h, p.tc_cb.data(), p.tc_cb.size() * 4);
  h = fnv1a(h, p.tc_a.data(), p.tc_a.size() * 2);
  h = fnv1a(h, p.tcp_steps.data(), p.tcp_steps.size());
  p.digest = h;
  p.build_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return SPARSE_OK;
}

}  // namespace srt
