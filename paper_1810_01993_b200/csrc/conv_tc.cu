// Implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// The reference computes every convolution of the training step in
// pkg/src/deskdl/model/_kernels_py.py:44-83 (im2col + sgemm) or
// _convkernels.pyx:16-71 (direct loops), NCHW fp32.  Here the same three
// products run NHWC bf16 with fp32 accumulation in TMEM:
//
//   fprop / dgrad  M = pixels (128-pixel rectangular box), N = output channels,
//                  K = taps x input channels.  Each K block is one TMA box of the
//                  input shifted by the tap offset; TMA's out-of-bounds zero fill
//                  implements the "same" padding and any dilation.  dgrad is the
//                  same kernel over dy with tap-flipped, ci/co-swapped weights.
//   wgrad          M = (tap, ci) rows (two 64-channel shifted boxes), N = output
//                  channels, K = pixels; both operands MN-major.  Split-K over
//                  pixel boxes, fp32 partials, deterministic reduction.
//
// Warp roles (192 threads, one CTA per SM, persistent over tiles):
//   warp 0  TMA producer      warp 1  MMA issuer + TMEM owner
//   warps 2-5 epilogue (TMEM -> registers -> fused epilogue -> global)
// Two TMEM accumulator stages let the epilogue of tile i overlap the MMAs of i+1.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "internal.h"
#include "sm100.cuh"

namespace b2 {

constexpr int BM = 128;

// Programmatic dependent launch for the persistent tensor-core kernels (B2DL_PDL=0 disables).
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
static int launch_tc(void (*kern)(KArgs...), int grid, int block, int smem, cudaStream_t st, int cluster,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) {
    fprintf(stderr, "b2dl: CUDA error %s\n", cudaGetErrorString(e));
    return B2DL_E_CUDA;
  }
  return B2DL_OK;
}
constexpr int SMEM_BUDGET = 200 * 1024;

__host__ __device__ constexpr uint32_t tmem_cols_for(int n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}
// CG = 2: a CTA pair (cluster of 2 on one TPC) computes a 256-pixel x BN tile with
// cta_group::2 MMAs; each CTA stages its own 128-pixel A box and half of B's BN rows, so the
// operand bytes per FLOP drop by a third against a single-CTA 128 x BN tile.
template <int BN, int KBLK, bool BMN = false, int CG = 1>
struct FpropCfg {
  static constexpr int A_BYTES = BM * KBLK * 2;
  // MN-major B (master-layout weights): 64-channel-wide chunks of KBLK K rows
  static constexpr int B_CHUNK = 64 * KBLK * 2;
  static constexpr int NBC = (BN < 64 ? 1 : BN / 64) / CG;  // chunks staged by this CTA
  static constexpr int B_BYTES = BMN ? NBC * B_CHUNK : BN / CG * KBLK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = tmem_cols_for(2 * BN);
  static constexpr int CW = BN < 32 ? BN : 32;  // epilogue chunk (TMEM columns per load)
};

// Shared memory: [A stages][B stages][epilogue buffers][barriers].  The stage count is chosen
// per launch: whatever the epilogue's operand buffers leave of the 227 KB opt-in limit.
constexpr int SMEM_MAX = 232448;
constexpr int FPROP_MAX_STAGES = 8;
constexpr int SMEM_FIXED = 1024 + 512;  // alignment slack + barriers / TMEM slot
// TMA epilogue: one 32-pixel x 32-channel bf16 box per chunk, 64-byte rows, 64B swizzle.
// Per warp: two operand slots of up to two operands each (residual / mask / accumulated y,
// loaded one chunk ahead), and two output buffers (stores drain while the next chunk runs).
constexpr int EPI_LEGACY_BYTES = 8 * 32 * 80;

struct FpropParams {
  int n, h, w;
  int bw, bh, tiles_x, tiles_y;
  int num_m_tiles, num_n_tiles, num_tiles;
  int kw, dil, pad_top, pad_left;
  int num_cblk, num_kb, cin_pad;
  int cout;
  void* y;
  long long y_stride;
  int y_f32;
  const float* bias;
  const b2h* res;
  long long res_stride;
  const b2h* mask;
  long long mask_stride;
  int relu, accumulate, vec_ok;
  int b_mode;  // 0 packed [cout][taps][cin_pad]; 1 master HWIO, MN-major; 2 master HWIO, dgrad (flipped taps)
  int taps;
  int stages;          // operand pipeline depth
  int b_region;        // bytes of the B stages, rounded up to 1 KB
  int epi_bytes;       // epilogue buffer bytes
  int tma_epi;         // 1: TMA-staged epilogue (operands + output through swizzled boxes)
  int epi_nops;        // operands per chunk in the TMA epilogue (residual, mask, accumulated y)
  int epi_slots;       // operand slots per sub-group (prefetch depth + 1)
  int epi_pw;          // 1: per-warp epilogue boxes (32 pixels x 32 channels; no sub-group barrier)
  int epi_obufs;       // output buffers per sub-group (2; per-warp mode up to 4)
  int rt_cs;           // row-tap kernel: width (pixels) of the wide input box whose column taps are
                       // descriptor offsets (8 + (kw - 1) dil); 0: one 8-pixel box per column tap
  int dbg_epi;         // development: 1 = epilogue only drains TMEM (wrong results; timing aid)
  int bias_vec;        // bias 16-byte aligned
  int in_stride;       // input pixels per output pixel (strided reads of the input)
  int y_phase;         // output is a phase view of a larger tensor: TMA epilogue only
  float* bn_part;      // batch-norm statistics of the stored output: [row][2][cout] fp32 sum, sum of squares
  int bn_per_cta;      // 1: one row per CTA accumulated over its tiles (single N tile); 0: one row per M tile
  // Batch-norm backward statistics (this launch writes g = d loss / d y of a BN's output y =
  // relu(scale z + shift)): the mask operand is the BN input z, the relu mask is recomputed as
  // scale z + shift > 0, and rows of (sum g, sum g * xhat) with xhat = (z - mean) rstd are written.
  const float* bnb_stats;  // [4][cout]: mean, rstd, scale, shift
  float* bnb_part;         // [row][2][cout]; rows = 4 per CTA (per-CTA mode) or 4 per M tile
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  uint32_t a = smem_u32(p);
  return p + ((1024 - (a & 1023)) & 1023);
}

// ---- epilogue staging: each epilogue warp owns a 32-row x CW-column bf16 tile in shared
// memory (80-byte row pitch, bank-conflict free).  A thread holds one accumulator row (one
// pixel); global traffic goes through cooperative transfers in which 4 (or 2) lanes move one
// row's 64 (32) contiguous bytes, so every warp access is a set of full 32-byte sectors.
constexpr int EPI_ROW = 80;
constexpr int EPI_WARP_BYTES = 32 * EPI_ROW;

template <int CW>
struct CoopRows {
  static constexpr int PIECES = CW / 8;         // 16-byte pieces per row
  static constexpr int ROWS_PER_IT = 32 / PIECES;
  long long pix[PIECES];
  bool ok[PIECES];
};

template <int CW>
__device__ __forceinline__ void coop_load(const b2h* base, long long stride, int c0, int cout,
                                          const CoopRows<CW>& L, uint8_t* st, bool nc) {
  using R = CoopRows<CW>;
  const int lane = lane_id(), piece = lane % R::PIECES;
  const bool pv = c0 + piece * 8 < cout;
#pragma unroll
  for (int k = 0; k < R::PIECES; ++k) {
    uint4 u = make_uint4(0, 0, 0, 0);
    if (L.ok[k] && pv) {
      const uint4* src = reinterpret_cast<const uint4*>(base + L.pix[k] * stride + c0 + piece * 8);
      u = nc ? __ldg(src) : *src;
    }
    *reinterpret_cast<uint4*>(st + (k * R::ROWS_PER_IT + lane / R::PIECES) * EPI_ROW + piece * 16) = u;
  }
}
template <int CW>
__device__ __forceinline__ void coop_store(b2h* base, long long stride, int c0, int cout,
                                           const CoopRows<CW>& L, const uint8_t* st) {
  using R = CoopRows<CW>;
  const int lane = lane_id(), piece = lane % R::PIECES;
  const bool pv = c0 + piece * 8 < cout;
#pragma unroll
  for (int k = 0; k < R::PIECES; ++k)
    if (L.ok[k] && pv)
      *reinterpret_cast<uint4*>(base + L.pix[k] * stride + c0 + piece * 8) =
          *reinterpret_cast<const uint4*>(st + (k * R::ROWS_PER_IT + lane / R::PIECES) * EPI_ROW + piece * 16);
}
template <int CW>
__device__ __forceinline__ void row_get(const uint8_t* st, float* v) {
  const uint8_t* r = st + lane_id() * EPI_ROW;
#pragma unroll
  for (int q = 0; q < CW / 8; ++q) {
    const uint4 u = *reinterpret_cast<const uint4*>(r + q * 16);
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[q * 8 + 2 * e] = bf16lo(w4[e]);
      v[q * 8 + 2 * e + 1] = bf16hi(w4[e]);
    }
  }
}
template <int CW>
__device__ __forceinline__ void row_put(uint8_t* st, const float* v) {
  uint8_t* r = st + lane_id() * EPI_ROW;
#pragma unroll
  for (int q = 0; q < CW / 8; ++q) {
    uint4 u;
    u.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
    u.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
    u.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
    u.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
    *reinterpret_cast<uint4*>(r + q * 16) = u;
  }
}

// bf16 output with aligned views and cout % 8 == 0: coalesced through the staging tile
// Register prefetch of one cooperative 32 x CW tile (the epilogue's first global operand),
// issued before the accumulator is ready so the DRAM latency overlaps the MMA main loop.
template <int CW>
__device__ __forceinline__ void coop_prefetch(const b2h* base, long long stride, int c0, int cout,
                                              const CoopRows<CW>& L, uint4* r) {
  using R = CoopRows<CW>;
  const int piece = lane_id() % R::PIECES;
  const bool pv = c0 + piece * 8 < cout;
#pragma unroll
  for (int k = 0; k < R::PIECES; ++k)
    r[k] = (L.ok[k] && pv) ? __ldg(reinterpret_cast<const uint4*>(base + L.pix[k] * stride + c0 + piece * 8))
                           : make_uint4(0, 0, 0, 0);
}
template <int CW>
__device__ __forceinline__ void coop_stash(const uint4* r, uint8_t* st) {
  using R = CoopRows<CW>;
  const int lane = lane_id(), piece = lane % R::PIECES;
#pragma unroll
  for (int k = 0; k < R::PIECES; ++k)
    *reinterpret_cast<uint4*>(st + (k * R::ROWS_PER_IT + lane / R::PIECES) * EPI_ROW + piece * 16) = r[k];
}

// The first of (residual, mask) present is the prefetched operand `pre` (may be null).
template <int CW>
__device__ __forceinline__ void fprop_epilogue_vec(const FpropParams& p, float* v, int c0, const CoopRows<CW>& L,
                                                   uint8_t* st, const uint4* pre) {
  if (p.bias) {  // one coalesced load per warp, broadcast by shuffles
    const int lane = lane_id();
    const float b = (lane < CW && c0 + lane < p.cout) ? __ldg(p.bias + c0 + lane) : 0.f;
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] += __shfl_sync(0xffffffffu, b, i);
  }
  float t[CW];
  if (p.res) {
    if (pre)
      coop_stash<CW>(pre, st);
    else
      coop_load<CW>(p.res, p.res_stride, c0, p.cout, L, st, true);
    __syncwarp();
    row_get<CW>(st, t);
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] += t[i];
    __syncwarp();
  }
  if (p.relu) {
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  if (p.mask) {
    if (pre && !p.res)
      coop_stash<CW>(pre, st);
    else
      coop_load<CW>(p.mask, p.mask_stride, c0, p.cout, L, st, true);
    __syncwarp();
    row_get<CW>(st, t);
#pragma unroll
    for (int i = 0; i < CW; ++i)
      if (!(t[i] > 0.f)) v[i] = 0.f;
    __syncwarp();
  }
  b2h* y = reinterpret_cast<b2h*>(p.y);
  if (p.accumulate) {
    coop_load<CW>(y, p.y_stride, c0, p.cout, L, st, false);
    __syncwarp();
    row_get<CW>(st, t);
#pragma unroll
    for (int i = 0; i < CW; ++i) v[i] += t[i];
    __syncwarp();
  }
  row_put<CW>(st, v);
  __syncwarp();
  coop_store<CW>(y, p.y_stride, c0, p.cout, L, st);
  __syncwarp();
}

template <int CW>
__device__ __forceinline__ void fprop_epilogue_scalar(const FpropParams& p, float* v, long long pix, int c0) {
  const int nvalid = min(CW, p.cout - c0);
  if (p.bias) {
#pragma unroll
    for (int i = 0; i < CW; ++i)
      if (i < nvalid) v[i] += __ldg(p.bias + c0 + i);
  }
  // general (scalar) path: ragged channel counts, fp32 output, unaligned views
#pragma unroll
  for (int i = 0; i < CW; ++i) {
    if (i >= nvalid) break;
    float x = v[i];
    if (p.res) x += h_to_f(p.res[pix * p.res_stride + c0 + i]);
    if (p.relu) x = fmaxf(x, 0.f);
    if (p.mask && !(h_to_f(p.mask[pix * p.mask_stride + c0 + i]) > 0.f)) x = 0.f;
    if (p.y_f32) {
      float* d = reinterpret_cast<float*>(p.y) + pix * p.y_stride + c0 + i;
      *d = p.accumulate ? *d + x : x;
    } else {
      b2h* d = reinterpret_cast<b2h*>(p.y) + pix * p.y_stride + c0 + i;
      if (p.accumulate) x += h_to_f(*d);
      *d = f_to_h(x);
    }
  }
}

constexpr int FPROP_THREADS = 320;  // TMA warp, MMA warp, 8 epilogue warps

// swizzled (64B) rows of an epilogue box: lane r's 16-byte piece k sits at piece k ^ ((r >> 1) & 3)
__device__ __forceinline__ void box_row_get(const uint8_t* box, float* t) {
  const int r = lane_id();
  const uint8_t* row = box + r * 64;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 u = *reinterpret_cast<const uint4*>(row + ((k ^ ((r >> 1) & 3)) << 4));
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      t[k * 8 + 2 * e] = bf16lo(w4[e]);
      t[k * 8 + 2 * e + 1] = bf16hi(w4[e]);
    }
  }
}
__device__ __forceinline__ void box_row_put(uint8_t* box, const float* v) {
  const int r = lane_id();
  uint8_t* row = box + r * 64;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint4 u;
    u.x = pack_bf16x2(v[k * 8 + 0], v[k * 8 + 1]);
    u.y = pack_bf16x2(v[k * 8 + 2], v[k * 8 + 3]);
    u.z = pack_bf16x2(v[k * 8 + 4], v[k * 8 + 5]);
    u.w = pack_bf16x2(v[k * 8 + 6], v[k * 8 + 7]);
    *reinterpret_cast<uint4*>(row + ((k ^ ((r >> 1) & 3)) << 4)) = u;
  }
}

// TMA epilogue, EW warps = EW / 4 sub-groups of 4 warps (one per TMEM lane quarter).  A
// sub-group owns every (EW / 4)-th 32-column chunk of a tile; one chunk of the whole 128-pixel
// tile is one 8 KB TMA box (32 channels x the tile's pixel box, 64-byte swizzled rows), so a
// tile moves in few, large TMA operations: operands arrive one chunk ahead, the four warps pack
// their 32 rows into a shared output box, meet at a named barrier, and one thread stores it.
constexpr int EPI_CHUNK = 128 * 64;  // 128 pixels x 32 bf16 channels
// per sub-group: `slots` operand slots of nops chunks (operands run slots-1 chunks ahead) + 2
// output buffers
__host__ __device__ constexpr int epi_sub_bytes(int nops, int slots = 2, int obufs = 2) {
  return (slots * nops + obufs) * EPI_CHUNK;
}
constexpr int EPI_MAX_SLOTS = 4;

// ST: statistics epilogue variant (compile time, so the plain kernels carry none of its registers):
// 0 none, 1 batch-norm forward statistics (bn_part), 2 batch-norm backward statistics (bnb_part)
template <int BN, int CG, int EW, int ST = 0>
__device__ __forceinline__ void fprop_epilogue_tma(const FpropParams& p, const CUtensorMap* tmY, const CUtensorMap* tmR,
                                                   const CUtensorMap* tmM, uint32_t tmem_base, uint64_t* tfull,
                                                   uint64_t* tempty, uint64_t* inbar, uint8_t* epi, int warp, int rank,
                                                   int unit0, int units) {
  constexpr int SUBS = EW / 4;                 // sub-groups
  constexpr int NCH = BN / 32;                 // 32-column chunks per tile
  constexpr int NJ = (NCH + SUBS - 1) / SUBS;  // chunks per sub-group
  const int lane = lane_id();
  const int per_img = p.tiles_x * p.tiles_y;
  const int ew = warp - 2;
  const int q = warp & 3;
  const int sub = ew >> 2;
  const bool leader = (q == 0) && (lane == 0);  // warp with lane quarter 0 of the sub-group
  // Per-warp mode (epi_pw, not with forward statistics, which read all four quarters back): each
  // warp moves its own 32 rows of a chunk as one 32-pixel x 32-channel box -- the same bytes of the
  // same swizzled buffers -- with its own operand barriers and bulk groups, so the four warps of a
  // sub-group never rendezvous; the tensor maps carry the per-warp box (host side).
  const bool pw = ST != 1 && p.epi_pw;
  const bool issuer = pw ? lane == 0 : leader;
  const int qoff = pw ? q * (EPI_CHUNK / 4) : 0;
  const int wdx = pw ? (32 * q) % p.bw : 0, wdy = pw ? (32 * q) / p.bw : 0;
  const uint32_t box_tx = pw ? EPI_CHUNK / 4 : EPI_CHUNK;
  const int nops = p.epi_nops;
  const int S = p.epi_slots;   // operand slots: loads run S-1 chunks ahead of use
  const int OB = pw ? p.epi_obufs : 2;
  uint8_t* sbuf = epi + sub * epi_sub_bytes(nops, S, OB);
  uint8_t* obuf = sbuf + S * nops * EPI_CHUNK;
  uint64_t* ib = pw ? inbar + 2 * ew : inbar + EPI_MAX_SLOTS * sub;   // pw: S <= 2 (host)
  auto locate = [&](int tile, int& img, int& x, int& y, int& nt) {
    const int pmt = tile / p.num_n_tiles;
    nt = tile - pmt * p.num_n_tiles;
    const int mt = pmt * CG + rank;
    img = mt / per_img;
    const int r = mt - img * per_img;
    const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
    y = ty * p.bh;
    x = tx * p.bw;
  };
  auto chunks = [&](int nt) {  // valid chunks of this sub-group in a tile of N-tile nt
    int n = 0;
#pragma unroll
    for (int j = 0; j < NJ; ++j)
      if (SUBS * j + sub < NCH && nt * BN + (SUBS * j + sub) * 32 < p.cout) n = j + 1;
    return n;
  };
  auto issue = [&](int tile, int j, int slot) {
    // per-warp mode: called by the converged warp, one elected lane (lane 0) issues -- no
    // single-thread issue loop around each TMA instruction; it also owns the bulk groups
    if (pw ? elect_one_sync() : leader) {
      int img, x, y, nt;
      locate(tile, img, x, y, nt);
      x += wdx;
      y += wdy;
      const int c0 = nt * BN + (SUBS * j + sub) * 32;
      uint8_t* dst = sbuf + slot * nops * EPI_CHUNK + qoff;
      fence_proxy_async();
      mbar_arrive_expect_tx(&ib[slot], nops * box_tx);
      int o = 0;
      if (p.res) tma_load_4d(dst + (o++) * EPI_CHUNK, tmR, &ib[slot], c0, x, y, img);
      if (p.mask) tma_load_4d(dst + (o++) * EPI_CHUNK, tmM, &ib[slot], c0, x, y, img);
      if (p.accumulate) tma_load_4d(dst + o * EPI_CHUNK, tmY, &ib[slot], c0, x, y, img);
    }
  };
  auto release = [&](int as) {  // accumulator stage fully read: hand it back to the MMA warp
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (CG == 2)
        mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
      else
        mbar_arrive(&tempty[as]);
    }
  };
  auto sub_sync = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(1 + sub) : "memory"); };
  const int row = q * 32 + lane;          // tile row (pixel) of this thread
  const int swz = (lane >> 1) & 3;        // 64B-swizzle phase of the row
  // operand issue cursor (leader thread only): walks the consumer's (tile, chunk) sequence S-1
  // items ahead, skipping tiles in which this sub-group has no chunk.  Only the last N tile can
  // be partial, so a tile's chunk count follows from its N index, tracked without divisions.
  const int nv_full = chunks(0), nv_last = chunks(p.num_n_tiles - 1);
  const int units_nt = units % p.num_n_tiles;
  int itile = unit0, int_nt = unit0 % p.num_n_tiles, ij = 0, islot = 0;
  auto nv_at = [&](int ntv) { return ntv == p.num_n_tiles - 1 ? nv_last : nv_full; };
  auto step_tile = [&]() {
    itile += units;
    int_nt += units_nt;
    if (int_nt >= p.num_n_tiles) int_nt -= p.num_n_tiles;
  };
  // (every lane keeps the cursor: warp-uniform, cheap)
  while (itile < p.num_tiles && nv_at(int_nt) == 0) step_tile();
  auto issue_next = [&]() {
    if (!nops || itile >= p.num_tiles || !(pw || leader)) return;
    issue(itile, ij, islot);
    islot = islot + 1 == S ? 0 : islot + 1;
    if (++ij >= nv_at(int_nt)) {
      ij = 0;
      do {
        step_tile();
      } while (itile < p.num_tiles && nv_at(int_nt) == 0);
    }
  };
  for (int k = 0; k < S - 1 && !p.dbg_epi; ++k) issue_next();
  float bn_acc[NJ];
  float bb_acc[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) bn_acc[j] = bb_acc[j][0] = bb_acc[j][1] = 0.f;
  uint32_t phbits = 0;   // wait parity per slot
  int slot = 0, ob = 0, it = 0;
  for (int tile = unit0; tile < p.num_tiles; tile += units, ++it) {
    const int as = it & 1;
    const uint32_t ap = (it >> 1) & 1;
    int img, x, y, nt;
    locate(tile, img, x, y, nt);
    const int nv = chunks(nt);
    mbar_wait(&tfull[as], ap);
    tc_fence_after();
    const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN;
    if (p.dbg_epi) {
      release(as);
      continue;
    }
#pragma unroll 1
    for (int j = 0; j < NJ; ++j) {
      if (j >= nv) break;  // uniform over the sub-group
      if (pw) __syncwarp();   // the slot refilled next was read by this warp's lanes last chunk
      issue_next();        // keeps S-1 chunks of operands in flight
      const int c0 = nt * BN + (SUBS * j + sub) * 32;
      uint32_t cur[32];
      tmem_ld_issue_x32(tbase + (SUBS * j + sub) * 32, cur);
      tmem_ld_wait();
      if (j == nv - 1) release(as);
      const uint8_t* in = sbuf + slot * nops * EPI_CHUNK;
      if (nops) {
        mbar_wait(&ib[slot], (phbits >> slot) & 1u);
        phbits ^= 1u << slot;
      }
      uint8_t* ochunk = obuf + ob * EPI_CHUNK;
      const float4* bias4 = p.bias ? reinterpret_cast<const float4*>(p.bias + c0) : nullptr;
      float bstat[64];   // BN backward statistics of this row's 32 channels (only with bnb_stats)
      const bool pix_ok = img < p.n && y + row / p.bw < p.h && x + (row % p.bw) < p.w;
      if (pw) {   // this buffer's store (OB chunks ago) must have read it out
        if (lane == 0) {
          if (OB >= 4)
            bulk_wait_read<3>();
          else if (OB == 3)
            bulk_wait_read<2>();
          else
            bulk_wait_read<1>();
        }
        __syncwarp();
      }
      if constexpr (ST != 2) {
        // operation-major over the chunk's 32 values: one uniform branch per operand per chunk,
        // operand pointers fixed per chunk (the per-piece form below re-derives both per 8 values)
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(cur[e]);
        auto poff = [&](int k) { return row * 64 + ((k ^ swz) << 4); };
        auto add16 = [&](const uint8_t* src) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint4 u = *reinterpret_cast<const uint4*>(src + poff(k));
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * k + 2 * e] += bf16lo(w4[e]);
              v[8 * k + 2 * e + 1] += bf16hi(w4[e]);
            }
          }
        };
        if (bias4) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (c0 + 8 * k < p.cout) {  // TMA epilogue: bias 16-byte aligned, cout % 8 == 0
              const float4 b0 = __ldg(bias4 + 2 * k), b1 = __ldg(bias4 + 2 * k + 1);
              v[8 * k + 0] += b0.x;
              v[8 * k + 1] += b0.y;
              v[8 * k + 2] += b0.z;
              v[8 * k + 3] += b0.w;
              v[8 * k + 4] += b1.x;
              v[8 * k + 5] += b1.y;
              v[8 * k + 6] += b1.z;
              v[8 * k + 7] += b1.w;
            }
        }
        const uint8_t* mop = in + (p.res ? EPI_CHUNK : 0);   // operand order: residual, mask, y
        if (p.res) add16(in);
        if (p.relu) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = fmaxf(v[e], 0.f);
        }
        if (p.mask && p.accumulate) {   // mask before the accumulated value: per element
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint4 u = *reinterpret_cast<const uint4*>(mop + poff(k));
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (!(bf16lo(w4[e]) > 0.f)) v[8 * k + 2 * e] = 0.f;
              if (!(bf16hi(w4[e]) > 0.f)) v[8 * k + 2 * e + 1] = 0.f;
            }
          }
        }
        if (p.accumulate) add16(mop + (p.mask ? EPI_CHUNK : 0));
        uint32_t pkw[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pkw[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
        if (p.mask && !p.accumulate) {   // relu mask on the packed pairs (same bits as zeroing)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint4 u = *reinterpret_cast<const uint4*>(mop + poff(k));
            pkw[4 * k + 0] &= pos_mask_h2(u.x);
            pkw[4 * k + 1] &= pos_mask_h2(u.y);
            pkw[4 * k + 2] &= pos_mask_h2(u.z);
            pkw[4 * k + 3] &= pos_mask_h2(u.w);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<uint4*>(ochunk + poff(k)) =
              make_uint4(pkw[4 * k], pkw[4 * k + 1], pkw[4 * k + 2], pkw[4 * k + 3]);
      } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // 8-column pieces
        const int poff = row * 64 + ((k ^ swz) << 4);
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(cur[8 * k + e]);
        if (bias4 && c0 + 8 * k < p.cout) {  // TMA epilogue: bias 16-byte aligned, cout % 8 == 0
          const float4 b0 = __ldg(bias4 + 2 * k);
          const float4 b1 = __ldg(bias4 + 2 * k + 1);
          v[0] += b0.x;
          v[1] += b0.y;
          v[2] += b0.z;
          v[3] += b0.w;
          v[4] += b1.x;
          v[5] += b1.y;
          v[6] += b1.z;
          v[7] += b1.w;
        }
        int o = 0;
        if (p.res) {
          const uint4 u = *reinterpret_cast<const uint4*>(in + (o++) * EPI_CHUNK + poff);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[2 * e] += bf16lo(w4[e]);
            v[2 * e + 1] += bf16hi(w4[e]);
          }
        }
        if (p.relu) {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
        }
        float zf[8];
        if (p.mask) {
          const uint4 u = *reinterpret_cast<const uint4*>(in + (o++) * EPI_CHUNK + poff);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
          if constexpr (ST == 2) {   // mask operand = BN input z: relu mask = scale z + shift > 0
            const float4* sc4 = reinterpret_cast<const float4*>(p.bnb_stats + 2 * p.cout + c0 + 8 * k);
            const float4* sh4 = reinterpret_cast<const float4*>(p.bnb_stats + 3 * p.cout + c0 + 8 * k);
            const float4 sa = __ldg(sc4), sb = __ldg(sc4 + 1), ha = __ldg(sh4), hb = __ldg(sh4 + 1);
            const float scl[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
            const float shf[8] = {ha.x, ha.y, ha.z, ha.w, hb.x, hb.y, hb.z, hb.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              zf[2 * e] = bf16lo(w4[e]);
              zf[2 * e + 1] = bf16hi(w4[e]);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (!(fmaf(zf[e], scl[e], shf[e]) > 0.f)) v[e] = 0.f;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              if (!(bf16lo(w4[e]) > 0.f)) v[2 * e] = 0.f;
              if (!(bf16hi(w4[e]) > 0.f)) v[2 * e + 1] = 0.f;
            }
          }
        }
        if (p.accumulate) {
          const uint4 u = *reinterpret_cast<const uint4*>(in + o * EPI_CHUNK + poff);
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[2 * e] += bf16lo(w4[e]);
            v[2 * e + 1] += bf16hi(w4[e]);
          }
        }
        uint4 pk;
        pk.x = pack_bf16x2(v[0], v[1]);
        pk.y = pack_bf16x2(v[2], v[3]);
        pk.z = pack_bf16x2(v[4], v[5]);
        pk.w = pack_bf16x2(v[6], v[7]);
        *reinterpret_cast<uint4*>(ochunk + poff) = pk;
        if constexpr (ST == 2) {   // this pixel's (g, g * xhat) of the STORED g, channel-major pairs
          const float4* mu4 = reinterpret_cast<const float4*>(p.bnb_stats + c0 + 8 * k);
          const float4* rs4 = reinterpret_cast<const float4*>(p.bnb_stats + p.cout + c0 + 8 * k);
          const float4 ma = __ldg(mu4), mb = __ldg(mu4 + 1), ra = __ldg(rs4), rb = __ldg(rs4 + 1);
          const float mu[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};
          const float rs[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
          const uint32_t pkw[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float g = (e & 1) ? bf16hi(pkw[e >> 1]) : bf16lo(pkw[e >> 1]);
            const bool ok = pix_ok;
            bstat[2 * (8 * k + e)] = ok ? g : 0.f;
            bstat[2 * (8 * k + e) + 1] = ok ? g * ((zf[e] - mu[e]) * rs[e]) : 0.f;
          }
        }
      }
      }
      if constexpr (ST == 2) {
        // reduce-scatter over the 32 lanes (rows): lane l ends with channel l's (sum g, sum g xhat)
#pragma unroll
        for (int half = 32, bit = 16; half >= 2; half >>= 1, bit >>= 1) {
          const bool hi = (lane & bit) != 0;
#pragma unroll
          for (int e = 0; e < half; ++e) {
            const float send = hi ? bstat[e] : bstat[e + half];
            const float keep = hi ? bstat[e + half] : bstat[e];
            bstat[e] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
          }
        }
        if (p.bn_per_cta) {
          bb_acc[j][0] += bstat[0];
          bb_acc[j][1] += bstat[1];
        } else if (c0 + lane < p.cout) {
          const int mt = (tile / p.num_n_tiles) * CG + rank;
          if (mt < p.num_m_tiles) {
            const long long row = static_cast<long long>(mt) * 4 + q;
            p.bnb_part[(row * 2) * p.cout + c0 + lane] = bstat[0];
            p.bnb_part[(row * 2 + 1) * p.cout + c0 + lane] = bstat[1];
          }
        }
      }
      fence_proxy_async();
      if (pw) {
        __syncwarp();
        if (elect_one_sync()) {   // lane 0 of the converged warp
          tma_store_4d(tmY, ochunk + qoff, c0, x + wdx, y + wdy, img);
          bulk_commit();
        }
      } else {
        // the other output buffer (next chunk's) must be read out by its store before anyone
        // packs into it: its store was the only one outstanding before this chunk's
        if (leader) bulk_wait_read<0>();
        sub_sync();
        if (leader) {
          tma_store_4d(tmY, ochunk, c0, x, y, img);
          bulk_commit();
        }
      }
      if constexpr (ST == 1) {
        // Batch-norm statistics of this chunk (training-mode BN after the conv):
        // per-channel sum and sum of squares of the STORED bf16 values over the tile's valid
        // pixels, read back from the packed output box while its TMA store drains.  Warp q takes
        // the 8 channels of 16-byte piece q over rows lane + 32 m; a reduce-scatter butterfly
        // leaves sum / sum-of-squares value (lane >> 1) in lane pair (2i, 2i+1) -- fixed order, no
        // shared scratch, no extra barrier (the box is rewritten only after the next sub_sync).
        float v16[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v16[e] = 0.f;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int r = lane + 32 * m;
          const int ry = r / p.bw, rx = r - ry * p.bw;
          if (img < p.n && y + ry < p.h && x + rx < p.w) {
            const uint4 u = *reinterpret_cast<const uint4*>(ochunk + r * 64 + ((q ^ ((r >> 1) & 3)) << 4));
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a0 = bf16lo(w4[e]), a1 = bf16hi(w4[e]);
              v16[2 * e] += a0;
              v16[8 + 2 * e] = fmaf(a0, a0, v16[8 + 2 * e]);
              v16[2 * e + 1] += a1;
              v16[8 + 2 * e + 1] = fmaf(a1, a1, v16[8 + 2 * e + 1]);
            }
          }
        }
#pragma unroll
        for (int half = 8, bit = 16; half >= 1; half >>= 1, bit >>= 1) {
          const bool hi = (lane & bit) != 0;
#pragma unroll
          for (int e = 0; e < half; ++e) {
            const float send = hi ? v16[e] : v16[e + half];
            const float keep = hi ? v16[e + half] : v16[e];
            v16[e] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
          }
        }
        v16[0] += __shfl_xor_sync(0xffffffffu, v16[0], 1);
        if (p.bn_per_cta) {
          bn_acc[j] += v16[0];   // same channels in every tile (one N tile): fold across tiles
        } else {
          const int mt = (tile / p.num_n_tiles) * CG + rank;
          const int idx = lane >> 1, ch = c0 + 8 * q + (idx & 7);
          if ((lane & 1) == 0 && mt < p.num_m_tiles && ch < p.cout)
            p.bn_part[(static_cast<long long>(mt) * 2 + (idx >> 3)) * p.cout + ch] = v16[0];
        }
      }
      ob = ob + 1 == OB ? 0 : ob + 1;
      slot = slot + 1 == S ? 0 : slot + 1;
    }
    if (nv == 0) release(as);
  }
  if (ST == 2 && p.bn_per_cta) {   // this CTA's 4 rows (one per lane quarter), in tile order
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int ch = (SUBS * j + sub) * 32 + lane;
      if (SUBS * j + sub < NCH && ch < p.cout) {
        const long long row = static_cast<long long>(blockIdx.x) * 4 + q;
        p.bnb_part[(row * 2) * p.cout + ch] = bb_acc[j][0];
        p.bnb_part[(row * 2 + 1) * p.cout + ch] = bb_acc[j][1];
      }
    }
  }
  if (ST == 1 && p.bn_per_cta) {   // this CTA's row: its tiles' statistics, in tile order
    const int idx = lane >> 1;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int ch = (SUBS * j + sub) * 32 + 8 * q + (idx & 7);
      if ((lane & 1) == 0 && SUBS * j + sub < NCH && ch < p.cout)
        p.bn_part[(static_cast<long long>(blockIdx.x) * 2 + (idx >> 3)) * p.cout + ch] = bn_acc[j];
    }
  }
  if (issuer) bulk_wait<0>();
  __syncwarp();
}

// Epilogue role of the fprop kernels (8 warps, two per TMEM lane quarter splitting the tile's
// column chunks): TMEM -> registers -> bias / residual / relu / mask / accumulate -> global.
template <int BN, int CG, int ST = 0>
__device__ __forceinline__ void fprop_epilogue_role(const FpropParams& p, const CUtensorMap* tmY, const CUtensorMap* tmR,
                                                    const CUtensorMap* tmM, uint32_t tmem_base, uint64_t* tfull,
                                                    uint64_t* tempty, uint64_t* inbar, uint8_t* epi, int warp,
                                                    int rank, int unit0, int units) {
  constexpr int CW = BN < 32 ? BN : 32;
  const int lane = lane_id();
  const int per_img = p.tiles_x * p.tiles_y;
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    const int row = q * 32 + lane;
    const int ry = row / p.bw, rx = row - ry * p.bw;
    constexpr int NCH = BN / CW;
    constexpr int NJ = (NCH + 1) / 2;
    if constexpr (CW == 32) {
      if (p.tma_epi) {
        fprop_epilogue_tma<BN, CG, 8, ST>(p, tmY, tmR, tmM, tmem_base, tfull, tempty, inbar, epi, warp, rank, unit0,
                                      units);
        return;
      }
    }
    {
    uint8_t* st = epi + ew * EPI_WARP_BYTES;
    const bool vec = p.vec_ok && !p.y_f32 && (p.cout % 8) == 0;
    using R = CoopRows<CW>;
    int it = 0;
    for (int tile = unit0; tile < p.num_tiles; tile += units, ++it) {
      const int as = it & 1;
      const uint32_t ap = (it >> 1) & 1;
      const int pmt = tile / p.num_n_tiles, nt = tile - pmt * p.num_n_tiles;
      const int mt = pmt * CG + rank;
      const int img = mt / per_img, r = mt - img * per_img;
      const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
      const int yy = ty * p.bh + ry, xx = tx * p.bw + rx;
      const bool valid = img < p.n && yy < p.h && xx < p.w;  // odd pair count: the last odd CTA idles
      const long long pix = (static_cast<long long>(img) * p.h + yy) * p.w + xx;
      R L;
#pragma unroll
      for (int k = 0; k < R::PIECES; ++k) {
        const int rr = q * 32 + k * R::ROWS_PER_IT + lane / R::PIECES;
        const int cy = ty * p.bh + rr / p.bw, cx = tx * p.bw + rr % p.bw;
        L.ok[k] = img < p.n && cy < p.h && cx < p.w;
        L.pix[k] = (static_cast<long long>(img) * p.h + cy) * p.w + cx;
      }
      // prefetch the first global epilogue operand of all of this warp's chunks
      uint4 pre[NJ][R::PIECES];
      const b2h* pbase = p.res ? p.res : p.mask;
      const long long pstride = p.res ? p.res_stride : p.mask_stride;
      if (vec && pbase) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int c0 = nt * BN + (2 * j + half) * CW;
          if (2 * j + half < NCH && c0 < p.cout) coop_prefetch<CW>(pbase, pstride, c0, p.cout, L, pre[j]);
        }
      }
      mbar_wait(&tfull[as], ap);
      tc_fence_after();
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int ch = 2 * j + half;
        if (ch >= NCH) break;  // warp-uniform
        uint32_t cur[CW];
        if constexpr (CW == 32)
          tmem_ld_issue_x32(tbase + ch * CW, cur);
        else
          tmem_ld_issue_x16(tbase + ch * CW, cur);
        tmem_ld_wait();
        float v[CW];
#pragma unroll
        for (int i = 0; i < CW; ++i) v[i] = __uint_as_float(cur[i]);
        const int c0 = nt * BN + ch * CW;
        if (c0 < p.cout) {
          if (vec)
            fprop_epilogue_vec<CW>(p, v, c0, L, st, pbase ? pre[j] : nullptr);
          else if (valid)
            fprop_epilogue_scalar<CW>(p, v, pix, c0);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2)
          mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
        else
          mbar_arrive(&tempty[as]);
      }
    }
    }
}

// EW epilogue warps: 8, or 16 for the TMA epilogue (twice the warps to hide its latency chain)
template <int BN, int KBLK, bool BMN, int CG, int EW, int ST = 0>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    conv_fprop_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                      const __grid_constant__ CUtensorMap tmM, const FpropParams p) {
  using C = FpropCfg<BN, KBLK, BMN, CG>;
  const int STAGES = p.stages;
  constexpr uint32_t LAYOUT = KBLK == 64 ? LAYOUT_SW128 : KBLK == 32 ? LAYOUT_SW64 : LAYOUT_SW32;
  constexpr uint32_t SBO = KBLK * 2 * 8;  // 8 rows of KBLK bf16
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* epi = sB + p.b_region;  // 1 KB aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + p.epi_bytes);
  uint64_t* empty = full + FPROP_MAX_STAGES;
  uint64_t* tfull = empty + FPROP_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;  // two operand-slot barriers per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inbar + 2 * EW);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  // CTA pair: rank 0 issues the MMAs and owns the operand-full / accumulator-empty barriers
  const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], EW * CG);
    }
    for (int s = 0; s < 2 * EW; ++s) mbar_init(&inbar[s], 1);
    if (p.tma_epi) {
      tma_prefetch(&tmY);
      if (p.res) tma_prefetch(&tmR);
      if (p.mask) tma_prefetch(&tmM);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2)
      tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    else
      tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: let the next kernel's CTAs start theirs; wait for our inputs
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.tiles_x * p.tiles_y;
  const int unit0 = blockIdx.x / CG, units = gridDim.x / CG;

  if (warp == 0) {
    {   // converged producer warp: waits and coordinates warp-uniform, one elected lane issues
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = unit0; tile < p.num_tiles; tile += units) {
        const int pmt = tile / p.num_n_tiles, nt = tile - pmt * p.num_n_tiles;
        const int mt = pmt * CG + rank;
        const int img = mt / per_img, r = mt - img * per_img;
        const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
        const int y0 = ty * p.bh, x0 = tx * p.bw, n0 = nt * BN + rank * (BN / CG);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const int tap = kb / p.num_cblk, cb = kb - tap * p.num_cblk;
          const int i = tap / p.kw, j = tap - i * p.kw;
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int ax = x0 * p.in_stride + j * p.dil - p.pad_left, ay = y0 * p.in_stride + i * p.dil - p.pad_top;
          if (!elect_one_sync()) {
            // the other lanes only keep the stage / phase walk
          } else if constexpr (CG == 2) {
            // both CTAs' loads complete on the even CTA's barrier, which expects both halves
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            tma_load_4d_pair(a_dst, &tmA, fb, cb * KBLK, ax, ay, img);
            if constexpr (BMN) {
#pragma unroll
              for (int qq = 0; qq < C::NBC; ++qq)
                tma_load_3d_pair(b_dst + qq * C::B_CHUNK, &tmB, fb, n0 + qq * 64, cb * KBLK, tap);
            } else if (p.b_mode == 2) {
              tma_load_3d_pair(b_dst, &tmB, fb, cb * KBLK, n0, p.taps - 1 - tap);
            } else {
              tma_load_2d_pair(b_dst, &tmB, fb, tap * p.cin_pad + cb * KBLK, n0);
            }
          } else {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_4d(a_dst, &tmA, &full[stage], cb * KBLK, ax, ay, img);
            if constexpr (BMN) {  // master HWIO weights: box (64 co, KBLK ci, 1 tap) per 64 output channels
#pragma unroll
              for (int qq = 0; qq < C::NBC; ++qq)
                tma_load_3d(b_dst + qq * C::B_CHUNK, &tmB, &full[stage], n0 + qq * 64, cb * KBLK, tap);
            } else if (p.b_mode == 2) {  // dgrad from master HWIO: box (KBLK co, BN ci, flipped tap)
              tma_load_3d(b_dst, &tmB, &full[stage], cb * KBLK, n0, p.taps - 1 - tap);
            } else {
              tma_load_2d(b_dst, &tmB, &full[stage], tap * p.cin_pad + cb * KBLK, n0);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // converged warp, elected issuer (see the row-tap kernel): no per-MMA single-thread issue loop
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM * CG, BN, false, BMN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = unit0; tile < p.num_tiles; tile += units, ++it) {
        const int as = it & 1;
        const uint32_t ap = (it >> 1) & 1;
        mbar_wait(&tempty[as], ap ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < KBLK / 16; ++k) {
              const uint64_t ad = make_sdesc(a0 + k * 32, 16, SBO, LAYOUT);
              const uint64_t bd = BMN ? make_sdesc(b0 + k * 2048, C::B_CHUNK, 1024, LAYOUT_SW128)
                                      : make_sdesc(b0 + k * 32, 16, SBO, LAYOUT);
              if constexpr (CG == 2)
                umma_bf16_pair(d, ad, bd, idesc, (kb | k) != 0);
              else
                umma_bf16(d, ad, bd, idesc, (kb | k) != 0);
            }
            if constexpr (CG == 2)
              umma_commit_pair(&empty[stage]);
            else
              umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) {
          if constexpr (CG == 2)
            umma_commit_pair(&tfull[as]);
          else
            umma_commit(&tfull[as]);
        }
        __syncwarp();
      }
    }
  } else {
    if constexpr (EW == 16)
      fprop_epilogue_tma<BN, CG, 16, ST>(p, &tmY, &tmR, &tmM, tmem_base, tfull, tempty, inbar, epi, warp, rank, unit0,
                                     units);
    else
      fprop_epilogue_role<BN, CG, ST>(p, &tmY, &tmR, &tmM, tmem_base, tfull, tempty, inbar, epi, warp, rank, unit0,
                                  units);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ row-window halo fprop
// The narrow-input stem in row-window mode (b2dl_conv_args.window): an 8 x 16-pixel tile needs
// kh tap rows of the window image, i.e. one tall (16 + kh - 1)-row box per 64-channel K half,
// loaded once and addressed per tap row at a 1 KB offset (one SW128 atom).  The
// weights of all tap rows (kh x 64-wide K halves x 64 output channels) stay resident in
// shared memory, so per tile only the tall input boxes move: ~7x less operand traffic than
// streaming one 128-pixel box + weights per (tap row, K half).
constexpr int HALO_BW = 8, HALO_BH = 16, HALO_BN = 64;
constexpr int HALO_BBOX = HALO_BN * 64 * 2;  // one (tap row, K half) weight box: 64 co x 64 k

template <int ST>
__global__ void __launch_bounds__(FPROP_THREADS, 1)
    conv_halo_fprop_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                           const __grid_constant__ CUtensorMap tmM, const FpropParams p) {
  const int taps = p.taps, nh = p.num_cblk;
  const int a_stage = (HALO_BH + taps - 1) * HALO_BW * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sB = smem;
  uint8_t* sA = smem + taps * nh * HALO_BBOX;
  uint8_t* epi = sA + p.stages * a_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + p.epi_bytes);
  uint64_t* empty = full + FPROP_MAX_STAGES;
  uint64_t* tfull = empty + FPROP_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;
  uint64_t* bfull = inbar + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);
    }
    for (int s = 0; s < 16; ++s) mbar_init(&inbar[s], 1);
    mbar_init(bfull, 1);
    tma_prefetch(&tmY);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * HALO_BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: let the next kernel's CTAs start theirs; wait for our inputs
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.tiles_x * p.tiles_y;

  if (warp == 0) {
    {   // converged producer warp, elected issuer
      if (elect_one_sync()) {
        mbar_arrive_expect_tx(bfull, taps * nh * HALO_BBOX);
        for (int i = 0; i < taps; ++i)
          for (int h = 0; h < nh; ++h)
            tma_load_2d(sB + (i * nh + h) * HALO_BBOX, &tmB, bfull, i * p.cin_pad + h * 64, 0);
      }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int img = tile / per_img, r = tile - img * per_img;
        const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
        for (int h = 0; h < nh; ++h) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one_sync()) {
            mbar_arrive_expect_tx(&full[stage], a_stage);
            tma_load_4d(sA + stage * a_stage, &tmA, &full[stage], h * 64, tx * HALO_BW, ty * HALO_BH - p.pad_top,
                        img);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {   // converged warp, elected issuer (see the row-tap kernel)
      constexpr uint32_t idesc = make_idesc_bf16(BM, HALO_BN, false, false);
      mbar_wait(bfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
        const int as = it & 1;
        const uint32_t ap = (it >> 1) & 1;
        mbar_wait(&tempty[as], ap ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * HALO_BN;
        for (int h = 0; h < nh; ++h) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          // descriptors advance by (byte offset >> 4) in their start-address field
          const uint64_t ad0 = make_sdesc(smem_u32(sA + stage * a_stage), 16, 1024, LAYOUT_SW128);
          const uint64_t bd0 = make_sdesc(smem_u32(sB + h * HALO_BBOX), 16, 1024, LAYOUT_SW128);
          if (elect_one_sync()) {
            for (int i = 0; i < taps; ++i) {
              const uint64_t ai = ad0 + ((i * HALO_BW * 128) >> 4);  // tap row i: the box shifted down i rows
              const uint64_t bi = bd0 + ((i * nh * HALO_BBOX) >> 4);
#pragma unroll
              for (int k = 0; k < 4; ++k) umma_bf16(d, ai + 2 * k, bi + 2 * k, idesc, (h | i | k) != 0);
            }
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(&tfull[as]);
        __syncwarp();
      }
    }
  } else {
    fprop_epilogue_role<HALO_BN, 1, ST>(p, &tmY, &tmR, &tmM, tmem_base, tfull, tempty, inbar, epi, warp, 0, blockIdx.x,
                                    gridDim.x);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * HALO_BN);
  }
}

// ------------------------------------------------------------------ row-tap fprop (narrow N)
// Narrow convs (forward N = BN <= 64, e.g. the growth-32 5x5 dense layers of the Tiramisu; dgrads
// up to N = 256 over a narrow K): with one 128-pixel box per (tap, K block) the operand loads, not
// the MMAs, bound the kernel (each input element crosses L2 -> SM kh*kw times for only 2*BN FLOPs
// per byte).  Here an 8 x 16-pixel tile loads, per (column tap j, channel block), ONE tall box of
// 8 x (16 + (kh-1) dil) pixels and the kh row taps address it at i*dil image-row offsets, with the
// kh weight boxes of that column streamed in the same stage: kh times fewer activation loads.
// With resident weights one wide box of (8 + (kw-1) dil) columns serves the column taps as well.
constexpr int RT_BW = 8, RT_BH = 16;

// KB = channels per K block (64, or 32 for 17..32-channel inputs: SW64, 512-byte image rows).  When
// all the weights fit (p.b_region > 0) they are loaded once and stay resident; the stages then carry
// only the tall input boxes.
// CG = 2: a CTA pair (cluster of 2) runs two vertically adjacent tiles as one M = 256 MMA; each CTA
// stages its own tall box and half of the weight rows (BN / 2), and the even CTA issues
// 256 x BN x 16 instructions -- half the MMA issue count per FLOP, which bounds the N = 32 kernel.
template <int BN, int KB, int CG = 1>
__global__ void __launch_bounds__(FPROP_THREADS, 1)
    conv_rowtap_fprop_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                             const __grid_constant__ CUtensorMap tmM, const FpropParams p, int kh) {
  constexpr int ROW = RT_BW * KB * 2;              // bytes per image row of the tall box
  constexpr uint32_t LAYOUT = KB == 64 ? LAYOUT_SW128 : LAYOUT_SW64;
  constexpr uint32_t SBO = 8 * KB * 2;             // 8 rows of KB bf16
  const int row_b = p.rt_cs ? p.rt_cs * KB * 2 : ROW;   // bytes per image row of the staged box
  const int a_box = (RT_BH + (kh - 1) * p.dil) * row_b;        // bytes the TMA box delivers
  const int a_stage = (a_box + 1023) / 1024 * 1024;               // 1 KB-aligned stage buffers
  const int b_box = (BN / CG) * KB * 2;          // this CTA's weight rows of one (tap, K block)
  const bool resident = p.b_region > 0;
  const int stage_bytes = a_stage + (resident ? 0 : kh * b_box);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sW = smem;                                // resident weights [tap][cblk] boxes
  uint8_t* sS = smem + (resident ? p.b_region : 0);  // stages: [A tall box][kh weight boxes]
  uint8_t* epi = sS + p.stages * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + p.epi_bytes);
  uint64_t* empty = full + FPROP_MAX_STAGES;
  uint64_t* tfull = empty + FPROP_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* inbar = tempty + 2;
  uint64_t* bfull = inbar + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8 * CG);
    }
    for (int s = 0; s < 16; ++s) mbar_init(&inbar[s], 1);
    mbar_init(bfull, 1);
    tma_prefetch(&tmY);
    if (p.res) tma_prefetch(&tmR);
    if (p.mask) tma_prefetch(&tmM);
    fence_barrier_init();
  }
  constexpr uint32_t TCOLS = tmem_cols_for(2 * BN);
  if (warp == 1) {
    if constexpr (CG == 2)
      tmem_alloc_pair(tmem_slot, TCOLS);
    else
      tmem_alloc(tmem_slot, TCOLS);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.tiles_x * p.tiles_y;
  // stages per tile: (column tap, channel block); with the wide box and resident weights one box
  // per channel block serves every column tap (descriptor start + j * dil pixels)
  const bool reuse = p.rt_cs && resident;
  const int nsteps = reuse ? p.num_cblk : p.kw * p.num_cblk;
  const int unit0 = blockIdx.x / CG, units = gridDim.x / CG;
  const int n0 = rank * (BN / CG);        // this CTA's weight rows

  if (warp == 0) {
    {   // converged producer warp: waits and coordinates warp-uniform, one elected lane issues
      if (resident && elect_one_sync()) {
        if constexpr (CG == 2) {   // both halves complete on the even CTA's barrier
          if (rank == 0) mbar_arrive_expect_tx(bfull, 2 * p.taps * p.num_cblk * b_box);
          const uint32_t fb = mapa_shared(smem_u32(bfull), 0);
          for (int t = 0; t < p.taps; ++t)
            for (int cb = 0; cb < p.num_cblk; ++cb)
              tma_load_2d_pair(sW + (t * p.num_cblk + cb) * b_box, &tmB, fb, t * p.cin_pad + cb * KB, n0);
        } else {
          mbar_arrive_expect_tx(bfull, p.taps * p.num_cblk * b_box);
          for (int t = 0; t < p.taps; ++t)
            for (int cb = 0; cb < p.num_cblk; ++cb)
              tma_load_2d(sW + (t * p.num_cblk + cb) * b_box, &tmB, bfull, t * p.cin_pad + cb * KB, 0);
        }
      }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = unit0; tile < p.num_tiles; tile += units) {
        const int mt = tile * CG + rank;   // an odd last pair's second tile is past the end: zero fill
        const int img = mt / per_img, r = mt - img * per_img;
        const int ty = r / p.tiles_x, tx = r - ty * p.tiles_x;
        for (int st = 0; st < nsteps; ++st) {
          const int j = reuse ? 0 : st / p.num_cblk, cb = st - j * p.num_cblk;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* dst = sS + stage * stage_bytes;
          const int ax = tx * RT_BW + (p.rt_cs ? 0 : j * p.dil) - p.pad_left, ay = ty * RT_BH - p.pad_top;
          if (elect_one_sync()) {
            if constexpr (CG == 2) {
              if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (stage_bytes - (a_stage - a_box)));
              const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
              tma_load_4d_pair(dst, &tmA, fb, cb * KB, ax, ay, img);
              if (!resident)
                for (int i = 0; i < kh; ++i)
                  tma_load_2d_pair(dst + a_stage + i * b_box, &tmB, fb, (i * p.kw + j) * p.cin_pad + cb * KB, n0);
            } else {
              mbar_arrive_expect_tx(&full[stage], stage_bytes - (a_stage - a_box));
              tma_load_4d(dst, &tmA, &full[stage], cb * KB, ax, ay, img);
              if (!resident)
                for (int i = 0; i < kh; ++i)
                  tma_load_2d(dst + a_stage + i * b_box, &tmB, &full[stage], (i * p.kw + j) * p.cin_pad + cb * KB,
                              0);
            }
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp walks the schedule (waits, descriptors: warp-uniform); one elected lane issues
    // the MMAs and their commits -- no per-instruction single-thread issue loop around each UTCHMMA
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(BM * CG, BN, false, false);
      if (resident) mbar_wait(bfull, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = unit0; tile < p.num_tiles; tile += units, ++it) {
        const int as = it & 1;
        const uint32_t ap = (it >> 1) & 1;
        mbar_wait(&tempty[as], ap ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int st = 0; st < nsteps; ++st) {
          const int j0 = reuse ? 0 : st / p.num_cblk, cb = st - j0 * p.num_cblk;
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sS + stage * stage_bytes);
          if (elect_one_sync()) {
            for (int jj = 0; jj < (reuse ? p.kw : 1); ++jj) {
              const int j = j0 + jj;
              // wide box: column tap j starts j * dil pixels (KB * 2 bytes each) into every box row;
              // the swizzle follows the address bits, so no descriptor base offset is involved
              const int cs = p.rt_cs ? j * p.dil : 0;
              const uint64_t ad0 = make_sdesc(a0 + cs * KB * 2, 16, p.rt_cs ? row_b : SBO, LAYOUT);
              for (int i = 0; i < kh; ++i) {
                // row tap i: the tall box shifted down i*dil image rows (whole swizzle atoms);
                // descriptors advance by (byte offset >> 4) in their start-address field
                const uint64_t ai = ad0 + ((i * p.dil * row_b) >> 4);
                const uint32_t b0 = resident ? smem_u32(sW + ((i * p.kw + j) * p.num_cblk + cb) * b_box)
                                             : a0 + a_stage + i * b_box;
                const uint64_t bi = make_sdesc(b0, 16, SBO, LAYOUT);
#pragma unroll
                for (int k = 0; k < KB / 16; ++k) {
                  if constexpr (CG == 2)
                    umma_bf16_pair(d, ai + 2 * k, bi + 2 * k, idesc, (st | jj | i | k) != 0);
                  else
                    umma_bf16(d, ai + 2 * k, bi + 2 * k, idesc, (st | jj | i | k) != 0);
                }
              }
            }
            if constexpr (CG == 2)
              umma_commit_pair(&empty[stage]);
            else
              umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) {
          if constexpr (CG == 2)
            umma_commit_pair(&tfull[as]);
          else
            umma_commit(&tfull[as]);
        }
        __syncwarp();
      }
    }
  } else {
    fprop_epilogue_role<BN, CG>(p, &tmY, &tmR, &tmM, tmem_base, tfull, tempty, inbar, epi, warp, rank, unit0,
                                units);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_pair(tmem_base, TCOLS);
    else
      tmem_dealloc(tmem_base, TCOLS);
  }
}

// ------------------------------------------------------------------ wgrad
// D[(tap, ci)][co] = sum_p x[p + off(tap), ci] * dy[p, co].  A CTA tile covers NACC x 128
// (tap, ci) rows -- NXC x-chunks of XW channels in NACC TMEM accumulators -- against BN output
// channels over KP-pixel K blocks.  XW = 64: SW128 MN-major chunks, two accumulators sharing
// every dy stage (a third less operand traffic per FLOP than one 128-row tile).  XW = 16 (the
// 16-channel input of the stem): SW32 chunks, no zero-padded channels, 256-pixel K blocks so
// the 49 per-tap boxes are few and large.
// The epilogue warps, idle during the main loop, also fold the dy tiles of the row-0 tile
// into per-channel column sums: the bias gradient (ops.py:172-175) costs no extra pass.
template <int BN, int XW>
struct WgradCfg {
  static constexpr int KP = XW == 16 ? 256 : 64;          // pixels per K block
  static constexpr int NACC = XW == 16 ? 1 : 2;           // 128-row TMEM accumulators
  static constexpr int XCHUNK = XW * KP * 2;              // XW channels x KP pixels, bf16
  static constexpr int DCHUNK = 64 * KP * 2;              // 64 out channels x KP pixels
  static constexpr int NXC = NACC * 128 / XW;             // x-chunks per tile
  static constexpr int NB = BN < 64 ? 1 : BN / 64;
  static constexpr int A_BYTES = NXC * XCHUNK;
  static constexpr int B_BYTES = NB * DCHUNK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (SMEM_BUDGET / STAGE_BYTES) > 8 ? 8 : (SMEM_BUDGET / STAGE_BYTES);
  static constexpr uint32_t TMEM_COLS = tmem_cols_for(NACC * BN);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int CW = BN < 32 ? BN : 32;
  static constexpr uint32_t XLAYOUT = XW == 64 ? LAYOUT_SW128 : LAYOUT_SW32;
  static constexpr uint32_t XSBO = 8 * XW * 2;            // 8 pixel rows
  static constexpr uint32_t XKSTEP = 16 * XW * 2;         // 16 pixel rows = one UMMA K step
  static constexpr int KSTEPS = KP / 16;
};

struct WgradParams {
  int n, h, w;
  int bwk, bhk, pbx, pby, num_pb;
  int kw, dil, pad_top, pad_left;
  int cblk, num_x_chunks;
  int m_tiles, n_tiles, splits, num_tiles, pb_per_split;
  int cin, cout;
  long long krows;  // taps * cin
  float* ws;        // [splits][krows][cout]
  float* bsum;      // [splits][cout] partial column sums of dy, or nullptr
  int xg;           // x chunks per TMA op (5-D map, channel blocks as an outer box dim); 0 = 4-D map
  int dyg;          // dy chunks per TMA op (5-D map); 0 = 4-D map
};

template <int BN, int XW>
__global__ void __launch_bounds__(192, 1)
    conv_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                      const WgradParams p) {
  using C = WgradCfg<BN, XW>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmDY);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 epilogue warps (dy column sums)
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: let the next kernel's CTAs start theirs; wait for our inputs
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.pbx * p.pby;

  if (warp == 0) {
    {   // converged producer warp, elected issuer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        const int mt = tile % p.m_tiles;
        const int rest = tile / p.m_tiles;
        const int nt = rest % p.n_tiles, split = rest / p.n_tiles;
        const int pb_lo = split * p.pb_per_split, pb_hi = min(p.num_pb, pb_lo + p.pb_per_split);
        const int c_lo = mt * C::NXC;
        const int nxc = min(C::NXC, p.num_x_chunks - c_lo);
        const int tx_bytes = C::B_BYTES + nxc * C::XCHUNK;
        for (int pb = pb_lo; pb < pb_hi; ++pb) {
          const int img = pb / per_img, r = pb - img * per_img;
          const int by = r / p.pbx, bx = r - by * p.pbx;
          const int x0 = bx * p.bwk, y0 = by * p.bhk;
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one_sync()) {
          mbar_arrive_expect_tx(&full[stage], tx_bytes);
          // few large TMA ops: a 5-D map loads xg (dyg) 64-channel chunks of one tap per op
          const int xstep = p.xg ? p.xg : 1;
          for (int c = 0; c < nxc; c += xstep) {
            const int chunk = c_lo + c;
            const int tap = chunk / p.cblk, cb = chunk - tap * p.cblk;
            const int i = tap / p.kw, j = tap - i * p.kw;
            if (p.xg)
              tma_load_5d(sA + stage * C::A_BYTES + c * C::XCHUNK, &tmX, &full[stage], 0,
                          x0 + j * p.dil - p.pad_left, y0 + i * p.dil - p.pad_top, img, cb);
            else
              tma_load_4d(sA + stage * C::A_BYTES + c * C::XCHUNK, &tmX, &full[stage], cb * XW,
                          x0 + j * p.dil - p.pad_left, y0 + i * p.dil - p.pad_top, img);
          }
          if (p.dyg) {
            tma_load_5d(sB + stage * C::B_BYTES, &tmDY, &full[stage], 0, x0, y0, img, nt * BN / 64);
          } else {
#pragma unroll
            for (int qq = 0; qq < C::NB; ++qq)
              tma_load_4d(sB + stage * C::B_BYTES + qq * C::DCHUNK, &tmDY, &full[stage], nt * BN + qq * 64, x0, y0,
                          img);
          }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {   // converged warp, elected issuer (see the row-tap fprop kernel)
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, true, true);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
        const int mt = tile % p.m_tiles;
        const int rest = tile / p.m_tiles;
        const int split = rest / p.n_tiles;
        const int pb_lo = split * p.pb_per_split, pb_hi = min(p.num_pb, pb_lo + p.pb_per_split);
        const bool second = C::NACC == 2 && (mt * C::NXC + C::NXC / 2) < p.num_x_chunks;
        mbar_wait(tempty, (it & 1) ^ 1);
        tc_fence_after();
        for (int pb = pb_lo; pb < pb_hi; ++pb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < C::KSTEPS; ++k) {
              const uint32_t acc = (pb != pb_lo) || (k != 0);
              const uint64_t bd = make_sdesc(b0 + k * 2048, C::DCHUNK, 1024, LAYOUT_SW128);
              const uint64_t ad0 = make_sdesc(a0 + k * C::XKSTEP, C::XCHUNK, C::XSBO, C::XLAYOUT);
              umma_bf16(tmem_base, ad0, bd, idesc, acc);
              if (second) {
                const uint64_t ad1 =
                    make_sdesc(a0 + (C::NXC / 2) * C::XCHUNK + k * C::XKSTEP, C::XCHUNK, C::XSBO, C::XLAYOUT);
                umma_bf16(tmem_base + BN, ad1, bd, idesc, acc);
              }
            }
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one_sync()) umma_commit(tfull);
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    // column-sum ownership: thread et sums output channels 2*et, 2*et+1 of the dy tile
    const int cs_chunk = et / 32, cs_word = et % 32;
    const bool cs_active = 2 * et < (C::NB * 64 < BN ? C::NB * 64 : BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++it) {
      const int mt = tile % p.m_tiles;
      const int rest = tile / p.m_tiles;
      const int nt = rest % p.n_tiles, split = rest / p.n_tiles;
      const int pb_lo = split * p.pb_per_split, pb_hi = min(p.num_pb, pb_lo + p.pb_per_split);
      // every m-tile of a (split, n-tile) group sums an interleaved 1/m_tiles of the K blocks
      const bool do_sum = p.bsum != nullptr && cs_active;
      float s0 = 0.f, s1 = 0.f;
      for (int pb = pb_lo; pb < pb_hi; ++pb) {
        mbar_wait(&full[stage], phase);
        if (do_sum && (pb - pb_lo) % p.m_tiles == mt) {
          // dy chunk: KP pixel rows of 128 B (64 channels), 16-byte units XOR-swizzled by row % 8
          const uint8_t* base = sB + stage * C::B_BYTES + cs_chunk * C::DCHUNK;
          const int unit = cs_word >> 2, sub = (cs_word & 3) * 4;
#pragma unroll 8
          for (int r = 0; r < C::KP; ++r) {
            const uint32_t v = *reinterpret_cast<const uint32_t*>(base + r * 128 + ((unit ^ (r & 7)) << 4) + sub);
            s0 += bf16lo(v);
            s1 += bf16hi(v);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (do_sum) {
        const int co = nt * BN + 2 * et;
        float* dst = p.bsum + (static_cast<long long>(split) * p.m_tiles + mt) * p.cout;
        if (co < p.cout) dst[co] = s0;
        if (co + 1 < p.cout) dst[co + 1] = s1;
      }
      mbar_wait(tfull, it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int hh = 0; hh < C::NACC; ++hh) {
        const int row = hh * 128 + q * 32 + lane;  // tile row = (x-chunk, channel within chunk)
        const int chunk = mt * C::NXC + row / XW;
        const int tap = chunk / p.cblk;
        const int ci = (chunk - tap * p.cblk) * XW + (row % XW);
        const bool valid = chunk < p.num_x_chunks && ci < p.cin;
        float* dst =
            p.ws + (static_cast<long long>(split) * p.krows + static_cast<long long>(tap) * p.cin + ci) * p.cout;
#pragma unroll 1
        for (int ch = 0; ch < BN / C::CW; ++ch) {
          float v[32];
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + hh * BN + ch * C::CW;
          if constexpr (C::CW == 32)
            tmem_ld_32x32b_x32(taddr, v);
          else
            tmem_ld_32x32b_x16(taddr, v);
          const int c0 = nt * BN + ch * C::CW;
          if (valid && c0 < p.cout) {
            const int nvalid = min(C::CW, p.cout - c0);
            if (nvalid == C::CW && (p.cout & 3) == 0) {
#pragma unroll
              for (int e = 0; e < C::CW; e += 4)
                *reinterpret_cast<float4*>(dst + c0 + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < C::CW; ++e)
                if (e < nvalid) dst[c0 + e] = v[e];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// batched segment reduction (deterministic, fixed order over parts)
// ------------------------------------------------------------------ row-window halo wgrad
// dW[(tap row i, k)][co] = sum_p xwin[p + i rows][k] * dy[p][co] for the row-window stem.  A
// K block is an 8 x 16-pixel block: one tall (16 + kh - 1)-row x box per 64-wide K half serves
// all kh tap rows (row offset i = 1 KB), against one dy box.  kh accumulators of 128 (k) x 64
// (co) live in TMEM for the CTA's whole pixel range (split-K over CTAs, one partial each).
constexpr int HW_BW = 8, HW_BH = 16;  // pixel block (one K block = 128 pixels)

__global__ void __launch_bounds__(192, 1)
    conv_halo_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                           const WgradParams p, int taps, int stages) {
  const int xbox = (HW_BH + taps - 1) * HW_BW * 128;  // one tall x box (64-wide K half)
  const int stage_bytes = 2 * xbox + HW_BW * HW_BH * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + FPROP_MAX_STAGES;
  uint64_t* tfull = empty + FPROP_MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* bred = reinterpret_cast<float*>(tmem_slot + 4);  // [64] bias half-sums

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int split = blockIdx.x;
  const int pb_lo = split * p.pb_per_split;
  const int pb_hi = min(p.num_pb, pb_lo + p.pb_per_split);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmDY);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 epilogue warps (dy column sums)
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done: let the next kernel's CTAs start theirs; wait for our inputs
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.pbx * p.pby;

  if (warp == 0) {
    {   // converged producer warp, elected issuer
      int stage = 0;
      uint32_t phase = 0;
      for (int pb = pb_lo; pb < pb_hi; ++pb) {
        const int img = pb / per_img, r = pb - img * per_img;
        const int by = r / p.pbx, bx = r - by * p.pbx;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one_sync()) {
          mbar_arrive_expect_tx(&full[stage], stage_bytes);
          uint8_t* st = smem + stage * stage_bytes;
          for (int h = 0; h < 2; ++h)
            tma_load_4d(st + h * xbox, &tmX, &full[stage], h * 64, bx * HW_BW, by * HW_BH - p.pad_top, img);
          tma_load_4d(st + 2 * xbox, &tmDY, &full[stage], 0, bx * HW_BW, by * HW_BH, img);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    {   // converged warp, elected issuer (see the row-tap fprop kernel)
      constexpr uint32_t idesc = make_idesc_bf16(128, 64, true, true);
      int stage = 0;
      uint32_t phase = 0;
      for (int pb = pb_lo; pb < pb_hi; ++pb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t x0 = smem_u32(smem + stage * stage_bytes);
        const uint64_t ad0 = make_sdesc(x0, xbox, 1024, LAYOUT_SW128);
        const uint64_t bd0 = make_sdesc(x0 + 2 * xbox, 16384, 1024, LAYOUT_SW128);
        const uint32_t acc = pb > pb_lo;
        if (elect_one_sync()) {
          for (int i = 0; i < taps; ++i) {
            const uint64_t ai = ad0 + ((i * HW_BW * 128) >> 4);
#pragma unroll
            for (int k = 0; k < HW_BW * HW_BH / 16; ++k)  // 16 pixels (2 KB) per K step
              umma_bf16(tmem_base + i * 64, ai + k * 128, bd0 + k * 128, idesc, acc | k);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one_sync()) umma_commit(tfull);
      __syncwarp();
    }
  } else {
    const int t = threadIdx.x - 64;  // 0..127
    const int co = t & 63, ph = t >> 6;
    float bs = 0.f;
    int stage = 0;
    uint32_t phase = 0;
    for (int pb = pb_lo; pb < pb_hi; ++pb) {
      mbar_wait(&full[stage], phase);
      if (p.bsum) {
        const uint8_t* dyt = smem + stage * stage_bytes + 2 * xbox;
#pragma unroll 8
        for (int px = ph * 64; px < ph * 64 + 64; ++px)
          bs += h_to_f(*reinterpret_cast<const b2h*>(
              dyt + px * 128 + ((((co >> 3) ^ (px & 7))) << 4) + (co & 7) * 2));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    // bias partial of this split: the two pixel halves meet in shared memory
    if (ph == 1) bred[co] = bs;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (ph == 0 && p.bsum && co < p.cout) p.bsum[static_cast<long long>(split) * p.cout + co] = bs + bred[co];
    // weight partial: lane = k row of the 128-row accumulators
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int k = q * 32 + lane;
    float* out = p.ws + static_cast<long long>(split) * p.krows * p.cout;
    for (int i = 0; i < taps; ++i) {
      float v[64];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + i * 64, v);
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + i * 64 + 32, v + 32);
      if (k < p.cin) {
        float* row = out + (static_cast<long long>(i) * p.cin + k) * p.cout;
        if (p.cout == 64) {
#pragma unroll
          for (int c = 0; c < 64; c += 4) *reinterpret_cast<float4*>(row + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c < p.cout) row[c] = v[c];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------------------ row-tap wgrad (narrow N)
// dW[(i, j, ci)][co] for narrow outputs (cout <= 64: the growth-32 dense layers, 3x3 64-channel
// convs): a CTA owns two (column tap j, 64-channel block) combinations -- the two 64-row halves of a 128-row M tile, LBO =
// one tall box -- over a range of 8 x 16-pixel K blocks, with one TMEM accumulator per tap row i.
// Per K block it loads two tall x boxes (16 + (kh-1) dil rows) and one dy box, and every tap row
// reads the tall boxes at an i*dil KB offset: kh times fewer x loads than a box per tap.  Partial
// layout = the generic wgrad's ([split][tap][cin][cout], bias sums [split][cout] from tile 0).
template <int BN>
__global__ void __launch_bounds__(192, 1)
    conv_rowtap_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmDY,
                             const WgradParams p, int kh, int stages, int tiles) {
  const int xbox = (HW_BH + (kh - 1) * p.dil) * HW_BW * 128;  // one tall x box (64 channels)
  const int stage_bytes = 2 * xbox + HW_BW * HW_BH * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + FPROP_MAX_STAGES;
  uint64_t* tfull = empty + FPROP_MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* bred = reinterpret_cast<float*>(tmem_slot + 4);  // [64] bias half-sums

  const int warp = threadIdx.x >> 5;
  const int lane = lane_id();
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int ncombo = p.kw * p.cblk;   // (column tap, channel block) combinations, two per tile
  const int c0 = 2 * tile, nh = c0 + 1 < ncombo ? 2 : 1;
  const int pb_lo = split * p.pb_per_split;
  const int pb_hi = min(p.num_pb, pb_lo + p.pb_per_split);
  const bool do_bias = p.bsum != nullptr && tile == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmDY);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + 4);  // MMA commit + the 4 epilogue warps (dy column sums)
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  constexpr int COLS = 512;
  if (warp == 1) tmem_alloc(tmem_slot, COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();
  const int per_img = p.pbx * p.pby;

  if (warp == 0) {
    {   // converged producer warp, elected issuer
      int stage = 0;
      uint32_t phase = 0;
      for (int pb = pb_lo; pb < pb_hi; ++pb) {
        const int img = pb / per_img, r = pb - img * per_img;
        const int by = r / p.pbx, bx = r - by * p.pbx;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one_sync()) {
          mbar_arrive_expect_tx(&full[stage], stage_bytes - (2 - nh) * xbox);
          uint8_t* st = smem + stage * stage_bytes;
          for (int h = 0; h < nh; ++h) {   // a missing second half computes rows nobody writes back
            const int jj = (c0 + h) / p.cblk, cb = (c0 + h) - jj * p.cblk;
            tma_load_4d(st + h * xbox, &tmX, &full[stage], cb * 64, bx * HW_BW + jj * p.dil - p.pad_left,
                        by * HW_BH - p.pad_top, img);
          }
          tma_load_4d(st + 2 * xbox, &tmDY, &full[stage], 0, bx * HW_BW, by * HW_BH, img);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    {   // converged warp, elected issuer (see the row-tap fprop kernel)
      constexpr uint32_t idesc = make_idesc_bf16(128, BN, true, true);
      int stage = 0;
      uint32_t phase = 0;
      for (int pb = pb_lo; pb < pb_hi; ++pb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t x0 = smem_u32(smem + stage * stage_bytes);
        const uint64_t ad0 = make_sdesc(x0, xbox, 1024, LAYOUT_SW128);
        const uint64_t bd0 = make_sdesc(x0 + 2 * xbox, 16384, 1024, LAYOUT_SW128);
        const uint32_t acc = pb > pb_lo;
        if (elect_one_sync()) {
          for (int i = 0; i < kh; ++i) {
            const uint64_t ai = ad0 + ((i * p.dil * HW_BW * 128) >> 4);
#pragma unroll
            for (int k = 0; k < HW_BW * HW_BH / 16; ++k)  // 16 pixels (2 KB) per K step
              umma_bf16(tmem_base + i * BN, ai + k * 128, bd0 + k * 128, idesc, acc | k);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one_sync()) umma_commit(tfull);
      __syncwarp();
    }
  } else {
    const int t = threadIdx.x - 64;  // 0..127
    const int co = t & 63, ph = t >> 6;
    float bs = 0.f;
    int stage = 0;
    uint32_t phase = 0;
    for (int pb = pb_lo; pb < pb_hi; ++pb) {
      mbar_wait(&full[stage], phase);
      if (do_bias) {
        const uint8_t* dyt = smem + stage * stage_bytes + 2 * xbox;
#pragma unroll 8
        for (int px = ph * 64; px < ph * 64 + 64; ++px)
          bs += h_to_f(*reinterpret_cast<const b2h*>(
              dyt + px * 128 + ((((co >> 3) ^ (px & 7))) << 4) + (co & 7) * 2));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (ph == 1) bred[co] = bs;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (ph == 0 && do_bias && co < p.cout) p.bsum[static_cast<long long>(split) * p.cout + co] = bs + bred[co];
    // weight partial: TMEM lane = (half, channel) row of the 128-row accumulators
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int cmb = c0 + row / 64;
    const int j = cmb / p.cblk;
    const int ci = (cmb - j * p.cblk) * 64 + (row & 63);
    float* out = p.ws + static_cast<long long>(split) * p.krows * p.cout;
    for (int i = 0; i < kh; ++i) {
      float v[BN];
      if constexpr (BN == 64) {
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + i * BN, v);
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + i * BN + 32, v + 32);
      } else {
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + i * BN, v);
      }
      if (cmb < ncombo && ci < p.cin) {
        float* dst = out + (static_cast<long long>(i * p.kw + j) * p.cin + ci) * p.cout;
        if (p.cout == BN) {
#pragma unroll
          for (int c = 0; c < BN; c += 4) *reinterpret_cast<float4*>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < BN; ++c)
            if (c < p.cout) dst[c] = v[c];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, COLS);
  }
}

__global__ void reduce_segments_kernel(const b2dl_segment* __restrict__ segs, float* __restrict__ base) {
  const b2dl_segment sg = segs[blockIdx.y];
  float* dst = base + sg.dst_off;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const bool vec = (sg.n & 3) == 0 && ((reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (sg.parts >= 16 && sg.n <= (vec ? 16384 : 4096) && blockDim.x == 256) {
    // short rows, many partials (bias column sums: splits x m-tiles rows; the head's 4 x #SMs
    // parts): G = 256 / cols thread groups each sum every G-th partial of a column, then group 0
    // folds the G group sums in order -- a fixed tree (deterministic) with G independent load
    // chains instead of one
    __shared__ float4 red[256];
    const long long nu = vec ? sg.n >> 2 : sg.n;   // 16-byte or 4-byte units per row
    int cols = sg.parts >= 64 ? 8 : 32;
    while (cols > 1 && cols / 2 >= nu) cols >>= 1;
    const int groups = 256 / cols;
    const int col = threadIdx.x % cols, g = threadIdx.x / cols;
    const float4* src4 = reinterpret_cast<const float4*>(sg.src);
    float4* dst4 = reinterpret_cast<float4*>(dst);
    for (long long c0 = static_cast<long long>(blockIdx.x) * cols; c0 < nu; c0 += static_cast<long long>(gridDim.x) * cols) {
      const long long i = c0 + col;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < nu) {
#pragma unroll 4
        for (int k = g; k < sg.parts; k += groups) {
          if (vec) {
            const float4 v = __ldcs(src4 + k * nu + i);
            s.x += v.x;
            s.y += v.y;
            s.z += v.z;
            s.w += v.w;
          } else {
            s.x += __ldcs(sg.src + k * nu + i);
          }
        }
      }
      red[threadIdx.x] = s;
      __syncthreads();
      if (g == 0 && i < nu) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sg.accumulate) {
          if (vec) t = dst4[i];
          else t.x = dst[i];
        }
        for (int u = 0; u < groups; ++u) {
          const float4 v = red[u * cols + col];
          t.x += v.x;
          t.y += v.y;
          t.z += v.z;
          t.w += v.w;
        }
        if (vec) dst4[i] = t;
        else dst[i] = t.x;
      }
      __syncthreads();
    }
    return;
  }
  if (vec) {
    // 16-byte lanes, 8 partial rows in flight per thread (same per-element summation order)
    const long long n4 = sg.n >> 2;
    const float4* src4 = reinterpret_cast<const float4*>(sg.src);
    float4* dst4 = reinterpret_cast<float4*>(dst);
    for (long long i = t0; i < n4; i += stride) {
      float4 s = sg.accumulate ? dst4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      int k = 0;
      for (; k + 8 <= sg.parts; k += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src4 + (k + u) * n4 + i);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s.x += v[u].x;
          s.y += v[u].y;
          s.z += v[u].z;
          s.w += v[u].w;
        }
      }
      for (; k < sg.parts; ++k) {
        const float4 v = __ldcs(src4 + k * n4 + i);
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      dst4[i] = s;
    }
    return;
  }
  for (long long i = t0; i < sg.n; i += stride) {
    float s = sg.accumulate ? dst[i] : 0.f;
    const float* src = sg.src + i;
    int k = 0;
    for (; k + 4 <= sg.parts; k += 4) {
      const float a = __ldg(src + (k + 0) * sg.n), b = __ldg(src + (k + 1) * sg.n);
      const float c = __ldg(src + (k + 2) * sg.n), d = __ldg(src + (k + 3) * sg.n);
      s += a;
      s += b;
      s += c;
      s += d;
    }
    for (; k < sg.parts; ++k) s += __ldg(src + k * sg.n);
    dst[i] = s;
  }
}

// out[c] (+)= sum_s part[s][c]   (fixed order)
__global__ void bias_reduce_kernel(const float* __restrict__ part, int splits, int c, float* __restrict__ out,
                                   int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= c) return;
  float s = accumulate ? out[i] : 0.f;
  for (int k = 0; k < splits; ++k) s += part[static_cast<long long>(k) * c + i];
  out[i] = s;
}

// dw[k][co] (+)= sum_s ws[s][k][co]   (fixed summation order -> deterministic)
__global__ void wgrad_reduce_kernel(const float* __restrict__ ws, float* __restrict__ dw, long long total,
                                    int splits, int accumulate) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = accumulate ? dw[i] : 0.f;
    for (int k = 0; k < splits; ++k) s += ws[k * total + i];
    dw[i] = s;
  }
}

// ------------------------------------------------------------------ host side
struct FpropMaps {
  CUtensorMap a, b, y, r, m;
};

// Development knobs (defaults are the measured choice): B2DL_EW16_NOPS = most epilogue operands
// for which 16 epilogue warps are used; B2DL_EPI_SLOTS_<EW>_<nops> = operand slots.
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && e[0] ? atoi(e) : dflt;
}
static int ew16_max_nops() {
  static const int v = env_int("B2DL_EW16_NOPS", 2);
  return v;
}
// B2DL_EPI_PW: per-warp TMA epilogue boxes (fprop_epilogue_tma)
static bool epi_pw_enabled() {
  static const int v = env_int("B2DL_EPI_PW", 1);
  return v != 0;
}
static int epi_obufs_for(int ew, int nops) {
  static int cache[2][4] = {{-1, -1, -1, -1}, {-1, -1, -1, -1}};
  int& c = cache[ew == 16][nops & 3];
  if (c < 0) {
    char name[40];
    snprintf(name, sizeof(name), "B2DL_EPI_OBUFS_%d_%d", ew, nops);
    c = std::max(2, std::min(4, env_int(name, 2)));
  }
  return c;
}
static int epi_slots_for(int ew, int nops) {
  static int cache[2][4] = {{-1, -1, -1, -1}, {-1, -1, -1, -1}};
  int& c = cache[ew == 16][nops & 3];
  if (c < 0) {
    char name[40];
    snprintf(name, sizeof(name), "B2DL_EPI_SLOTS_%d_%d", ew, nops);
    // 16 warps x 2 operands: one slot (no prefetch) -- the 4 sub-groups' buffers otherwise leave
    // the main loop too few stages (measured on the 1/8-resolution 1x1 dgrads: 107 -> 95 us)
    c = std::max(1, std::min(EPI_MAX_SLOTS, env_int(name, ew == 16 && nops >= 2 ? 1 : 2)));
  }
  return c;
}

template <int BN, int KBLK, bool BMN, int CG, int EW = 8, int ST = 0>
static int launch_fprop(const FpropMaps& t, FpropParams p, cudaStream_t st) {
  using C = FpropCfg<BN, KBLK, BMN, CG>;
  auto kern = conv_fprop_kernel<BN, KBLK, BMN, CG, EW, ST>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) != cudaSuccess)
      return B2DL_E_CUDA;
    attr_set = true;
  }
  if (C::CW != 32) p.tma_epi = 0;
  if (p.y_phase && !p.tma_epi) return B2DL_E_VALUE;
  p.epi_nops = p.tma_epi ? (p.res != nullptr) + (p.mask != nullptr) + (p.accumulate != 0) : 0;
  // operand prefetch depth (slots - 1 chunks ahead).  Measured: a third slot does not speed up
  // the epilogue-bound 1x1 layers (their chunks wait on instruction latency, not on the loads)
  // and costs operand stages, so two it is.
  p.epi_slots = epi_slots_for(EW, p.epi_nops);
  if (!p.tma_epi || ST == 1) p.epi_pw = 0;
  if (p.epi_pw) p.epi_slots = std::min(p.epi_slots, 2);   // two operand barriers per epilogue warp
  p.epi_obufs = p.epi_pw ? epi_obufs_for(EW, p.epi_nops) : 2;
  p.dbg_epi = env_int("B2DL_DBG_EPI", 0);
  p.epi_bytes = p.tma_epi ? (EW / 4) * epi_sub_bytes(p.epi_nops, p.epi_slots, p.epi_obufs) : EPI_LEGACY_BYTES;
  if (p.bn_part && !p.tma_epi) return B2DL_E_VALUE;
  // deepest operand pipeline that fits beside the epilogue buffers
  p.stages = 1;
  for (int s = FPROP_MAX_STAGES; s >= 1; --s) {
    const int b_region = (s * C::B_BYTES + 1023) / 1024 * 1024;
    if (s * C::A_BYTES + b_region + p.epi_bytes + SMEM_FIXED <= SMEM_MAX) {
      p.stages = s;
      break;
    }
  }
  p.b_region = (p.stages * C::B_BYTES + 1023) / 1024 * 1024;
  const int smem = p.stages * C::A_BYTES + p.b_region + p.epi_bytes + SMEM_FIXED;
  const int grid = CG * std::min(p.num_tiles, num_sms() / CG);
  p.bn_per_cta = p.num_n_tiles == 1;   // must match b2dl_conv_fprop_bn_rows
  const int rc = launch_tc(kern, grid, 64 + 32 * EW, smem, st, CG, t.a, t.b, t.y, t.r, t.m, p);
  return rc ? rc : check_launch();
}

template <int BN, int XW>
static int launch_wgrad(const CUtensorMap& tx, const CUtensorMap& tdy, const WgradParams& p, cudaStream_t st) {
  using C = WgradCfg<BN, XW>;
  auto kern = conv_wgrad_kernel<BN, XW>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess)
      return B2DL_E_CUDA;
    attr_set = true;
  }
  const int grid = std::min(p.num_tiles, num_sms());
  const int rc = launch_tc(kern, grid, 192, C::SMEM, st, 1, tx, tdy, p);
  return rc ? rc : check_launch();
}

// CTA-pair fprop/dgrad for 256-wide tiles; B2DL_FPROP_PAIRS=0 selects single-CTA tiles
static bool fprop_pairs_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_FPROP_PAIRS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CTA-pair tiles for 128-wide N (B2DL_FPROP_PAIR128=1).  Off by default: at N = 128 the pair's
// per-SM operand reads (4 KB A + 2 KB B per 64-cycle MMA) outrun shared memory, measured ~25 %
// slower than a 256-wide pair on the 1/8-resolution ASPP convs.
static bool fprop_pair128_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_FPROP_PAIR128");
    return e && e[0] == '1';
  }();
  return on;
}

// 16 epilogue warps for TMA-epilogue launches with <= 1 operand; B2DL_EW16=0 keeps 8
static bool ew16_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_EW16");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int pick_bn(int cout) {
  if (cout > 128) return 256;
  if (cout > 64) return 128;
  if (cout > 32) return 64;
  if (cout > 16) return 32;
  return 16;
}

// TMA-staged fprop epilogue; B2DL_TMA_EPILOGUE=0 selects the register/shared-memory path
static bool tma_epilogue_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_TMA_EPILOGUE");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool view_aligned(const b2dl_act& a, int elem_bytes) {
  return (reinterpret_cast<uintptr_t>(a.ptr) % 16 == 0) && ((static_cast<long long>(a.c_stride) * elem_bytes) % 16 == 0);
}

// Row-window stem through the halo kernel: packed weights, <= 64 output channels, <= 7 tap
// rows, a 64- or 128-wide folded K, bf16 output through the TMA epilogue.
static int launch_halo_fprop(const b2dl_conv_args* a, const b2dl_act& xv, cudaStream_t st) {
  const b2dl_act& y = a->y;
  FpropParams p{};
  p.n = y.n;
  p.h = y.h;
  p.w = y.w;
  p.bw = HALO_BW;
  p.bh = HALO_BH;
  p.tiles_x = cdiv(y.w, HALO_BW);
  p.tiles_y = cdiv(y.h, HALO_BH);
  p.num_m_tiles = y.n * p.tiles_x * p.tiles_y;
  p.num_n_tiles = 1;
  p.num_tiles = p.num_m_tiles;
  p.kw = 1;
  p.dil = 1;
  p.pad_top = a->pad_top;
  p.cin_pad = b2dl_cin_pad(xv.c);
  p.num_cblk = p.cin_pad / 64;
  p.taps = a->kh;
  p.num_kb = p.taps * p.num_cblk;
  p.cout = a->cout;
  p.y = y.ptr;
  p.y_stride = y.c_stride;
  p.bias = a->bias;
  p.bias_vec = a->bias && (reinterpret_cast<uintptr_t>(a->bias) % 16 == 0);
  p.res = reinterpret_cast<const b2h*>(a->residual.ptr);
  p.res_stride = a->residual.c_stride;
  p.mask = reinterpret_cast<const b2h*>(a->mask.ptr);
  p.mask_stride = a->mask.c_stride;
  p.relu = a->relu;
  p.accumulate = a->accumulate;
  p.vec_ok = 1;
  p.tma_epi = 1;
  p.epi_nops = (p.res != nullptr) + (p.mask != nullptr) + (p.accumulate != 0);
  p.epi_slots = 2;
  p.bn_part = a->bn_partial;
  p.epi_bytes = 2 * epi_sub_bytes(p.epi_nops, 2);
  const int a_stage = (HALO_BH + p.taps - 1) * HALO_BW * 128;
  const int b_region = p.taps * p.num_cblk * HALO_BBOX;
  p.stages = std::min(FPROP_MAX_STAGES, (SMEM_MAX - SMEM_FIXED - b_region - p.epi_bytes) / a_stage);
  if (p.stages < 2) return B2DL_E_NOT_IMPLEMENTED;
  const int smem = b_region + p.stages * a_stage + p.epi_bytes + SMEM_FIXED;

  FpropMaps t;
  const int bwx = p.bw, bhx = p.bh;  // epilogue boxes: 32 channels x the whole tile
  const uint64_t ktot = static_cast<uint64_t>(p.taps) * p.cin_pad;
  const uint64_t wd[2] = {ktot, static_cast<uint64_t>(a->cout)};
  const uint64_t wsd[1] = {ktot * 2};
  const uint32_t wb[2] = {64u, static_cast<uint32_t>(HALO_BN)};
  if (window_map(&t.a, a->x, xv.c, y.w, 64, HALO_BW, HALO_BH + p.taps - 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tiled(&t.b, B2H_TMA, 2, const_cast<void*>(a->w_packed), wd, wsd, wb,
                   CU_TENSOR_MAP_SWIZZLE_128B) ||
      act_map(&t.y, y, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B) ||
      (p.res && act_map(&t.r, a->residual, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B)) ||
      (p.mask && act_map(&t.m, a->mask, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B)))
    return B2DL_E_ALIGN;
  auto kern = p.bn_part ? conv_halo_fprop_kernel<1> : conv_halo_fprop_kernel<0>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[p.bn_part != nullptr]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) != cudaSuccess)
      return B2DL_E_CUDA;
    attr_set[p.bn_part != nullptr] = true;
  }
  const int grid = std::min(p.num_tiles, num_sms());
  p.bn_per_cta = 1;
  const int rc = launch_tc(kern, grid, FPROP_THREADS, smem, st, 1, t.a, t.b, t.y, t.r, t.m, p);
  return rc ? rc : check_launch();
}

// Row-tap path for narrow outputs (B2DL_ROWTAP=0 disables): packed weights, cout <= 128 (<= 256
// over a <= 64-channel input), >= B2DL_ROWTAP_MINK (3) tap rows, bf16 output through the TMA
// epilogue.
static bool rowtap_enabled() {
  static const bool on = [] {
    const char* e = getenv("B2DL_ROWTAP");
    return !(e && e[0] == '0');
  }();
  return on;
}
static int rowtap_min_kh() {   // fewest tap rows for the row-tap kernels (B2DL_ROWTAP_MINK, default 3)
  static const int v = [] {
    const char* e = getenv("B2DL_ROWTAP_MINK");
    return e && e[0] ? atoi(e) : 3;
  }();
  return v;
}
static bool rowtap_resident_enabled() {   // B2DL_ROWTAP_RESIDENT=0: always stream the weights
  static const bool on = [] {
    const char* e = getenv("B2DL_ROWTAP_RESIDENT");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool rowtap_fprop_ok(const b2dl_conv_args* a, const b2dl_act& x) {
  const b2dl_act& y = a->y;
  const int nops = (a->residual.ptr != nullptr) + (a->mask.ptr != nullptr) + (a->accumulate != 0);
  return rowtap_enabled() && !a->window && a->w_mode == 0 && a->w_packed && a->kh >= rowtap_min_kh() &&
         (a->cout <= 128 || (a->cout <= 256 && x.c <= 64)) &&   // wide N only over a narrow K
         a->cout % 8 == 0 && x.c > 16 && RT_BH + (a->kh - 1) * a->dilation <= 256 &&
         (a->in_stride <= 1) && (a->out_stride <= 1) && !a->bn_partial && !a->bnb_stats &&
         (!a->bias || (reinterpret_cast<uintptr_t>(a->bias) % 16 == 0)) && !a->y_f32 && view_aligned(y, 2) &&
         nops <= 2 && (!a->residual.ptr || view_aligned(a->residual, 2)) &&
         (!a->mask.ptr || view_aligned(a->mask, 2)) && tma_epilogue_enabled();
}

static int launch_rowtap_fprop(const b2dl_conv_args* a, const b2dl_act& x, cudaStream_t st) {
  const b2dl_act& y = a->y;
  const int bn = a->cout <= 32 ? 32 : a->cout <= 64 ? 64 : a->cout <= 128 ? 128 : 256;
  FpropParams p{};
  p.n = y.n;
  p.h = y.h;
  p.w = y.w;
  p.bw = RT_BW;
  p.bh = RT_BH;
  p.tiles_x = cdiv(y.w, RT_BW);
  p.tiles_y = cdiv(y.h, RT_BH);
  p.num_m_tiles = y.n * p.tiles_x * p.tiles_y;
  p.num_n_tiles = 1;
  // CTA pairs (M = 256 per MMA) unless B2DL_ROWTAP_PAIRS=0 or there is a single tile
  static const int pairs_on = env_int("B2DL_ROWTAP_PAIRS", 1);
  const int cg = pairs_on && p.num_m_tiles >= 2 ? 2 : 1;
  p.num_tiles = cdiv(p.num_m_tiles, cg);
  p.kw = a->kw;
  p.dil = a->dilation;
  p.pad_top = a->pad_top;
  p.pad_left = a->pad_left;
  // K block: a 17..32-channel input needs only half a block.  (32-channel blocks for the 96 / 160 /
  // 224-channel inputs too -- a quarter less MMA work at 96 -- measured 2.6 % slower on config 4.)
  const int kb = x.c <= 32 ? 32 : 64;
  p.cin_pad = b2dl_cin_pad(x.c);      // packed weights' K stride per tap
  p.num_cblk = cdiv(x.c, kb);
  p.taps = a->kh * a->kw;
  p.num_kb = p.taps * p.num_cblk;
  p.cout = a->cout;
  p.y = y.ptr;
  p.y_stride = y.c_stride;
  p.bias = a->bias;
  p.bias_vec = a->bias != nullptr;
  p.res = reinterpret_cast<const b2h*>(a->residual.ptr);
  p.res_stride = a->residual.c_stride;
  p.mask = reinterpret_cast<const b2h*>(a->mask.ptr);
  p.mask_stride = a->mask.c_stride;
  p.relu = a->relu;
  p.accumulate = a->accumulate;
  p.vec_ok = 1;
  p.tma_epi = 1;
  p.epi_nops = (p.res != nullptr) + (p.mask != nullptr) + (p.accumulate != 0);
  p.epi_slots = 2;
  p.epi_bytes = 2 * epi_sub_bytes(p.epi_nops, 2);
  // wide box: 8 + (kw - 1) dil pixels per row (B2DL_RT_COLSHIFT=2: 16, 0: off; SW128 and SW64
  // alike); the 8-row core matrices then start at any pixel row, which the address-based
  // swizzle allows
  static const int rt_cs_env = env_int("B2DL_RT_COLSHIFT", 1);
  const int wide = RT_BW + (a->kw - 1) * a->dilation;
  p.rt_cs = (rt_cs_env && wide <= 2 * RT_BW) ? (rt_cs_env == 2 ? 2 * RT_BW : wide) : 0;
  const int box_rows = RT_BH + (a->kh - 1) * a->dilation;
  // (stage buffers 1 KB aligned: a wide SW64 box on a 256-byte boundary read back wrong in pairs)
  int a_stage = (box_rows * (p.rt_cs ? p.rt_cs : RT_BW) * kb * 2 + 1023) / 1024 * 1024;
  const int b_box = (bn / cg) * kb * 2;   // per CTA: a pair splits the weight rows
  // weights resident when they fit beside >= 3 input stages, else streamed with each stage
  const int w_bytes = (p.taps * p.num_cblk * b_box + 1023) / 1024 * 1024;
  const int room = SMEM_MAX - SMEM_FIXED - p.epi_bytes;
  p.b_region = (w_bytes + 3 * a_stage <= room && rowtap_resident_enabled()) ? w_bytes : 0;
  if (!p.b_region && p.rt_cs) {   // the wide box pays only when it is reused (resident weights)
    p.rt_cs = 0;
    a_stage = (box_rows * RT_BW * kb * 2 + 1023) / 1024 * 1024;
    p.b_region = (w_bytes + 3 * a_stage <= room && rowtap_resident_enabled()) ? w_bytes : 0;
  }
  const int stage_bytes = a_stage + (p.b_region ? 0 : a->kh * b_box);
  p.stages = std::min(FPROP_MAX_STAGES, (room - p.b_region) / stage_bytes);
  if (p.stages < 2) return B2DL_E_NOT_IMPLEMENTED;
  const int smem = p.b_region + p.stages * stage_bytes + p.epi_bytes + SMEM_FIXED;

  FpropMaps t;
  const uint64_t ktot = static_cast<uint64_t>(p.taps) * p.cin_pad;
  const uint64_t wd[2] = {ktot, static_cast<uint64_t>(a->cout)};
  const uint64_t wsd[1] = {ktot * 2};
  const uint32_t wb[2] = {static_cast<uint32_t>(kb), static_cast<uint32_t>(bn / cg)};
  const CUtensorMapSwizzle sw = kb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  if (act_map(&t.a, x, kb, p.rt_cs ? p.rt_cs : RT_BW, RT_BH + (a->kh - 1) * a->dilation, sw) ||
      encode_tiled(&t.b, B2H_TMA, 2, const_cast<void*>(a->w_packed), wd, wsd, wb, sw) ||
      act_map(&t.y, y, 32, RT_BW, RT_BH, CU_TENSOR_MAP_SWIZZLE_64B) ||
      (p.res && act_map(&t.r, a->residual, 32, RT_BW, RT_BH, CU_TENSOR_MAP_SWIZZLE_64B)) ||
      (p.mask && act_map(&t.m, a->mask, 32, RT_BW, RT_BH, CU_TENSOR_MAP_SWIZZLE_64B)))
    return B2DL_E_ALIGN;
  decltype(&conv_rowtap_fprop_kernel<32, 64>) kern;
#define B2_RT(BNV, KBV, CGV) conv_rowtap_fprop_kernel<BNV, KBV, CGV>
  if (cg == 2)
    kern = bn == 32    ? (kb == 64 ? B2_RT(32, 64, 2) : B2_RT(32, 32, 2))
           : bn == 64  ? (kb == 64 ? B2_RT(64, 64, 2) : B2_RT(64, 32, 2))
           : bn == 128 ? (kb == 64 ? B2_RT(128, 64, 2) : B2_RT(128, 32, 2))
                       : (kb == 64 ? B2_RT(256, 64, 2) : B2_RT(256, 32, 2));
  else
    kern = bn == 32    ? (kb == 64 ? B2_RT(32, 64, 1) : B2_RT(32, 32, 1))
           : bn == 64  ? (kb == 64 ? B2_RT(64, 64, 1) : B2_RT(64, 32, 1))
           : bn == 128 ? (kb == 64 ? B2_RT(128, 64, 1) : B2_RT(128, 32, 1))
                       : (kb == 64 ? B2_RT(256, 64, 1) : B2_RT(256, 32, 1));
#undef B2_RT
  static bool attr_set[16] = {};
  const int ai = (cg == 2) * 8 + (bn == 32 ? 0 : bn == 64 ? 2 : bn == 128 ? 4 : 6) + (kb == 64);
  if (!attr_set[ai]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) != cudaSuccess)
      return B2DL_E_CUDA;
    attr_set[ai] = true;
  }
  const int grid = cg * std::min(p.num_tiles, num_sms() / cg);
  const int rc = launch_tc(kern, grid, FPROP_THREADS, smem, st, cg, t.a, t.b, t.y, t.r, t.m, p, static_cast<int>(a->kh));
  return rc ? rc : check_launch();
}

static bool halo_fprop_ok(const b2dl_conv_args* a, const b2dl_act& xv) {
  const b2dl_act& y = a->y;
  const int nops = (a->residual.ptr != nullptr) + (a->mask.ptr != nullptr) + (a->accumulate != 0);
  return a->window && a->w_mode == 0 && a->w_packed && a->cout <= HALO_BN && a->cout % 8 == 0 && a->kh <= 7 &&
         (!a->bias || (reinterpret_cast<uintptr_t>(a->bias) % 16 == 0)) &&
         a->dilation == 1 && xv.c > 16 && xv.c <= 128 && !a->y_f32 && view_aligned(y, 2) && nops <= 2 &&
         (!a->residual.ptr || view_aligned(a->residual, 2)) && (!a->mask.ptr || view_aligned(a->mask, 2)) &&
         tma_epilogue_enabled();
}

}  // namespace b2

using namespace b2;

extern "C" int b2dl_cin_pad(int cin) { return cin <= 16 ? 16 : round_up(cin, 64); }

namespace b2 {
// Row-window mode: the virtual input (kw-folded channels over the output width); validates
// the haloed storage of x.
static int window_view(const b2dl_act& x, int window, int kw, int pad_left, int out_w, b2dl_act* xv) {
  *xv = x;
  if (!window) return B2DL_OK;
  if (window < 1 || kw != 1 || pad_left != 0 || x.c != x.c_stride || x.w < out_w + window - 1)
    return B2DL_E_VALUE;
  xv->c = window * x.c;
  xv->w = out_w;
  return B2DL_OK;
}
}  // namespace b2

namespace b2 {
static int fprop_kblk(const b2dl_conv_args* a, const b2dl_act& x) {
  if (x.c <= 16) return 16;
  // (the statistics epilogue variants are instantiated for 64-channel K blocks only)
  if (x.c <= 32 && a->w_mode != 0 && !a->window && !a->bn_partial && !a->bnb_stats) return 32;
  return 64;
}
// N tile width and CTA pairing of a b2dl_conv_fprop launch (shared with b2dl_conv_fprop_bn_rows)
// Output tile width of the generic fprop (tile = bw x (128 / bw) pixels).  A strided input
// (the upsampled conv's dgrad reads dy at s_in x the output resolution) re-reads the kernel's
// (k - 1)-pixel halo of every tile, so it takes squarer tiles (B2DL_STRIDED_BW caps the width).
static int fprop_tile_w(int w, int s_in) {
  int bw = pow2_divisor(w, 128);
  if (bw < 8 && w >= 8) bw = std::min(128, 1 << (31 - __builtin_clz(w)));
  while (bw * s_in > 256) bw >>= 1;   // strided input box: traversal extent <= 256
  if (s_in > 1) {
    static const int cap = env_int("B2DL_STRIDED_BW", 0);
    if (cap >= 8 && bw > cap) bw = cap;
  }
  return bw;
}

static void fprop_choose(const b2dl_conv_args* a, const b2dl_act& x, int kblk, int* bn_out, int* cg_out) {
  int bn = a->block_n ? a->block_n : pick_bn(a->cout);
  // 256- and 128-wide N tiles run as CTA pairs (256 pixels x BN per pair)
  auto pair_ok = [&](int b) {
    return (b == 256 || (b == 128 && fprop_pair128_enabled())) && kblk == 64 && fprop_pairs_enabled();
  };
  int cg = pair_ok(bn) ? 2 : 1;
  if (!a->block_n && (bn == 256 || bn == 128) && kblk == 64) {
    // wave quantisation: pick the (N tile, pairing) that fills the persistent grid best,
    // weighted by the relative speed of each tile shape
    const int bw = fprop_tile_w(x.w, a->in_stride > 0 ? a->in_stride : 1);
    const long long mt = static_cast<long long>(x.n) * cdiv(x.w, bw) * cdiv(x.h, BM / bw);
    // ... and by the share of computed columns that are real output channels (N padding)
    auto score = [&](int b, int g, double speed) {
      const long long units = (mt + g - 1) / g * cdiv(a->cout, b), slots = num_sms() / g;
      const long long waves = (units + slots - 1) / slots;
      const double cols = static_cast<double>(a->cout) / (cdiv(a->cout, b) * b);
      return speed * cols * static_cast<double>(units) / (waves * slots);
    };
    struct Cand {
      int b, g;
      double speed;
    };
    // relative speeds measured with tools/prof_tiles.py: 128-wide tiles run at ~0.6 of the 256-wide
    // pair on long-K (tensor-bound) launches, but at par on short-K (epilogue / HBM-bound) ones
    // (e.g. 96 -> 320 channels at full resolution: 404 us on 128-wide tiles, 487 us on 256-pairs)
    const int taps = a->kh * a->kw;
    const bool short_k = taps * cdiv(x.c, kblk) <= 4;
    const Cand cands[3] = {{256, 2, 1.0}, {128, 2, short_k ? 0.85 : 0.6}, {128, 1, short_k ? 1.0 : 0.7}};
    double best = -1.0;
    for (const Cand& c : cands) {
      if (c.b > bn || (c.g == 2 && !pair_ok(c.b)) || (c.b == 256 && a->cout <= 128)) continue;
      const double sc = score(c.b, c.g, c.speed);
      if (sc > best) {
        best = sc;
        bn = c.b;
        cg = c.g;
      }
    }
  }

  *bn_out = bn;
  *cg_out = cg;
}
}  // namespace b2

extern "C" int b2dl_conv_fprop_bn_rows(const b2dl_conv_args* a) {
  // mirrors the tiling b2dl_conv_fprop picks (halo stem: 8 x 16 pixels; else a 128-pixel box):
  // one statistics row per CTA when the launch has a single N tile, else one per M tile
  if (!a) return -B2DL_E_VALUE;
  b2dl_act y = a->y;
  const int s_out = a->out_stride > 0 ? a->out_stride : 1;
  if (s_out > 1) {
    y.h /= s_out;
    y.w /= s_out;
  }
  b2dl_act x;
  if (window_view(a->x, a->window, a->kw, a->pad_left, y.w, &x)) return -B2DL_E_VALUE;
  const int s_in = a->in_stride > 0 ? a->in_stride : 1;
  if (s_in > 1) {
    x.h = y.h;
    x.w = y.w;
  }
  if (halo_fprop_ok(a, x)) return std::min(y.n * cdiv(y.w, HALO_BW) * cdiv(y.h, HALO_BH), num_sms());
  const int bw = fprop_tile_w(x.w, s_in);
  const int m_tiles = x.n * cdiv(x.w, bw) * cdiv(x.h, BM / bw);
  int bn, cg;
  fprop_choose(a, x, fprop_kblk(a, x), &bn, &cg);
  const int n_tiles = cdiv(a->cout, bn);
  if (n_tiles > 1) return m_tiles;
  return cg * std::min(cdiv(m_tiles, cg) * n_tiles, num_sms() / cg);
}

extern "C" int b2dl_conv_fprop(const b2dl_conv_args* a, void* stream) {
  if (!a || !a->x.ptr || !a->y.ptr || a->w_mode < 0 || a->w_mode > 2) return B2DL_E_VALUE;
  b2dl_act y = a->y;
  const int s_out = a->out_stride > 0 ? a->out_stride : 1;
  if (s_out > 1) {   // phase view: the kernel tiles the (h/f, w/f) output; the store map is strided
    if (s_out > 8 || a->out_phase_h < 0 || a->out_phase_h >= s_out || a->out_phase_w < 0 ||
        a->out_phase_w >= s_out || y.h % s_out || y.w % s_out || a->residual.ptr || a->mask.ptr || a->accumulate ||
        a->y_f32 || a->window || a->in_stride > 1)
      return B2DL_E_VALUE;
    y.h /= s_out;
    y.w /= s_out;
  }
  b2dl_act x;
  if (window_view(a->x, a->window, a->kw, a->pad_left, y.w, &x)) return B2DL_E_VALUE;
  const int s_in = a->in_stride > 0 ? a->in_stride : 1;
  if (s_in > 1 && (a->window || x.h != s_in * y.h || x.w != s_in * y.w || s_in > 8)) return B2DL_E_VALUE;
  if (s_in > 1) {   // the kernel tiles the output; the input map is strided (checked above)
    x.h = y.h;
    x.w = y.w;
  }
  if (x.n != y.n || x.h != y.h || x.w != y.w || y.c != a->cout) return B2DL_E_VALUE;
  if (a->kh < 1 || a->kw < 1 || a->dilation < 1 || a->cout < 1 || x.c < 1) return B2DL_E_VALUE;
  if (!view_aligned(x, 2)) return B2DL_E_ALIGN;
  if (halo_fprop_ok(a, x)) return launch_halo_fprop(a, x, as_stream(stream));
  if (rowtap_fprop_ok(a, x)) {   // (too little shared memory for 2 stages: the generic kernel below)
    const int rc = launch_rowtap_fprop(a, x, as_stream(stream));
    if (rc != B2DL_E_NOT_IMPLEMENTED) return rc;
  }
  // K block: 16 channels for narrow inputs, 32 for 17..32-channel inputs read through master
  // weights (e.g. the dgrad over a growth-32 dense layer's dy: half the padded MMA work of a
  // 64-wide block), else 64
  const int kblk = fprop_kblk(a, x);
  const int cin_pad = kblk == 32 ? 32 : b2dl_cin_pad(x.c);
  int bn, cg;
  fprop_choose(a, x, kblk, &bn, &cg);

  FpropParams p{};
  p.n = x.n;
  p.h = x.h;
  p.w = x.w;
  p.in_stride = s_in;
  p.bw = fprop_tile_w(x.w, s_in);
  p.bh = BM / p.bw;
  p.tiles_x = cdiv(x.w, p.bw);
  p.tiles_y = cdiv(x.h, p.bh);
  p.num_m_tiles = x.n * p.tiles_x * p.tiles_y;
  p.num_n_tiles = cdiv(a->cout, bn);
  p.num_tiles = cdiv(p.num_m_tiles, cg) * p.num_n_tiles;  // scheduling units: tiles or tile pairs
  p.kw = a->kw;
  p.dil = a->dilation;
  p.pad_top = a->pad_top;
  p.pad_left = a->pad_left;
  p.num_cblk = cin_pad / kblk;
  p.num_kb = a->kh * a->kw * p.num_cblk;
  p.cin_pad = cin_pad;
  p.cout = a->cout;
  p.y = y.ptr;
  p.y_stride = y.c_stride;
  p.y_f32 = a->y_f32;
  p.bias = a->bias;
  p.res = reinterpret_cast<const b2h*>(a->residual.ptr);
  p.res_stride = a->residual.c_stride;
  p.mask = reinterpret_cast<const b2h*>(a->mask.ptr);
  p.mask_stride = a->mask.c_stride;
  p.relu = a->relu;
  p.accumulate = a->accumulate;
  p.vec_ok = view_aligned(y, a->y_f32 ? 4 : 2) && (!p.res || view_aligned(a->residual, 2)) &&
             (!p.mask || view_aligned(a->mask, 2));

  FpropMaps t;
  const CUtensorMapSwizzle sw = kblk == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                : kblk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                             : CU_TENSOR_MAP_SWIZZLE_32B;
  if (a->window ? window_map(&t.a, a->x, x.c, y.w, kblk, p.bw, p.bh, sw)
                : s_in > 1 ? act_map_strided(&t.a, a->x, kblk, p.bw, p.bh, s_in, sw)
                           : act_map(&t.a, x, kblk, p.bw, p.bh, sw))
    return B2DL_E_ALIGN;
  const int mode = a->w_mode;
  p.b_mode = mode;
  p.taps = a->kh * a->kw;
  if (mode == 0) {
    if (!a->w_packed) return B2DL_E_VALUE;
    const uint64_t ktot = static_cast<uint64_t>(a->kh) * a->kw * cin_pad;
    const uint64_t wd[2] = {ktot, static_cast<uint64_t>(a->cout)};
    const uint64_t ws[1] = {ktot * 2};
    const uint32_t wb[2] = {static_cast<uint32_t>(kblk), static_cast<uint32_t>(bn / cg)};
    if (encode_tiled(&t.b, B2H_TMA, 2, const_cast<void*>(a->w_packed), wd, ws, wb, sw))
      return B2DL_E_ALIGN;
  } else {
    // master HWIO bf16 [taps][cin_f][cout_f] of the forward conv; fprop: cin_f = x.c, cout_f = cout;
    // dgrad: the forward conv's cin is our cout and its cout our input channel count
    if (!a->w_master) return B2DL_E_VALUE;
    const uint64_t cf = mode == 1 ? static_cast<uint64_t>(a->cout) : static_cast<uint64_t>(x.c);
    const uint64_t kf = mode == 1 ? static_cast<uint64_t>(x.c) : static_cast<uint64_t>(a->cout);
    if ((cf * 2) % 16 || (reinterpret_cast<uintptr_t>(a->w_master) & 15)) return B2DL_E_ALIGN;
    const uint64_t wd[3] = {cf, kf, static_cast<uint64_t>(p.taps)};
    const uint64_t ws[2] = {cf * 2, cf * kf * 2};
    if (mode == 1) {
      const uint32_t wb[3] = {64u, static_cast<uint32_t>(kblk), 1u};
      if (encode_tiled(&t.b, B2H_TMA, 3, const_cast<void*>(a->w_master), wd, ws, wb,
                       CU_TENSOR_MAP_SWIZZLE_128B))
        return B2DL_E_ALIGN;
    } else {
      const uint32_t wb[3] = {static_cast<uint32_t>(kblk), static_cast<uint32_t>(bn / cg), 1u};
      if (encode_tiled(&t.b, B2H_TMA, 3, const_cast<void*>(a->w_master), wd, ws, wb, sw))
        return B2DL_E_ALIGN;
    }
  }

  // TMA epilogue: bf16 output (and operands) through 32-pixel x 32-channel swizzled boxes
  p.bias_vec = a->bias && (reinterpret_cast<uintptr_t>(a->bias) % 16 == 0);
  p.tma_epi = p.vec_ok && !p.y_f32 && (a->cout % 8) == 0 && bn >= 32 && tma_epilogue_enabled() &&
              (!a->bias || p.bias_vec) &&
              ((p.res != nullptr) + (p.mask != nullptr) + (p.accumulate != 0)) <= 2;
  p.y_phase = s_out > 1;
  if (p.y_phase && !p.tma_epi) return B2DL_E_VALUE;
  p.bn_part = a->bn_partial;
  if (p.bn_part && (p.y_phase || !p.tma_epi)) return B2DL_E_VALUE;
  p.bnb_stats = a->bnb_stats;
  p.bnb_part = a->bnb_partial;
  if ((p.bnb_stats != nullptr) != (p.bnb_part != nullptr)) return B2DL_E_VALUE;
  if (p.bnb_stats && (!p.tma_epi || p.y_phase || !p.mask || p.res || p.accumulate ||
                      (reinterpret_cast<uintptr_t>(p.bnb_stats) & 15) || (a->cout & 7)))
    return B2DL_E_VALUE;
  if (p.tma_epi) {
    // epilogue boxes: 32 channels x the whole tile, or x one warp's 32 pixels (per-warp mode)
    p.epi_pw = epi_pw_enabled() && !p.bn_part;
    const int bwx = p.epi_pw ? std::min(p.bw, 32) : p.bw, bhx = p.epi_pw ? 32 / bwx : p.bh;
    if ((s_out > 1 ? act_map_phase(&t.y, a->y, s_out, a->out_phase_h, a->out_phase_w, 32, bwx, bhx,
                                   CU_TENSOR_MAP_SWIZZLE_64B)
                   : act_map(&t.y, y, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B)) ||
        (p.res && act_map(&t.r, a->residual, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B)) ||
        (p.mask && act_map(&t.m, a->mask, 32, bwx, bhx, CU_TENSOR_MAP_SWIZZLE_64B))) {
      if (p.y_phase || p.bn_part) return B2DL_E_ALIGN;
      p.tma_epi = 0;
    }
  }

  cudaStream_t st = as_stream(stream);
#define B2_FPROP(BNV, KB)                                                                \
  if (bn == BNV && kblk == KB)                                                           \
    return mode == 1 ? launch_fprop<BNV, KB, true, 1>(t, p, st) : launch_fprop<BNV, KB, false, 1>(t, p, st);
  const int nops = (p.res != nullptr) + (p.mask != nullptr) + (p.accumulate != 0);
  // 16 epilogue warps where the epilogue dominates (short K); long-K launches keep the deeper
  // operand ring that 8 warps' smaller buffers leave room for
  if (p.bn_part || p.bnb_stats) {   // statistics epilogues: 8 epilogue warps, 64-wide K blocks
    const int stv = p.bn_part ? 1 : 2;
    // forward statistics on short-K launches: 16 epilogue warps, as for the plain epilogue
    if (stv == 1 && p.tma_epi && nops <= ew16_max_nops() && p.num_kb <= 16 && ew16_enabled() &&
        env_int("B2DL_ST_EW16", 1)) {
      if (cg == 2 && bn == 256)
        return mode == 1 ? launch_fprop<256, 64, true, 2, 16, 1>(t, p, st) : launch_fprop<256, 64, false, 2, 16, 1>(t, p, st);
      if (cg == 1 && bn == 256)
        return mode == 1 ? launch_fprop<256, 64, true, 1, 16, 1>(t, p, st) : launch_fprop<256, 64, false, 1, 16, 1>(t, p, st);
      if (cg == 1 && bn == 128)
        return mode == 1 ? launch_fprop<128, 64, true, 1, 16, 1>(t, p, st) : launch_fprop<128, 64, false, 1, 16, 1>(t, p, st);
    }
#define B2_FPROP_ST(BNV, CGV, STV)                                                                    \
  if (bn == BNV && cg == CGV && kblk == 64 && stv == STV)                                             \
    return mode == 1 ? launch_fprop<BNV, 64, true, CGV, 8, STV>(t, p, st)                             \
                     : launch_fprop<BNV, 64, false, CGV, 8, STV>(t, p, st);
    B2_FPROP_ST(256, 2, 1)
    B2_FPROP_ST(128, 2, 1)
    B2_FPROP_ST(256, 1, 1)
    B2_FPROP_ST(128, 1, 1)
    B2_FPROP_ST(64, 1, 1)
    B2_FPROP_ST(32, 1, 1)
    B2_FPROP_ST(256, 2, 2)
    B2_FPROP_ST(128, 2, 2)
    B2_FPROP_ST(256, 1, 2)
    B2_FPROP_ST(128, 1, 2)
    B2_FPROP_ST(64, 1, 2)
    B2_FPROP_ST(32, 1, 2)
#undef B2_FPROP_ST
    return B2DL_E_VALUE;
  }
  if (p.tma_epi && nops <= ew16_max_nops() && kblk == 64 && p.num_kb <= 16 && ew16_enabled()) {
    if (cg == 2 && bn == 256)
      return mode == 1 ? launch_fprop<256, 64, true, 2, 16>(t, p, st) : launch_fprop<256, 64, false, 2, 16>(t, p, st);
    if (cg == 1 && bn == 256)
      return mode == 1 ? launch_fprop<256, 64, true, 1, 16>(t, p, st) : launch_fprop<256, 64, false, 1, 16>(t, p, st);
    if (cg == 1 && bn == 128)
      return mode == 1 ? launch_fprop<128, 64, true, 1, 16>(t, p, st) : launch_fprop<128, 64, false, 1, 16>(t, p, st);
  }
  if (cg == 2 && bn == 256)
    return mode == 1 ? launch_fprop<256, 64, true, 2>(t, p, st) : launch_fprop<256, 64, false, 2>(t, p, st);
  if (cg == 2 && bn == 128)
    return mode == 1 ? launch_fprop<128, 64, true, 2>(t, p, st) : launch_fprop<128, 64, false, 2>(t, p, st);
  B2_FPROP(256, 64)
  B2_FPROP(128, 64)
  B2_FPROP(64, 64)
  B2_FPROP(32, 64)
  B2_FPROP(16, 64)
  B2_FPROP(256, 32)
  B2_FPROP(128, 32)
  B2_FPROP(64, 32)
  B2_FPROP(32, 32)
  B2_FPROP(16, 32)
  B2_FPROP(256, 16)
  B2_FPROP(128, 16)
  B2_FPROP(64, 16)
  B2_FPROP(32, 16)
  B2_FPROP(16, 16)
#undef B2_FPROP
  return B2DL_E_VALUE;
}

namespace b2 {
struct WgradPlan {
  WgradParams p;
  int bn, xw;
  int halo;  // row-window stem kernel
  size_t ws_bytes, bsum_bytes;
};
static int plan_wgrad(const b2dl_wgrad_args* a, WgradPlan* out) {
  const b2dl_act& dy = a->dy;
  b2dl_act x;
  if (window_view(a->x, a->window, a->kw, a->pad_left, dy.w, &x)) return B2DL_E_VALUE;
  if (x.n != dy.n || x.h != dy.h || x.w != dy.w) return B2DL_E_VALUE;
  out->halo = 0;
  if (a->window && dy.c <= 64 && a->kh <= 8 && x.c > 16 && x.c <= 128 && a->dilation == 1) {
    // row-window stem: 8 x 16-pixel K blocks, one split (partial) per CTA
    WgradParams p{};
    p.n = x.n;
    p.h = x.h;
    p.w = x.w;
    p.bwk = HW_BW;
    p.bhk = HW_BH;
    p.pbx = cdiv(x.w, HW_BW);
    p.pby = cdiv(x.h, HW_BH);
    p.num_pb = x.n * p.pbx * p.pby;
    p.kw = 1;
    p.dil = 1;
    p.pad_top = a->pad_top;
    p.cin = x.c;
    p.cout = dy.c;
    p.krows = static_cast<long long>(a->kh) * x.c;
    p.m_tiles = 1;
    p.n_tiles = 1;
    const int splits = std::min(num_sms(), p.num_pb);
    p.pb_per_split = cdiv(p.num_pb, splits);
    p.splits = cdiv(p.num_pb, p.pb_per_split);
    p.num_tiles = p.splits;
    out->p = p;
    out->bn = 64;
    out->xw = 64;
    out->halo = 1;
    out->ws_bytes = static_cast<size_t>(p.splits) * p.krows * p.cout * sizeof(float);
    out->bsum_bytes = static_cast<size_t>(p.splits) * p.cout * sizeof(float);
    return B2DL_OK;
  }
  // (from 3 tap rows: the 3x3 64->64 stage-0 wgrads take 21 instead of 42 us at 2 x 288 x 192)
  if (!a->window && rowtap_enabled() && dy.c <= 64 && a->kh >= rowtap_min_kh() &&
      a->kh * (dy.c <= 32 ? 32 : 64) <= 512 &&
      x.c > 16 && HW_BH + (a->kh - 1) * a->dilation <= 256) {
    // row-tap wgrad (narrow N): a unit = (column tap, pair of 64-channel blocks, pixel split)
    WgradParams p{};
    p.n = x.n;
    p.h = x.h;
    p.w = x.w;
    p.bwk = HW_BW;
    p.bhk = HW_BH;
    p.pbx = cdiv(x.w, HW_BW);
    p.pby = cdiv(x.h, HW_BH);
    p.num_pb = x.n * p.pbx * p.pby;
    p.kw = a->kw;
    p.dil = a->dilation;
    p.pad_top = a->pad_top;
    p.pad_left = a->pad_left;
    p.cblk = cdiv(x.c, 64);
    p.cin = x.c;
    p.cout = dy.c;
    p.krows = static_cast<long long>(a->kh) * a->kw * x.c;
    p.m_tiles = 1;
    p.n_tiles = 1;
    const int tiles = (a->kw * p.cblk + 1) / 2;
    // one unit per CTA, all resident in one wave (a 149th unit would double the kernel's time)
    int splits = a->splits > 0 ? a->splits : std::max(1, num_sms() / tiles);
    splits = std::min(splits, p.num_pb);
    p.pb_per_split = cdiv(p.num_pb, splits);
    p.splits = cdiv(p.num_pb, p.pb_per_split);
    p.num_tiles = tiles * p.splits;
    out->p = p;
    out->bn = dy.c <= 32 ? 32 : 64;
    out->xw = 64;
    out->halo = 2;
    out->ws_bytes = static_cast<size_t>(p.splits) * p.krows * p.cout * sizeof(float);
    out->bsum_bytes = static_cast<size_t>(p.splits) * p.cout * sizeof(float);
    return B2DL_OK;
  }
  WgradParams p{};
  p.n = x.n;
  p.h = x.h;
  p.w = x.w;
  const int kp = x.c <= 16 ? 256 : 64;  // WgradCfg<.., XW>::KP
  p.bwk = pow2_divisor(x.w, kp);
  if (p.bwk < 8 && x.w >= 8) p.bwk = std::min(kp, 1 << (31 - __builtin_clz(x.w)));
  p.bhk = kp / p.bwk;
  p.pbx = cdiv(x.w, p.bwk);
  p.pby = cdiv(x.h, p.bhk);
  p.num_pb = x.n * p.pbx * p.pby;
  p.kw = a->kw;
  p.dil = a->dilation;
  p.pad_top = a->pad_top;
  p.pad_left = a->pad_left;
  const int xw = x.c <= 16 ? 16 : 64;
  p.cblk = cdiv(x.c, xw);
  p.num_x_chunks = a->kh * a->kw * p.cblk;
  p.cin = x.c;
  p.cout = dy.c;
  p.krows = static_cast<long long>(a->kh) * a->kw * x.c;
  const int bn = pick_bn(dy.c);
  p.m_tiles = cdiv(p.num_x_chunks, xw == 16 ? 8 : 4);  // WgradCfg::NXC
  p.n_tiles = cdiv(dy.c, bn);
  int splits = a->splits;
  if (splits <= 0) {
    // split-K count minimising  waves x (K blocks per split) x t_kb  +  partial traffic / HBM:
    // more splits fill the persistent grid (#SMs), but every split writes (and the batched
    // reduction re-reads) a krows x cout fp32 partial.  t_kb ~ 0.7 us for a 256-wide tile
    // (two 128 x 256 x 64 MMA blocks), proportional to the tile width.
    const int base = p.m_tiles * p.n_tiles;
    const int sms = num_sms();
    const int smax = std::max(1, std::min(sms, p.num_pb / 4));
    const double t_kb = 0.7e-6 * std::max(bn, 32) / 256.0;
    const double part_bytes = static_cast<double>(p.krows) * p.cout * 4.0 * 2.0;
    double best = 1e30;
    splits = 1;
    for (int s = 1; s <= smax; ++s) {
      const long long tiles = static_cast<long long>(base) * s;
      const long long waves = (tiles + sms - 1) / sms;
      const double t = waves * std::ceil(static_cast<double>(p.num_pb) / s) * t_kb + s * part_bytes / 6.0e12;
      if (t < best * 0.999) {
        best = t;
        splits = s;
      }
    }
  }
  splits = std::min(splits, p.num_pb);
  p.pb_per_split = cdiv(p.num_pb, splits);
  p.splits = cdiv(p.num_pb, p.pb_per_split);  // no empty splits
  p.num_tiles = p.m_tiles * p.n_tiles * p.splits;
  out->p = p;
  out->bn = bn;
  out->xw = xw;
  out->ws_bytes = static_cast<size_t>(p.splits) * p.krows * p.cout * sizeof(float);
  out->bsum_bytes = static_cast<size_t>(p.splits) * p.m_tiles * p.cout * sizeof(float);
  return B2DL_OK;
}
}  // namespace b2

extern "C" size_t b2dl_wgrad_workspace_size(const b2dl_wgrad_args* a) {
  WgradPlan pl;
  if (!a || plan_wgrad(a, &pl)) return 0;
  return align_up(pl.ws_bytes, 256) + align_up(pl.bsum_bytes, 256);
}

extern "C" int b2dl_conv_wgrad(const b2dl_wgrad_args* a, void* stream) {
  if (!a || !a->x.ptr || !a->dy.ptr || !a->dw) return B2DL_E_VALUE;
  if (!view_aligned(a->x, 2) || !view_aligned(a->dy, 2)) return B2DL_E_ALIGN;
  WgradPlan pl;
  int rc = plan_wgrad(a, &pl);
  if (rc) return rc;
  const size_t need = b2dl_wgrad_workspace_size(a);
  if (!a->workspace || a->workspace_bytes < need) return B2DL_E_VALUE;
  pl.p.ws = reinterpret_cast<float*>(a->workspace);
  const bool defer = a->defer_reduce != 0;
  pl.p.bsum = a->bias_grad ? reinterpret_cast<float*>(reinterpret_cast<char*>(a->workspace) +
                                                      align_up(pl.ws_bytes, 256))
                           : nullptr;
  CUtensorMap tx, tdy;
  cudaStream_t st = as_stream(stream);
  if (pl.halo == 2) {
    const int kh = a->kh;
    const int xrows = HW_BH + (kh - 1) * a->dilation;
    if (act_map(&tx, a->x, 64, HW_BW, xrows, CU_TENSOR_MAP_SWIZZLE_128B) ||
        act_map(&tdy, a->dy, 64, HW_BW, HW_BH, CU_TENSOR_MAP_SWIZZLE_128B))
      return B2DL_E_ALIGN;
    const int stage_bytes = 2 * xrows * HW_BW * 128 + HW_BW * HW_BH * 128;
    const int stages = std::min(FPROP_MAX_STAGES, (SMEM_MAX - SMEM_FIXED) / stage_bytes);
    if (stages < 2) return B2DL_E_NOT_IMPLEMENTED;
    const int tiles = (a->kw * pl.p.cblk + 1) / 2;
    auto kern = pl.bn == 32 ? conv_rowtap_wgrad_kernel<32> : conv_rowtap_wgrad_kernel<64>;
    static bool attr_set[2] = {false, false};
    if (!attr_set[pl.bn == 64]) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) != cudaSuccess)
        return B2DL_E_CUDA;
      attr_set[pl.bn == 64] = true;
    }
    rc = launch_tc(kern, pl.p.num_tiles, 192, stages * stage_bytes + SMEM_FIXED, st, 1, tx, tdy, pl.p, kh, stages,
                   tiles);
    if (!rc) rc = check_launch();
    if (rc) return rc;
  } else if (pl.halo) {
    const int taps = a->kh;
    if (window_map(&tx, a->x, pl.p.cin, a->dy.w, 64, HW_BW, HW_BH + taps - 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
        act_map(&tdy, a->dy, 64, HW_BW, HW_BH, CU_TENSOR_MAP_SWIZZLE_128B))
      return B2DL_E_ALIGN;
    const int stage_bytes = 2 * (HW_BH + taps - 1) * HW_BW * 128 + HW_BW * HW_BH * 128;
    const int stages = std::min(FPROP_MAX_STAGES, (SMEM_MAX - SMEM_FIXED) / stage_bytes);
    static bool attr_set = false;
    if (!attr_set) {
      if (cudaFuncSetAttribute(conv_halo_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX) !=
          cudaSuccess)
        return B2DL_E_CUDA;
      attr_set = true;
    }
    rc = launch_tc(conv_halo_wgrad_kernel, pl.p.splits, 192, stages * stage_bytes + SMEM_FIXED, st, 1, tx, tdy,
                   pl.p, taps, stages);
    if (!rc) rc = check_launch();
    if (rc) return rc;
  } else {
    // x: 5-D map (64-ch inner, W, H, N, channel block) when chunks of one tap can be grouped
    pl.p.xg = 0;
    if (a->window) {
      if (pl.xw != 64 || window_map(&tx, a->x, a->window * a->x.c, a->dy.w, 64, pl.p.bwk, pl.p.bhk,
                                    CU_TENSOR_MAP_SWIZZLE_128B))
        return B2DL_E_ALIGN;
    } else if (pl.xw == 64 && a->x.c % 64 == 0) {
      const int cblk = a->x.c / 64;
      const int g = cblk % 4 == 0 ? 4 : (cblk % 2 == 0 ? 2 : 1);
      if (g > 1) {
        if (act_map5(&tx, a->x, pl.p.bwk, pl.p.bhk, g)) return B2DL_E_ALIGN;
        pl.p.xg = g;
      }
    }
    if (!a->window && !pl.p.xg && act_map(&tx, a->x, pl.xw, pl.p.bwk, pl.p.bhk,
                            pl.xw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B))
      return B2DL_E_ALIGN;
    pl.p.dyg = 0;
    const int nbw = pl.bn < 64 ? 1 : pl.bn / 64;
    if (nbw > 1 && a->dy.c % pl.bn == 0) {
      if (act_map5(&tdy, a->dy, pl.p.bwk, pl.p.bhk, nbw)) return B2DL_E_ALIGN;
      pl.p.dyg = nbw;
    } else if (act_map(&tdy, a->dy, 64, pl.p.bwk, pl.p.bhk, CU_TENSOR_MAP_SWIZZLE_128B)) {
      return B2DL_E_ALIGN;
    }
#define B2_WG(BNV)                                                                                      \
  case BNV:                                                                                             \
    rc = pl.xw == 64 ? launch_wgrad<BNV, 64>(tx, tdy, pl.p, st) : launch_wgrad<BNV, 16>(tx, tdy, pl.p, st); \
    break;
    switch (pl.bn) {
      B2_WG(256)
      B2_WG(128)
      B2_WG(64)
      B2_WG(32)
      default:
        rc = pl.xw == 64 ? launch_wgrad<16, 64>(tx, tdy, pl.p, st) : launch_wgrad<16, 16>(tx, tdy, pl.p, st);
        break;
    }
  }
#undef B2_WG
  if (rc) return rc;
  if (defer) return B2DL_OK;
  const long long total = pl.p.krows * pl.p.cout;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 4LL * num_sms()));
  wgrad_reduce_kernel<<<blocks, 256, 0, st>>>(pl.p.ws, a->dw, total, pl.p.splits, a->accumulate);
  rc = check_launch();
  if (rc) return rc;
  if (a->bias_grad) {
    bias_reduce_kernel<<<cdiv(pl.p.cout, 128), 128, 0, st>>>(pl.p.bsum, pl.p.splits * pl.p.m_tiles, pl.p.cout,
                                                             a->bias_grad, a->accumulate);
    rc = check_launch();
  }
  return rc;
}

extern "C" int b2dl_wgrad_partials(const b2dl_wgrad_args* a, int* w_parts, int* b_parts, size_t* b_offset) {
  if (!a || !w_parts || !b_parts || !b_offset) return B2DL_E_VALUE;
  WgradPlan pl;
  const int rc = plan_wgrad(a, &pl);
  if (rc) return rc;
  *w_parts = pl.p.splits;
  *b_parts = pl.p.splits * pl.p.m_tiles;
  *b_offset = align_up(pl.ws_bytes, 256);
  return B2DL_OK;
}

extern "C" int b2dl_reduce_segments(const b2dl_segment* segs, int nseg, int64_t max_n, float* dst_base,
                                    void* stream) {
  if (!segs || nseg < 1 || !dst_base) return B2DL_E_VALUE;
  // fill the GPU (~8 blocks per SM) whether the table holds one conv's two segments or many
  const long long want = std::max<long long>(1, (8LL * num_sms() + nseg - 1) / nseg);
  // (short segments are reduced 8 columns per block, see the kernel)
  const int bx = static_cast<int>(std::max<long long>(1, std::min<long long>(std::max((max_n / 4 + 255) / 256, (max_n + 7) / 8), want)));
  dim3 grid(bx, nseg);
  reduce_segments_kernel<<<grid, 256, 0, as_stream(stream)>>>(segs, dst_base);
  return check_launch();
}
