// TMA-fed, warp-specialised, persistent tcgen05 GEMM for the dense layers of
// bf16-context training ("the loss is back-propagated to update the
// weights"): every forward layer and every dgrad whose output is 64 < N <= 256
// wide and whose activation operand A is row-major fp32 (the layers bench.py's
// C3 step spends most of its time in).
//
//   C[M, N] = epi( A[M, K] . B[K, N] ),  epi = + bias, + resid, ReLU, ReLU' mask,
//                                               accumulate (C += .), as EpiParams
//
// Precision is the training path's bf16x3 (R37): A = Ah + Al (hi = truncated
// bf16, lo = RN_bf16(A - hi)), B likewise (the per-call weight image of
// bimg_kernel), A.B ~= Ah.Bh + Ah.Bl + Al.Bh with fp32 accumulation in TMEM.
//
// Why this kernel: the register-staged GEMM it replaces (tc_gemm_bimg_kernel)
// moved 373 MB per 204,800 x 256 launch at 2.2 TB/s -- its loader threads
// could keep only one 16 KB k-block in flight per CTA.  Here every byte of HBM
// traffic is a tensor-memory-accelerator copy issued ahead of use:
//   warp 0      TMA producer: A tiles [128 rows x 32 k] fp32 (128B swizzle)
//               into a 3-deep ring;
//   warps 2-5   converters: fp32 tile -> bf16 hi / lo in the K-major canonical
//               UMMA layout (the k-block's 32 KB weight image arrives by a 1-D
//               bulk copy the producer issues with the A tile, 3 deep);
//   warp 1      MMA issuer: 6 x tcgen05.mma (M=128, N=256, K=16) per k-block
//               into one of two TMEM accumulators (512 columns), so the
//               epilogue of tile i overlaps the main loop of tile i+1;
//   warps 6-13  epilogue, two per TMEM lane quarter, each independent of the
//               others: thread = tile row = TMEM lane; per 16-column chunk the
//               residual / mask / old-C input arrives by TMA (a 3-deep ring
//               per warp, 64B swizzle, [32 rows x 16 cols] boxes), the result
//               replaces it in the same stage and leaves by TMA store.
// Measured by skipping parts (TLP_TMA_DEBUG): a first epilogue with two
// 128-thread barriers per chunk ran 4-5x longer than the main loop; storing
// rows straight from registers (32 rows, 16 B each per warp instruction) made
// the stores half of the kernel; per-warp TMA boxes fix both.
// Tiles (128 rows) are walked persistently, one CTA per SM.
#include "tlp_internal.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

namespace {

constexpr int TM = 128, TN = 256, TK = 32;
#ifndef TLP_TMA_SA  // ring depths (A/B experiments: -DTLP_TMA_SA=.. etc.)
#define TLP_TMA_SA 3
#define TLP_TMA_SB 3
#define TLP_TMA_SC 2
#endif
constexpr int SA = TLP_TMA_SA;               // fp32 A ring (TMA)
constexpr int SB = TLP_TMA_SB;               // B image ring (bulk copies, issued with A)
constexpr int SC = TLP_TMA_SC;               // converted A hi/lo ring (MMA operands)
constexpr int SE = 3;                        // epilogue input ring per warp (16-column chunks)
constexpr int EC = 16;                       // epilogue chunk columns
constexpr uint32_t A_BYTES = TM * TK * 4;    // 16 KB fp32 tile
constexpr uint32_t AH_BYTES = TM * TK * 2;   // 8 KB bf16
constexpr uint32_t B_BYTES = 2 * TN * TK * 2;  // 32 KB hi | lo image block
constexpr uint32_t C_STAGE = 2 * AH_BYTES;   // 16 KB hi | lo
constexpr int EW = 8;                        // epilogue warps
constexpr uint32_t E_BYTES = 32 * EC * 4;    // 2 KB: one warp's 32 rows x 16 columns of the input
constexpr uint32_t OFF_A = 0;
constexpr uint32_t OFF_B = OFF_A + SA * A_BYTES;
constexpr uint32_t OFF_C = OFF_B + SB * B_BYTES;
constexpr uint32_t OFF_E = OFF_C + SC * C_STAGE;
constexpr uint32_t OFF_BAR = OFF_E + EW * SE * E_BYTES;
constexpr uint32_t SMEM_USED = OFF_BAR + 512;
constexpr uint32_t SMEM_ALLOC = SMEM_USED + 1024;  // manual 1 KB alignment of the base
constexpr int THREADS = 448;  // warp 0 TMA, 1 MMA, 2-5 converters, 6-13 epilogue
static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
static_assert(SE >= 3, "the two-input epilogue uses stages 0-1 (inputs) and 2 (output)");

struct TmaArgs {
  int64_t M, N, K;
  int ntiles;            // row blocks x ntn
  int ntn;               // 256-wide column blocks (N > 256 only when N % 256 == 0)
  const uint8_t* img;    // bf16 hi/lo weight image, [ntn][K/32][hi 16 KB | lo 16 KB]
  float* C;              // [M, ldc] output (and the old values when accumulating)
  int64_t ldc;
  const float* bias;     // [N] or null
  int n_in;              // epilogue inputs by TMA: 0, 1 or 2
  int in_kind[2];        // 0 = residual (added before ReLU), 1 = mask, 2 = old C (accumulate)
  int relu, mask_after, accumulate, has_mask;
  int dbg;  // timing experiments only (TLP_TMA_DEBUG): 1 = no epilogue work, 2 = no conversion,
            // 3 = no epilogue stores, 4 = no TMEM loads
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// PAIR (experiment, TLP_TMA_PAIR=1; off by default): clusters of two CTAs run tcgen05
// cta_group::2 -- one M = 256 MMA per instruction over a 256-row tile pair,
// each CTA holding its own 128 A rows and HALF of the weight image block (the
// N rows [128 rank, 128 rank + 128)); the rank-0 CTA issues, commits arrive in
// both CTAs.  Per 256 rows the weight image crosses L2 once instead of twice
// and the MMA issue count halves -- the single-CTA kernel's main loop waited
// for operands ~45% of the time (A 16 KB + B 32 KB per k-block and CTA).
// Correct (training parity green in this mode) but SLOWER: every launch of the
// C3 step took 1.2-1.5x longer (QKV forward 410 -> 554 us under ncu, step 3.60
// -> 4.41 ms), also with a 5-deep converted-A ring; the leader's per-k-block
// wait on both CTAs' conversions and on the relayed half-block arrivals is on
// the critical path.
template <int NIN, bool PAIR>  // epilogue inputs (a.n_in), specialised: the epilogue bounds the kernel
__global__ void __launch_bounds__(THREADS, 1) tma_gemm_kernel(const __grid_constant__ CUtensorMap mA,
                                                              const __grid_constant__ CUtensorMap mIn0,
                                                              const __grid_constant__ CUtensorMap mIn1,
                                                              const __grid_constant__ CUtensorMap mOut,
                                                              const TmaArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sb = (sraw + 1023u) & ~1023u;  // 1 KB aligned (128B-swizzle atoms)
  uint8_t* smem = smem_raw + (sb - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // pair: the weight ring holds half blocks (hi 8 KB | lo 8 KB), twice as many
  // pair: half blocks (hi 8 KB | lo 8 KB) in SB stages, and the 48 KB this
  // frees deepens the converted-A ring (SC -> 5): the leader's MMAs wait on
  // both CTAs' conversions, so the ring must cover a cross-CTA round trip
  constexpr int NSB = SB;
  constexpr uint32_t BSTG = PAIR ? B_BYTES / 2 : B_BYTES;
  constexpr int SCN = PAIR ? 5 : SC;
  constexpr uint32_t OFF_CK = OFF_B + NSB * BSTG;
  constexpr uint32_t OFF_EK = OFF_CK + SCN * C_STAGE;
  constexpr uint32_t OFF_BK = OFF_EK + EW * SE * E_BYTES;
  static_assert(OFF_BK + 512 <= SMEM_USED, "pair layout fits the single-CTA budget");
  const uint32_t bar = sb + OFF_BK;
  const uint32_t a_full = bar, a_empty = a_full + 8 * SA;
  const uint32_t b_full = a_empty + 8 * SA, b_empty = b_full + 8 * NSB;
  const uint32_t c_empty = b_empty + 8 * NSB, conv_full = c_empty + 8 * SCN;
  const uint32_t acc_full = conv_full + 8 * SCN, acc_empty = acc_full + 16, e_full = acc_empty + 16;
  const uint32_t b_peer = e_full + 8 * EW * SE;  // [NSB] pair: the peer's half block landed
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + OFF_BK + 480);
  const int nk = (int)((a.K + TK - 1) / TK);
  const int nch = (int)((min(a.N, (int64_t)TN) + EC - 1) / EC);  // chunks per tile
  const uint32_t rank = PAIR ? tc::cl_rank() : 0u;
  const uint32_t P2 = PAIR ? 2u : 1u;  // CTAs whose threads arrive on the leader's barriers
  // tile walk: single -> 128-row tiles blockIdx.x + k gridDim.x; pair -> 256-row
  // tile pairs (cluster + k clusters), this CTA's rows = row block 2 mt2 + rank
  const int wstart = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int wstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nwalk = a.ntiles;  // host: tile pairs when PAIR
  auto row_block = [&](int tile) { return PAIR ? 2 * (tile / a.ntn) + (int)rank : tile / a.ntn; };

  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) { tc::mbar_init(a_full + 8 * i, 1); tc::mbar_init(a_empty + 8 * i, 4); }
    for (int i = 0; i < NSB; ++i) {
      tc::mbar_init(b_full + 8 * i, 1); tc::mbar_init(b_empty + 8 * i, 1); tc::mbar_init(b_peer + 8 * i, 1);
    }
    for (int i = 0; i < SCN; ++i) { tc::mbar_init(c_empty + 8 * i, 1); tc::mbar_init(conv_full + 8 * i, 4 * P2); }
    for (int i = 0; i < 2; ++i) { tc::mbar_init(acc_full + 8 * i, 1); tc::mbar_init(acc_empty + 8 * i, EW * P2); }
    for (int i = 0; i < EW * SE; ++i) tc::mbar_init(e_full + 8 * i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) tc::tmem_alloc_pair(tc::smem_u32(tptr), 512);
    else tc::tmem_alloc(tc::smem_u32(tptr), 512);
  }
  tc::tc_fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  // arrivals on the leader's barriers (the peer's go through the cluster window)
  auto arrive_leader = [&](uint32_t b) {
    if (PAIR && rank != 0) tc::mbar_arrive_cluster(tc::map_cluster(b, 0));
    else tc::mbar_arrive(b);
  };
  pdl_wait();  // setup above overlapped the previous kernel's tail (TLP_LAUNCH_PDL)
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: A tiles + weight image blocks
    if (lane == 0) {
      int s = 0, t = 0;
      uint32_t ph = 0, pb = 0;
      for (int tile = wstart; tile < nwalk; tile += wstep) {
        // column block fastest: the CTAs working on one row block at a time
        // share its A tiles through L2
        const int mt = row_block(tile), nb = tile % a.ntn;
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(a_empty + 8 * s, ph ^ 1);
          tc::mbar_arrive_expect_tx(a_full + 8 * s, A_BYTES);
          tc::tma_load_2d(sb + OFF_A + s * A_BYTES, &mA, kb * TK, mt * TM, a_full + 8 * s);
          if (++s == SA) { s = 0; ph ^= 1; }
          tc::mbar_wait(b_empty + 8 * t, pb ^ 1);
          tc::mbar_arrive_expect_tx(b_full + 8 * t, BSTG);
          const uint8_t* blk = a.img + ((size_t)nb * nk + kb) * B_BYTES;
          if (PAIR) {  // this CTA's N half of the hi and of the lo block
            tc::bulk_g2s(sb + OFF_B + t * BSTG, blk + rank * (B_BYTES / 4), B_BYTES / 4, b_full + 8 * t);
            tc::bulk_g2s(sb + OFF_B + t * BSTG + B_BYTES / 4, blk + B_BYTES / 2 + rank * (B_BYTES / 4),
                         B_BYTES / 4, b_full + 8 * t);
          } else {
            tc::bulk_g2s(sb + OFF_B + t * BSTG, blk, B_BYTES, b_full + 8 * t);
          }
          if (++t == NSB) { t = 0; pb ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (pair: the leader;
    // the peer's lane 0 relays "my half block landed" to the leader)
    if (PAIR && rank != 0 && lane == 0) {
      int sbk = 0;
      uint32_t pb = 0;
      const uint32_t peer0 = tc::map_cluster(b_peer, 0);
      for (int tile = wstart; tile < nwalk; tile += wstep)
        for (int kb = 0; kb < nk; ++kb) {
          tc::mbar_wait(b_full + 8 * sbk, pb);
          tc::mbar_arrive_cluster(peer0 + 8 * sbk);
          if (++sbk == NSB) { sbk = 0; pb ^= 1; }
        }
    }
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = tc::idesc_bf16(PAIR ? 2 * TM : TM, TN);
      int s = 0, t = 0, sbk = 0;
      uint32_t ph = 0, pb = 0;
      auto wait = [&](uint32_t b, uint32_t par) {
        if (PAIR) tc::mbar_wait_cluster(b, par); else tc::mbar_wait(b, par);
      };
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t en) {
        if (PAIR) tc::mma_bf16_pair(d, ad, bd, idesc, en); else tc::mma_bf16(d, ad, bd, idesc, en);
      };
      auto commit = [&](uint32_t b) {
        if (PAIR) tc::mma_commit_pair(b); else tc::mma_commit(b);
      };
      for (int tile = wstart; tile < nwalk; tile += wstep, ++t) {
        const int buf = t & 1;
        wait(acc_empty + 8 * buf, ((t >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(buf * TN);
        for (int kb = 0; kb < nk; ++kb) {
          wait(conv_full + 8 * s, ph);
          tc::mbar_wait(b_full + 8 * sbk, pb);
          if (PAIR) tc::mbar_wait_cluster(b_peer + 8 * sbk, pb);
          tc::tc_fence_after();
          const uint32_t ah = sb + OFF_CK + s * C_STAGE, al = ah + AH_BYTES;
          const uint32_t bh = sb + OFF_B + sbk * BSTG, bl = bh + BSTG / 2;
#pragma unroll
          for (int ks = 0; ks < TK / 16; ++ks) {
            const uint64_t dah = tc::smem_desc(ah + ks * 256, 128, 512), dal = tc::smem_desc(al + ks * 256, 128, 512);
            const uint64_t dbh = tc::smem_desc(bh + ks * 256, 128, 512), dbl = tc::smem_desc(bl + ks * 256, 128, 512);
            mma(d, dal, dbh, (kb > 0 || ks > 0) ? 1u : 0u);  // Al.Bh
            mma(d, dah, dbl, 1u);                          // Ah.Bl
            mma(d, dah, dbh, 1u);                          // Ah.Bh
          }
          commit(c_empty + 8 * s);
          commit(b_empty + 8 * sbk);
          if (++s == SCN) { s = 0; ph ^= 1; }
          if (++sbk == NSB) { sbk = 0; pb ^= 1; }
        }
        commit(acc_full + 8 * buf);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------ converters (128 threads)
    const int cw = warp - 2;
    int sa = 0, sc = 0;
    uint32_t pa = 0, pc = 0;
    for (int tile = wstart; tile < nwalk; tile += wstep) {
      for (int kb = 0; kb < nk; ++kb) {
        tc::mbar_wait(a_full + 8 * sa, pa);
        tc::mbar_wait(c_empty + 8 * sc, pc ^ 1);  // the MMAs of this stage's last use are done
        const uint32_t cst = OFF_CK + sc * C_STAGE;
        const uint8_t* src = smem + OFF_A + sa * A_BYTES;
        uint8_t* hi = smem + cst;
        uint8_t* lo = hi + AH_BYTES;
#pragma unroll
        for (int it = 0; it < (a.dbg == 2 ? 0 : 8); ++it) {
          // 8 rows x 4 16-byte chunks per warp instruction: conflict-free reads of
          // the 128B-swizzled tile (chunk j of row r at j ^ (r & 7)) and
          // conflict-free 8-byte stores into the canonical layout
          const int task = it * 4 + cw;
          const int rg = task >> 1, jb = (task & 1) * 4;
          const int r = rg * 8 + (lane & 7), j = jb + (lane >> 3);
          const float4 v = *reinterpret_cast<const float4*>(src + r * 128 + ((j ^ (r & 7)) << 4));
          const uint32_t x0 = __float_as_uint(v.x), x1 = __float_as_uint(v.y);
          const uint32_t x2 = __float_as_uint(v.z), x3 = __float_as_uint(v.w);
          const uint32_t h0 = __byte_perm(x0, x1, 0x7632), h1 = __byte_perm(x2, x3, 0x7632);
          const uint32_t l0 = tc::pack_bf16(v.x - __uint_as_float(x0 & 0xffff0000u),
                                            v.y - __uint_as_float(x1 & 0xffff0000u));
          const uint32_t l1 = tc::pack_bf16(v.z - __uint_as_float(x2 & 0xffff0000u),
                                            v.w - __uint_as_float(x3 & 0xffff0000u));
          const uint32_t off = rg * 512 + (j >> 1) * 128 + (r & 7) * 16 + (j & 1) * 8;
          *reinterpret_cast<uint2*>(hi + off) = make_uint2(h0, h1);
          *reinterpret_cast<uint2*>(lo + off) = make_uint2(l0, l1);
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::mbar_arrive(a_empty + 8 * sa);
          arrive_leader(conv_full + 8 * sc);
        }
        if (++sa == SA) { sa = 0; pa ^= 1; }
        if (++sc == SCN) { sc = 0; pc ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (8 warps, 2 per TMEM lane quarter)
    // Warp (q, hh) owns rows 32q..32q+31 (thread = row = TMEM lane) and the
    // 16-column chunks c = hh, hh + 2, ...  It needs no other warp: its input
    // boxes [32 rows x 16 cols] arrive by TMA on its own mbarriers (SE deep,
    // issued ahead), and it stores its results straight from registers
    // (64 contiguous bytes per row and chunk; L2 merges the sectors).
    const int ew = warp - 6;
    const int q = warp & 3, hh = ew >> 2;
    const int r = 32 * q + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const uint32_t my_e = e_full + 8 * SE * ew;
    const uint32_t my_buf = sb + OFF_EK + (uint32_t)ew * SE * E_BYTES;
    const int nmine = (nch - hh + 1) / 2;  // chunks per tile for this warp
    const long long tiles_mine = nwalk > wstart ? (nwalk - 1 - wstart) / wstep + 1 : 0;
    const long long total = tiles_mine * nmine;
    // One input (n_in <= 1): stage g % SE holds chunk g's input, then its result
    // for the TMA store; the input of chunk g + SE - 1 is loaded into stage
    // (g - 1) % SE once the store of chunk g - 1 has finished reading it.
    // Two inputs (old C + ReLU' mask): stages 0-1 hold both inputs of one chunk
    // (re-armed for chunk g + 1 as soon as they are in registers), stage 2 is
    // the output staging buffer.
    constexpr bool two = NIN == 2;
    auto issue_in = [&](long long g) {  // this warp's g-th chunk overall
      if (NIN == 0 || g >= total) return;
      const int tile = wstart + (int)(g / nmine) * wstep;
      const int mt = row_block(tile), c0 = (tile % a.ntn) * TN;
      const int c = hh + 2 * (int)(g % nmine);
      const int se = two ? 0 : (int)(g % SE);
      tc::mbar_arrive_expect_tx(my_e + 8 * se, (uint32_t)NIN * E_BYTES);
      tc::tma_load_2d(my_buf + se * E_BYTES, &mIn0, c0 + c * EC, mt * TM + 32 * q, my_e + 8 * se);
      if (two) tc::tma_load_2d(my_buf + E_BYTES, &mIn1, c0 + c * EC, mt * TM + 32 * q, my_e);
    };
    if (lane == 0)
      for (long long g = 0; g < (two ? 1 : SE - 1); ++g) issue_in(g);
    long long g = 0;
    int t = 0;
    const int sw = (lane >> 1) & 3;  // 64B swizzle of box row `lane`: chunk j at j ^ ((lane >> 1) & 3)
    for (int tile = wstart; tile < nwalk; tile += wstep, ++t) {
      const int buf = t & 1;
      const int mt = row_block(tile), c0 = (tile % a.ntn) * TN;
      tc::mbar_wait(acc_full + 8 * buf, (t >> 1) & 1);
      tc::tc_fence_after();
      for (int c = hh; c < (a.dbg == 1 ? 0 : nch); c += 2, ++g) {
        float v[16];
        if (a.dbg != 4) tc::tmem_ld16(tl + (uint32_t)(buf * TN + c * EC), v);
        else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        float b[16];
        if (a.bias) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(a.bias + c0 + c * EC) + i);
            b[4 * i] = x.x; b[4 * i + 1] = x.y; b[4 * i + 2] = x.z; b[4 * i + 3] = x.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) b[i] = 0.f;
        }
        const int se = two ? 0 : (int)(g % SE);
        const int so = two ? 2 : se;  // output staging stage
        uint8_t* stage = smem + (my_buf - sb) + se * E_BYTES + lane * 64;
        uint8_t* ostage = smem + (my_buf - sb) + so * E_BYTES + lane * 64;
        float in[NIN > 0 ? NIN : 1][16];
        if (NIN > 0) {
          tc::mbar_wait(my_e + 8 * se, (uint32_t)((two ? g : g / SE) & 1));
#pragma unroll
          for (int s2 = 0; s2 < NIN; ++s2) {
            {
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const float4 x = *reinterpret_cast<const float4*>(stage + s2 * E_BYTES + ((jj ^ sw) << 4));
                in[s2][4 * jj] = x.x; in[s2][4 * jj + 1] = x.y; in[s2][4 * jj + 2] = x.z; in[s2][4 * jj + 3] = x.w;
              }
            }
          }
          if (two) {
            __syncwarp();
            if (lane == 0) {
              issue_in(g + 1);          // both input slots are in registers: prefetch the next chunk
              tc::bulk_wait_read<0>();  // the output stage's previous store has read it
            }
            __syncwarp();
          }
        }
        tc::tmem_wait_ld();
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float resid = 0.f, mask = 1.f, old = 0.f;
#pragma unroll
          for (int s2 = 0; s2 < NIN; ++s2) {
            {
              if (a.in_kind[s2] == 0) resid = in[s2][i];
              else if (a.in_kind[s2] == 1) mask = in[s2][i];
              else old = in[s2][i];
            }
          }
          float x = v[i] + b[i] + resid;
          if (a.relu) x = fmaxf(x, 0.f);
          if (a.has_mask && !a.mask_after) x = mask > 0.f ? x : 0.f;
          x += old;
          if (a.has_mask && a.mask_after) x = mask > 0.f ? x : 0.f;
          y[i] = x;
        }
        // one input: the result replaces the input in the same (swizzled)
        // stage -- the last store from it (chunk g - SE) finished reading
        // before the input of chunk g was loaded into it
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          *reinterpret_cast<float4*>(ostage + ((jj ^ sw) << 4)) =
              make_float4(y[4 * jj], y[4 * jj + 1], y[4 * jj + 2], y[4 * jj + 3]);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.dbg != 3) {
            tc::tma_store_2d(&mOut, c0 + c * EC, mt * TM + 32 * q, my_buf + so * E_BYTES);
            tc::bulk_commit();
          }
          if (!two) {
            tc::bulk_wait_read<1>();  // chunk g - 1's store has read its stage
            issue_in(g + SE - 1);     // -> that stage takes the input of chunk g + SE - 1
          }
        }
        __syncwarp();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(acc_empty + 8 * buf);
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    if (PAIR) tc::tmem_dealloc_pair(tmem, 512);
    else tc::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- weight gradients
// dW[Mf, Nf] (+ db = 1^T dY as row Mf) of one row slice, Mf, Nf <= 256:
//   A = X^T (X [rows][Mf], MN-major), B = dY (dY [rows][Nf], MN-major),
// both arriving by TMA as [32 rows x 32 cols] fp32 boxes with the 128B/32B-atom
// swizzle -- exactly the MN-major SWIZZLE_128B_BASE32B UMMA operand layout, the
// one kind::tf32 accepts for MN-major operands -- and consumed as
// kind::tf32 (the tensor core reads the fp32 bits and drops the low 13
// mantissa bits: no conversion pass, no second copy; R52).  One CTA per row
// slice owns the whole 256 x 256 fp32 accumulator (two M = 128 halves, 512
// TMEM columns), so X and dY are read from HBM exactly once; the bias
// gradient is summed in fp32 on the CUDA cores from the same staged dY tiles.
// Partials [slice][Mf + 1][Nf] leave by TMA store and are reduced in a fixed
// order by the caller (deterministic).
constexpr int WK = 32;                       // rows per k-block (4 tf32 k-steps)
constexpr int WS = 3;                        // stages
constexpr uint32_t WBOX = 32 * 32 * 4;       // one [32 x 32] fp32 box, 4 KB
constexpr uint32_t WSTAGE = 16 * WBOX;       // X 8 boxes | dY 8 boxes = 64 KB
constexpr uint32_t W_OFF_BAR = WS * WSTAGE;
constexpr uint32_t W_SMEM = W_OFF_BAR + 256 + 1024;
constexpr int W_THREADS = 192;               // warp 0 TMA, 1 MMA, 2-5 column sums + epilogue
static_assert(W_SMEM <= 232448, "wgrad shared memory budget");

struct WgradArgs {
  int64_t R, kslice;
  int Mf, Nf, Z;
  int64_t cy0;                               // dY column of product j = blockIdx.x: cy0 * j
  float* part;                               // [J][Z][Mf + 1][Nf]
  int dbg;                                   // TLP_TMA_WGRAD_DEBUG (diagnostics)
};

template <bool COLSUM>
__global__ void __launch_bounds__(W_THREADS, 1) tma_wgrad_kernel(const __grid_constant__ CUtensorMap mX,
                                                                 const __grid_constant__ CUtensorMap mY,
                                                                 const __grid_constant__ CUtensorMap mP,
                                                                 const WgradArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = tc::smem_u32(smem_raw);
  const uint32_t sb = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sb - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x, z = blockIdx.y;
  const uint32_t full = sb + W_OFF_BAR, empty = full + 8 * WS, done = empty + 8 * WS;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + W_OFF_BAR + 128);
  const int64_t r0 = (int64_t)z * a.kslice;
  const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(a.kslice, a.R - r0));
  const int nkb = (int)((rows + WK - 1) / WK);
  const int nbx = a.Mf / 32, nby = a.Nf / 32, nmh = (a.Mf + 127) / 128;
  const int cy = (int)(a.cy0 * j);
  if (threadIdx.x == 0) {
    for (int i = 0; i < WS; ++i) {
      tc::mbar_init(full + 8 * i, 1);
      tc::mbar_init(empty + 8 * i, COLSUM ? 5 : 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tc::smem_u32(tptr), 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tptr;
  pdl_wait();  // setup above overlapped the previous kernel's tail (TLP_LAUNCH_PDL)
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(empty + 8 * s, ph ^ 1);
        tc::mbar_arrive_expect_tx(full + 8 * s, (uint32_t)(nbx + nby) * WBOX);
        const int row = (int)(r0 + (int64_t)kb * WK);
        const uint32_t st = sb + s * WSTAGE;
        for (int i = 0; i < nbx; ++i) tc::tma_load_2d(st + i * WBOX, &mX, 32 * i, row, full + 8 * s);
        for (int i = 0; i < nby; ++i) tc::tma_load_2d(st + (8 + i) * WBOX, &mY, cy + 32 * i, row, full + 8 * s);
        if (++s == WS) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, (uint32_t)a.Nf, 1u, 1u);
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(full + 8 * s, ph);
        tc::tc_fence_after();
        const uint32_t st = sb + s * WSTAGE;
#pragma unroll
        for (int ks = 0; ks < WK / 8; ++ks) {
          // MN-major SWIZZLE_128B_BASE32B: LBO = next 32-element MN block (next
          // box), SBO = next 4 K rows (the 32B atom's K extent); a k-step = 8 rows
          const uint64_t bd = tc::smem_desc_sw128_32b(st + 8 * WBOX + ks * 1024, WBOX, 512);
          for (int mh = 0; mh < nmh; ++mh) {
            const uint64_t ad = tc::smem_desc_sw128_32b(st + mh * 4 * WBOX + ks * 1024, WBOX, 512);
            tc::mma_tf32(tmem + 256u * mh, ad, bd, idesc, (kb > 0 || ks > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(empty + 8 * s);
        if (++s == WS) { s = 0; ph ^= 1; }
      }
      tc::mma_commit(done);
    }
  } else {
    // ---- warps 2..5: fp32 column sums of dY while the tiles stream, then the epilogue
    const int et = threadIdx.x - 64;
    float cs[2] = {0.f, 0.f};
    if (COLSUM) {
      int s = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(full + 8 * s, ph);
        const uint8_t* yb = smem + s * WSTAGE + 8 * WBOX;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int n = et + 128 * i;
          if (n < a.Nf) {
            const uint8_t* box = yb + (n >> 5) * WBOX;
            const int ch = (n & 31) >> 3, el = (n & 7) * 4;  // 32-byte chunk, byte in it
            float acc = cs[i];
#pragma unroll 8
            for (int r = 0; r < WK; ++r)  // fixed order
              acc += *reinterpret_cast<const float*>(box + r * 128 + ((ch ^ (r & 3)) << 5) + el);
            cs[i] = acc;
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(empty + 8 * s);
        if (++s == WS) { s = 0; ph ^= 1; }
      }
    }
    const int q = warp & 3;
    const int prow = (j * a.Z + z) * (a.Mf + 1);  // first partial row of (j, z)
    if (nkb > 0) {
      tc::mbar_wait(done, 0);
      tc::tc_fence_after();
    }
    // staging: two 4 KB boxes per warp in the (now idle) stage 0
    const uint32_t stg = sb + (uint32_t)(warp - 2) * 2 * WBOX;
    uint8_t* stg_p = smem + (stg - sb);
    int nb = 0;
    for (int mh = 0; mh < nmh; ++mh) {
      if (mh * 128 + 32 * q >= a.Mf) break;
      for (int cb = 0; cb < nby; ++cb, ++nb) {
        float v[32];
        if (nkb > 0) {
          tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 256u * mh + 32u * cb, v);
          tc::tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (a.dbg == 1) {  // diagnostics: direct stores of the accumulator rows
          float* d = a.part + (int64_t)(prow + mh * 128 + 32 * q + lane) * a.Nf + 32 * cb;
          for (int i = 0; i < 32; ++i) d[i] = v[i];
          continue;
        }
        if (a.dbg == 2) {  // diagnostics: accumulator lane / column pattern
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = (float)(1000 * (32 * q + lane) + 32 * cb + i);
        }
        if (lane == 0) tc::bulk_wait_read<1>();  // this staging box's previous store has read it
        __syncwarp();
        uint8_t* row = stg_p + (nb & 1) * WBOX + lane * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(row + ((c ^ (lane & 7)) << 4)) =
              make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tc::tma_store_2d(&mP, 32 * cb, prow + mh * 128 + 32 * q, stg + (nb & 1) * WBOX);
          tc::bulk_commit();
        }
      }
    }
    if (COLSUM) {
      float* dst = a.part + (int64_t)(prow + a.Mf) * a.Nf;
#pragma unroll
      for (int i = 0; i < 2; ++i)
        if (et + 128 * i < a.Nf) dst[et + 128 * i] = cs[i];
    }
    if (lane == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// fp32 [rows][ld] matrix, box [box_rows][box_cols]
bool make_map(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, uint32_t box_cols,
              uint32_t box_rows, CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_ok(const void* p, int64_t ld) {
  return p && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 4 == 0;
}

}  // namespace

// Returns TLP_ERR_UNSUPPORTED (nothing launched) when the call does not fit the
// kernel; the caller then uses the register-staged path.
tlp_status tc_gemm_tma(tlp_ctx* ctx, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                       const uint8_t* img, float* C, int64_t ldc, const EpiParams& e, cudaStream_t s) {
  static const char* env = getenv("TLP_TMA_GEMM");
  if (env && env[0] == '0') return TLP_ERR_UNSUPPORTED;
  if (!(N > 64 && (N <= TN || N % TN == 0) && N % EC == 0 && K > 0 && M > 0 &&
        cdiv(M, TM) * cdiv(N, TN) <= (int64_t)INT32_MAX / 2))
    return TLP_ERR_UNSUPPORTED;
  if (!tma_ok(A, lda) || !tma_ok(C, ldc)) return TLP_ERR_UNSUPPORTED;
  TmaArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.ntn = (int)cdiv(N, TN);
  a.ntiles = (int)(cdiv(M, TM) * a.ntn);
  a.img = img;
  a.bias = e.bias;
  a.relu = e.relu ? 1 : 0;
  a.mask_after = e.mask_after ? 1 : 0;
  a.accumulate = e.accumulate ? 1 : 0;
  a.has_mask = e.mask ? 1 : 0;
  static const char* dbg = getenv("TLP_TMA_DEBUG");
  a.dbg = dbg ? atoi(dbg) : 0;
  a.C = C;
  a.ldc = ldc;
  const float* ins[2] = {nullptr, nullptr};
  int64_t lds[2] = {0, 0};
  auto add_in = [&](const float* p, int64_t ld, int kind) {
    if (a.n_in == 2) return false;
    ins[a.n_in] = p; lds[a.n_in] = ld; a.in_kind[a.n_in] = kind; ++a.n_in;
    return tma_ok(p, ld);
  };
  if (e.resid && !add_in(e.resid, e.ldr, 0)) return TLP_ERR_UNSUPPORTED;
  if (e.accumulate && !add_in(C, ldc, 2)) return TLP_ERR_UNSUPPORTED;
  if (e.mask && !add_in(e.mask, e.ldm, 1)) return TLP_ERR_UNSUPPORTED;
  if (e.bias && (reinterpret_cast<uintptr_t>(e.bias) & 15)) return TLP_ERR_UNSUPPORTED;
  CUtensorMap mA, mI0, mI1, mO;
  if (!make_map(&mA, A, K, M, lda, TK, TM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mO, C, N, M, ldc, EC, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return TLP_ERR_UNSUPPORTED;
  mI0 = mO;
  mI1 = mO;
  if (a.n_in > 0 && !make_map(&mI0, ins[0], N, M, lds[0], EC, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return TLP_ERR_UNSUPPORTED;
  if (a.n_in > 1 && !make_map(&mI1, ins[1], N, M, lds[1], EC, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return TLP_ERR_UNSUPPORTED;
  static const char* penv = getenv("TLP_TMA_PAIR");  // cta_group::2 pairs (experiment, default off)
  const bool pair = penv && penv[0] == '1' && ctx->num_sms >= 2 && M > TM;
  if (pair) {
    a.ntiles = (int)(cdiv(M, 2 * TM) * a.ntn);  // 256-row tile pairs
    const int grid = 2 * (int)std::min<int64_t>(a.ntiles, ctx->num_sms / 2);
    // (the three kernels share one function-pointer type: no per-call-site
    // static here -- TLP_SMEM_ATTR would then cover only the first of them)
    auto launch = [&](auto kern) -> cudaError_t {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_ALLOC);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3(THREADS);
      cfg.dynamicSmemBytes = SMEM_ALLOC;
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      static const char* ppdl = getenv("TLP_TMA_PAIR_PDL");  // cluster + PDL launch (experiment)
      cfg.numAttrs = (ppdl && ppdl[0] == '1' && pdl_enabled()) ? 2 : 1;
      return cudaLaunchKernelEx(&cfg, kern, mA, mI0, mI1, mO, a);
    };
    cudaError_t le = a.n_in == 0 ? launch(tma_gemm_kernel<0, true>)
                   : a.n_in == 1 ? launch(tma_gemm_kernel<1, true>) : launch(tma_gemm_kernel<2, true>);
    if (le != cudaSuccess) {
      ctx->last_error = std::string("CUDA launch (tma_gemm pair): ") + cudaGetErrorString(le);
      return TLP_ERR_CUDA;
    }
    TLP_LAUNCH_CHECK();
    return TLP_OK;
  }
  const int grid = (int)std::min<int64_t>(a.ntiles, ctx->num_sms);
  if (a.n_in == 0) {
    TLP_SMEM_ATTR((tma_gemm_kernel<0, false>), SMEM_ALLOC);
    TLP_LAUNCH_PDL((tma_gemm_kernel<0, false>), grid, THREADS, SMEM_ALLOC, s, mA, mI0, mI1, mO, a);
  } else if (a.n_in == 1) {
    TLP_SMEM_ATTR((tma_gemm_kernel<1, false>), SMEM_ALLOC);
    TLP_LAUNCH_PDL((tma_gemm_kernel<1, false>), grid, THREADS, SMEM_ALLOC, s, mA, mI0, mI1, mO, a);
  } else {
    TLP_SMEM_ATTR((tma_gemm_kernel<2, false>), SMEM_ALLOC);
    TLP_LAUNCH_PDL((tma_gemm_kernel<2, false>), grid, THREADS, SMEM_ALLOC, s, mA, mI0, mI1, mO, a);
  }
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

// Weight (+ bias) gradient partials of J products sharing X (dY_j = columns
// [j cy0, j cy0 + Nf) of dY): part[j][z][Mf + colsum][Nf] for row slices of
// kslice rows.  TLP_ERR_UNSUPPORTED (nothing launched) when the shapes or
// alignments do not fit; the caller then uses the bf16x3 register-staged kernel.
tlp_status tc_wgrad_tma(tlp_ctx* ctx, int64_t R, int64_t Mf, int64_t Nf, const float* X, int64_t ldx,
                        const float* dY, int64_t ldy, float* part, int Z, int64_t kslice, bool colsum,
                        int J, int64_t cy0, cudaStream_t s) {
  static const char* env = getenv("TLP_TMA_WGRAD");
  if (env && env[0] == '0') return TLP_ERR_UNSUPPORTED;
  if (!(Mf % 32 == 0 && Mf >= 32 && Mf <= 256 && Nf % 32 == 0 && Nf >= 32 && Nf <= 256 && R > 0 &&
        R <= (int64_t)INT32_MAX - WK && kslice % WK == 0 && Z >= 1 && J >= 1 && J <= 8))
    return TLP_ERR_UNSUPPORTED;
  if (!tma_ok(X, ldx) || !tma_ok(dY, ldy) || !tma_ok(part, Nf) || (J > 1 && cy0 % 4 != 0))
    return TLP_ERR_UNSUPPORTED;
  CUtensorMap mX, mY, mP;
  const int64_t ycols = (J - 1) * cy0 + Nf;
  if (!make_map(&mX, X, Mf, R, ldx, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      !make_map(&mY, dY, ycols, R, ldy, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      !make_map(&mP, part, Nf, (int64_t)J * Z * (Mf + 1), Nf, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return TLP_ERR_UNSUPPORTED;
  static const char* dbg = getenv("TLP_TMA_WGRAD_DEBUG");
  WgradArgs a{R, kslice, (int)Mf, (int)Nf, Z, cy0, part, dbg ? atoi(dbg) : 0};
  const dim3 grid((unsigned)J, (unsigned)Z);
  if (colsum) {
    TLP_SMEM_ATTR(tma_wgrad_kernel<true>, W_SMEM);
    TLP_LAUNCH_PDL(tma_wgrad_kernel<true>, grid, W_THREADS, W_SMEM, s, mX, mY, mP, a);
  } else {
    TLP_SMEM_ATTR(tma_wgrad_kernel<false>, W_SMEM);
    TLP_LAUNCH_PDL(tma_wgrad_kernel<false>, grid, W_THREADS, W_SMEM, s, mX, mY, mP, a);
  }
  TLP_LAUNCH_CHECK();
  return TLP_OK;
}

bool make_tmap_f32_2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld,
                      uint32_t box_cols, uint32_t box_rows, int swizzle) {
  if (!base || (reinterpret_cast<uintptr_t>(base) & 15) || (ld * 4) % 16 || rows < 1) return false;
  return make_map(m, base, cols, rows, ld, box_cols, box_rows, static_cast<CUtensorMapSwizzle>(swizzle));
}
