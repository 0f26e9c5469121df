// tc_gemm.cu — warp-specialized persistent tcgen05 GEMM for the SP/HP tile
// classes of the Cholesky (see tc_gemm.cuh), plus the panel producers that
// write the sender-side operand mirrors.
//
// CTA = 384 threads: warp 0 issues TMA, warp 1 issues tcgen05.mma (one
// elected lane), warp 2 owns the TMEM allocation, warps 4-11 run the epilogue
// (TMEM lane quarter = warp % 4, two warps per quarter splitting the columns
// so every SM sub-partition has two epilogue warps to hide latency). Two TMEM accumulators let the epilogue of
// sub-tile t overlap the MMAs of sub-tile t+1. Each work item is a 128 x BN
// sub-tile of one b x b output tile with K = b.
#include <cstdlib>
#include <random>
#include <vector>

#include "tc_gemm.cuh"
#include "ozaki.cuh"
#include "tcgen05.cuh"

namespace sphemu_gpu {

// ---------------------------------------------------------------------------
// Host: tensor maps
// ---------------------------------------------------------------------------
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      throw Error(SPHEMU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

}  // namespace

CUtensorMap make_map_strided(const void* base, int64_t rows, int64_t cols, int64_t row_bytes, int elem_bytes,
                             int box_rows, int swizzle_bytes) {
  CUtensorMap m;
  const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(swizzle_bytes / elem_bytes), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SPHEMU_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}
namespace {
// Row-major [rows x cols] array, box = 128 bytes of K x box_rows rows, SW128.
CUtensorMap make_map(const void* base, int64_t rows, int64_t cols, int elem_bytes, int box_rows,
                     int swizzle_bytes = 128) {
  return make_map_strided(base, rows, cols, cols * elem_bytes, elem_bytes, box_rows, swizzle_bytes);
}

}  // namespace

// The C-operand view of the tile arena for the update epilogue: the arena
// as [bytes / (esz b)] rows of b elements (every tile offset is a multiple
// of esz b bytes), one map per C class width, 32-row TMA boxes.
void PanelFormats::set_arena(const void* base, int64_t bytes, int b_) {
  m_c16 = make_map_strided(base, bytes / (2 * b_), b_, 2 * static_cast<int64_t>(b_), 2, 32);
  m_c32 = make_map_strided(base, bytes / (4 * b_), b_, 4 * static_cast<int64_t>(b_), 4, 32);
}

void PanelFormats::alloc(int nt_, int b_, const std::vector<uint8_t>& pmap, int hp_format_, bool f16x3_,
                         const int* rowexp_) {
  f16x3 = f16x3_;
  need_tf32 = !f16x3_;
  need_p16 = false;
  for (uint8_t p : pmap) need_p16 |= (p == SPHEMU_PREC_HP);  // pmap holds SPHEMU_PREC_* per tile
  rowexp = rowexp_;
  nt = nt_;
  b = b_;
  hp_format = hp_format_;
  bn = (b % 256 == 0) ? 256 : 128;
  const int64_t rows = static_cast<int64_t>(nt - 1) * b;
  const size_t elems = static_cast<size_t>(rows) * b;
  p_hi.alloc(elems);
  p_lo.alloc(elems);
  p16.alloc(elems);
  in_hi.alloc(elems);
  in_lo.alloc(elems);
  l_hi.alloc(static_cast<size_t>(b) * b);
  l_lo.alloc(static_cast<size_t>(b) * b);
  const int bn_tf32 = 128;  // tf32x3 uses 128-wide N tiles (smem budget)
  m_phi_a = make_map(p_hi.get(), rows, b, 4, TC_BM);
  m_plo_a = make_map(p_lo.get(), rows, b, 4, TC_BM);
  m_phi_b = make_map(p_hi.get(), rows, b, 4, bn_tf32);
  m_plo_b = make_map(p_lo.get(), rows, b, 4, bn_tf32);
  m_p16_a = make_map(p16.get(), rows, b, 2, TC_BM);
  m_p16_b = make_map(p16.get(), rows, b, 2, bn);
  m_inhi_a = make_map(in_hi.get(), rows, b, 4, TC_BM);
  m_inlo_a = make_map(in_lo.get(), rows, b, 4, TC_BM);
  m_lhi_b = make_map(l_hi.get(), b, b, 4, bn_tf32);
  m_llo_b = make_map(l_lo.get(), b, b, 4, bn_tf32);
  if (f16x3 || hp_format == SPHEMU_HP_BF16) {  // FP16x3 panel (opt-in) / the BF16x2 panel's operands
    in16_hi.alloc(elems);
    in16_lo.alloc(elems);
    l16_hi.alloc(static_cast<size_t>(b) * b);
    l16_lo.alloc(static_cast<size_t>(b) * b);
    lexp.alloc(b);
    m_in16hi_a = make_map(in16_hi.get(), rows, b, 2, TC_BM);
    m_in16lo_a = make_map(in16_lo.get(), rows, b, 2, TC_BM);
    m_l16hi_b = make_map(l16_hi.get(), b, b, 2, 128);
    m_l16lo_b = make_map(l16_lo.get(), b, b, 2, 128);
  }
  if (f16x3) {
    h_hi.alloc(elems);
    h_lo.alloc(elems);
    m_hhi_a = make_map(h_hi.get(), rows, b, 2, TC_BM, 128);
    m_hlo_a = make_map(h_lo.get(), rows, b, 2, TC_BM, 128);
    m_hhi_b = make_map(h_hi.get(), rows, b, 2, bn, 128);
    m_hlo_b = make_map(h_lo.get(), rows, b, 2, bn, 128);
  }
}

// ---------------------------------------------------------------------------
// Device: the persistent warp-specialized GEMM
// ---------------------------------------------------------------------------
// OP_BF16X2: A one bf16 operand, B a bf16 hi/lo split (2 MMAs): the BF16-class panel TRSM
enum : int { OP_F16 = 0, OP_BF16 = 1, OP_TF32X3 = 2, OP_F16X3 = 3, OP_BF16X2 = 4 };
enum : int { MODE_UPDATE = 0, MODE_PANEL = 1 };

struct TcArgs {
  TileStore ts;
  const int2* list;  // output tiles (i, j); panel mode: (i, k)
  const int* crow;   // update mode: per list entry, the tile's first row in the C tensor map
  int64_t items;     // list entries * sub-tiles per entry
  int k;
  int b;
  int sub_n;         // b / BN
  int sub_per;       // (b / 128) * sub_n
  double* p64;
  float* p_hi;
  float* p_lo;
  uint16_t* p16;
  uint16_t* h_hi;    // fp16 split of the row-scaled panel (FP16x3 path)
  uint16_t* h_lo;
  const int* rowexp; // per global row: power-of-two scale exponent
  int lb;            // logical tile size (global row = tile * lb + local row)
  int hp_format;
  const int* fail;
  unsigned* sat;
  int dbg;           // diagnostics only (SPHEMU_TC_DBG): 1 = skip the C epilogue, 2 = also skip the MMAs
  int opt;           // tuning switches (SPHEMU_TC_OPT): 1 = C prefetch to L2 (TMA, one item ahead),
                     // 4 = operands evict_first (not evict_last), 8 = C through L2 normally (not streaming),
                     // 16 = operands evict_normal, 32 = operands evict_last on a 0.5 fraction
  int* counter;      // non-null: items are claimed dynamically (atomicAdd), zeroed before the launch
  const int* lexp;   // FP16x3 panel: per output column (Linv row) power-of-two exponent
  const int* yield;  // non-null: stop claiming items once *yield != 0 (dynamic scheduling only)
  int k2;            // update mode: second panel step of a merged two-step update (-1 = none)
  uint8_t* s8;       // panel mode: INT8 DP digit rows to write (nullptr = none; p64 may then be nullptr)
};

template <int OPK>
struct OpTraits {
  static constexpr bool kSplit = (OPK == OP_TF32X3 || OPK == OP_F16X3);
  static constexpr bool kBsplit = (OPK == OP_BF16X2);  // only B carries a lo part
  static constexpr bool kTf32 = (OPK == OP_TF32X3);
  static constexpr int kElem = kTf32 ? 4 : 2;
  // smem row of K per stage (swizzle width). 64-byte rows (SWIZZLE_64B, twice
  // the stages) were measured slower for FP16x3 than 128-byte rows.
  static constexpr int kRowBytes = 128;
  static constexpr int kBK = kRowBytes / kElem;  // K elements per stage
  static constexpr int kUK = kTf32 ? 8 : 16;    // K per tcgen05.mma
  static constexpr int kFmt = (OPK == OP_F16 || OPK == OP_F16X3) ? 0 : ((OPK == OP_BF16 || OPK == OP_BF16X2) ? 1 : 2);
};

// CG = 2: a CTA pair (cluster of 2) runs cta_group::2 MMAs of M = 256: each
// CTA stages its own 128 rows of A and half of the BN rows of B per stage
// and holds its 128 accumulator rows in its own TMEM.
template <int BN, int OPK, int MODE, int CG = 1>
struct TcLayout {
  using T = OpTraits<OPK>;
  static constexpr bool kUpd = (MODE == MODE_UPDATE);
  static constexpr int kA = TC_BM * T::kRowBytes;          // bytes of one A buffer
  static constexpr int kB = (BN / CG) * T::kRowBytes;      // bytes of one B buffer (this CTA's rows)
  static constexpr int kStage = (T::kSplit ? 2 : 1) * (kA + kB) + (T::kBsplit ? kB : 0);
  // Update mode stages the C tile through shared memory: per epilogue warp
  // a ring of kRing TMA boxes (32 rows x 128 bytes each).
#ifndef SPH_TC_RING
#define SPH_TC_RING 1
#endif
#ifndef SPH_TC_RING2
#define SPH_TC_RING2 3
#endif
#ifndef SPH_TC_RING_SPLIT128
#define SPH_TC_RING_SPLIT128 1
#endif
  // Epilogue warps: 8 (two per TMEM lane quarter), or 16 for the CTA-pair
  // 16-bit update (four per quarter, one 64-column box each): that epilogue
  // is latency-bound, and more warps per sub-partition hide the C box round
  // trip better than a deeper per-warp ring, which would cost operand stages
  // (measured at N = 98 304 dpsphp/bf16: HP update 798 TFLOP/s vs 758 with 8
  // warps and a 3-box ring; single CTAs with 16 warps drop to 3 stages, 633).
#ifndef SPH_TC_EPI16
#define SPH_TC_EPI16 1
#endif
#ifndef SPH_TC_RING16
#define SPH_TC_RING16 1
#endif
#ifndef SPH_TC_REGC
#define SPH_TC_REGC 1  // register-staged C boxes (see the epilogue); 0 = TMA load/store ring
#endif
  static constexpr bool kWide = kUpd && !T::kSplit && BN == 256 && CG == 2 && SPH_TC_EPI16;
  static constexpr int kEpi = kWide ? 16 : TC_EPI_WARPS;
  static constexpr int kThreads = 32 * (4 + kEpi);
  static constexpr int kRing =
      kUpd ? ((kWide || SPH_TC_REGC) ? (SPH_TC_REGC ? 1 : SPH_TC_RING16)
                    : ((CG == 2 && !T::kSplit) ? SPH_TC_RING2
                                               : ((T::kSplit && BN == 128) ? SPH_TC_RING_SPLIT128 : SPH_TC_RING)))
           : 0;
  static constexpr int kStages = (232448 - 2048 - kEpi * kRing * 32 * 128) / kStage > 6
                                     ? 6
                                     : (232448 - 2048 - kEpi * kRing * 32 * 128) / kStage;
  static constexpr int kCBox = 32 * 128;
  static constexpr int kCBytes = kEpi * kRing * kCBox;
  static constexpr int kSmem = kStages * kStage + kCBytes + 1024 /*align*/ + 1024 /*barriers + schedule*/;
  static constexpr int kAcc = (512 / BN) > 4 ? 4 : (512 / BN);  // TMEM accumulators in flight (512 columns)
  static constexpr int kTmemCols = kAcc * BN;
  static_assert(kSmem <= 232448, "shared memory budget");
};

template <int BN, int OPK, int MODE, int CG>
__global__ void __launch_bounds__(TcLayout<BN, OPK, MODE, CG>::kThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap mA_hi, const __grid_constant__ CUtensorMap mA_lo,
              const __grid_constant__ CUtensorMap mB_hi, const __grid_constant__ CUtensorMap mB_lo,
              const __grid_constant__ CUtensorMap mC, const __grid_constant__ CUtensorMap mA2_hi,
              const __grid_constant__ CUtensorMap mA2_lo, const __grid_constant__ CUtensorMap mB2_hi,
              const __grid_constant__ CUtensorMap mB2_lo, const TcArgs args) {
  using T = OpTraits<OPK>;
  using Lay = TcLayout<BN, OPK, MODE, CG>;
  static_assert(CG == 1 || MODE == MODE_UPDATE, "CTA pairs run the trailing update only");
  constexpr int S = Lay::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* cbuf = smem + S * Lay::kStage;  // 1024-aligned (stages are multiples of 1024 bytes)
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + Lay::kCBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + Lay::kAcc;
  uint64_t* cfull = tempty + Lay::kAcc;  // [epilogue warp][kRing]
  uint64_t* sfull = cfull + Lay::kEpi * Lay::kRing;  // dynamic schedule ring: producer -> consumers
  uint64_t* sempty = sfull + 4;                          // consumers (MMA warp + epilogue warps) -> producer
  int* sched = reinterpret_cast<int*>(sempty + 4);       // [4] claimed items (-1 = none left)
  int* wcache = sched + 4;                               // [kEpi][4] epilogue copies
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wcache + Lay::kEpi * 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // An earlier POTRF failed: read once per CTA (the chain's kernel may set
  // the flag between two threads' reads) so the CTA leaves as a whole; a
  // pair uses the leader's read for both CTAs (below, after the cluster
  // barrier that publishes the peer's mbarriers).
  __shared__ int s_fail;
  if constexpr (CG == 1) {
    if (threadIdx.x == 0) s_fail = *(volatile const int*)args.fail;
    __syncthreads();
    if (s_fail >= 0) return;
  }
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;  // 0 = pair leader (issues the MMAs)
  const int64_t cid = blockIdx.x / CG, ncl = gridDim.x / CG;  // work is strided over clusters

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < Lay::kAcc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * Lay::kEpi);  // one arrive per epilogue warp of each CTA
    }
    for (int s = 0; s < Lay::kEpi * Lay::kRing; ++s) mbar_init(&cfull[s], 1);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&sfull[s], 1);
      // consumers: the MMA warp + the epilogue warps; a pair's leader also
      // counts the peer's producer and epilogue warps (remote arrivals)
      mbar_init(&sempty[s], CG == 2 ? 2 + 2 * Lay::kEpi : 1 + Lay::kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA_hi);
    tma_prefetch(&mB_hi);
    if (MODE == MODE_UPDATE && args.k2 >= 0) {
      tma_prefetch(&mA2_hi);
      tma_prefetch(&mB2_hi);
      if (T::kSplit) {
        tma_prefetch(&mA2_lo);
        tma_prefetch(&mB2_lo);
      }
    }
    if (MODE == MODE_UPDATE) tma_prefetch(&mC);
    if (T::kSplit) {
      tma_prefetch(&mA_lo);
      tma_prefetch(&mB_lo);
    }
  }
  if (warp == 2) {
    if constexpr (CG == 2) tmem_alloc_cg2(tmem_holder, Lay::kTmemCols);
    else tmem_alloc(tmem_holder, Lay::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if constexpr (CG == 2) {
    if (rank == 0 && threadIdx.x == 0) {
      const int f = *(volatile const int*)args.fail;
      s_fail = f;
      st_cluster_u32(mapa_shared(&s_fail, 1), static_cast<uint32_t>(f));
    }
    cluster_sync_all();
    if (s_fail >= 0) {
      if (warp == 2) tmem_dealloc_cg2(tmem_base, Lay::kTmemCols);
      return;
    }
  }

  const int kblocks = args.b / T::kBK;
  const int halves = (MODE == MODE_UPDATE && args.k2 >= 0) ? 2 : 1;  // merged two-step update
  const int64_t items = args.items;
  // Work items: statically strided over clusters, or (CG = 1 with a counter)
  // claimed one by one by the producer and handed to the MMA and epilogue
  // warps through a 4-slot ring, so CTAs that start late (SMs still held by a
  // concurrent kernel) simply find less work left.
  // Dynamic claims: CTAs (or pair leaders) take items from an atomic counter;
  // a leader hands each item to its peer through the peer's ring slot.
  const bool dyn = args.counter != nullptr;
  auto static_item = [&](int64_t n) -> int64_t {
    const int64_t w = cid + n * ncl;
    return w < items ? w : -1;
  };
  auto ring_take = [&](int64_t n) -> int64_t {  // consumer side; caller decides who arrives
    const int slot = static_cast<int>(n & 3);
    if constexpr (CG == 2) mbar_wait_cluster(&sfull[slot], static_cast<uint32_t>((n >> 2) & 1));
    else mbar_wait(&sfull[slot], static_cast<uint32_t>((n >> 2) & 1));
    return static_cast<int64_t>(*(volatile int*)&sched[slot]);
  };
  auto ring_release = [&](int64_t n) {  // one consumer's arrival on the (leader's) empty slot
    if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(&sempty[n & 3], 0));
    else mbar_arrive(&sempty[n & 3]);
  };

  auto decode = [&](int64_t w, int& i, int& j, int& m0, int& n0) {
    const int2 ij = args.list[w / args.sub_per];
    const int sub = static_cast<int>(w % args.sub_per);
    i = ij.x;
    j = ij.y;
    m0 = (sub / args.sub_n) * (TC_BM * CG) + static_cast<int>(rank) * TC_BM;
    n0 = (sub % args.sub_n) * BN;
  };

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // SPHEMU_TC_OPT A/B tests: bit 2 evict_first, bit 16 evict_normal, bit 32 evict_last on half the lines
      const uint64_t keep = (args.opt & 4)    ? l2_evict_first()
                            : (args.opt & 16) ? l2_evict_normal()
                            : (args.opt & 32) ? l2_evict_last_half()
                                              : l2_evict_last();
      // Update mode, opt-in (SPHEMU_TC_OPT bit 1): pull the C sub-tile of the
      // next work item into L2 while this one's MMAs run. Off by default: the
      // epilogue's register-staged C loads run a box ahead anyway, and the
      // prefetched C lines evicted the panel operands every item re-reads
      // (C2 47.4 -> 46.2 ms, n = 64 800 dpsp 233.5 -> 220.0 ms, C3 891.5 ->
      // 829.0 ms without it; tools/gpu_tasks.sh sweep with SPHEMU_TC_OPT).
      // The next item's list entry and C row are loaded while this item's
      // first stages are in flight (a dependent global load here would stall
      // the TMA issue at every item boundary).
      auto prefetch_c = [&](int64_t wi, int2 ij, int crow) {
        if (MODE != MODE_UPDATE || SPH_DBG(args) == 1 || SPH_DBG(args) == 2 || SPH_DBG(args) == 5 || !(args.opt & 1) || wi >= items)
          return;
        constexpr int kEszP = T::kSplit ? 4 : 2;
        (void)ij;
        const int sub = static_cast<int>(wi % args.sub_per);
        const int tm = (sub / args.sub_n) * (TC_BM * CG) + static_cast<int>(rank) * TC_BM;
        const int tn = (sub % args.sub_n) * BN;
#pragma unroll 1
        for (int rq = 0; rq < TC_BM; rq += 32)
#pragma unroll 1
          for (int cx = 0; cx < BN; cx += 128 / kEszP) tma_prefetch_l2_2d(&mC, tn + cx, crow + tm + rq);
      };
      auto fetch = [&]() -> int64_t {
        // a yield request stops new claims; claimed items are always processed
        if (args.yield && *(volatile const int*)args.yield) return -1;
        const int64_t v = atomicAdd(args.counter, 1);
        return v < items ? v : -1;
      };
      auto publish = [&](int64_t n, int64_t v) {
        const int slot = static_cast<int>(n & 3);
        if constexpr (CG == 2) {
          mbar_wait_cluster(&sempty[slot], static_cast<uint32_t>(((n >> 2) & 1) ^ 1));
          sched[slot] = static_cast<int>(v);
          st_cluster_u32(mapa_shared(&sched[slot], 1), static_cast<uint32_t>(v));
          mbar_arrive(&sfull[slot]);
          mbar_arrive_cluster(mapa_shared(&sfull[slot], 1));  // release.cluster: orders the remote store
        } else {
          mbar_wait(&sempty[slot], static_cast<uint32_t>(((n >> 2) & 1) ^ 1));
          sched[slot] = static_cast<int>(v);
          mbar_arrive(&sfull[slot]);  // release: the slot write is visible to the consumers
        }
      };
      // A pair's peer producer is a consumer of the leader's claims.
      auto claim_item = [&](int64_t n) -> int64_t {
        if (CG == 2 && rank != 0) {
          const int64_t v = ring_take(n);
          ring_release(n);
          return v;
        }
        const int64_t v = fetch();
        publish(n, v);
        return v;
      };
      // A pair's leader claims one item further ahead, so the peer finds its
      // next item already published at the top of each item (the claim's
      // atomic and the cross-CTA handoff stay off the peer's TMA issue).
      constexpr bool kAhead = CG == 2;
      int64_t w = dyn ? claim_item(0) : static_item(0);
      int64_t w_ahead = (dyn && kAhead && rank == 0 && w >= 0) ? claim_item(1) : -1;
      int2 ij_cur = w >= 0 ? args.list[w / args.sub_per] : make_int2(0, 0);
      int crow_cur = (MODE == MODE_UPDATE && w >= 0) ? args.crow[w / args.sub_per] : 0;
      prefetch_c(w >= 0 ? w : items, ij_cur, crow_cur);
      for (int64_t n = 0; w >= 0; ++n) {
        int64_t w_next;
        if (dyn && kAhead && rank == 0) {
          w_next = w_ahead;
          w_ahead = w_next >= 0 ? claim_item(n + 2) : -1;
        } else {
          w_next = dyn ? claim_item(n + 1) : static_item(n + 1);
        }
        const int sub = static_cast<int>(w % args.sub_per);
        const int i = ij_cur.x, j = ij_cur.y;
        const int m0 = (sub / args.sub_n) * (TC_BM * CG) + static_cast<int>(rank) * TC_BM;
        const int n0 = (sub % args.sub_n) * BN;
        int2 ij_nxt = ij_cur;
        int crow_nxt = crow_cur;
        const bool more = w_next >= 0;
        if (more) {
          ij_nxt = args.list[w_next / args.sub_per];
          if (MODE == MODE_UPDATE) crow_nxt = args.crow[w_next / args.sub_per];
        }
        // Merged update (k2 >= 0): K runs over panel k's b columns, then
        // panel k2's — C -= [P_k P_k2] [Q_k Q_k2]^T in one accumulator, one
        // C round trip for two steps.
        for (int kb2 = 0; kb2 < kblocks * halves; ++kb2) {
          const int hf = kb2 >= kblocks ? 1 : 0, kb = kb2 - hf * kblocks;
          const int kk = hf ? args.k2 : args.k;
          const CUtensorMap* ma_hi = hf ? &mA2_hi : &mA_hi;
          const CUtensorMap* ma_lo = hf ? &mA2_lo : &mA_lo;
          const CUtensorMap* mb_hi = hf ? &mB2_hi : &mB_hi;
          const CUtensorMap* mb_lo = hf ? &mB2_lo : &mB_lo;
          const int a_row = (i - kk - 1) * args.b + m0;
          const int b_row = (MODE == MODE_UPDATE) ? (j - kk - 1) * args.b + n0 + static_cast<int>(rank) * (BN / CG)
                                                  : n0;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * Lay::kStage;
          const int kx = kb * T::kBK;
          // The panel operands are re-read by every work item of the step
          // while the C tiles stream through once: keep them in L2.
          if constexpr (CG == 2) {
            // both CTAs' bytes complete on the leader's full barrier
            const uint32_t fb = mapa_shared(&full[stage], 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], CG * Lay::kStage);
            tma_load_2d_cg2_hint(ma_hi, fb, st, kx, a_row, keep);
            tma_load_2d_cg2_hint(mb_hi, fb, st + Lay::kA, kx, b_row, keep);
            if (T::kSplit) {
              tma_load_2d_cg2_hint(ma_lo, fb, st + Lay::kA + Lay::kB, kx, a_row, keep);
              tma_load_2d_cg2_hint(mb_lo, fb, st + 2 * Lay::kA + Lay::kB, kx, b_row, keep);
            }
          } else {
            mbar_arrive_expect_tx(&full[stage], Lay::kStage);
            tma_load_2d_hint(ma_hi, &full[stage], st, kx, a_row, keep);
            tma_load_2d_hint(mb_hi, &full[stage], st + Lay::kA, kx, b_row, keep);
            if (T::kSplit) {
              tma_load_2d_hint(ma_lo, &full[stage], st + Lay::kA + Lay::kB, kx, a_row, keep);
              tma_load_2d_hint(mb_lo, &full[stage], st + 2 * Lay::kA + Lay::kB, kx, b_row, keep);
            }
            if (T::kBsplit) tma_load_2d_hint(mb_lo, &full[stage], st + Lay::kA + Lay::kB, kx, b_row, keep);
          }
          if (kb2 == 1 && more) prefetch_c(w_next, ij_nxt, crow_nxt);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        ij_cur = ij_nxt;
        crow_cur = crow_nxt;
        w = w_next;
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ===== MMA issuer (single thread; the pair leader for CG = 2) =====
    constexpr uint32_t idesc = umma_idesc(T::kFmt, TC_BM * CG, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t n = 0;; ++n) {
      int64_t w;
      if (dyn) {
        w = ring_take(n);
        __syncwarp();
        if (lane == 0) ring_release(n);
      } else {
        w = static_item(n);
      }
      if (w < 0) break;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * BN;
      for (int kb = 0; kb < kblocks * halves; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0 && SPH_DBG(args) == 2) {
          if constexpr (CG == 2) umma_commit_cg2(&empty[stage]);
          else umma_commit(&empty[stage]);
        } else if (lane == 0) {
          uint8_t* st = smem + stage * Lay::kStage;
          const uint64_t a_hi = umma_desc_k<T::kRowBytes>(st);
          const uint64_t b_hi = umma_desc_k<T::kRowBytes>(st + Lay::kA);
#pragma unroll
          for (int kk = 0; kk < T::kBK / T::kUK; ++kk) {
            const uint64_t koff = (kk * T::kUK * T::kElem) >> 4;
            const uint32_t accum = (kb | kk) ? 1u : 0u;
            if constexpr (T::kTf32) {
              const uint64_t a_lo = umma_desc_k<T::kRowBytes>(st + Lay::kA + Lay::kB);
              const uint64_t b_lo = umma_desc_k<T::kRowBytes>(st + 2 * Lay::kA + Lay::kB);
              umma_tf32(d, a_lo + koff, b_hi + koff, idesc, accum);
              umma_tf32(d, a_hi + koff, b_lo + koff, idesc, 1u);
              umma_tf32(d, a_hi + koff, b_hi + koff, idesc, 1u);
            } else if constexpr (T::kSplit && CG == 2) {
              const uint64_t a_lo = umma_desc_k<T::kRowBytes>(st + Lay::kA + Lay::kB);
              const uint64_t b_lo = umma_desc_k<T::kRowBytes>(st + 2 * Lay::kA + Lay::kB);
              umma_f16_cg2(d, a_lo + koff, b_hi + koff, idesc, accum);
              umma_f16_cg2(d, a_hi + koff, b_lo + koff, idesc, 1u);
              umma_f16_cg2(d, a_hi + koff, b_hi + koff, idesc, 1u);
            } else if constexpr (T::kSplit) {
              const uint64_t a_lo = umma_desc_k<T::kRowBytes>(st + Lay::kA + Lay::kB);
              const uint64_t b_lo = umma_desc_k<T::kRowBytes>(st + 2 * Lay::kA + Lay::kB);
              umma_f16(d, a_lo + koff, b_hi + koff, idesc, accum);
              umma_f16(d, a_hi + koff, b_lo + koff, idesc, 1u);
              umma_f16(d, a_hi + koff, b_hi + koff, idesc, 1u);
            } else if constexpr (T::kBsplit) {
              const uint64_t b_lo = umma_desc_k<T::kRowBytes>(st + Lay::kA + Lay::kB);
              umma_f16(d, a_hi + koff, b_lo + koff, idesc, accum);
              umma_f16(d, a_hi + koff, b_hi + koff, idesc, 1u);
            } else if constexpr (CG == 2) {
              umma_f16_cg2(d, a_hi + koff, b_hi + koff, idesc, accum);
            } else {
              umma_f16(d, a_hi + koff, b_hi + koff, idesc, accum);
            }
          }
          if constexpr (CG == 2) umma_commit_cg2(&empty[stage]);
          else umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) {
        if constexpr (CG == 2) umma_commit_cg2(&tfull[acc]);
        else umma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++acc == Lay::kAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM -> registers -> tile storage (+ panel mirrors) =====
    const int q = warp & 3;         // TMEM lane quarter (hardware: warp % 4)
    constexpr int NG = Lay::kEpi / 4;  // warps per quarter, splitting the columns
    const int grp = (warp - 4) >> 2;
    const int row_in = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned sat_local = 0;
    const int b = args.b;
    // Update-mode C staging (see below): box geometry and the load ring.
    constexpr int kEsz = T::kSplit ? 4 : 2;        // storage bytes of the C class (SP fp32, HP 16-bit)
    constexpr int kBoxCols = 128 / kEsz;           // columns per 128-byte box row
    constexpr int kNBox = BN / kBoxCols / NG;      // boxes per warp per work item (box grp + NG bx)
    static_assert(MODE != MODE_UPDATE || kNBox * NG * kBoxCols == BN, "boxes split evenly over the warps");
    constexpr int R = Lay::kRing > 0 ? Lay::kRing : 1;
    uint8_t* cring = cbuf + (warp - 4) * R * Lay::kCBox;
    uint64_t* cf = cfull + (warp - 4) * R;
    int64_t gbox = 0, gissue = 0;  // next box to process / to load (sequence over this CTA's items)
    auto c_row = [&](int64_t wi) { return args.crow[wi / args.sub_per]; };  // tile's first arena row
    int* wc = wcache + (warp - 4) * 4;
    int64_t rn = 0;  // items read from the schedule ring so far (lane 0)
    auto item_lane0 = [&](int64_t idx) -> int64_t {  // lane 0 only
      if (dyn) {
        for (; rn <= idx; ++rn) {
          wc[rn & 3] = static_cast<int>(ring_take(rn));
          ring_release(rn);
        }
        return wc[idx & 3];
      }
      return static_item(idx);
    };
    auto issue_c = [&]() {  // lane 0: TMA-load the next C box into its ring slot
      const int64_t wi = item_lane0(gissue / kNBox);
      if (wi < 0) return;
      const int bx = grp + NG * static_cast<int>(gissue % kNBox);
      int ti, tj, tm, tn;
      decode(wi, ti, tj, tm, tn);
      const int slot = static_cast<int>(gissue % R);
      mbar_arrive_expect_tx(&cf[slot], Lay::kCBox);
      tma_load_2d(&mC, &cf[slot], cring + slot * Lay::kCBox, tn + bx * kBoxCols, c_row(wi) + tm + q * 32);
      ++gissue;
    };
#if SPH_TC_REGC
    // Register-staged C (default): each box is read from L2 by coalesced
    // 16-byte loads (4 rows x 128 B per instruction) one box ahead, so the
    // loads of the next box fly while this one is computed and across the
    // accumulator wait; the warp's 4 KB smem slot only transposes the box
    // between the coalesced order and the TMEM row-per-lane order, and the
    // result leaves by coalesced stores that nobody waits for.
    uint4 cpre[8];
    char* cpre_ptr = nullptr;  // this lane's first 16 B of the prefetched box (nullptr = none)
    const int64_t c_pitch = static_cast<int64_t>(args.ts.b) * (T::kSplit ? 4 : 2);
    auto load_box = [&](int64_t seq) {
      int64_t wi = -1;
      if (lane == 0) wi = item_lane0(seq / kNBox);
      wi = __shfl_sync(0xffffffffu, static_cast<int>(wi), 0);
      if (wi < 0) {
        cpre_ptr = nullptr;
        return;
      }
      const int bx = grp + NG * static_cast<int>(seq % kNBox);
      int ti, tj, tm, tn;
      decode(wi, ti, tj, tm, tn);
      const int64_t row0 = static_cast<int64_t>(c_row(wi)) + tm + q * 32 + (lane >> 3);
      cpre_ptr = args.ts.base + row0 * c_pitch + static_cast<int64_t>(tn + bx * kBoxCols) * (T::kSplit ? 4 : 2) +
                 (lane & 7) * 16;
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8)
        cpre[s8] = SPH_DBG(args) == 5 ? make_uint4(0, 0, 0, 0)
                                 : ((args.opt & 8) ? __ldcg(reinterpret_cast<const uint4*>(cpre_ptr + s8 * 4 * c_pitch))
                                                   : __ldcs(reinterpret_cast<const uint4*>(cpre_ptr + s8 * 4 * c_pitch)));
    };
    if (MODE == MODE_UPDATE) load_box(0);
#else
    if (MODE == MODE_UPDATE && lane == 0 && (SPH_DBG(args) == 0 || SPH_DBG(args) >= 3) && SPH_DBG(args) != 5)
      for (int s = 0; s < R; ++s) issue_c();
#endif
    for (int64_t n = 0;; ++n) {
      if (lane == 0) item_lane0(n);
      __syncwarp();
      const int64_t w = dyn ? static_cast<int64_t>(*(volatile int*)&wc[n & 3]) : static_item(n);
      __syncwarp();  // every lane has read the cache before lane 0 may overwrite it
      if (w < 0) break;
      int i, j, m0, n0;
      decode(w, i, j, m0, n0);
      void* tp = args.ts.tile(i, j);
      const int p = args.ts.tprec(i, j);
      if constexpr (MODE == MODE_UPDATE) {
        // C = round_p(C - acc). The C sub-tile streams through shared
        // memory by TMA: each epilogue warp owns a ring of kRing boxes of
        // 32 rows x 128 bytes (its TMEM lane quarter); loads run kRing - 1
        // boxes ahead (across work items), results go back in place and
        // leave by TMA store. Thread t handles row t of the box, reading
        // the 128B-swizzled row conflict-free. Element arithmetic: one
        // correctly rounded fp32 subtraction (== the FP64 subtract + round
        // of mpchol.cpp:311-312 up to the rare double-rounding tie), then
        // the storage rounding.
        // HP tiles of an F16 launch are fp16, of a BF16 launch bf16 (one class per launch).
        constexpr bool kBf = (OPK == OP_BF16);
        constexpr float kThr = kBf ? 3.3961514e38f : 65520.0f;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int bl = 0; bl < ((SPH_DBG(args) == 1 || SPH_DBG(args) == 2) ? 0 : kNBox); ++bl, ++gbox) {
          const int bx = grp + NG * bl;
#if SPH_TC_REGC
          (void)bx;
          const int slot = 0;
          char* const cur_ptr = cpre_ptr;
          // the first 32 accumulator columns come from TMEM while the box is transposed
          uint32_t v_first[32];
          tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + bx * kBoxCols, v_first);
          {
            const uint32_t sb = smem_addr(cring);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
              const int r = 4 * s8 + (lane >> 3);
              sts128(sb + r * 128 + (((lane & 7) ^ (r & 7)) << 4), cpre[s8]);
            }
          }
          __syncwarp();
          load_box(gbox + 1);
#else
          const int slot = static_cast<int>(gbox % R);
          if (SPH_DBG(args) != 5) mbar_wait(&cf[slot], static_cast<uint32_t>((gbox / R) & 1));
#endif
          const uint32_t row_s = smem_addr(cring + slot * Lay::kCBox) + lane * 128;
#pragma unroll
          for (int h = 0; h < (SPH_DBG(args) == 3 ? 0 : kBoxCols / 32); ++h) {
            uint32_t v[32];
#if SPH_TC_REGC
            if (h == 0) {
              tmem_wait_ld();
#pragma unroll
              for (int t = 0; t < 32; ++t) v[t] = v_first[t];
            } else
#endif
              tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + bx * kBoxCols + h * 32, v);
            if constexpr (OPK == OP_F16X3) {
              // operands were scaled by 2^e_row: undo exactly (powers of two)
              const int er = args.rowexp[min(i * args.lb + m0 + row_in, args.ts.n - 1)];
              const int cbase = j * args.lb + n0 + bx * kBoxCols + h * 32;
              const float rs = __int_as_float((127 - er) << 23);
              int ecs[32];
              if ((cbase & 3) == 0 && cbase + 31 < args.ts.n) {  // 8 vector loads instead of 32 scalar ones
#pragma unroll
                for (int t4 = 0; t4 < 8; ++t4) {
                  const int4 e4 = __ldg(reinterpret_cast<const int4*>(args.rowexp + cbase) + t4);
                  ecs[4 * t4] = e4.x;
                  ecs[4 * t4 + 1] = e4.y;
                  ecs[4 * t4 + 2] = e4.z;
                  ecs[4 * t4 + 3] = e4.w;
                }
              } else {
#pragma unroll
                for (int t = 0; t < 32; ++t) ecs[t] = __ldg(args.rowexp + min(cbase + t, args.ts.n - 1));
              }
#pragma unroll
              for (int t = 0; t < 32; ++t)
                v[t] = __float_as_uint(__uint_as_float(v[t]) * (rs * __int_as_float((127 - ecs[t]) << 23)));
            }
            if constexpr (kEsz == 4) {
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) {
                const uint32_t ptr = row_s + ((cc ^ (lane & 7)) << 4);
                uint4 cv = lds128(ptr);
                cv.x = __float_as_uint(__fsub_rn(__uint_as_float(cv.x), __uint_as_float(v[4 * cc + 0])));
                cv.y = __float_as_uint(__fsub_rn(__uint_as_float(cv.y), __uint_as_float(v[4 * cc + 1])));
                cv.z = __float_as_uint(__fsub_rn(__uint_as_float(cv.z), __uint_as_float(v[4 * cc + 2])));
                cv.w = __float_as_uint(__fsub_rn(__uint_as_float(cv.w), __uint_as_float(v[4 * cc + 3])));
                sts128(ptr, cv);
              }
            } else {
              // HP class: packed pairs, cvt.rn.satfinite clamps to +-max
              // finite exactly like half.hpp's saturation; values whose RNE
              // result would overflow are counted (|x| >= 65520 for fp16,
              // >= bf16's rounding threshold for bf16).
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) {
                const uint32_t ptr = row_s + (((h * 4 + cc) ^ (lane & 7)) << 4);
                uint4 raw = lds128(ptr);
                uint32_t* w2 = reinterpret_cast<uint32_t*>(&raw);
                float x[8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if constexpr (!kBf) {
                    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w2[u]));
                    x[2 * u] = f.x;
                    x[2 * u + 1] = f.y;
                  } else {
                    x[2 * u] = __uint_as_float(w2[u] << 16);
                    x[2 * u + 1] = __uint_as_float(w2[u] & 0xffff0000u);
                  }
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) x[e] = __fsub_rn(x[e], __uint_as_float(v[8 * cc + e]));
                // saturation count: one max-tree per 8 values, exact count only when one overflows
                const float m01 = fmaxf(fabsf(x[0]), fabsf(x[1])), m23 = fmaxf(fabsf(x[2]), fabsf(x[3]));
                const float m45 = fmaxf(fabsf(x[4]), fabsf(x[5])), m67 = fmaxf(fabsf(x[6]), fabsf(x[7]));
                if (fmaxf(fmaxf(m01, m23), fmaxf(m45, m67)) >= kThr) {
#pragma unroll
                  for (int e = 0; e < 8; ++e) sat_local += fabsf(x[e]) >= kThr;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  uint32_t packed;
                  if constexpr (!kBf)
                    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(packed) : "f"(x[2 * u + 1]), "f"(x[2 * u]));
                  else
                    asm("cvt.rn.satfinite.bf16x2.f32 %0, %1, %2;" : "=r"(packed) : "f"(x[2 * u + 1]), "f"(x[2 * u]));
                  w2[u] = packed;
                }
                sts128(ptr, raw);
              }
            }
          }
#if SPH_TC_REGC
          __syncwarp();
          {
            const uint32_t sb = smem_addr(cring);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) {
              const int r = 4 * s8 + (lane >> 3);
              const uint4 v = lds128(sb + r * 128 + (((lane & 7) ^ (r & 7)) << 4));
              if (SPH_DBG(args) != 4) {  // the C tile is not read again this step: stream it out
                if (args.opt & 8) __stcg(reinterpret_cast<uint4*>(cur_ptr + s8 * 4 * c_pitch), v);
                else __stcs(reinterpret_cast<uint4*>(cur_ptr + s8 * 4 * c_pitch), v);
              }
            }
          }
          __syncwarp();  // the slot is free for the next box
          continue;
#endif
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            int bi, bj, bm, bn;
            decode(w, bi, bj, bm, bn);
            if (SPH_DBG(args) != 3 && SPH_DBG(args) != 4)
              tma_store_2d(&mC, cring + slot * Lay::kCBox, bn + bx * kBoxCols, c_row(w) + bm + q * 32);
            bulk_commit();
            if (R == 1) {
              bulk_wait_read0();  // the single slot is free again
              issue_c();
            } else if (gbox >= 1) {
              bulk_wait_read1();  // box gbox-1 has left its slot: refill it
              issue_c();
            }
          }
          __syncwarp();
        }
      } else {
      const int r = m0 + row_in;
      const int64_t prow = (int64_t)(i - args.k - 1) * b + r;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      for (int c0 = 32 * grp; c0 < BN; c0 += 32 * NG) {
        uint32_t v[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c0, v);
        const int64_t e0 = (int64_t)r * b + n0 + c0;
        if constexpr (OPK == OP_F16X3) {
          // X = acc * 2^(-rowexp(row) - g(col)): exact power-of-two unscale of the scaled operands
          const int er = args.rowexp[min(i * args.lb + r, args.ts.n - 1)];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int g = __ldg(args.lexp + n0 + c0 + t);
            v[t] = __float_as_uint(__uint_as_float(v[t]) * __int_as_float((127 - er - g) << 23));
          }
        }
        {
          // Panel: X = B * Linv^T rounded through p(i, k); write the tile, the
          // FP64 mirror and the tensor mirrors, 8 columns (>= 32 B) per store.
#pragma unroll
          for (int t = 0; t < 32; t += 8) {
            const int64_t e = e0 + t;
            const int64_t pe = prow * b + n0 + c0 + t;
            double qv[8];
            uint16_t h16[8];
            float fq[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const double x = (double)__uint_as_float(v[t + u]);
              if (p == kSP) {
                fq[u] = __double2float_rn(x);
                qv[u] = (double)fq[u];
                unsigned dummy = 0;
                h16[u] = args.hp_format == SPHEMU_HP_BF16 ? __bfloat16_as_ushort(to_bf16_sat(qv[u], dummy))
                                                         : __half_as_ushort(to_half_sat(qv[u], dummy));
              } else if (p == kHP) {
                const __half hv = to_half_sat(x, sat_local);
                h16[u] = __half_as_ushort(hv);
                qv[u] = (double)__half2float(hv);
              } else {
                const __nv_bfloat16 hv = to_bf16_sat(x, sat_local);
                h16[u] = __bfloat16_as_ushort(hv);
                qv[u] = (double)__bfloat162float(hv);
              }
            }
            if (p == kSP) {
              float4* tf = reinterpret_cast<float4*>(static_cast<float*>(tp) + e);
              tf[0] = make_float4(fq[0], fq[1], fq[2], fq[3]);
              tf[1] = make_float4(fq[4], fq[5], fq[6], fq[7]);
            } else {
              *reinterpret_cast<uint4*>(static_cast<uint16_t*>(tp) + e) = *reinterpret_cast<const uint4*>(h16);
            }
            if (args.p64) {
              double2* pd = reinterpret_cast<double2*>(args.p64 + pe);
#pragma unroll
              for (int u = 0; u < 4; ++u) pd[u] = make_double2(qv[2 * u], qv[2 * u + 1]);
            }
            if (args.s8)  // the INT8 DP class's digits of this row, instead of the FP64 mirror
              oz_store8(args.s8 + prow * (OZ_DIGITS * static_cast<int64_t>(b)), n0 + c0 + t, qv,
                        oz_mu_of(args.rowexp[min(i * args.lb + r, args.ts.n - 1)]));
            if (args.p_hi) {
              float hi[8], lo[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) tf32_split((float)qv[u], hi[u], lo[u]);
              float4* ph = reinterpret_cast<float4*>(args.p_hi + pe);
              float4* pl = reinterpret_cast<float4*>(args.p_lo + pe);
              ph[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
              ph[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
              pl[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
              pl[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
            }
            if (args.p16) *reinterpret_cast<uint4*>(args.p16 + pe) = *reinterpret_cast<const uint4*>(h16);
            if (args.h_hi) {
              const int er = args.rowexp[min(i * args.lb + r, args.ts.n - 1)];
              uint16_t hh[8], hl[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) f16_split(qv[u], er, hh[u], hl[u]);
              *reinterpret_cast<uint4*>(args.h_hi + pe) = *reinterpret_cast<const uint4*>(hh);
              *reinterpret_cast<uint4*>(args.h_lo + pe) = *reinterpret_cast<const uint4*>(hl);
            }
          }
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // this warp is done with the accumulator (the leader's barrier for a pair)
        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(&tempty[acc], 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == Lay::kAcc) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (MODE == MODE_UPDATE && lane == 0) bulk_wait_all();
    sat_local = warp_sum_u32(sat_local);
    if (lane == 0 && sat_local) atomicAdd(args.sat, sat_local);
  }
  __syncthreads();
  if constexpr (CG == 2) {
    cluster_sync_all();  // both CTAs are done with the pair's TMEM
    if (warp == 2) tmem_dealloc_cg2(tmem_base, Lay::kTmemCols);
  } else {
    if (warp == 2) tmem_dealloc(tmem_base, Lay::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Panel producers
// ---------------------------------------------------------------------------
// tf32 splits of the panel TRSM inputs B_i (SP/HP-class panel tiles) and of
// Linv (blockIdx.y == 0 handles Linv, y >= 1 the list entries).
__global__ void k_panel_prep(TileStore ts, int k, const int2* list, const double* __restrict__ linv,
                             float* in_hi, float* in_lo, float* l_hi, float* l_lo, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int64_t bb = (int64_t)b * b;
  if (blockIdx.y == 0) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
      float hi, lo;
      tf32_split(__double2float_rn(linv[e]), hi, lo);
      l_hi[e] = hi;
      l_lo[e] = lo;
    }
    return;
  }
  const int i = list[blockIdx.y - 1].x;
  const void* tp = ts.tile(i, k);
  const int p = ts.tprec(i, k);
  const int64_t base = (int64_t)(i - k - 1) * bb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
    float hi, lo;
    tf32_split((float)load_elem(tp, p, e), hi, lo);
    in_hi[base + e] = hi;
    in_lo[base + e] = lo;
  }
}

// BF16-class panel TRSM inputs (OP_BF16X2): blockIdx.y == 0 splits Linv
// into bf16 hi + lo (the B operand, ~16 bits), y >= 1 copies each listed
// tile's bf16 bits into its panel rows (the A operand; the TRSM writes the
// tile in place, so it cannot read it there). X = B (Linv_hi + Linv_lo)^T
// carries ~2^-16 relative error before the epilogue rounds it to bf16.
__global__ void k_panel_prep_bf16x2(TileStore ts, int k, const int2* list, const double* __restrict__ linv,
                                    uint16_t* in16, uint16_t* l_hi, uint16_t* l_lo, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int64_t bb = (int64_t)b * b;
  if (blockIdx.y == 0) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
      const double x = linv[e];
      const __nv_bfloat16 hi = __double2bfloat16(x);
      const __nv_bfloat16 lo = __double2bfloat16(x - (double)__bfloat162float(hi));
      l_hi[e] = __bfloat16_as_ushort(hi);
      l_lo[e] = __bfloat16_as_ushort(lo);
    }
    return;
  }
  const int i = list[blockIdx.y - 1].x;
  const uint4* src = static_cast<const uint4*>(ts.tile(i, k));
  uint4* dst = reinterpret_cast<uint4*>(in16 + (int64_t)(i - k - 1) * bb);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb / 8; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

// FP16x3 panel TRSM inputs. With 2^(14 - rowexp[x]) ~ sqrt(A_xx) (k_rowexp):
//   B_s[r][c]   = B[r][c] 2^(rowexp[R] + rowexp[C] - 14)      |B_s| <~ 2^14
//   L_s[j][c]   = Linv[j][c] 2^(14 - rowexp[C] + g_j)        g_j: row max -> <= 2^14
// so (B_s L_s^T)[r][j] = X[r][j] 2^(rowexp[R] + g_j), undone exactly in the
// panel epilogue; hi + lo fp16 carry ~22 bits like a tf32 split.
__global__ void k_linv_prep16(const double* __restrict__ linv, int b, int k, int lb, int n, const int* rowexp,
                              uint16_t* l_hi, uint16_t* l_lo, int* lexp, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  __shared__ float red[32];
  const int j = blockIdx.x;
  float m = 0.f;
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    const int C = min(k * lb + c, n - 1);
    m = fmaxf(m, fabsf(ldexpf(__double2float_rn(linv[(int64_t)j * b + c]), 14 - rowexp[C])));
  }
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  m = red[0];
  int e = 0;
  if (m > 0.f) frexpf(m, &e);  // m = f 2^e, f in [0.5, 1)
  const int g = m > 0.f ? 14 - e : 0;
  if (threadIdx.x == 0) lexp[j] = g;
  for (int c = threadIdx.x; c < b; c += blockDim.x) {
    const int C = min(k * lb + c, n - 1);
    uint16_t hi, lo;
    f16_split(linv[(int64_t)j * b + c], 14 - rowexp[C] + g, hi, lo);
    l_hi[(int64_t)j * b + c] = hi;
    l_lo[(int64_t)j * b + c] = lo;
  }
}

__global__ void k_panel_prep16(TileStore ts, int k, const int2* list, const int* rowexp, uint16_t* in_hi,
                               uint16_t* in_lo, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int64_t bb = (int64_t)b * b;
  const int i = list[blockIdx.y].x;
  const void* tp = ts.tile(i, k);
  const int p = ts.tprec(i, k);
  const int64_t base = (int64_t)(i - k - 1) * bb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    const int R = min(i * ts.lb + r, ts.n - 1), Cc = min(k * ts.lb + c, ts.n - 1);
    uint16_t hi, lo;
    f16_split(load_elem(tp, p, e), rowexp[R] + rowexp[Cc] - 14, hi, lo);
    in_hi[base + e] = hi;
    in_lo[base + e] = lo;
  }
}

// DP-class panel tiles: P64 (already rounded) -> tile storage + mirrors.
__global__ void k_panel_finish_dp(TileStore ts, int k, const int2* list, const double* __restrict__ p64,
                                  float* p_hi, float* p_lo, uint16_t* p16, int hp_format, const int* fail,
                                  uint16_t* h_hi, uint16_t* h_lo, const int* rowexp, uint8_t* s8) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int64_t bb = (int64_t)b * b;
  const int i = list[blockIdx.y].x;
  void* tp = ts.tile(i, k);
  const int p = ts.tprec(i, k);
  const int64_t base = (int64_t)(i - k - 1) * bb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
    const double x = p64[base + e];  // already rounded through p(i, k): the store is exact
    unsigned none = 0;
    store_elem(tp, p, e, x, none);
    if (p_hi) {
      float hi, lo;
      tf32_split(__double2float_rn(x), hi, lo);
      p_hi[base + e] = hi;
      p_lo[base + e] = lo;
    }
    if (p16) {
      unsigned dummy = 0;
      p16[base + e] = hp_format == SPHEMU_HP_BF16 ? __bfloat16_as_ushort(to_bf16_sat(x, dummy))
                                                  : __half_as_ushort(to_half_sat(x, dummy));
    }
    if (h_hi) {
      const int r = (int)(e / b);
      f16_split(x, rowexp[min(i * ts.lb + r, ts.n - 1)], h_hi[base + e], h_lo[base + e]);
    }
  }
  if (s8) {  // INT8 DP digits of these rows: 8 consecutive elements per thread
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < bb / 8; g += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = g * 8;
      const int r = (int)(e / b), c = (int)(e % b);
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = p64[base + e + u];
      oz_store8(s8 + ((int64_t)(i - k - 1) * b + r) * (OZ_DIGITS * (int64_t)b), c, x,
                oz_mu_of(rowexp[min(i * ts.lb + r, ts.n - 1)]));
    }
  }
}

// DP-class panel tiles through FP64 DMMA (list variant of k_panel_trsm_fp64).
__global__ void __launch_bounds__(DG_THREADS) k_panel_trsm_fp64_list(TileStore ts, int k, const int2* list,
                                                                      const double* __restrict__ Linv,
                                                                      double* __restrict__ P64,
                                                                      const int* fail, unsigned* sat) {
  __shared__ DgSmem sm;
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int sub_per = b / DG_BM;
  const int i = list[blockIdx.x / sub_per].x;
  const int r0 = (blockIdx.x % sub_per) * DG_BM, c0 = blockIdx.y * DG_BN;
  TileRowAcc A{ts.tile(i, k), ts.tprec(i, k), b, r0, b, b};
  RowMajorK B{Linv + (int64_t)c0 * b, b, DG_BN, b};
  double acc[4][4][2];
  dgemm_64x64(A, B, b, sm, acc);
  double* out = P64 + (int64_t)(i - k - 1) * b * b;
  unsigned local = 0;
  const int p = ts.tprec(i, k);
  dg_for_each(acc, [&](int r, int c, double v) { out[(int64_t)(r0 + r) * b + c0 + c] = quantize_value(v, p, local); });
  flush_sat(local, sat);
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
namespace {

// The second panel's operand maps of a merged two-step update (unused otherwise).
struct Maps2 {
  const CUtensorMap *a_hi = nullptr, *a_lo = nullptr, *b_hi = nullptr, *b_lo = nullptr;
};

template <int BN, int OPK, int MODE, int CG = 1>
void launch_tc(const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& b_hi,
               const CUtensorMap& b_lo, const CUtensorMap& c_map, TcArgs args, cudaStream_t s, int max_ctas = 0,
               bool resume = false, Maps2 m2 = {}) {
  const CUtensorMap& a2_hi = m2.a_hi ? *m2.a_hi : a_hi;
  const CUtensorMap& a2_lo = m2.a_lo ? *m2.a_lo : a_lo;
  const CUtensorMap& b2_hi = m2.b_hi ? *m2.b_hi : b_hi;
  const CUtensorMap& b2_lo = m2.b_lo ? *m2.b_lo : b_lo;
  using Lay = TcLayout<BN, OPK, MODE, CG>;
  auto kern = k_tc_gemm<BN, OPK, MODE, CG>;
  smem_optin(reinterpret_cast<const void*>(kern), Lay::kSmem);
  if (args.counter && !resume) SPH_CUDA(cudaMemsetAsync(args.counter, 0, sizeof(int), s));
  const int cap = (max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms()) / CG;
  const int grid = CG * static_cast<int>(std::min<int64_t>(args.items, std::max(1, cap)));
  if constexpr (CG == 1) {
    kern<<<grid, Lay::kThreads, Lay::kSmem, s>>>(a_hi, a_lo, b_hi, b_lo, c_map, a2_hi, a2_lo, b2_hi, b2_lo, args);
  } else {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(Lay::kThreads);
    lc.dynamicSmemBytes = Lay::kSmem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    SPH_CUDA(cudaLaunchKernelEx(&lc, kern, a_hi, a_lo, b_hi, b_lo, c_map, a2_hi, a2_lo, b2_hi, b2_lo, args));
  }
  SPH_LAUNCH_CHECK();
}



}  // namespace

void tc_panel_trsm(const TileStore& ts, int k, const int2* d_dp, int64_t n_dp, const int2* d_lo,
                   int64_t n_lo, const double* linv, double* p64, PanelFormats& pf, const int* fail,
                   unsigned* sat, cudaStream_t s, int max_ctas, int* counter, const int2* d_bf, int64_t n_bf) {
  const int b = ts.b;
  if (n_dp) {
    k_panel_trsm_fp64_list<<<dim3(static_cast<unsigned>(n_dp * (b / DG_BM)), b / DG_BN), DG_THREADS, 0, s>>>(
        ts, k, d_dp, linv, p64, fail, sat);
    SPH_LAUNCH_CHECK();
    k_panel_finish_dp<<<dim3(std::max(1, b * b / (256 * 16)), static_cast<unsigned>(n_dp)), 256, 0, s>>>(
        ts, k, d_dp, p64, pf.tf32_hi(), pf.tf32_lo(), pf.half16(), pf.hp_format, fail,
        pf.f16x3 ? pf.h_hi.get() : nullptr, pf.h_lo.get(), pf.rowexp, pf.s8);
    SPH_LAUNCH_CHECK();
  }
  static const bool panel16 = [] {
    // FP16x3 panel TRSM: same speed as 3xTF32 here (the panel is latency-
    // bound) with a slightly larger backward error, so opt-in only.
    const char* e = std::getenv("SPHEMU_PANEL_F16X3");
    return e && e[0] == '1';
  }();
  const bool p16 = panel16 && pf.f16x3;
  if (n_lo && p16) {
    k_linv_prep16<<<b, 128, 0, s>>>(linv, b, k, ts.lb, ts.n, pf.rowexp, pf.l16_hi.get(), pf.l16_lo.get(),
                                     pf.lexp.get(), fail);
    SPH_LAUNCH_CHECK();
    k_panel_prep16<<<dim3(std::max(1, b * b / (256 * 16)), static_cast<unsigned>(n_lo)), 256, 0, s>>>(
        ts, k, d_lo, pf.rowexp, pf.in16_hi.get(), pf.in16_lo.get(), fail);
    SPH_LAUNCH_CHECK();
  } else if (n_lo) {
    k_panel_prep<<<dim3(std::max(1, b * b / (256 * 16)), static_cast<unsigned>(n_lo + 1)), 256, 0, s>>>(
        ts, k, d_lo, linv, pf.in_hi.get(), pf.in_lo.get(), pf.l_hi.get(), pf.l_lo.get(), fail);
    SPH_LAUNCH_CHECK();
  }
  auto panel_args = [&](const int2* list, int64_t cnt) {
    TcArgs a{};
    a.k2 = -1;
    a.ts = ts;
    a.list = list;
    a.k = k;
    a.b = b;
    a.sub_n = b / 128;
    a.sub_per = (b / TC_BM) * a.sub_n;
    a.items = cnt * a.sub_per;
    a.p64 = (pf.s8 || pf.no_p64) ? nullptr : p64;  // nothing reads the SP/HP rows' FP64 mirror then
    a.s8 = pf.s8;
    a.p_hi = pf.tf32_hi();
    a.p_lo = pf.tf32_lo();
    a.p16 = pf.half16();
    a.h_hi = pf.f16x3 ? pf.h_hi.get() : nullptr;
    a.h_lo = pf.h_lo.get();
    a.rowexp = pf.rowexp;
    a.lb = ts.lb;
    a.hp_format = pf.hp_format;
    a.fail = fail;
    a.sat = sat;
    a.counter = counter;
    a.lexp = pf.lexp.get();
    return a;
  };
  if (n_lo) {
    const TcArgs a = panel_args(d_lo, n_lo);
    if (p16)
      launch_tc<128, OP_F16X3, MODE_PANEL>(pf.m_in16hi_a, pf.m_in16lo_a, pf.m_l16hi_b, pf.m_l16lo_b, pf.m_l16hi_b, a, s,
                                           max_ctas);
    else
      launch_tc<128, OP_TF32X3, MODE_PANEL>(pf.m_inhi_a, pf.m_inlo_a, pf.m_lhi_b, pf.m_llo_b, pf.m_lhi_b, a, s,
                                            max_ctas);
  }
  if (n_bf) {  // BF16-class panel tiles: one bf16 operand x Linv's bf16 hi/lo, 2 MMAs per K step
    k_panel_prep_bf16x2<<<dim3(std::max(1, b * b / (256 * 16)), static_cast<unsigned>(n_bf + 1)), 256, 0, s>>>(
        ts, k, d_bf, linv, pf.in16_hi.get(), pf.l16_hi.get(), pf.l16_lo.get(), fail);
    SPH_LAUNCH_CHECK();
    const TcArgs a = panel_args(d_bf, n_bf);
    launch_tc<128, OP_BF16X2, MODE_PANEL>(pf.m_in16hi_a, pf.m_in16hi_a, pf.m_l16hi_b, pf.m_l16lo_b, pf.m_l16hi_b, a, s,
                                          max_ctas);
  }
}

void tc_update(const TileStore& ts, int k, int cls, int hp_format, const int2* list, const int* rows, int64_t cnt,
               const double* p64, PanelFormats& pf, const int* fail, unsigned* sat, cudaStream_t s,
               int max_ctas, int* counter, const int* yield, bool resume, int k2, PanelFormats* pf2) {
  (void)p64;
  TcArgs a{};
  a.k2 = (k2 >= 0 && pf2) ? k2 : -1;
  a.ts = ts;
  a.list = list;
  a.crow = rows;
  a.k = k;
  a.b = ts.b;
  a.hp_format = hp_format;
  a.fail = fail;
  a.sat = sat;
  a.rowexp = pf.rowexp;
  a.lb = ts.lb;
  static const int dbg = SPH_DBG_ENV("SPHEMU_TC_DBG");
  a.dbg = dbg;
  a.counter = counter;
  static const int opt = [] {
    const char* e = std::getenv("SPHEMU_TC_OPT");
    return e ? std::atoi(e) : 0;
  }();
  a.opt = opt;
  // CTA pairs (cta_group::2, M = 256) for the 256-wide kinds: bitwise
  // identical results. Default for the HP class, where the pair's smaller
  // operand stages leave room for 16 epilogue warps (update 820 vs 767
  // TFLOP/s single-CTA at N = 98 304 dpsphp/bf16), and for the SP class
  // (fp16x3): each CTA stages half of the B rows, so the shared-memory
  // traffic per MMA (TMA writes + operand reads) drops from ~147 to ~98
  // B/clk (C2 dpsp 51.8 -> 49.3 ms, n = 64 800 dpsp 275 -> 234 ms, C3
  // 916 -> 891 ms; SPHEMU_TC_CG_SP=1 restores single CTAs).
  static const int cg_env = [] {
    const char* e = std::getenv("SPHEMU_TC_CG");
    return e ? std::atoi(e) : 2;
  }();
  static const int cg_sp = [] {
    const char* e = std::getenv("SPHEMU_TC_CG_SP");
    return e ? std::atoi(e) : 2;
  }();
  static const int sp_bn = [] {
    const char* e = std::getenv("SPHEMU_SP_BN");
    return e ? std::atoi(e) : 256;
  }();
  const bool pair = (cls == SPHEMU_PREC_SP ? cg_sp : cg_env) == 2 && pf.bn == 256;
  // Dynamic claims for CTA pairs (the leader claims one item ahead and hands
  // it to its peer through the peer's ring slot): they let the pair yield
  // its SMs to the chain's panel, which pays off on short factorizations
  // (C2, nt = 64: 47.8 vs 48.8 ms at the best reserve of each) but costs
  // throughput on long ones (n = 64 800: 237.7 vs 233.9 ms; C3: 910 vs 897
  // ms). pf.pair_dyn_sp (the handle's choice, nt < 96) selects it for the SP
  // class; SPHEMU_TC_PAIR_DYN = 0 none, 1 the SP class, 2 all overrides.
  static const int pair_dyn_env = [] {
    const char* e = std::getenv("SPHEMU_TC_PAIR_DYN");
    return e ? std::atoi(e) : -1;
  }();
  const int pair_dyn = pair_dyn_env >= 0 ? pair_dyn_env : (pf.pair_dyn_sp ? 1 : 0);
  const bool dyn = counter != nullptr && (!pair || pair_dyn >= 2 || (pair_dyn == 1 && cls == SPHEMU_PREC_SP));
  a.counter = dyn ? counter : nullptr;
  if (resume && !dyn) return;  // statically scheduled launches never yield
  a.yield = dyn ? yield : nullptr;
  if (cls == SPHEMU_PREC_SP) {
    const int bn_sp = (pf.f16x3 && pf.bn == 256 && sp_bn == 256 && !pair) ? 256 : (pair ? 256 : 128);
    a.sub_n = ts.b / (pf.f16x3 ? bn_sp : 128);
    a.sub_per = (ts.b / (TC_BM * (pair && pf.f16x3 ? 2 : 1))) * a.sub_n;
    a.items = cnt * a.sub_per;
    if (pf.f16x3 && pair)
      launch_tc<256, OP_F16X3, MODE_UPDATE, 2>(pf.m_hhi_a, pf.m_hlo_a, pf.m_hhi_a, pf.m_hlo_a, pf.m_c32, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_hhi_a : nullptr, a.k2 >= 0 ? &pf2->m_hlo_a : nullptr, a.k2 >= 0 ? &pf2->m_hhi_a : nullptr, a.k2 >= 0 ? &pf2->m_hlo_a : nullptr});
    else if (pf.f16x3 && bn_sp == 256)
      launch_tc<256, OP_F16X3, MODE_UPDATE>(pf.m_hhi_a, pf.m_hlo_a, pf.m_hhi_b, pf.m_hlo_b, pf.m_c32, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_hhi_a : nullptr, a.k2 >= 0 ? &pf2->m_hlo_a : nullptr, a.k2 >= 0 ? &pf2->m_hhi_b : nullptr, a.k2 >= 0 ? &pf2->m_hlo_b : nullptr});
    else if (pf.f16x3)  // 128-wide N: B boxes of 128 rows (the A-side maps)
      launch_tc<128, OP_F16X3, MODE_UPDATE>(pf.m_hhi_a, pf.m_hlo_a, pf.m_hhi_a, pf.m_hlo_a, pf.m_c32, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_hhi_a : nullptr, a.k2 >= 0 ? &pf2->m_hlo_a : nullptr, a.k2 >= 0 ? &pf2->m_hhi_a : nullptr, a.k2 >= 0 ? &pf2->m_hlo_a : nullptr});
    else
      launch_tc<128, OP_TF32X3, MODE_UPDATE>(pf.m_phi_a, pf.m_plo_a, pf.m_phi_b, pf.m_plo_b, pf.m_c32, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_phi_a : nullptr, a.k2 >= 0 ? &pf2->m_plo_a : nullptr, a.k2 >= 0 ? &pf2->m_phi_b : nullptr, a.k2 >= 0 ? &pf2->m_plo_b : nullptr});
  } else {
    static const int hp_bn = [] {
      const char* e = std::getenv("SPHEMU_HP_BN");
      return e ? std::atoi(e) : 256;
    }();
    const int bn_hp = (pf.bn == 256 && hp_bn == 256) || pair ? 256 : 128;
    a.sub_n = ts.b / bn_hp;
    a.sub_per = (ts.b / (TC_BM * (pair ? 2 : 1))) * a.sub_n;
    a.items = cnt * a.sub_per;
    if (pair) {
      if (hp_format == SPHEMU_HP_BF16)
        launch_tc<256, OP_BF16, MODE_UPDATE, 2>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr});
      else
        launch_tc<256, OP_F16, MODE_UPDATE, 2>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr});
    } else if (bn_hp == 256) {
      if (hp_format == SPHEMU_HP_BF16)
        launch_tc<256, OP_BF16, MODE_UPDATE>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_b, pf.m_p16_b, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_b : nullptr, a.k2 >= 0 ? &pf2->m_p16_b : nullptr});
      else
        launch_tc<256, OP_F16, MODE_UPDATE>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_b, pf.m_p16_b, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_b : nullptr, a.k2 >= 0 ? &pf2->m_p16_b : nullptr});
    } else {  // 128-wide N: B boxes of 128 rows (the A-side map)
      if (hp_format == SPHEMU_HP_BF16)
        launch_tc<128, OP_BF16, MODE_UPDATE>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr});
      else
        launch_tc<128, OP_F16, MODE_UPDATE>(pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_p16_a, pf.m_c16, a, s, max_ctas, resume,
                  Maps2{a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr, a.k2 >= 0 ? &pf2->m_p16_a : nullptr});
    }
  }
}

// rng.hpp:12-39 uniform stream (mt19937_64, 53-bit in (0,1]) and
// mpchol.cpp:423-429's d_i = exp(0.6u - 0.3), pw[k] = pow(0.9, k).
void host_spd_factors(int n, uint64_t seed, double* d, double* pw, double rho) {
  std::mt19937_64 eng(seed);
  for (int i = 0; i < n; ++i) {
    const double u = static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
    d[i] = std::exp(0.6 * u - 0.3);
  }
  for (int k = 0; k < n; ++k) pw[k] = std::pow(rho, k);
}

}  // namespace sphemu_gpu
