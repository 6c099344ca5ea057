// filter_step.cuh -- K1: one step of the Chebyshev filter (Alg 2 line 3 / line 8) as a
// single fused kernel: a complex (Hp^H . Y_i) GEMM on the FP64 tensor cores (DMMA.8x8x4) fed by
// TMA-staged, 128B-swizzled shared-memory tiles, with the three-term-recurrence axpby, the degree
// masking and the finished-column store in the epilogue (no separate elementwise pass).
//
// Complex arithmetic, MODE below:
//  3M (default): P1 = sum Re h Re y, P2 = sum Im h Im y, P3 = sum (Re h - Im h)(Re y + Im y) from the
//    interleaved tiles plus two TMA-staged real planes; Re = P1 + P2, Im = P3 - P1 + P2 for conj(h) y.
//  4M: Hp (n x nloc, complex, column-major) is read as a real K-major matrix A' (nloc rows, K' = 2n),
//    Y_i as real K-major columns B' = (re, im, re, im, ...). The imaginary output column uses
//    B''_j = (im, -re, im, -re, ...) built in registers from the same shared tile (swap + sign), so
//    C = A' [B' B''] has (Re, Im) of output (r, j) in one thread's accumulator pair.
// Schedule: persistent CTAs (data-parallel tiles, then stream-K over the remaining k-iterations),
// thread 0 of each CTA issues the TMA loads; optional thread-block clusters (CL = 2, multicast H tile),
// 2 CTAs per SM (OCC = 2) and half stages (KH = 1) exist as measured alternatives.
#pragma once
#include "common.cuh"

namespace chfsi {

// stream-K tickets in the workspace (one int per tail tile and cluster rank)
constexpr int64_t kMaxTailTickets = 1024;

struct StepParams {
  int64_t nrows;        // output rows (nloc)
  int32_t num_kt;       // k-tiles per output tile (32 real = 16 complex contraction entries each)
  int32_t kt_per_rank;  // k-tiles per rank chunk of the B operand (== num_kt when p == 1)
  int32_t a_rank_stride;  // real-K offset between rank chunks in A (2 * nloc_per_rank)
  int32_t a3_rank_stride;  // 3M: K offset between rank chunks in the Re H - Im H plane (nloc rounded up to even)
  int32_t col0;         // first active complex column s_i
  int32_t col_end;      // k (one past the last active column)
  int32_t fin_end;      // columns [col0, fin_end) finish at this step and go to `out`
  int32_t b_col0;       // B-operand column coordinate of complex column col0
  int32_t flags;        // 1: read y_cur (c != 0), 2: read y_prev (b != 0)
  // persistent schedule (host-computed, see schedule_filter_step): tiles are numbered n-fastest;
  // CTA c owns the data-parallel tiles c, c + grid, ..., c + (dp_units - 1) grid, then the
  // stream-K iterations [sk_bounds[c], sk_bounds[c+1]) of the tail tiles tail_tile0.. (each tile =
  // num_kt iterations); a split tile is finished by the last of its contributors to arrive (ticket),
  // which sums the partial accumulators in k order. The bounds balance WORK, not iterations: an
  // iteration of a tile with fewer active column units is cheaper, and a CTA whose data-parallel
  // tiles carry less work takes a larger share of the tail (work-weighted stream-K).
  int32_t tiles_n;      // N tiles
  int32_t units_n;      // WNC-wide column units of the active block, split evenly over the N tiles
  int32_t grid;         // CTAs
  int32_t dp_units;     // full tiles per CTA
  int32_t tail_tile0;   // first stream-K tile
  int64_t tail_iters;   // (tiles - tail_tile0) * num_kt
  static constexpr int kMaxGrid = 296;  // schedule ids (CTAs, or clusters) a launch may use
  int32_t sk_bounds[kMaxGrid + 1];      // tail iteration ranges per CTA, non-decreasing, [0] = 0, [grid] = tail_iters
  double* partials;     // 2 slots per CTA
  int* tickets;         // one per tail tile, zero between launches
  double a, b, c;       // Y_{i+1} = a (acc - c y_cur) - b y_prev
  const double2* y_cur;
  int64_t ld_cur;
  const double2* y_prev;
  int64_t ld_prev;
  double2* y_next;      // may alias y_prev (same element, same thread: read then write)
  int64_t ld_next;
  double2* out;         // finished columns (caller's Y)
  int64_t ld_out;
  // p > 1: this rank's chunk of the next step's packed B operand. n_rdst = 1: the chunk in this rank's
  // buffer (completed by an allgather); n_rdst = nranks (peer push): the chunk in every rank's buffer,
  // stored through NVLink peer pointers by this epilogue, so the exchange overlaps the MMAs tile by
  // tile and only a barrier remains between steps. n_rdst = 0: none.
  static constexpr int kMaxRdst = 8;
  double2* r_dst[kMaxRdst];
  int32_t n_rdst;
  int64_t ld_r_next;
  // 3M mode: every B-operand column carries, after its 2*ld complex doubles, the real plane
  // y_r + y_i at double offset y3_off (state buffers) / y3_off_r (packed r_next) from the column start
  int64_t y3_off;
  int64_t y3_off_r;
  int* nonfinite;       // set to 1 if any written value is not finite (nullable)
};

constexpr int kBKHalf = 16;            // doubles per 128-byte swizzle row (one TMA box of the interleaved operands)

// MODE (the arithmetic of one step):
//  kReal: real symmetric (BNC, WNC count real columns, a plain real GEMM);
//  kZ4M:  complex Hermitian by the real embedding A' [B' B''] (BNC, WNC count complex columns; B'' in
//         registers): 4 real MACs per complex MAC;
//  kZ3M:  complex Hermitian by Gauss's 3-multiplication form: for conj(h) y with
//         h = a_r + i a_i, y = y_r + i y_i,  P1 = sum a_r y_r,  P2 = sum a_i y_i,
//         P3 = sum (a_r - a_i)(y_r + y_i);  Re = P1 + P2,  Im = P3 - P1 + P2  -- 3 real MACs per
//         complex MAC. The planes a_r - a_i (of H, once per call) and y_r + y_i (of Y, written by the
//         previous step's epilogue) are extra TMA operands, so the main loop has no FP64 add.
constexpr int kReal = 0, kZ4M = 1, kZ3M = 2;

// KH: 128-byte swizzle rows of the interleaved operands per stage (2: 16 complex K entries per stage; 1:
// half stages of 8 entries -- twice as many, finer-grained stages in the same shared memory, so a stage
// is refilled sooner after it is released; the 3M planes then use 64-byte rows with the 64B swizzle)
template <int BM, int BNC, int WM, int WNC, int STAGES, int MODE = kZ4M, int CL = 1, int KH = 2, int PW = 0>
struct FilterCfg {
  static constexpr bool kCplx = MODE != kReal;  // complex output columns
  static constexpr int kWarpsM = BM / WM;
  static constexpr int kWarpsN = BNC / WNC;
  static constexpr int kConsumerWarps = kWarpsM * kWarpsN;
  static constexpr int kConsumerThreads = kConsumerWarps * 32;
  // PW = 0: thread 0 doubles as the TMA producer; PW = 4: an extra warpgroup produces (one lane of it
  // issues the loads), its registers handed to the consumers with setmaxnreg
  static constexpr int kThreads = kConsumerThreads + 32 * PW;
  static constexpr int kMT = WM / 8;   // 8-row MMA tiles per warp
  static constexpr int kNT = MODE == kZ4M ? WNC / 4 : WNC / 8;  // 8-real-column MMA tiles per warp
  static constexpr int kNP = MODE == kZ3M ? 3 : 1;              // accumulator sets (P1, P2, P3)
  static constexpr int kKH = KH;
  static constexpr int kBKs = kBKHalf * KH;                     // real K doubles per stage
  static constexpr int kPlaneRow = 64 * KH;                     // bytes of one plane row per stage
  static constexpr int kA3 = MODE == kZ3M ? BM * kPlaneRow : 0;  // a_r - a_i plane
  // B regions start on 1024-byte boundaries (the 128B-swizzle pattern is taken from absolute shared
  // address bits, so a region must begin at an 8-row atom): BNC rows padded to a multiple of 8
  static constexpr int kBRow = ((BNC + 7) / 8) * 8 * 128;       // smem stride of one B swizzle region
  static constexpr int kB3 = MODE == kZ3M ? ((BNC + 7) / 8) * 8 * kPlaneRow : 0;  // y_r + y_i plane
  static constexpr int kABytes = KH * BM * 128 + kA3;
  static constexpr int kBBytes = KH * kBRow + kB3;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // bytes the stage's TMA boxes deliver (mbarrier transaction count)
  static constexpr int kTxBytes = KH * BM * 128 + kA3 + KH * BNC * 128 + (MODE == kZ3M ? BNC * kPlaneRow : 0);
  static_assert(kStageBytes % 1024 == 0, "stages must start on 128B-swizzle atoms");
  static constexpr int kSmemBytes = STAGES * kStageBytes + 2 * STAGES * 8 + 1024;  // + barriers + align
  static_assert(WM % 8 == 0 && WNC % (MODE == kZ4M ? 4 : 8) == 0 && BM % WM == 0 && BNC % WNC == 0, "tile shape");
  static_assert(BM <= 256 && BNC <= 256, "TMA box limit");
};

// 128B swizzle: 16-byte chunk c of row r lives at chunk (c ^ (r & 7)) (buffer 1024-byte aligned).
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// 64B swizzle (64-byte rows): 16-byte chunk c of row r lives at chunk c ^ ((r >> 1) & 3) (512-byte atoms)
__device__ __forceinline__ uint32_t swz64(int row, int chunk) {
  return static_cast<uint32_t>(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4));
}

// first iteration of CTA c in the stream-K tail
__device__ __forceinline__ int64_t sk_start(const StepParams& p, int64_t c) { return p.sk_bounds[c]; }
// CTA whose (non-empty) tail range contains iteration g: the last c with sk_bounds[c] <= g
__device__ __forceinline__ int64_t sk_owner(const StepParams& p, int64_t g) {
  int lo = 0, hi = p.grid - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.sk_bounds[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

template <int N>
struct IntC {
  static constexpr int value = N;
};

// balanced N split: N tile i covers column units [i*(U/T) + min(i, U%T), ...) of width U/T (+1 for
// the first U%T tiles), so every tile has (nearly) the same number of active warps and the stream-K
// split by iterations stays balanced; returns the first column (relative to col0) and the units
__device__ __forceinline__ int tile_cols(int ntile, int tiles_n, int units, int wnc, int* n_units) {
  const int base = units / tiles_n, extra = units % tiles_n;
  *n_units = base + (ntile < extra ? 1 : 0);
  return (ntile * base + (ntile < extra ? ntile : extra)) * wnc;
}

// conditional sign flip on the integer pipe: XOR of the high word with 0 or 0x80000000 (inline PTX so
// the compiler cannot turn it into an FP64 DADD, which would compete with the DMMAs)
__device__ __forceinline__ double xor_sign(double x, uint32_t mask) {
  int hi = __double2hiint(x);
  asm("xor.b32 %0, %0, %1;" : "+r"(hi) : "r"(mask));
  return __hiloint2double(hi, __double2loint(x));
}

// CL = 2: CTA pairs (thread-block clusters of 2 along N). The pair shares one M tile: each CTA loads
// half of every A box (rows [rank BM/2, (rank+1) BM/2) of H and of the plane) and multicasts it to both,
// so the H tile crosses L2 -> SM once per pair and the pair advances in k in lockstep; the persistent /
// stream-K schedule runs over pair tiles (tiles_n N tiles = tiles_n / 2 pair columns) and cluster ids.
// OCC: CTAs resident per SM (the persistent grid is OCC x SM count; 2 lets one CTA's MMAs cover the
// other's TMA waits)
// PW = 4: a dedicated producer warpgroup (the last four warps; one lane works) issues every TMA load as
// soon as the consumer warps have released a stage -- STAGES - 1 stages of lead instead of about one.
// Registers are allocated per warpgroup, so the launch gives every thread 65536 / kThreads; the producer
// warpgroup drops to kProdRegs with setmaxnreg and the consumers take kConsRegs
template <int BM, int BNC, int WM, int WNC, int STAGES, int MODE = kZ4M, int CL = 1, int OCC = 1, int KH = 2,
          int PW = 0>
__global__ void __launch_bounds__(FilterCfg<BM, BNC, WM, WNC, STAGES, MODE, 1, 2, PW>::kThreads, OCC)
    filter_step_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmA3, const __grid_constant__ CUtensorMap tmB3,
                       const StepParams p) {
  using Cfg = FilterCfg<BM, BNC, WM, WNC, STAGES, MODE, CL, KH, PW>;
  static_assert(PW == 0 || (PW == 4 && CL == 1 && Cfg::kConsumerWarps % 4 == 0), "producer warpgroup: single CTAs");
  // the CTA's register pool is kThreads x (its launch allocation, 65536 / kThreads rounded down to 8 for a
  // kernel this large -- launch_cfg verifies the compiled count before the first launch, since an
  // increase the pool cannot satisfy would block the consumers forever)
  constexpr int kProdRegs = 24;
  constexpr int kLaunchRegs = (65536 / Cfg::kThreads) / 8 * 8;
  constexpr int kConsRegs =
      PW ? ((kLaunchRegs * Cfg::kThreads - 32 * PW * kProdRegs) / Cfg::kConsumerThreads) / 8 * 8 : 0;
  static_assert(PW == 0 || kConsRegs <= 256, "setmaxnreg range");
  static_assert(CL == 1 || CL == 2, "cluster of 1 or 2");
  static_assert(KH == 2 || (KH == 1 && MODE == kZ3M), "half stages are built for the 3M planes");
  constexpr int kHalves = KH;
  constexpr int kBK = Cfg::kBKs;
  static_assert(BM % (8 * CL) == 0, "A box split");
  constexpr bool CPLX = MODE == kZ4M;  // the A' [B' B''] embedding
  constexpr int kNP = Cfg::kNP;
  // stream-K partial accumulators: 3M publishes (Re, Im) = (P1 + P2, P3 - P1 + P2) -- the epilogue's
  // combination is linear, so partial sums of it are exact partials -- 2 sets instead of 3
  constexpr int kPS = MODE == kZ3M ? 2 : kNP;
  constexpr int kAcc = kPS * Cfg::kMT * Cfg::kNT * 2;  // partial doubles per thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align to 1024 B (128B-swizzle atoms) by pointer arithmetic on the shared array, so the compiler
  // keeps the shared address space and emits LDS (an integer round-trip would give generic LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  __shared__ int s_ticket;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // the consumer warps' own barrier (the producer warp of PW = 1 never joins the split-tile fix-up)
  auto consumer_sync = [&]() {
    if constexpr (PW == 0)
      __syncthreads();
    else
      asm volatile("bar.sync 1, %0;" ::"n"(Cfg::kConsumerThreads) : "memory");
  };
  const int64_t cta = blockIdx.x / CL;        // schedule id (cluster id when CL = 2)
  const int crank = (int)(blockIdx.x % CL);    // rank in the cluster (1-D grid, cluster dims (CL,1,1))
  const int64_t pcta = blockIdx.x;             // physical CTA: owner of partial-accumulator slots
  // schedule tile (pair tile when CL = 2) -> this CTA's output tile (m-major, tiles_n N tiles)
  auto cta_tile = [&](int T) -> int {
    if constexpr (CL == 1) {
      return T;
    } else {
      const int tnp = p.tiles_n / CL;
      return (T / tnp) * p.tiles_n + (T % tnp) * CL + crank;
    }
  };
  const int KT = p.num_kt;
  const int64_t t_beg = sk_start(p, cta);
  const int64_t t_end = sk_start(p, cta + 1);
  const int64_t dp_iters = (int64_t)p.dp_units * KT;
  const int64_t my_iters = dp_iters + (t_end - t_beg);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps * CL);  // CL = 2: both CTAs release a stage
    }
    fence_barrier_init();
  }
  __syncthreads();
  if constexpr (CL == 2) cluster_sync();  // the peer's barriers exist before any multicast lands

  // CTA-local iteration j -> (tile, k-tile)
  auto coords = [&](int64_t j, int& tile, int& kt) {
    if (j < dp_iters) {
      tile = (int)(cta + (j / KT) * p.grid);
      kt = (int)(j % KT);
    } else {
      const int64_t g = t_beg + (j - dp_iters);
      tile = p.tail_tile0 + (int)(g / KT);
      kt = (int)(g % KT);
    }
  };
  // TMA producer. PW = 4: one lane of the producer warpgroup refills each stage as soon as every
  // consumer warp has released it (STAGES - 1 stages of lead). PW = 0: thread 0, itself a consumer,
  // refills one iteration behind its own progress, so it blocks only if another warp is more than one
  // k-tile behind. Either way the producer walks the CTA's iterations in order with an incremental
  // cursor and runs across tile boundaries, so the next tile's first stages stream in during an
  // epilogue. The cursor lives in shared memory: one thread touches it, and keeping it out of the
  // register file leaves the consumers their full budget
  __shared__ struct {
    int64_t j;
    int tile, kt, dp_left, stage;
  } pc;
  int64_t& pc_j = pc.j;
  int& pc_tile = pc.tile;
  int& pc_kt = pc.kt;
  int& pc_dp_left = pc.dp_left;
  int& pc_stage = pc.stage;
  auto pc_init = [&]() {
    if (pc_dp_left > 0) {
      pc_tile = (int)cta;
      pc_kt = 0;
    } else {
      pc_tile = p.tail_tile0 + (int)(t_beg / KT);
      pc_kt = (int)(t_beg % KT);
    }
  };
  // load k-tile kt of schedule tile T into stage st
  auto load_stage = [&](int T, int kt, int st) {
    const int tile = cta_tile(T);
    const int m0 = (tile / p.tiles_n) * BM;
    int nu;
    const int bcol = p.b_col0 + tile_cols(tile % p.tiles_n, p.tiles_n, p.units_n, WNC, &nu);
    uint8_t* sa = smem + st * Cfg::kStageBytes;
    uint8_t* sb = sa + Cfg::kABytes;
    mbar_arrive_expect_tx(&full[st], Cfg::kTxBytes);  // CL = 2: includes the peer's multicast half
    const int q = kt / p.kt_per_rank;
    const int t = kt - q * p.kt_per_rank;
    const int ka = q * p.a_rank_stride + t * kBK;
    const int kb = t * kBK;
    // plane K coordinate: rank chunks of the plane start on even entries (a3_rank_stride = nloc rounded
    // up to even) -- a TMA box starting 8 bytes off a 16-byte boundary traps
    const int ka3 = q * p.a3_rank_stride + t * (kBK / 2);
#pragma unroll
    for (int h = 0; h < kHalves; ++h) {
      if constexpr (CL == 1) {
        tma_load_2d(sa + h * BM * 128, &tmA, ka + h * kBKHalf, m0, &full[st]);
      } else {
        tma_load_2d_mc(sa + h * BM * 128 + crank * (BM / CL) * 128, &tmA, ka + h * kBKHalf, m0 + crank * (BM / CL),
                       &full[st], (uint16_t)((1u << CL) - 1));
      }
      tma_load_3d(sb + h * Cfg::kBRow, &tmB, kb + h * kBKHalf, bcol, q, &full[st]);
    }
    if constexpr (MODE == kZ3M) {  // the real planes: 16 complex entries = one 128-byte row
      if constexpr (CL == 1) {
        tma_load_2d(sa + kHalves * BM * 128, &tmA3, ka3, m0, &full[st]);
      } else {
        tma_load_2d_mc(sa + kHalves * BM * 128 + crank * (BM / CL) * Cfg::kPlaneRow, &tmA3, ka3, m0 + crank * (BM / CL),
                       &full[st], (uint16_t)((1u << CL) - 1));
      }
      tma_load_3d(sb + kHalves * Cfg::kBRow, &tmB3, kb / 2, bcol, q, &full[st]);
    }
  };
  auto produce = [&]() {  // load iteration pc_j into stage pc_stage, then advance the cursor
    load_stage(pc_tile, pc_kt, pc_stage);
    ++pc_j;
    if (++pc_stage == STAGES) pc_stage = 0;
    if (++pc_kt == KT) {
      pc_kt = 0;
      if (pc_dp_left > 0) {
        if (--pc_dp_left > 0) {
          pc_tile += p.grid;
        } else {
          pc_init();
        }
      } else {
        ++pc_tile;
      }
    }
  };
  const int producer_thread = PW ? Cfg::kConsumerThreads : 0;
  if ((int)threadIdx.x == producer_thread) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if constexpr (MODE == kZ3M) {
      tma_prefetch(&tmA3);
      tma_prefetch(&tmB3);
    }
    pc_j = 0;
    pc_stage = 0;
    pc_dp_left = p.dp_units;
    pc_init();
    while (pc_j < STAGES && pc_j < my_iters) produce();
  }
  if constexpr (PW == 4) {
    if (warp >= Cfg::kConsumerWarps) {  // the producer warpgroup: refill every stage as soon as it is released
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
      if (warp == Cfg::kConsumerWarps && lane == 0) {
        uint32_t ph = 0;  // parity of the stage's current use
        for (int64_t it = STAGES; it < my_iters; ++it) {
          const int st = (int)(it % STAGES);
          if (st == 0) ph ^= 1u;
          mbar_wait(&empty[st], ph ^ 1u);  // consumers released iteration it - STAGES
          produce();
        }
      }
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsRegs));
  }

  const int wm = warp % Cfg::kWarpsM;
  const int wn = warp / Cfg::kWarpsM;
  const int g = lane >> 2;   // MMA group (row of A / column of B within the 8-wide tile)
  const int qd = lane & 3;   // thread in group (k index; output column pair)
  const bool odd = (g & 1);  // this lane feeds an imaginary-part (B'') column
  const uint32_t sign_mask = odd ? 0x80000000u : 0u;
  const int a_row0 = wm * WM + g;
  // B smem row of this lane's first MMA column: complex -> complex column (lane >> 3), the lane pair
  // (2c, 2c+1) building (B', B''); real -> real column g
  const int b_row0 = CPLX ? wn * WNC + (lane >> 3) : wn * WNC + g;  // 3M: complex column g
  bool bad = false;

  double acc[Cfg::kMT][Cfg::kNT][2];
  double acc2[MODE == kZ3M ? Cfg::kMT : 1][MODE == kZ3M ? Cfg::kNT : 1][2];  // 3M: P2
  double acc3[MODE == kZ3M ? Cfg::kMT : 1][MODE == kZ3M ? Cfg::kNT : 1][2];  // 3M: P3
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
      for (int jj = 0; jj < Cfg::kNT; ++jj) {
        acc[i][jj][0] = acc[i][jj][1] = 0.0;
        if constexpr (MODE == kZ3M) acc2[i][jj][0] = acc2[i][jj][1] = acc3[i][jj][0] = acc3[i][jj][1] = 0.0;
      }
  };
  // accumulator element x of set s (s = 0: P1 / the only set, 1: P2, 2: P3) -- flat view for stream-K
  auto acc_ref = [&](int sset, int i, int jj, int e) -> double& {
    if constexpr (MODE == kZ3M) {
      if (sset == 1) return acc2[i][jj][e];
      if (sset == 2) return acc3[i][jj][e];
    }
    return acc[i][jj][e];
  };

  // fused epilogue: three-term recurrence, degree masking, finished-column store
  auto store_val = [&](int col, int64_t r, double v) {  // real: one value of column col
    const double* yc = reinterpret_cast<const double*>(p.y_cur);
    const double* yp = reinterpret_cast<const double*>(p.y_prev);
    if (p.flags & 1) v -= p.c * yc[(int64_t)col * p.ld_cur + r];
    v *= p.a;
    if (p.flags & 2) v -= p.b * yp[(int64_t)col * p.ld_prev + r];
    bad |= !isfinite(v);
    if (col < p.fin_end) {
      reinterpret_cast<double*>(p.out)[(int64_t)col * p.ld_out + r] = v;
    } else {
      reinterpret_cast<double*>(p.y_next)[(int64_t)col * p.ld_next + r] = v;
      for (int q = 0; q < p.n_rdst; ++q)
        reinterpret_cast<double*>(p.r_dst[q])[(int64_t)(col - p.fin_end) * p.ld_r_next + r] = v;
    }
  };
  // 3M: one complex output (vr, vi) of column col; also writes the y_r + y_i plane of the next operand
  auto store_z3 = [&](int col, int64_t r, double vr, double vi) {
    if (p.flags & 1) {
      const double2 yc = p.y_cur[(int64_t)col * p.ld_cur + r];
      vr -= p.c * yc.x;
      vi -= p.c * yc.y;
    }
    vr *= p.a;
    vi *= p.a;
    if (p.flags & 2) {
      const double2 yp = p.y_prev[(int64_t)col * p.ld_prev + r];
      vr -= p.b * yp.x;
      vi -= p.b * yp.y;
    }
    bad |= !(isfinite(vr) && isfinite(vi));
    const double2 v = make_double2(vr, vi);
    if (col < p.fin_end) {
      p.out[(int64_t)col * p.ld_out + r] = v;
    } else {
      double2* yn = p.y_next + (int64_t)col * p.ld_next;
      yn[r] = v;
      reinterpret_cast<double*>(yn)[p.y3_off + r] = vr + vi;
      for (int q = 0; q < p.n_rdst; ++q) {
        double2* rn = p.r_dst[q] + (int64_t)(col - p.fin_end) * p.ld_r_next;
        rn[r] = v;
        reinterpret_cast<double*>(rn)[p.y3_off_r + r] = vr + vi;
      }
    }
  };
  // packed: the 3M accumulators hold (Re, Im) in (acc, acc2) after a stream-K reduction
  auto epilogue = [&](int tile, bool packed) {
    const int m0 = (tile / p.tiles_n) * BM;
    int nu;
    const int c0 = tile_cols(tile % p.tiles_n, p.tiles_n, p.units_n, WNC, &nu);
    if (wn >= nu) return;  // this warp's columns belong to the next tile
    const int col_base = p.col0 + c0 + wn * WNC + (CPLX ? qd : 2 * qd);  // (unused by 3M)
#pragma unroll
    for (int i = 0; i < Cfg::kMT; ++i) {
      const int64_t r = (int64_t)m0 + wm * WM + i * 8 + g;
      if (r >= p.nrows) continue;
#pragma unroll
      for (int j = 0; j < Cfg::kNT; ++j) {
        if constexpr (MODE == kZ3M) {
          // lane owns complex columns col, col + 1 of row r: Re = P1 + P2, Im = P3 - P1 + P2
          const int col = p.col0 + c0 + wn * WNC + j * 8 + 2 * qd;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (col + e >= p.col_end) continue;
            if (packed)
              store_z3(col + e, r, acc[i][j][e], acc2[i][j][e]);
            else
              store_z3(col + e, r, acc[i][j][e] + acc2[i][j][e], (acc3[i][j][e] - acc[i][j][e]) + acc2[i][j][e]);
          }
          continue;
        }
        if constexpr (MODE == kReal) {
          const int col = col_base + j * 8;
          if (col < p.col_end) store_val(col, r, acc[i][j][0]);
          if (col + 1 < p.col_end) store_val(col + 1, r, acc[i][j][1]);
          continue;
        }
        const int col = col_base + j * 4;
        if (col >= p.col_end) continue;
        double vr = acc[i][j][0], vi = acc[i][j][1];
        if (p.flags & 1) {
          const double2 yc = p.y_cur[(int64_t)col * p.ld_cur + r];
          vr -= p.c * yc.x;
          vi -= p.c * yc.y;
        }
        vr *= p.a;
        vi *= p.a;
        if (p.flags & 2) {
          const double2 yp = p.y_prev[(int64_t)col * p.ld_prev + r];
          vr -= p.b * yp.x;
          vi -= p.b * yp.y;
        }
        const double2 v = make_double2(vr, vi);
        bad |= !(isfinite(vr) && isfinite(vi));
        if (col < p.fin_end) {
          p.out[(int64_t)col * p.ld_out + r] = v;
        } else {
          p.y_next[(int64_t)col * p.ld_next + r] = v;
          for (int q = 0; q < p.n_rdst; ++q) p.r_dst[q][(int64_t)(col - p.fin_end) * p.ld_r_next + r] = v;
        }
      }
    }
  };

  int64_t j = 0;  // CTA-local iteration (global across tiles)
  int stage = 0;   // j % STAGES
  uint32_t phase = 0;  // (j / STAGES) & 1
  while (j < my_iters) {
    int T, kbeg;
    coords(j, T, kbeg);
    const int tile = cta_tile(T);  // this CTA's output tile
    // this work unit: k-tiles [kbeg, kend) of `tile`
    int kend = KT;
    if (j >= dp_iters) {
      const int64_t g0 = t_beg + (j - dp_iters);
      const int64_t tile_end_g = (g0 / KT + 1) * KT;
      kend = (int)(KT - (tile_end_g - (t_end < tile_end_g ? t_end : tile_end_g)));
    }
    zero_acc();

    // Active 8-column MMA tiles of this warp (4 complex columns under 4M): a warp whose columns all lie
    // past the active block (ragged last N tile) skips its MMAs, and the warp holding the block's last,
    // partly active column unit skips the MMA tiles of its inactive half -- the DMMA pipe is shared per
    // SM sub-partition, so neither the padding unit nor the padding half costs tensor-core time.
    // NA is a compile-time count (kNT, kNT / 2 or 0) so the k-loop keeps its full unrolling.
    int nu;
    const int tc0 = tile_cols(tile % p.tiles_n, p.tiles_n, p.units_n, WNC, &nu);
    const int wcols = min(nu * WNC, p.col_end - p.col0 - tc0) - wn * WNC;
    constexpr bool kHalfOk = Cfg::kNT % 2 == 0;
    const int na = wcols <= 0 ? 0 : (kHalfOk && 2 * wcols <= WNC) ? Cfg::kNT / 2 : Cfg::kNT;
    // the MMAs of one stage for NA active MMA tiles (the branch stays inside the k-loop so the loop
    // control keeps to the uniform datapath)
    auto mma_stage = [&](auto na_tag, const uint8_t* sa, const uint8_t* sb) {
      constexpr int NA = decltype(na_tag)::value;
      if constexpr (MODE == kZ3M) {
        const uint8_t* a3 = sa + kHalves * BM * 128;
        const uint8_t* b3 = sb + kHalves * Cfg::kBRow;
#pragma unroll
        for (int h = 0; h < kHalves; ++h) {
          const uint8_t* ah = sa + h * BM * 128;
          const uint8_t* bh = sb + h * Cfg::kBRow;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            // P1, P2: complex entry 2*qd + sub of this half -> (a_r, a_i) and (y_r, y_i) in one LDS.128
            const int chunk = 2 * qd + sub;
            double2 av[Cfg::kMT], bv[NA];
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i) av[i] = *reinterpret_cast<const double2*>(ah + swz(a_row0 + i * 8, chunk));
#pragma unroll
            for (int jj = 0; jj < NA; ++jj) bv[jj] = *reinterpret_cast<const double2*>(bh + swz(b_row0 + jj * 8, chunk));
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], av[i].x, bv[jj].x);
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc2[i][jj][0], acc2[i][jj][1], av[i].y, bv[jj].y);
          }
          // P3: plane entries 2c, 2c+1 of chunk c. KH = 2: c = 2qd + h of the 128-byte row (h = 0, 1
          // cover all 16 entries; even/odd chunks for the two rows of a quarter-warp keep the LDS.128
          // conflict-free under the 128B swizzle, c' = c ^ (row & 7)). KH = 1: c = qd of the 64-byte row
          // (64B swizzle: c' = c ^ ((row >> 1) & 3); rows g, g+1 of a quarter-warp land in opposite
          // 64-byte halves of the bank space -> conflict-free)
          {
            double2 cv[Cfg::kMT], dv[NA];
            if constexpr (KH == 2) {
              const int chunk = 2 * qd + h;
#pragma unroll
              for (int i = 0; i < Cfg::kMT; ++i) cv[i] = *reinterpret_cast<const double2*>(a3 + swz(a_row0 + i * 8, chunk));
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dv[jj] = *reinterpret_cast<const double2*>(b3 + swz(b_row0 + jj * 8, chunk));
            } else {
#pragma unroll
              for (int i = 0; i < Cfg::kMT; ++i) cv[i] = *reinterpret_cast<const double2*>(a3 + swz64(a_row0 + i * 8, qd));
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dv[jj] = *reinterpret_cast<const double2*>(b3 + swz64(b_row0 + jj * 8, qd));
            }
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc3[i][jj][0], acc3[i][jj][1], cv[i].x, dv[jj].x);
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc3[i][jj][0], acc3[i][jj][1], cv[i].y, dv[jj].y);
          }
        }
      } else {
#pragma unroll
        for (int h = 0; h < kHalves; ++h) {
          const uint8_t* ah = sa + h * BM * 128;
          const uint8_t* bh = sb + h * Cfg::kBRow;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            // k-steps 2*sub, 2*sub+1 of this half: lane qd covers doubles 4*qd + 2*sub + {0,1}
            const int chunk = 2 * qd + sub;
            double2 av[Cfg::kMT], bv[NA];
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i) av[i] = *reinterpret_cast<const double2*>(ah + swz(a_row0 + i * 8, chunk));
#pragma unroll
            for (int jj = 0; jj < NA; ++jj) {
              if constexpr (CPLX) {
                // B' (even g): (re, im) as stored; B'' (odd g): (im, -re) -- two lane-offset LDS.64 do the
                // swap, one integer XOR the sign (no select, no FP64 op)
                const double* y = reinterpret_cast<const double*>(bh + swz(b_row0 + jj * 4, chunk));
                bv[jj].x = y[odd ? 1 : 0];
                bv[jj].y = xor_sign(y[odd ? 0 : 1], sign_mask);
              } else {
                bv[jj] = *reinterpret_cast<const double2*>(bh + swz(b_row0 + jj * 8, chunk));
              }
            }
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], av[i].x, bv[jj].x);
#pragma unroll
            for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
              for (int jj = 0; jj < NA; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], av[i].y, bv[jj].y);
          }
        }
      }
    };
    for (int kt = kbeg; kt < kend; ++kt, ++j) {
      const int s = stage;
      mbar_wait(&full[s], phase);
      const uint8_t* sa = smem + s * Cfg::kStageBytes;
      const uint8_t* sb = sa + Cfg::kABytes;
      if (na == Cfg::kNT)
        mma_stage(IntC<Cfg::kNT>{}, sa, sb);
      else if (kHalfOk && na == Cfg::kNT / 2)
        mma_stage(IntC<(kHalfOk ? Cfg::kNT / 2 : Cfg::kNT)>{}, sa, sb);
      __syncwarp();
      if (lane == 0) {
        if constexpr (CL == 1) {
          mbar_arrive(&empty[s]);
        } else {  // release the stage in both CTAs: either may multicast into it next
#pragma unroll
          for (int q = 0; q < CL; ++q) mbar_arrive_cluster(&empty[s], (uint32_t)q);
        }
      }
      // refill the stage of iteration j - 1 (stage pc_stage, phase of j - 1) with iteration pc_j
      if (PW == 0 && threadIdx.x == 0 && j >= 1 && *(volatile int64_t*)&pc_j < my_iters) {
        const uint32_t prev_phase = (s == 0) ? (phase ^ 1u) : phase;
        mbar_wait(&empty[pc_stage], prev_phase);
        produce();
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }

    if (kbeg == 0 && kend == KT) {
      epilogue(tile, false);
      continue;
    }
    // ---- split tile: publish the partial accumulator; the last contributor finishes the tile ----
    const int u = T - p.tail_tile0;  // schedule (pair) tile of the stream-K tail
    const int64_t U0 = (int64_t)u * KT, U1 = U0 + KT;
    const int my_slot = (t_beg / KT == u) ? 0 : 1;
    double* mine = p.partials + ((pcta * 2 + my_slot) * kAcc) * (int64_t)Cfg::kThreads;
#pragma unroll
    for (int ps = 0; ps < kPS; ++ps)
#pragma unroll
      for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
        for (int jj = 0; jj < Cfg::kNT; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double v;
            if constexpr (MODE == kZ3M)
              v = ps == 0 ? acc[i][jj][e] + acc2[i][jj][e] : (acc3[i][jj][e] - acc[i][jj][e]) + acc2[i][jj][e];
            else
              v = acc_ref(ps, i, jj, e);
            __stcg(mine + (((ps * Cfg::kMT + i) * Cfg::kNT + jj) * 2 + e) * Cfg::kThreads + threadIdx.x, v);
          }
    __threadfence();
    consumer_sync();
    const int64_t c_lo = sk_owner(p, U0), c_hi = sk_owner(p, U1 - 1);
    int nseg = 0;
    for (int64_t c = c_lo; c <= c_hi; ++c)
      if (sk_start(p, c + 1) > sk_start(p, c)) ++nseg;
    if (threadIdx.x == 0) s_ticket = atomicAdd(&p.tickets[u * CL + crank], 1);
    consumer_sync();
    if (s_ticket != nseg - 1) continue;  // not the last contributor
    __threadfence();
    zero_acc();
    for (int64_t c = c_lo; c <= c_hi; ++c) {  // fixed k order: deterministic sum
      const int64_t cs = sk_start(p, c);
      if (sk_start(p, c + 1) <= cs) continue;
      const int slot = (cs / KT == u) ? 0 : 1;
      const double* src = p.partials + (((c * CL + crank) * 2 + slot) * kAcc) * (int64_t)Cfg::kThreads;
#pragma unroll
      for (int ps = 0; ps < kPS; ++ps)
#pragma unroll
        for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
          for (int jj = 0; jj < Cfg::kNT; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              acc_ref(ps, i, jj, e) += __ldcg(src + (((ps * Cfg::kMT + i) * Cfg::kNT + jj) * 2 + e) * Cfg::kThreads + threadIdx.x);
    }
    epilogue(tile, MODE == kZ3M);
    if (threadIdx.x == 0) p.tickets[u * CL + crank] = 0;  // ready for the next launch (stream ordered)
  }
  if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
  // neither CTA of a pair leaves while the other may still multicast into it or arrive on its barriers
  if constexpr (CL == 2) cluster_sync();
  // peer push: this thread's NVLink stores are ordered before the inter-step barrier's signal
  if (p.n_rdst > 1) __threadfence_system();
}

// host launcher: picks the tile configuration for the step shape; returns cudaError_t
struct TileChoice {
  int id;
  int cluster;  // CTAs per thread-block cluster (2: A-multicast pairs)
  int occ;      // CTAs resident per SM (persistent grid = occ x SMs)
  int kh;       // 128-byte swizzle rows per stage (real K per stage = 16 kh doubles)
  int bm, bnc;
  int threads;  // CTA size of the variant
  int acc;      // accumulator doubles per thread (partial-slot size = acc * threads doubles)
  int wnc;      // complex columns per warp (column-unit width of the balanced N split)
  double cost;  // model time of the step (choose_*: comparable between the 3M and 4M families)
};
TileChoice choose_filter_tile(int64_t nrows, int64_t ncols, int num_sms);
// Fill the persistent-schedule fields of p (tiles_n .. tail_iters) for variant t on num_sms SMs.
void schedule_filter_step(const TileChoice& t, int num_sms, StepParams& p);
// workspace the schedule needs: partial slots (doubles) and tickets (ints)
size_t filter_partials_doubles(const TileChoice& t, int num_sms);
// tmA3 / tmB3: the 3M planes (ignored by the other modes)
cudaError_t launch_filter_step(const TileChoice& t, const CUtensorMap& tmA, const CUtensorMap& tmB,
                               const CUtensorMap& tmA3, const CUtensorMap& tmB3, const StepParams& p,
                               cudaStream_t stream);
// real-symmetric variants (ids >= 100)
TileChoice choose_filter_tile_real(int64_t nrows, int64_t ncols, int num_sms);
// complex 3M variants (ids >= 200)
TileChoice choose_filter_tile_z3(int64_t nrows, int64_t ncols, int num_sms);

}  // namespace chfsi
