// filter_step.cuh -- K1: one step of the Chebyshev filter (Alg 2 line 3 / line 8) as a
// single fused kernel: a complex (Hp^H . Y_i) GEMM on the FP64 tensor cores (DMMA.8x8x4) fed by
// TMA-staged, 128B-swizzled shared-memory tiles, with the three-term-recurrence axpby, the degree
// masking and the finished-column store in the epilogue (no separate elementwise pass).
//
// Complex -> real embedding: Hp (n x nloc, complex, column-major) is read as a real
// K-major matrix A' (nloc rows, K' = 2n), Y_i as real K-major columns B' = (re, im, re, im, ...).
// The imaginary output column uses B''_j = (im, -re, im, -re, ...) built in registers from the same
// shared tile (swap + sign), so C = A' [B' B''] has (Re, Im) of output (r, j) in one thread's
// accumulator pair:  Re = sum a_q c_q + b_q d_q,  Im = sum a_q d_q - b_q c_q  for conj(h) * y.
#pragma once
#include "common.cuh"

namespace chfsi {

struct StepParams {
  int64_t nrows;        // output rows (nloc)
  int32_t num_kt;       // k-tiles (32 real = 16 complex contraction entries each)
  int32_t kt_per_rank;  // k-tiles per rank chunk of the B operand (== num_kt when p == 1)
  int32_t a_rank_stride;  // real-K offset between rank chunks in A (2 * nloc_per_rank)
  int32_t col0;         // first active complex column s_i
  int32_t col_end;      // k (one past the last active column)
  int32_t fin_end;      // columns [col0, fin_end) finish at this step and go to `out`
  int32_t b_col0;       // B-operand column coordinate of complex column col0
  int32_t flags;        // 1: read y_cur (c != 0), 2: read y_prev (b != 0)
  double a, b, c;       // Y_{i+1} = a (acc - c y_cur) - b y_prev
  const double2* y_cur;
  int64_t ld_cur;
  const double2* y_prev;
  int64_t ld_prev;
  double2* y_next;      // may alias y_prev (same element, same thread: read then write)
  int64_t ld_next;
  double2* out;         // finished columns (caller's Y)
  int64_t ld_out;
  double2* r_next;      // p > 1: this rank's chunk of the next step's packed B operand (nullable)
  int64_t ld_r_next;
  int* nonfinite;       // set to 1 if any written value is not finite (nullable)
};

constexpr int kBKHalf = 16;            // doubles per 128-byte swizzle row
constexpr int kHalves = 2;             // two swizzle rows per stage -> 32 real K per stage
constexpr int kBK = kBKHalf * kHalves;  // real K per stage

template <int BM, int BNC, int WM, int WNC, int STAGES>
struct FilterCfg {
  static constexpr int kWarpsM = BM / WM;
  static constexpr int kWarpsN = BNC / WNC;
  static constexpr int kConsumerWarps = kWarpsM * kWarpsN;
  static constexpr int kThreads = kConsumerWarps * 32;  // thread 0 doubles as the TMA producer
  static constexpr int kMT = WM / 8;   // 8-row MMA tiles per warp
  static constexpr int kNT = WNC / 4;  // 8-real-column (4 complex) MMA tiles per warp
  static constexpr int kABytes = kHalves * BM * 128;
  static constexpr int kBBytes = kHalves * BNC * 128;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 2 * STAGES * 8 + 1024;  // + barriers + align
  static_assert(WM % 8 == 0 && WNC % 4 == 0 && BM % WM == 0 && BNC % WNC == 0, "tile shape");
  static_assert(BM <= 256 && BNC <= 256, "TMA box limit");
};

// 128B swizzle: 16-byte chunk c of row r lives at chunk (c ^ (r & 7)) (buffer 1024-byte aligned).
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
}

template <int BM, int BNC, int WM, int WNC, int STAGES>
__global__ void __launch_bounds__(FilterCfg<BM, BNC, WM, WNC, STAGES>::kThreads, 1)
    filter_step_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const StepParams p) {
  using Cfg = FilterCfg<BM, BNC, WM, WNC, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x;  // n fastest: CTAs sharing an H row block run together (L2 reuse)
  const int m_tile = blockIdx.y;
  const int m0 = m_tile * BM;
  const int bcol = p.b_col0 + n_tile * BNC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // TMA producer = thread 0 (a dedicated producer warp would round the CTA to 12 warps of register
  // allocation and cap consumers at 168 registers). Stage s of k-tile kt is refilled with k-tile
  // kt + STAGES once every consumer warp has released it; thread 0 refills one iteration behind its
  // own progress, so it blocks only if another warp is more than one k-tile behind.
  auto produce = [&](int kt) {
    const int s = kt % STAGES;
    uint8_t* sa = smem + s * Cfg::kStageBytes;
    uint8_t* sb = sa + Cfg::kABytes;
    mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
    const int q = kt / p.kt_per_rank;
    const int t = kt - q * p.kt_per_rank;
    const int ka = q * p.a_rank_stride + t * kBK;
    const int kb = t * kBK;
#pragma unroll
    for (int h = 0; h < kHalves; ++h) {
      tma_load_2d(sa + h * BM * 128, &tmA, ka + h * kBKHalf, m0, &full[s]);
      tma_load_3d(sb + h * BNC * 128, &tmB, kb + h * kBKHalf, bcol, q, &full[s]);
    }
  };
  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int kt = 0; kt < STAGES && kt < p.num_kt; ++kt) produce(kt);
  }

  // ===== consumers: DMMA main loop =====
  const int wm = warp % Cfg::kWarpsM;
  const int wn = warp / Cfg::kWarpsM;
  const int g = lane >> 2;   // MMA group (row of A / column of B within the 8-wide tile)
  const int qd = lane & 3;   // thread in group (k index; output column pair)
  const bool odd = (g & 1);  // this lane feeds an imaginary-part (B'') column
  const int a_row0 = wm * WM + g;
  const int b_row0 = wn * WNC + (lane >> 3);

  double acc[Cfg::kMT][Cfg::kNT][2];
#pragma unroll
  for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::kNT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < p.num_kt; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint8_t* sa = smem + s * Cfg::kStageBytes;
    const uint8_t* sb = sa + Cfg::kABytes;
#pragma unroll
    for (int h = 0; h < kHalves; ++h) {
      const uint8_t* ah = sa + h * BM * 128;
      const uint8_t* bh = sb + h * BNC * 128;
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        // k-steps 2*sub, 2*sub+1 of this half: lane qd covers doubles 4*qd + 2*sub + {0,1}
        const int chunk = 2 * qd + sub;
        double2 av[Cfg::kMT], bv[Cfg::kNT];
#pragma unroll
        for (int i = 0; i < Cfg::kMT; ++i) {
          const int r = a_row0 + i * 8;
          av[i] = *reinterpret_cast<const double2*>(ah + swz(r, chunk));
        }
#pragma unroll
        for (int j = 0; j < Cfg::kNT; ++j) {
          const int r = b_row0 + j * 4;
          const double2 y = *reinterpret_cast<const double2*>(bh + swz(r, chunk));
          // B' (even g): (re, im) as stored; B'' (odd g): (im, -re)
          bv[j].x = odd ? y.y : y.x;
          bv[j].y = odd ? -y.x : y.y;
        }
#pragma unroll
        for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::kNT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i].x, bv[j].x);
#pragma unroll
        for (int i = 0; i < Cfg::kMT; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::kNT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i].y, bv[j].y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (threadIdx.x == 0 && kt >= 1) {
      const int kr = kt - 1 + STAGES;
      if (kr < p.num_kt) {
        mbar_wait(&empty[(kt - 1) % STAGES], ((kt - 1) / STAGES) & 1);
        produce(kr);
      }
    }
  }

  // ===== fused epilogue: three-term recurrence, degree masking, finished-column store =====
  const int col_base = p.col0 + n_tile * BNC + wn * WNC + qd;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < Cfg::kMT; ++i) {
    const int64_t r = (int64_t)m0 + wm * WM + i * 8 + g;
    if (r >= p.nrows) continue;
#pragma unroll
    for (int j = 0; j < Cfg::kNT; ++j) {
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
        if (p.r_next) p.r_next[(int64_t)(col - p.fin_end) * p.ld_r_next + r] = v;
      }
    }
  }
  if (bad && p.nonfinite) atomicOr(p.nonfinite, 1);
}

// host launcher: picks the tile configuration for the step shape; returns cudaError_t
struct TileChoice {
  int id;
  int bm, bnc;
};
TileChoice choose_filter_tile(int64_t nrows, int64_t ncols, int num_sms);
cudaError_t launch_filter_step(const TileChoice& t, const CUtensorMap& tmA, const CUtensorMap& tmB,
                               const StepParams& p, cudaStream_t stream);

}  // namespace chfsi
