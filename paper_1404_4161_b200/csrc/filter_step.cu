// filter_step.cu -- instantiations and launcher of K1 (see filter_step.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "filter_step_launch.cuh"

namespace chfsi {

namespace {

struct Variant {
  int id, bm, bnc, wnc, threads, acc;
  double eff;       // per-flop efficiency relative to the family's best full-width variant (measured)
  int cluster = 1;  // 2: CTA pairs multicasting the shared H tile
  int occ = 1;      // CTAs per SM
  int kh = 2;       // 128-byte swizzle rows per stage (1: half stages)
};
// 4M (real embedding) variants; ids are the launch_filter_step cases
// The variants the step model never selects (for any width 1..2048 and panel height 64..32768: 4M 0, 2,
// 4, 8, 15; 3M 201-204, 206, 209, 210, 220, 227; real 100, 101) are built only with -DCHFSI_K1_AB (their
// A/B measurements stay in profiles/r01_*_variants.log, r01_cluster_ab.log, r01_occ2_ab.log,
// r01_halfstage_ab.log).
constexpr Variant kVariants[] = {
#ifdef CHFSI_K1_AB
    {0, 128, 32, 16, 256, 32, 0.930},  // 8 warps, warp tile 32 x 16
    {2, 128, 64, 32, 256, 64, 0.940},  // 8 warps, warp tile 32 x 32
    {4, 128, 64, 16, 512, 32, 0.950},  // 16 warps (4 per SMSP), warp tile 32 x 16
    {8, 128, 64, 16, 256, 64, 0.900},  // 8 warps, warp tile 64 x 16 (measured slower; kept for sweeps)
    {15, 256, 8, 4, 256, 16, 0.750},   // 8 warps (4 x 2), warp tile 64 x 4
#endif
    {1, 64, 64, 16, 256, 32, 0.920},   // 8 warps, warp tile 32 x 16
    {3, 64, 32, 16, 128, 32, 0.700},   // 4 warps
    {5, 128, 16, 16, 256, 16, 0.900},  // 8 warps, warp tile 16 x 16 (narrow blocks; best at k_a = 16)
    {6, 128, 32, 8, 512, 16, 0.960},   // 16 warps, warp tile 32 x 8
    {7, 128, 48, 16, 384, 32, 1.000},  // 12 warps, warp tile 32 x 16 (34.9 TF/s at n=13000, k=624)
    {9, 256, 32, 16, 256, 64, 0.970},  // 8 warps, warp tile 64 x 16, BM 256 (best at exact 32-column fits)
    // narrow (HBM-bound) steps, warp tile 32 or 64 x 4 complex columns (no padding at k_a = 4, 8, 12);
    // eff from n = 16384, 10 steps (profiles/r01_narrow_variants.log): k_a = 4: v10 6.60 ms (6.5 TB/s);
    // k_a = 8: v13 6.99 ms, v14 7.80, v12 9.06, v11 9.83; k_a = 12: v14 9.63, v12 9.91
    {10, 256, 4, 4, 256, 8, 0.800},    // 8 warps (8 x 1), warp tile 32 x 4
    {11, 128, 8, 4, 256, 8, 0.600},    // 8 warps (4 x 2), warp tile 32 x 4
    {12, 128, 12, 4, 384, 8, 0.700},   // 12 warps (4 x 3), warp tile 32 x 4
    {13, 256, 8, 4, 512, 8, 0.850},    // 16 warps (8 x 2), warp tile 32 x 4
    {14, 256, 12, 4, 384, 16, 0.820},  // 12 warps (4 x 3), warp tile 64 x 4
};
// 3M variants: accumulators are 3 sets (P1, P2, P3) of (WM/8) x (WNC/8) 8x8 tiles. eff: rates relative
// to 200, fitted to the r02 width tables (every variant at every width, n = 13000 and 4096;
// profiles/r02_width_table_pw*.jsonl): with its producer warpgroup (r02) 200 is the fastest tile at 198 of
// 231 widths, and these efficiencies make the step model's picks cost <= 0.05 % more than the per-width
// best. 16-warp tiles cannot take a producer warpgroup (640 threads leave the consumers < 128 registers).
constexpr Variant kVariantsZ3[] = {
    {200, 128, 48, 16, 512, 48, 1.0},      // 12 consumer warps + a producer warpgroup
    {207, 64, 64, 16, 512, 24, 0.88},       // 16 warps, warp tile 16 x 16, 4 stages
    {208, 128, 32, 8, 512, 24, 0.83},       // 16 warps, warp tile 32 x 8, 3 stages
#ifdef CHFSI_K1_AB
    {239, 128, 48, 16, 384, 48, 0.97},  // z200 without the producer warpgroup
    {201, 128, 32, 16, 256, 48, 0.93}, {202, 128, 16, 8, 256, 24, 0.72},
    {203, 64, 64, 16, 256, 48, 0.925}, {204, 192, 32, 16, 384, 48, 0.67},
    {210, 128, 48, 16, 384, 48, 0.5, 2},  // z200 as multicast CTA pairs (A/B measurement; not chosen yet)
    {206, 64, 48, 16, 192, 48, 0.5, 1, 2},  // 6 warps, 2 stages, 2 CTAs per SM (A/B measurement)
    {209, 128, 48, 16, 384, 48, 0.5},       // z200 with 2 stages (pipeline-depth probe, never chosen)
    {220, 128, 48, 16, 384, 48, 0.5, 1, 1, 1},   // z200 in 6 half stages (A/B measurement)
    {227, 64, 64, 16, 512, 24, 0.5, 1, 1, 1},    // z207 in 8 half stages (A/B measurement)
#endif
};
// real-symmetric variants (columns are real columns; kNT = WNC / 8). eff fitted to the r02 width table
// (every variant at widths 28..636, n = 13000; profiles/r02_width_table_real.jsonl): with a producer
// warpgroup 135 / 133 / 132 run 34.0-35.2 TF/s at k = 624 against 33.2-33.8 without (r02_ab_pw_real.log),
// and these efficiencies make the step model's picks cost 0.007 % more than the per-width best (3.3 %
// with the r01 set 102-105).
constexpr Variant kVariantsReal[] = {
#ifdef CHFSI_K1_AB
    {100, 128, 96, 32, 384, 32, 0.955}, {101, 128, 64, 32, 256, 32, 0.94},
    {102, 128, 32, 16, 256, 16, 0.87},  {103, 192, 64, 32, 384, 32, 0.97}, {105, 128, 48, 16, 384, 16, 0.97},
#endif
    {104, 128, 64, 16, 512, 16, 0.98},   // 16 warps (no room for a producer warpgroup)
    {132, 128, 32, 16, 384, 16, 0.97},   // 8 consumer warps + a producer warpgroup
    {133, 192, 64, 32, 512, 32, 1.0},    // 12 consumer warps + a producer warpgroup
    {135, 128, 48, 16, 512, 16, 1.0},    // 12 consumer warps + a producer warpgroup
};

// Model time of one step of `ncols` active columns over `nrows` rows for variant V, in units of a
// full-efficiency 4M column-row (8 n flops at 34.9 TF/s):
//  compute: the balanced N split gives the N tiles `per` or `per - 1` warp-column units; the work-
//           weighted persistent schedule charges the average tile (units / tn + woff per iteration,
//           against per + woff for a full one);
//           active warps in a tile cover latency as g(warps): >= 12 -> 1, 8..11 -> 0.85, 4..7 -> 0.6,
//           relative to the variant's own warp count (its measured eff already includes that);
//           `speed` = the family's best full-width rate relative to 4M (3M: 45.5 / 34.9)
//  memory:  H streamed once per step per N tile column (re-reads mostly from L2: +25 % per extra N
//           tile), `hbm_cols` = the column count at which the family's compute time equals its H
//           stream at ~5.9 TB/s (4M: 16 B / entry -> 11.8; 3M: 24 B / entry -> 17.7)
// Calibrated on profiles/r01_mid_width_variants.log and r01_narrow_variants.log.
constexpr double kSkWoff = 0.75;  // per-iteration cost of a tile's stage traffic, in column units (measured A/B)

static double warp_cover(int warps) { return warps >= 12 ? 1.0 : warps >= 8 ? 0.85 : warps >= 4 ? 0.6 : 0.4; }

// Column units a step of `ncols` active columns costs under variant (wnc, mma_cols): the block's last
// unit counts one half when only its first half is active and the warp tile holds an even number of
// MMA tiles (the kernel then skips the inactive half's MMAs; mma_cols = 8 real / 3M columns, 4 complex
// columns under 4M)
static double work_units(int64_t ncols, int wnc, int mma_cols) {
  const int64_t units = (ncols + wnc - 1) / wnc;
  const int64_t rag = ncols % wnc;
  const bool half = (wnc / mma_cols) % 2 == 0 && rag != 0 && 2 * rag <= wnc;
  return (double)units - (half ? 0.5 : 0.0);
}

static double step_cost(const Variant& V, int64_t nrows, int64_t ncols, double speed, double hbm_cols,
                        int mma_cols) {
  const int64_t tm = (nrows + V.bm - 1) / V.bm;
  const int64_t units = (ncols + V.wnc - 1) / V.wnc;
  const int64_t tn = (ncols + V.bnc - 1) / V.bnc;
  const int64_t per = (units + tn - 1) / tn;
  const int warps = V.threads / 32;
  const int warps_m = warps / (V.bnc / V.wnc);
  const double cover = warp_cover((int)per * warps_m) / warp_cover(warps);
  // work-weighted stream-K (schedule_filter_step): the step costs the average tile, (work / tn + woff)
  // per iteration, against a full tile's (per + woff); without weighting every tile costs the widest
  const double wu = work_units(ncols, V.wnc, mma_cols);
  const double fill = (wu / (double)tn + kSkWoff) / ((double)per + kSkWoff);
  const double cols = (double)(tn * per * V.wnc) * (wu != (double)(tn * per) ? fill : 1.0);
  const double rows = (double)tm * V.bm;
  const double compute = rows * cols / (V.eff * cover * speed);
  const double memory = rows * hbm_cols * (1.0 + 0.25 * (double)(tn - 1));
  // + 10 % of the compute term: between variants that all hit the HBM floor, the one with less
  // padded tensor work keeps more slack (and wins)
  return (compute > memory ? compute : memory) + 0.1 * compute;
}

template <size_t N>
static TileChoice choose(const Variant (&vs)[N], const char* env, int64_t nrows, int64_t ncols, double speed,
                         double hbm_cols, int mma_cols) {
  // test hook: the environment variable forces one variant (parity tests cover every instantiation)
  const char* fs = getenv(env);
  const int forced = fs ? atoi(fs) : -1;
  int best = -1;
  double best_cost = 1e300;
  for (size_t v = 0; v < N; ++v) {
    if (forced >= 0 && vs[v].id != forced) continue;
    const double cost = step_cost(vs[v], nrows, ncols, speed, hbm_cols, mma_cols);
    if (best < 0 || cost < best_cost * 0.999) {
      best_cost = cost;
      best = (int)v;
    }
  }
  if (best < 0) {  // a forced variant that is not built (-DCHFSI_K1_AB): the launch reports an invalid value
    const Variant& V = vs[0];
    return TileChoice{forced, V.cluster, V.occ, V.kh, V.bm, V.bnc, V.threads, V.acc, V.wnc, 1e300};
  }
  const Variant& V = vs[best];
  return TileChoice{V.id, V.cluster, V.occ, V.kh, V.bm, V.bnc, V.threads, V.acc, V.wnc, best_cost};
}

}  // namespace

TileChoice choose_filter_tile(int64_t nrows, int64_t ncols, int num_sms) {
  (void)num_sms;  // the persistent stream-K schedule removes wave quantisation
  return choose(kVariants, "CHFSI_FILTER_VARIANT", nrows, ncols, 1.0, 11.8, 4);
}

TileChoice choose_filter_tile_z3(int64_t nrows, int64_t ncols, int num_sms) {
  (void)num_sms;
  return choose(kVariantsZ3, "CHFSI_FILTER_VARIANT_Z3", nrows, ncols, 45.5 / 34.9, 17.7, 8);
}

TileChoice choose_filter_tile_real(int64_t nrows, int64_t ncols, int num_sms) {
  (void)num_sms;  // real: 2 n flops per column-row; speed / memory in the same relative units
  return choose(kVariantsReal, "CHFSI_FILTER_VARIANT_REAL", nrows, ncols, 1.0, 20.0, 8);
}

void schedule_filter_step(const TileChoice& t, int num_sms, StepParams& p) {
  const int64_t ncols = p.col_end - p.col0;
  const int64_t cl = t.cluster;
  const int64_t tm = (p.nrows + t.bm - 1) / t.bm;
  int64_t tn = (ncols + t.bnc - 1) / t.bnc;
  tn = (tn + cl - 1) / cl * cl;  // pairs: an even number of N tiles (the balanced split spreads the units)
  p.units_n = (int32_t)((ncols + t.wnc - 1) / t.wnc);
  const int64_t tiles = tm * (tn / cl);  // schedule tiles (pair tiles when cl = 2)
  const int64_t iters = tiles * p.num_kt;
  const int64_t slots = (int64_t)num_sms * t.occ / cl;  // schedule ids (clusters)
  int64_t grid = iters < slots ? iters : slots;
  if (grid > StepParams::kMaxGrid) grid = StepParams::kMaxGrid;  // the sk_bounds table's capacity
  p.tiles_n = (int32_t)tn;
  p.grid = (int32_t)grid;
  int64_t dp = tiles / grid;
  const int64_t rem = tiles - dp * grid;
  // Small remainder: the rem tail tiles would each be split over grid / rem contributors, and the last
  // of them sums all their partial accumulators serially (measured: 74 contributors cost 133 us on a
  // 1.5 ms step). Folding one data-parallel wave into the stream-K tail gives every CTA 1..1.5 tiles of
  // tail work, so a tail tile has at most two contributors (DP + "two-tile" stream-K hybrid).
  // CHFSI_SK_HYBRID=0 turns it off (A/B and test hook, read per call).
  const char* hy = getenv("CHFSI_SK_HYBRID");
  const bool hybrid = !(hy && hy[0] == '0');
  if (hybrid && dp >= 1 && rem > 0 && 2 * rem < grid && (rem + grid) * cl <= kMaxTailTickets) --dp;
  p.dp_units = (int32_t)dp;
  p.tail_tile0 = (int32_t)(p.dp_units * grid);
  p.tail_iters = (tiles - p.tail_tile0) * p.num_kt;
  // Work-weighted stream-K. The balanced N split gives tile column n either `base + 1` or `base` active
  // column units; an iteration's cost is modelled as (units + woff) -- a warp with no units skips its
  // MMAs, while the stage's TMA and barrier work is paid regardless (woff, in units). With the data-
  // parallel tiles assigned c, c + grid, ... a CTA can own only full-unit tiles (e.g. every even CTA
  // when tn = 2), so equal iteration counts leave the kernel as slow as if every tile were full. The
  // tail ranges compensate: each CTA gets (total work / grid - its data-parallel work) of the tail.
  // CHFSI_SK_WEIGHT=0 restores the equal split; CHFSI_SK_WOFF sets woff (A/B hooks, read per call).
  const int64_t KT = p.num_kt, tail_tiles = tiles - p.tail_tile0;
  const int64_t ntn = tn / cl;  // schedule tile columns
  const int64_t U = p.units_n, base = U / tn, extra = U % tn;
  const char* we = getenv("CHFSI_SK_WEIGHT");
  const char* wo = getenv("CHFSI_SK_WOFF");
  // the block's last N tile is half a unit cheaper when the kernel skips the inactive half of its last
  // unit (work_units)
  const double half = (double)U - work_units(ncols, t.wnc, t.id < 100 ? 4 : 8);
  const bool weighted = !(we && we[0] == '0') && cl == 1 && (extra != 0 || half != 0.0);
  const double woff = wo ? atof(wo) : kSkWoff;
  // Per-unit speed of a tile one warp column short of full (u = bnc / wnc - 1) relative to a full tile:
  // measured 1.1 -- its fewer warps per SM sub-partition run their MMAs slightly faster per unit
  // (profiles/r02_ab_cover.txt: against 1.0, 0.5 % less K1 time over 24 mid widths of the c2 mix, full
  // width unchanged; 0.8 / 0.9 were 1-2 % slower). CHFSI_SK_C2 / CHFSI_SK_C1 set the speed of tiles one /
  // two units short (A/B hooks, read once)
  static const double cov_env = getenv("CHFSI_SK_C2") ? atof(getenv("CHFSI_SK_C2")) : 1.1;
  const double cov_short1 = t.id == 200 ? cov_env : 1.0;  // measured on the workhorse z200 only
  static const double cov_short2 = getenv("CHFSI_SK_C1") ? atof(getenv("CHFSI_SK_C1")) : 1.0;
  const int64_t wn_full = t.bnc / t.wnc;
  auto cost = [&](int64_t tile) {  // per-iteration cost of schedule tile `tile`
    const int64_t n = tile % ntn;
    const int64_t u = base + (n < extra ? 1 : 0);
    const double cov = u == wn_full - 1 ? cov_short1 : u == wn_full - 2 ? cov_short2 : 1.0;
    return ((double)u - (n == ntn - 1 ? half : 0.0)) / cov + woff;
  };
  p.sk_bounds[0] = 0;
  if (!weighted || tail_tiles == 0) {
    for (int64_t c = 1; c <= grid; ++c) p.sk_bounds[c] = (int32_t)((c * p.tail_iters) / grid);
    return;
  }
  std::vector<double> dpw(grid, 0.0);
  double total = 0.0;
  for (int64_t c = 0; c < grid; ++c) {
    for (int64_t r = 0; r < dp; ++r) dpw[c] += cost(c + r * grid) * (double)KT;
    total += dpw[c];
  }
  double tail_work = 0.0;
  for (int64_t u = 0; u < tail_tiles; ++u) tail_work += cost(p.tail_tile0 + u) * (double)KT;
  total += tail_work;
  const double target = total / (double)grid;
  double want_sum = 0.0;
  std::vector<double> want(grid);
  for (int64_t c = 0; c < grid; ++c) want_sum += (want[c] = std::max(0.0, target - dpw[c]));
  // walk the tail, closing CTA c's range once its (normalised) share of the work is reached: whole tiles
  // at a time, then the iteration inside the tile where the share ends (each iteration goes to the side
  // it overlaps more)
  int64_t g = 0;  // tail iteration cursor
  double acc = 0.0, goal = 0.0;
  for (int64_t c = 0; c < grid; ++c) {
    goal += want[c] * tail_work / want_sum;
    while (g < p.tail_iters) {
      const int64_t u = g / KT, left = (u + 1) * KT - g;  // iterations left in the cursor's tile
      const double w = cost(p.tail_tile0 + u);
      if (acc + w * (double)left <= goal) {  // the rest of the tile fits the share
        acc += w * (double)left;
        g += left;
        continue;
      }
      const int64_t take = std::max<int64_t>(0, std::min<int64_t>(left, (int64_t)std::floor((goal - acc) / w + 0.5)));
      acc += w * (double)take;
      g += take;
      break;
    }
    p.sk_bounds[c + 1] = (int32_t)(c + 1 == grid ? p.tail_iters : g);
  }
}

size_t filter_partials_doubles(const TileChoice& t, int num_sms) {
  return (size_t)2 * num_sms * t.occ * t.acc * t.threads;
}

cudaError_t launch_filter_step(const TileChoice& t, const CUtensorMap& tmA, const CUtensorMap& tmB,
                               const CUtensorMap& tmA3, const CUtensorMap& tmB3, const StepParams& p,
                               cudaStream_t stream) {
  if (t.id >= 200) return launch_filter_z3(t.id, tmA, tmB, tmA3, tmB3, p, stream);
  if (t.id >= 100) return launch_filter_real(t.id, tmA, tmB, tmA3, tmB3, p, stream);
  return launch_filter_z4(t.id, tmA, tmB, tmA3, tmB3, p, stream);
}

}  // namespace chfsi
