// filter_step.cu -- instantiations and launcher of K1 (see filter_step.cuh).
#include <cstdlib>

#include "filter_step.cuh"

namespace chfsi {

namespace {

template <int BM, int BNC, int WM, int WNC, int STAGES, int MODE = kZ4M>
cudaError_t launch_cfg(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                       const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
  using Cfg = FilterCfg<BM, BNC, WM, WNC, STAGES, MODE>;
  auto kern = filter_step_kernel<BM, BNC, WM, WNC, STAGES, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<p.grid, Cfg::kThreads, Cfg::kSmemBytes, stream>>>(tmA, tmB, tmA3, tmB3, p);
  return cudaGetLastError();
}

struct Variant {
  int bm, bnc, wnc;
  double eff;   // relative per-flop efficiency of the variant (measured)
  int threads;  // CTA size
  int acc;      // accumulator doubles per thread
};
constexpr Variant kVariants[] = {
    {128, 32, 16, 0.930, 256, 32},  // 0: 8 warps, warp tile 32 x 16
    {64, 64, 16, 0.920, 256, 32},   // 1: 8 warps, warp tile 32 x 16
    {128, 64, 32, 0.940, 256, 64},  // 2: 8 warps, warp tile 32 x 32
    {64, 32, 16, 0.700, 128, 32},   // 3: 4 warps
    {128, 64, 16, 0.950, 512, 32},  // 4: 16 warps (4 per SMSP), warp tile 32 x 16
    {128, 16, 16, 0.800, 256, 16},  // 5: 8 warps, warp tile 16 x 16 (narrow blocks)
    {128, 32, 8, 0.960, 512, 16},   // 6: 16 warps, warp tile 32 x 8
    {128, 48, 16, 1.000, 384, 32},  // 7: 12 warps, warp tile 32 x 16 (34.9 TF/s at n=13000, k=624)
    {128, 64, 16, 0.900, 256, 64},  // 8: 8 warps, warp tile 64 x 16 (measured slower; kept for sweeps)
    {256, 32, 16, 0.970, 256, 64},  // 9: 8 warps, warp tile 64 x 16, BM 256 (best at exact 32-column fits)
};

}  // namespace

TileChoice choose_filter_tile(int64_t nrows, int64_t ncols, int num_sms) {
  // test hook: CHFSI_FILTER_VARIANT forces one variant (parity tests cover every instantiation)
  const char* fs = getenv("CHFSI_FILTER_VARIANT");
  const int forced = fs ? atoi(fs) : -1;
  const int nvar = (int)(sizeof(kVariants) / sizeof(kVariants[0]));
  if (forced >= 0 && forced < nvar)
    return TileChoice{forced, kVariants[forced].bm, kVariants[forced].bnc, kVariants[forced].threads,
                      kVariants[forced].acc, kVariants[forced].wnc};
  // the persistent stream-K schedule removes wave quantisation: minimise padded work / efficiency
  // (efficiencies: measured full-width rates relative to the best variant)
  int best = 0;
  double best_cost = 1e300;
  for (int v = 0; v < nvar; ++v) {
    const int64_t tm = (nrows + kVariants[v].bm - 1) / kVariants[v].bm;
    // balanced N split in warp-tile units: every tile has `per` active warp columns; idle warps skip
    // their MMAs but are not free (model: 30 % of full cost), and fewer than two
    // active warps per SM sub-partition lose latency hiding (profiles/r01_filter_variants)
    const Variant& V = kVariants[v];
    const int64_t units = (ncols + V.wnc - 1) / V.wnc;
    const int64_t tn = (ncols + V.bnc - 1) / V.bnc;
    const int64_t per = (units + tn - 1) / tn;
    const int warps_m = V.threads / 32 / (V.bnc / V.wnc);
    const double active_warps = (double)per * warps_m;
    const double occ = active_warps >= 8 ? 1.0 : 0.6 + 0.05 * active_warps;
    const double cols = 0.3 * (double)(tn * per * V.wnc) + 0.7 * (double)ncols;
    const double cost = (double)tm * V.bm * cols / (V.eff * occ);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = v;
    }
  }
  (void)num_sms;
  return TileChoice{best, kVariants[best].bm, kVariants[best].bnc, kVariants[best].threads, kVariants[best].acc,
                    kVariants[best].wnc};
}

TileChoice choose_filter_tile_real(int64_t nrows, int64_t ncols, int num_sms) {
  (void)num_sms;
  struct RV {
    int id, bm, bnc, wnc, threads, acc;
    double eff;
  };
  static const RV rv[] = {{100, 128, 96, 32, 384, 32, 1.0}, {101, 128, 64, 32, 256, 32, 0.97},
                          {102, 128, 32, 16, 256, 16, 0.93}};
  const char* fs = getenv("CHFSI_FILTER_VARIANT_REAL");
  const int forced = fs ? atoi(fs) : -1;
  int best = 0;
  double best_cost = 1e300;
  for (int v = 0; v < 3; ++v) {
    if (forced >= 0 && rv[v].id != forced) continue;
    const int64_t tm = (nrows + rv[v].bm - 1) / rv[v].bm;
    const int64_t units = (ncols + rv[v].wnc - 1) / rv[v].wnc;
    const int64_t tn = (ncols + rv[v].bnc - 1) / rv[v].bnc;
    const int64_t per = (units + tn - 1) / tn;
    const double cols = 0.3 * (double)(tn * per * rv[v].wnc) + 0.7 * (double)ncols;
    const double cost = (double)tm * rv[v].bm * cols / rv[v].eff;
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = v;
    }
  }
  return TileChoice{rv[best].id, rv[best].bm, rv[best].bnc, rv[best].threads, rv[best].acc, rv[best].wnc};
}

TileChoice choose_filter_tile_z3(int64_t nrows, int64_t ncols, int num_sms) {
  (void)num_sms;
  // 3M variants: accumulators are 3 sets (P1, P2, P3) of (WM/8) x (WNC/8) 8x8 tiles
  struct ZV {
    int id, bm, bnc, wnc, threads, acc;
    double eff;
  };
  // eff: measured full-width rates relative to 200 (n = 13000, k = 624: 45.2 / 42.0 / 32.4 / 41.8 /
  // 30.2 TF/s ZGEMM-equivalent; profiles/r01_z3_variants.log)
  static const ZV zv[] = {{200, 128, 48, 16, 384, 48, 1.0},  {201, 128, 32, 16, 256, 48, 0.93},
                          {202, 128, 16, 8, 256, 24, 0.72},  {203, 64, 64, 16, 256, 48, 0.925},
                          {204, 192, 32, 16, 384, 48, 0.67}};
  const int nv = (int)(sizeof(zv) / sizeof(zv[0]));
  const char* fs = getenv("CHFSI_FILTER_VARIANT_Z3");
  const int forced = fs ? atoi(fs) : -1;
  int best = 0;
  double best_cost = 1e300;
  for (int v = 0; v < nv; ++v) {
    if (forced >= 0 && zv[v].id != forced) continue;
    const int64_t tm = (nrows + zv[v].bm - 1) / zv[v].bm;
    const int64_t units = (ncols + zv[v].wnc - 1) / zv[v].wnc;
    const int64_t tn = (ncols + zv[v].bnc - 1) / zv[v].bnc;
    const int64_t per = (units + tn - 1) / tn;
    const int warps_m = zv[v].threads / 32 / (zv[v].bnc / zv[v].wnc);
    const double active_warps = (double)per * warps_m;
    const double occ = active_warps >= 8 ? 1.0 : 0.6 + 0.05 * active_warps;
    const double cols = 0.3 * (double)(tn * per * zv[v].wnc) + 0.7 * (double)ncols;
    const double cost = (double)tm * zv[v].bm * cols / (zv[v].eff * occ);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = v;
    }
  }
  return TileChoice{zv[best].id, zv[best].bm, zv[best].bnc, zv[best].threads, zv[best].acc, zv[best].wnc};
}

void schedule_filter_step(const TileChoice& t, int num_sms, StepParams& p) {
  const int64_t ncols = p.col_end - p.col0;
  const int64_t tm = (p.nrows + t.bm - 1) / t.bm, tn = (ncols + t.bnc - 1) / t.bnc;
  p.units_n = (int32_t)((ncols + t.wnc - 1) / t.wnc);
  const int64_t tiles = tm * tn;
  const int64_t iters = tiles * p.num_kt;
  const int64_t grid = iters < num_sms ? iters : num_sms;
  p.tiles_n = (int32_t)tn;
  p.grid = (int32_t)grid;
  p.dp_units = (int32_t)(tiles / grid);
  p.tail_tile0 = (int32_t)(p.dp_units * grid);
  p.tail_iters = (tiles - p.tail_tile0) * p.num_kt;
}

size_t filter_partials_doubles(const TileChoice& t, int num_sms) { return (size_t)2 * num_sms * t.acc * t.threads; }

cudaError_t launch_filter_step(const TileChoice& t, const CUtensorMap& tmA, const CUtensorMap& tmB,
                               const CUtensorMap& tmA3, const CUtensorMap& tmB3, const StepParams& p,
                               cudaStream_t stream) {
#define LC(BM, BNC, WM, WNC, ST, MODE) launch_cfg<BM, BNC, WM, WNC, ST, MODE>(tmA, tmB, tmA3, tmB3, p, stream)
  switch (t.id) {
    case 0:
      return LC(128, 32, 32, 16, 5, kZ4M);
    case 1:
      return LC(64, 64, 32, 16, 6, kZ4M);
    case 2:
      return LC(128, 64, 32, 32, 4, kZ4M);
    case 3:
      return LC(64, 32, 32, 16, 8, kZ4M);
    case 4:
      return LC(128, 64, 32, 16, 4, kZ4M);
    case 5:
      return LC(128, 16, 16, 16, 6, kZ4M);
    case 6:
      return LC(128, 32, 32, 8, 5, kZ4M);
    case 7:
      return LC(128, 48, 32, 16, 4, kZ4M);
    case 8:
      return LC(128, 64, 64, 16, 4, kZ4M);
    case 9:
      return LC(256, 32, 64, 16, 3, kZ4M);
    // real symmetric (columns are real columns)
    case 100:
      return LC(128, 96, 32, 32, 3, kReal);
    case 101:
      return LC(128, 64, 32, 32, 4, kReal);
    case 102:
      return LC(128, 32, 32, 16, 5, kReal);
    // complex 3M (columns are complex columns)
    case 200:
      return LC(128, 48, 32, 16, 3, kZ3M);
    case 201:
      return LC(128, 32, 32, 16, 3, kZ3M);
    case 202:
      return LC(128, 16, 32, 8, 3, kZ3M);
    case 203:
      return LC(64, 64, 32, 16, 4, kZ3M);
    case 204:
      return LC(192, 32, 32, 16, 2, kZ3M);
    default:
      return cudaErrorInvalidValue;
  }
#undef LC
}

}  // namespace chfsi
