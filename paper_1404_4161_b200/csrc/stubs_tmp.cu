#include "ctx.cuh"
extern "C" {
chfsi_status chfsi_lanczos_bounds(chfsi_ctx ctx, int64_t, int64_t, int64_t, const void*, int64_t, int32_t, uint64_t,
                                  double*, double*, double*) { chfsi::set_err(ctx, "not implemented"); return CHFSI_ERR_ARG; }
chfsi_status chfsi_qr(chfsi_ctx ctx, int64_t, int64_t, int64_t, void*, int64_t, int64_t, int64_t, int32_t*) { chfsi::set_err(ctx, "not implemented"); return CHFSI_ERR_ARG; }
chfsi_status chfsi_rayleigh_ritz(chfsi_ctx ctx, int64_t, int64_t, int64_t, const void*, int64_t, void*, int64_t, int64_t,
                                 double, double*, double*) { chfsi::set_err(ctx, "not implemented"); return CHFSI_ERR_ARG; }
chfsi_status chfsi_solve_sequence(chfsi_ctx ctx, int64_t, int64_t, int64_t, int32_t, chfsi_get_h, void*, const chfsi_opts*,
                                  void*, int64_t, double*, double*, chfsi_report*) { chfsi::set_err(ctx, "not implemented"); return CHFSI_ERR_ARG; }
}
