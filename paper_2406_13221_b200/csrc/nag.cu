// nag.cu — fused enhanced-NAG iteration (enctrain.py:344-398 loop body).
#include "../../include/helr_ckks.h"
#include "ctx.cuh"

extern "C" int helr_nag_iteration(helr_ctx* ctx, const uint64_t* z, int blocks, int log_g, int log_m,
                                  const uint64_t* w, const uint64_t* v, const uint64_t* bbar, int bbar_level, int lw,
                                  const uint64_t* rlk, const uint64_t* const* rot_keys, const uint64_t* mask_pt,
                                  const uint64_t* consts, uint64_t* w_out, uint64_t* v_out, void* stream) {
    (void)ctx; (void)z; (void)blocks; (void)log_g; (void)log_m; (void)w; (void)v; (void)bbar; (void)bbar_level;
    (void)lw; (void)rlk; (void)rot_keys; (void)mask_pt; (void)consts; (void)w_out; (void)v_out; (void)stream;
    set_error("helr_nag_iteration: not built yet");
    return HELR_EINVAL;
}
