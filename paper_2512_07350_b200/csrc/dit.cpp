// dit.cpp — placeholder until the DiT lands (returns LP_ERR_INVALID_ARGUMENT).
#include "common.cuh"
using namespace lpb200;
extern "C" {
int lp_dit_reserve(lp_dit*, int64_t) { set_last_error("DiT not built"); return LP_ERR_INVALID_ARGUMENT; }
int lp_dit_cfg_predict(lp_dit*, const void*, const int64_t*, int, int, double, void*, void*) {
    set_last_error("DiT not built");
    return LP_ERR_INVALID_ARGUMENT;
}
}
