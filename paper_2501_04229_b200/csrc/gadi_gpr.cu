// gadi_gpr.cu — GPR alpha predictor (placeholder until the device path lands).
#include "../../include/gadi_cuda.h"
extern "C" {
int gadi_gpr_fit(const double*, const double*, int32_t, const gadi_gpr_opts*, gadi_gpr**) { return GADI_E_UNSUPPORTED; }
int gadi_gpr_predict(gadi_gpr*, const double*, int32_t, double*, double*) { return GADI_E_UNSUPPORTED; }
int gadi_gpr_params(const gadi_gpr*, double*, double*, double*, double*, double*) { return GADI_E_UNSUPPORTED; }
int gadi_gpr_destroy(gadi_gpr*) { return GADI_OK; }
}
