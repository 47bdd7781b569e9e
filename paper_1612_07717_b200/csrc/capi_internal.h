// capi_internal.h — host helpers shared by capi.cu and drivers.cu.  Not public.
#pragma once

#include <cstdint>
#include <string>

#include "../../include/ablmc_b200.h"

namespace ablmc_host {

const char* set_error(const std::string& msg);
int validate(const ablmc_problem* pr);
int smoothing_polynomial(int r, double* coeffs);
int64_t dim_of(const ablmc_problem* pr);
double lambda_at(double x, const ablmc_model_params& p);

}  // namespace ablmc_host
