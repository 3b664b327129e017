// vc3_rt.h — host runtime shared by the translation units of the library
// (defined in vc3_kernels.cu): CUDA status bookkeeping, layout validation,
// the by-value parameter block and the device-resident decode tables.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "../../include/vc3_b200.h"
#include "vc3_device.cuh"

namespace vc3 {
namespace rt {

int cuda_status(cudaError_t e);        // VC3_OK or VC3_ERR_CUDA (records the error)
int launch_status();                   // cuda_status(cudaGetLastError())
int current_device();
int sm_count();
bool layout_ok(const vc3_layout& L);
Params make_params(const vc3_layout& L);
bool is_default_layout(const vc3_layout& L);
int get_table(const Params& P, const double2** out);  // nullptr when !P.table_mode
// the reference's own decode tables + the measured decode tolerance (exact modes)
int get_full_table(const Params& P, const double2** out);
double full_table_tolerance(const Params& P);  // host copy of the measured tolerance
size_t table_smem(const Params& P);
int ensure_smem(const void* func, size_t bytes);       // opt in to > 48 KB dynamic smem

}  // namespace rt
}  // namespace vc3
