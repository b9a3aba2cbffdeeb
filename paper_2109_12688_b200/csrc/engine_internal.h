// Private entry points shared between engine.cu and multi.cpp (not part of the ABI).
#pragma once

#include "dreg_cuda.h"

extern "C" {
int dregb_register_batch_records(dreg_cuda_ctx* c, int n_pairs, const float* const* targets,
                                 const float* const* sources, dreg_dims3 dims, const dreg_reg_cfg* cfg,
                                 float* const* phi_out, float* const* warped_out, dreg_pair_result* results,
                                 dreg_pair_record* rec_dev, int pair_base, int device_tag);
}
