/*
 * dreg_synth.h -- host-side synthetic inputs (libdreg_synth.so).  Input generation,
 * not on the registration path.
 *
 *  - dreg_synth_pair / _batch: the BASELINE.json config phantoms.
 *  - dreg_synth_case / _salt_pepper: the reference's own synthetic cases
 *    (synth.hpp: make_translate_case, make_sphere_ellipsoid_case,
 *    make_random_smooth_case, add_salt_pepper), byte-identical to the reference,
 *    used by the CLI's `synth` subcommand (tools/dreg.cpp:207-226).
 * All volumes are x-fastest; labels are u16.  Status 0 ok, 2 invalid argument.
 */
#ifndef DREG_SYNTH_H
#define DREG_SYNTH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DREG_CASE_TRANSLATE 0
#define DREG_CASE_SPHERE_ELLIPSOID 1
#define DREG_CASE_RANDOM_SMOOTH 2

int dreg_synth_pair(int config, uint32_t seed, int nx, int ny, int nz, float* fixed, float* moving);
int dreg_synth_batch(int config, uint32_t seed0, int n, int nx, int ny, int nz, float* fixed, float* moving,
                     int threads);
/* shift: 3 doubles (translate case; NULL = the CLI default {3, 0, 0}); labels nullable */
int dreg_synth_case(int kind, int nx, int ny, int nz, const double* shift, uint32_t seed, float* target,
                    float* source, uint16_t* target_labels, uint16_t* source_labels);
int dreg_synth_salt_pepper(float* vol, size_t voxels, double fraction, uint32_t seed);

#ifdef __cplusplus
}
#endif

#endif /* DREG_SYNTH_H */
