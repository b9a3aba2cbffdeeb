// dreg_b200/synth.hpp -- the reference's synthetic cases (synth.hpp) over
// libdreg_synth.so (include/dreg_synth.h); byte-identical outputs.  Link -ldreg_synth.
#pragma once

#include <cstdint>
#include <stdexcept>

#include "dreg_b200/dreg.hpp"
#include "dreg_synth.h"

namespace dreg {

struct SynthPair {
    ScalarVolume target;  // I0
    ScalarVolume source;  // I1
    LabelVolume target_labels;
    LabelVolume source_labels;
};

namespace b200_detail {
inline SynthPair make_case(int kind, Dims3 dims, const double* shift, std::uint32_t seed) {
    const Spacing3 unit{1.0, 1.0, 1.0};
    SynthPair p{ScalarVolume(dims, unit), ScalarVolume(dims, unit), LabelVolume(dims, unit), LabelVolume(dims, unit)};
    if (dreg_synth_case(kind, dims.x, dims.y, dims.z, shift, seed, p.target.data.data(), p.source.data.data(),
                        p.target_labels.labels.data(), p.source_labels.labels.data()) != 0)
        throw std::invalid_argument("synth: invalid case arguments");
    return p;
}
}  // namespace b200_detail

inline SynthPair make_translate_case(Dims3 dims, const Vec3& shift) {
    const double s[3] = {shift.x, shift.y, shift.z};
    return b200_detail::make_case(DREG_CASE_TRANSLATE, dims, s, 0);
}
inline SynthPair make_sphere_ellipsoid_case(Dims3 dims) {
    return b200_detail::make_case(DREG_CASE_SPHERE_ELLIPSOID, dims, nullptr, 0);
}
inline SynthPair make_random_smooth_case(Dims3 dims, std::uint32_t seed) {
    return b200_detail::make_case(DREG_CASE_RANDOM_SMOOTH, dims, nullptr, seed);
}
inline void add_salt_pepper(ScalarVolume& vol, double fraction, std::uint32_t seed) {
    dreg_synth_salt_pepper(vol.data.data(), vol.data.size(), fraction, seed);
}

}  // namespace dreg
