// Reference-style C++ client of the drop-in header: the same calls a dreg user makes
// (proj/tests/test_registration.cpp / test_admm.cpp idioms), compiled against
// include/dreg_b200/dreg.hpp and linked with libdreg_cuda.so.  Exit 0 = all checks pass.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>

#include "dreg_b200/dreg.hpp"

#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                   \
        }                                                               \
    } while (0)

static dreg::ScalarVolume blob(dreg::Dims3 d, double cx, double cy, double cz, double s) {
    dreg::ScalarVolume img(d, {1.0, 1.0, 1.0});
    for (int z = 0; z < d.z; ++z)
        for (int y = 0; y < d.y; ++y)
            for (int x = 0; x < d.x; ++x) {
                const double r2 = (x - cx) * (x - cx) + (y - cy) * (y - cy) + (z - cz) * (z - cz);
                img.at(x, y, z) = static_cast<float>(std::exp(-r2 / (2 * s * s)));
            }
    return img;
}

int main() {
    const dreg::Dims3 dims{24, 24, 24};
    const auto target = blob(dims, 11.5, 11.5, 11.5, 4.0);
    const auto source = blob(dims, 12.5, 11.5, 11.5, 4.0);

    dreg::SolverConfig solver;
    solver.data_term = 2;
    solver.lambda = 0.05;
    solver.theta = 0.5;
    solver.log_objective = false;
    auto cfg = dreg::make_registration_config(dreg::Profile::capped, solver, 1);
    cfg.max_admm_iters_per_level = {50};
    cfg.max_warps_per_level = {6};
    const auto res = dreg::register_pair(target, source, cfg);
    CHECK(res.velocity_count >= 1);
    CHECK(res.per_level.size() == 1);
    const auto& sad = res.per_level[0].mean_sad;
    for (std::size_t i = 1; i < sad.size(); ++i) CHECK(sad[i] <= sad[i - 1]);
    const auto js = dreg::jacobian_stats(res.phi);
    CHECK(js.pct_nonpositive == 0.0);
    CHECK(js.min_det > 0.0);

    // solve_velocity + diagnostics
    solver.max_iters = 20;
    solver.log_objective = true;
    const auto sv = dreg::solve_velocity(target, source, solver);
    CHECK(sv.diagnostics.iterations == 20);
    CHECK(sv.diagnostics.objective.size() == 20);
    CHECK(dreg::all_finite(sv.velocity));

    // error convention: invalid_argument and numeric_error
    bool threw = false;
    try {
        dreg::SolverConfig bad = solver;
        bad.theta = 0.0;
        dreg::validate(bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    auto nan_src = source;
    nan_src.data[7] = std::nanf("");
    try {
        dreg::register_pair(target, nan_src, cfg);
    } catch (const dreg::numeric_error&) {
        threw = true;
    }
    CHECK(threw);
    // io.hpp idioms (test_io.cpp): round trips, kind mismatch, report
    const auto dir = std::filesystem::temp_directory_path();
    const auto pphi = dir / "dreg_client_phi.dreg";
    dreg::write_volume(pphi, res.phi);
    const auto back = dreg::read_deformation(pphi);
    CHECK(back.disp.data == res.phi.disp.data);
    threw = false;
    try {
        (void)dreg::read_scalar(pphi);
    } catch (const dreg::io_error&) {
        threw = true;
    }
    CHECK(threw);
    const auto any = dreg::read_volume(pphi);
    CHECK(std::holds_alternative<dreg::VectorField>(any));

    // metrics.hpp idioms (test_metrics.cpp): label warp, dice, hausdorff
    dreg::LabelVolume tl(dims, {1.0, 1.0, 1.0}), sl(dims, {1.0, 1.0, 1.0});
    for (int z = 0; z < dims.z; ++z)
        for (int y = 0; y < dims.y; ++y)
            for (int x = 0; x < dims.x; ++x) {
                tl.at(x, y, z) = target.at(x, y, z) > 0.5f ? 1 : 0;
                sl.at(x, y, z) = source.at(x, y, z) > 0.5f ? 1 : 0;
            }
    const auto plbl = dir / "dreg_client_labels.dreg";
    dreg::write_volume(plbl, sl);
    CHECK(dreg::read_label(plbl).labels == sl.labels);
    const auto warped_lbl = dreg::warp_labels(sl, res.phi);
    const double d_before = dreg::dice(sl, tl, 1), d_after = dreg::dice(warped_lbl, tl, 1);
    CHECK(d_after >= d_before);
    CHECK(dreg::hausdorff_slice_avg(tl, tl, 1) == 0.0);
    dreg::RunReport report;
    report.dice[1] = d_after;
    report.hausdorff_mm[1] = dreg::hausdorff_slice_avg(warped_lbl, tl, 1);
    report.velocity_count = res.velocity_count;
    report.config = {"l2", 2, 0.05, 0.5, 1, "capped", 0.0, 0.02, 1e-6, dreg::thread_count()};
    const auto prep = dir / "dreg_client_report.json";
    dreg::write_report(prep, report);
    std::ifstream rf(prep);
    const std::string text((std::istreambuf_iterator<char>(rf)), std::istreambuf_iterator<char>());
    CHECK(text.find("\"velocity_count\": " + std::to_string(res.velocity_count)) != std::string::npos);

    // volume.hpp value-type API: Vec3 arithmetic, VectorField set / at / index,
    // Spacing3 equality, geometry validation (volume.cpp:15-22)
    {
        const dreg::Vec3 a{1.0, 2.0, 3.0}, b{0.5, -1.0, 2.0};
        CHECK((a + b).x == 1.5 && (a - b).y == 3.0 && (2.0 * a).z == 6.0 && (a * 0.5).x == 0.5);
        CHECK(a.dot(b) == 0.5 - 2.0 + 6.0 && a.squared_norm() == 14.0 && std::abs(a.norm() - std::sqrt(14.0)) < 1e-15);
        dreg::VectorField f(dims, {1.0, 1.0, 1.0});
        f.set(f.index(3, 4, 5), {0.25, -0.5, 1.0});
        CHECK(f.at(3, 4, 5).y == -0.5 && f.get(f.index(3, 4, 5)).z == 1.0);
        CHECK((dreg::Spacing3{1.0, 2.0, 3.0} == dreg::Spacing3{1.0, 2.0, 3.0}));
        CHECK(!(dreg::Spacing3{1.0, 2.0, 3.0} == dreg::Spacing3{1.0, 2.0, 2.5}));
        threw = false;
        try {
            dreg::ScalarVolume bad(dims, {1.0, 0.0, 1.0});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        // trilinear_sample (volume.hpp:107,110): lattice points are exact, clamping applies
        CHECK(dreg::trilinear_sample(target, dreg::Vec3{2.0, 3.0, 4.0}) == target.at(2, 3, 4));
        CHECK(dreg::trilinear_sample(target, dreg::Vec3{-5.0, 3.0, 4.0}) == target.at(0, 3, 4));
        const dreg::Vec3 fv = dreg::trilinear_sample(f, dreg::Vec3{3.0, 4.0, 5.0});
        CHECK(fv.x == 0.25 && fv.y == -0.5 && fv.z == 1.0);
        const double mid = dreg::trilinear_sample(target, dreg::Vec3{2.5, 3.0, 4.0});
        CHECK(std::abs(mid - 0.5 * (target.at(2, 3, 4) + target.at(3, 3, 4))) < 1e-7);
        // data_term_value (admm.hpp:68): v = 0 leaves rho = warped - target
        const auto grad = dreg::image_gradient(source);
        const dreg::VectorField zero(dims, {1.0, 1.0, 1.0});
        double l1 = 0.0;
        for (std::size_t i = 0; i < target.data.size(); ++i)
            l1 += std::abs(static_cast<double>(source.data[i]) - static_cast<double>(target.data[i]));
        CHECK(std::abs(dreg::data_term_value(target, source, grad, zero, 1) - l1) <= 1e-12 * l1);
        // w_update applies laplacian_symbol kernels and refuses any other kernel
        dreg::SolverConfig wc = solver;
        wc.lambda = 2.0;
        auto kern = dreg::laplacian_symbol(2, dims);
        const auto w = dreg::w_update(f, zero, kern, wc);
        CHECK(dreg::all_finite(w));
        kern.values[5] *= 1.5;
        threw = false;
        try {
            (void)dreg::w_update(f, zero, kern, wc);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }

    // B200 extension: the same pairs sharded over the box's GPUs (here: device 0),
    // NCCL all-gather of the per-pair records; results equal register_pair's
    {
        dreg::MultiDevice multi({0});
        std::vector<dreg_pair_record> rec;
        const auto mres = multi.register_batch({target, target}, {source, source}, cfg, &rec);
        CHECK(mres.size() == 2 && rec.size() == 2);
        for (int i = 0; i < 2; ++i) {
            CHECK(mres[i].phi.disp.data == res.phi.disp.data);
            CHECK(rec[i].pair == i && rec[i].velocity_count == res.velocity_count);
            CHECK(rec[i].folding_voxels == 0 && rec[i].min_det == js.min_det);
        }
    }

    std::printf("reference-style C++ client OK: velocity_count %d, min det %.4f\n", res.velocity_count, js.min_det);
    return 0;
}
