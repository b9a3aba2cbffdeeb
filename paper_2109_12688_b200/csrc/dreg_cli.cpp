// dreg -- command-line drop-in for the reference tool (proj/tools/dreg.cpp) over the
// B200 library.  Same subcommands, flags, defaults, validation, output lines and exit
// codes (0 success, 2 argument error, 3 I/O error, 4 numerical failure; errors print
// one `dreg: <category>: <reason>` line on stderr, dreg.cpp:286-319); every numerical
// step runs on the GPU through include/dreg_b200/dreg.hpp.
//
//   dreg [--threads N] register --target T --source S --out PHI --lambda L --theta TH
//        [--warped W] [--data-term l1|l2] [--order 1..3] [--levels 1..6]
//        [--profile capped|converged] [--tol X] [--seed-report R.json]
//        [--target-labels TL --source-labels SL]
//   dreg warp --in V --phi PHI --out O [--labels]
//   dreg evaluate --a A --b B --labels 1,2,...
//   dreg jacobian --phi PHI
//   dreg synth --case translate|blob|sphere-ellipsoid --dims M,N,H --out-prefix P
//        [--shift x,y,z] [--seed S] [--noise F]
//
// The reference parses with CLI11 (absent here); this parser accepts the same
// spellings: `--opt value`, `--opt=value`, comma-delimited lists, and the global
// --threads before or after the subcommand.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "dreg_b200/dreg.hpp"
#include "dreg_b200/synth.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitArgument = 2;
constexpr int kExitIo = 3;
constexpr int kExitNumeric = 4;

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string format6(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.6g", v);
    return buf;
}

// ---- a small option table ------------------------------------------------------------
struct Opt {
    std::string name;
    bool flag = false;      // takes no value
    bool required = false;
    int count = 1;          // values expected (0 = any number >= 1, comma or space separated)
    std::vector<std::string> values;
    bool seen = false;
};

struct Command {
    std::string name;
    std::map<std::string, Opt> opts;
    Opt& add(const std::string& n, bool required = false, int count = 1, bool flag = false) {
        Opt o;
        o.name = n;
        o.required = required;
        o.count = count;
        o.flag = flag;
        return opts[n] = o;
    }
    [[nodiscard]] bool has(const std::string& n) const { return opts.at(n).seen; }
    [[nodiscard]] const std::string& str(const std::string& n) const { return opts.at(n).values.at(0); }
};

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(item);
    if (!s.empty() && s.back() == ',') out.emplace_back();
    return out;
}

double to_double(const std::string& opt, const std::string& v) {
    char* end = nullptr;
    const double d = std::strtod(v.c_str(), &end);
    if (v.empty() || *end != '\0') throw ParseError(opt + ": " + v + " is not a number");
    return d;
}

long to_int(const std::string& opt, const std::string& v) {
    char* end = nullptr;
    const long n = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0') throw ParseError(opt + ": " + v + " is not an integer");
    return n;
}

void check_range(const std::string& opt, double v, double lo, double hi) {
    if (v < lo || v > hi)
        throw ParseError(opt + ": value " + format6(v) + " not in range [" + format6(lo) + " - " + format6(hi) + "]");
}

void check_member(const std::string& opt, const std::string& v, std::initializer_list<const char*> allowed) {
    for (const char* a : allowed)
        if (v == a) return;
    throw ParseError(opt + ": " + v + " not in {allowed set}");
}

// Parses argv[i..] into `cmd`, consuming the global --threads wherever it appears.
void parse_command(Command& cmd, int argc, char** argv, int i, int& threads) {
    while (i < argc) {
        std::string tok = argv[i++];
        std::string inline_val;
        bool has_inline = false;
        const auto eq = tok.find('=');
        if (tok.rfind("--", 0) == 0 && eq != std::string::npos) {
            inline_val = tok.substr(eq + 1);
            tok = tok.substr(0, eq);
            has_inline = true;
        }
        if (tok == "--threads") {
            const std::string v = has_inline ? inline_val : (i < argc ? argv[i++] : "");
            if (v.empty()) throw ParseError("--threads requires a value");
            threads = static_cast<int>(to_int("--threads", v));
            check_range("--threads", threads, 1, 256);
            continue;
        }
        auto it = cmd.opts.find(tok);
        if (it == cmd.opts.end()) throw ParseError("The following argument was not expected: " + tok);
        Opt& o = it->second;
        o.seen = true;
        if (o.flag) {
            if (has_inline) throw ParseError(tok + " takes no value");
            o.values = {"1"};
            continue;
        }
        std::vector<std::string> vals;
        if (has_inline) {
            for (auto& v : split(inline_val)) vals.push_back(v);
        }
        // values: further tokens up to the expected count (any count for lists)
        while (i < argc && (o.count == 0 || (int)vals.size() < o.count)) {
            const std::string next = argv[i];
            if (next.rfind("--", 0) == 0 && next.size() > 2 && !(next[2] >= '0' && next[2] <= '9')) break;
            if (next.rfind("-", 0) == 0 && next.size() > 1 && !(next[1] >= '0' && next[1] <= '9') && next[1] != '.')
                break;
            for (auto& v : split(next)) vals.push_back(v);
            ++i;
            if (o.count == 1) break;
        }
        if (vals.empty()) throw ParseError(tok + " requires a value");
        if (o.count > 0 && (int)vals.size() != o.count)
            throw ParseError(tok + ": expected " + std::to_string(o.count) + " values, got " +
                             std::to_string(vals.size()));
        o.values = vals;
    }
    for (const auto& [n, o] : cmd.opts)
        if (o.required && !o.seen) throw ParseError(n + " is required");
}

std::set<int> label_set(const dreg::LabelVolume& lbl) {
    std::set<int> out;
    for (auto v : lbl.labels)
        if (v != 0) out.insert(v);
    return out;
}

// ---- subcommands (dreg.cpp:93-226) ------------------------------------------------------
int run_register(const Command& c) {
    const std::string data_term = c.has("--data-term") ? c.str("--data-term") : "l1";
    const int order = c.has("--order") ? static_cast<int>(to_int("--order", c.str("--order"))) : 2;
    const double lambda = to_double("--lambda", c.str("--lambda"));
    const double theta = to_double("--theta", c.str("--theta"));
    const int levels = c.has("--levels") ? static_cast<int>(to_int("--levels", c.str("--levels"))) : 3;
    const std::string profile = c.has("--profile") ? c.str("--profile") : "capped";
    const double tol = c.has("--tol") ? to_double("--tol", c.str("--tol")) : -1.0;
    check_member("--data-term", data_term, {"l1", "l2"});
    check_range("--order", order, 1, 3);
    check_range("--levels", levels, 1, 6);
    check_member("--profile", profile, {"capped", "converged"});
    if (c.has("--tol") && tol < 0.0) throw ParseError("--tol: value must be non-negative");

    if (lambda < 0.0) throw std::invalid_argument("--lambda must be >= 0");
    if (theta <= 0.0) throw std::invalid_argument("--theta must be > 0");

    dreg::SolverConfig solver;
    solver.data_term = data_term == "l1" ? 1 : 2;
    solver.order = order;
    solver.lambda = lambda;
    solver.theta = theta;
    if (tol >= 0.0) solver.tol = tol;
    const auto prof = profile == "capped" ? dreg::Profile::capped : dreg::Profile::converged;
    const auto cfg = dreg::make_registration_config(prof, solver, levels);

    const dreg::ScalarVolume target = dreg::read_scalar(c.str("--target"));
    const dreg::ScalarVolume source = dreg::read_scalar(c.str("--source"));

    const dreg::RegistrationResult result = dreg::register_pair(target, source, cfg);
    dreg::write_volume(c.str("--out"), result.phi);
    if (c.has("--warped")) dreg::write_volume(c.str("--warped"), result.warped);

    if (c.has("--seed-report")) {
        dreg::RunReport report;
        report.runtime_seconds = result.elapsed_seconds;
        report.velocity_count = result.velocity_count;
        report.jacobian_pct_nonpositive = dreg::jacobian_stats(result.phi).pct_nonpositive;
        if (c.has("--target-labels") && c.has("--source-labels")) {
            const dreg::LabelVolume target_lbl = dreg::read_label(c.str("--target-labels"));
            const dreg::LabelVolume source_lbl = dreg::read_label(c.str("--source-labels"));
            const dreg::LabelVolume warped_lbl = dreg::warp_labels(source_lbl, result.phi);
            for (int label : label_set(target_lbl)) {
                report.dice[label] = dreg::dice(warped_lbl, target_lbl, label);
                report.hausdorff_mm[label] = dreg::hausdorff_slice_avg(warped_lbl, target_lbl, label);
            }
        }
        report.config = {data_term, order, lambda, theta, cfg.levels, profile, cfg.solver.tol,
                         cfg.warp_improvement_threshold, cfg.solver.epsilon, dreg::thread_count()};
        dreg::write_report(c.str("--seed-report"), report);
    }
    return kExitOk;
}

int run_warp(const Command& c) {
    const dreg::DeformationField phi = dreg::read_deformation(c.str("--phi"));
    if (c.has("--labels")) {
        const dreg::LabelVolume lbl = dreg::read_label(c.str("--in"));
        dreg::write_volume(c.str("--out"), dreg::warp_labels(lbl, phi));
    } else {
        const dreg::ScalarVolume img = dreg::read_scalar(c.str("--in"));
        dreg::write_volume(c.str("--out"), dreg::warp_image(img, phi));
    }
    return kExitOk;
}

int run_evaluate(const Command& c) {
    std::vector<int> labels;
    for (const auto& v : c.opts.at("--labels").values) labels.push_back(static_cast<int>(to_int("--labels", v)));
    const dreg::LabelVolume a = dreg::read_label(c.str("--a"));
    const dreg::LabelVolume b = dreg::read_label(c.str("--b"));
    if (!(a.dims == b.dims)) throw std::invalid_argument("dice: dimension mismatch");
    // every label in one upload (dreg_cuda_label_metrics); same values as the per-label calls
    std::vector<double> dice(labels.size()), hd(labels.size());
    std::vector<int> valid(labels.size());
    dreg::b200_detail::check(dreg_cuda_label_metrics(
        dreg::b200_detail::ctx(), a.labels.data(), b.labels.data(), dreg::b200_detail::D(a.dims),
        {a.spacing.x, a.spacing.y, a.spacing.z}, static_cast<int>(labels.size()), labels.data(), dice.data(),
        hd.data(), valid.data()));
    for (std::size_t j = 0; j < labels.size(); ++j) {
        std::cout << "label " << labels[j] << " dice " << format6(dice[j]) << " hausdorff_mm "
                  << (valid[j] ? format6(hd[j]) : std::string("nan")) << "\n";
    }
    return kExitOk;
}

int run_jacobian(const Command& c) {
    const dreg::DeformationField phi = dreg::read_deformation(c.str("--phi"));
    const dreg::JacobianStats stats = dreg::jacobian_stats(phi);
    std::cout << "pct_nonpositive " << format6(stats.pct_nonpositive) << " min_det " << format6(stats.min_det)
              << "\n";
    return kExitOk;
}

int run_synth(const Command& c) {
    const std::string kase = c.str("--case");
    check_member("--case", kase, {"translate", "blob", "sphere-ellipsoid"});
    std::vector<int> dims;
    for (const auto& v : c.opts.at("--dims").values) dims.push_back(static_cast<int>(to_int("--dims", v)));
    double shift[3] = {3.0, 0.0, 0.0};
    if (c.has("--shift"))
        for (int k = 0; k < 3; ++k) shift[k] = to_double("--shift", c.opts.at("--shift").values[k]);
    const long seed = c.has("--seed") ? to_int("--seed", c.str("--seed")) : 1;
    if (seed < 0 || seed > 4294967295L) throw ParseError("--seed: value out of range");
    const double noise = c.has("--noise") ? to_double("--noise", c.str("--noise")) : 0.0;
    check_range("--noise", noise, 0.0, 1.0);

    const dreg::Dims3 d{dims[0], dims[1], dims[2]};
    dreg::SynthPair pair;
    if (kase == "translate") pair = dreg::make_translate_case(d, {shift[0], shift[1], shift[2]});
    else if (kase == "blob") pair = dreg::make_random_smooth_case(d, static_cast<std::uint32_t>(seed));
    else pair = dreg::make_sphere_ellipsoid_case(d);
    if (noise > 0.0) dreg::add_salt_pepper(pair.source, noise, static_cast<std::uint32_t>(seed) + 17);
    const std::string prefix = c.str("--out-prefix");
    dreg::write_volume(prefix + "_target.dreg", pair.target);
    dreg::write_volume(prefix + "_source.dreg", pair.source);
    dreg::write_volume(prefix + "_target_labels.dreg", pair.target_labels);
    dreg::write_volume(prefix + "_source_labels.dreg", pair.source_labels);
    return kExitOk;
}

const char* kUsage =
    "dreg: diffeomorphic 3-D image registration (B200)\n"
    "Usage: dreg [--threads N] SUBCOMMAND [OPTIONS]\n"
    "Subcommands: register, warp, evaluate, jacobian, synth\n";

}  // namespace

int main(int argc, char** argv) {
    std::map<std::string, Command> cmds;
    {
        Command& r = cmds["register"];
        r.name = "register";
        r.add("--target", true);
        r.add("--source", true);
        r.add("--out", true);
        r.add("--warped");
        r.add("--data-term");
        r.add("--order");
        r.add("--lambda", true);
        r.add("--theta", true);
        r.add("--levels");
        r.add("--profile");
        r.add("--tol");
        r.add("--seed-report");
        r.add("--target-labels");
        r.add("--source-labels");
        Command& w = cmds["warp"];
        w.name = "warp";
        w.add("--in", true);
        w.add("--phi", true);
        w.add("--out", true);
        w.add("--labels", false, 1, true);
        Command& e = cmds["evaluate"];
        e.name = "evaluate";
        e.add("--a", true);
        e.add("--b", true);
        e.add("--labels", true, 0);
        Command& j = cmds["jacobian"];
        j.name = "jacobian";
        j.add("--phi", true);
        Command& s = cmds["synth"];
        s.name = "synth";
        s.add("--case", true);
        s.add("--dims", true, 3);
        s.add("--out-prefix", true);
        s.add("--shift", false, 3);
        s.add("--seed");
        s.add("--noise");
    }

    int threads = 1;
    Command* cmd = nullptr;
    try {
        int i = 1;
        while (i < argc && !cmd) {
            const std::string tok = argv[i];
            if (tok == "-h" || tok == "--help") {
                std::cout << kUsage;
                return kExitOk;
            }
            if (tok == "--threads" || tok.rfind("--threads=", 0) == 0) {
                std::string v;
                if (tok == "--threads") {
                    if (i + 1 >= argc) throw ParseError("--threads requires a value");
                    v = argv[i + 1];
                    i += 2;
                } else {
                    v = tok.substr(10);
                    i += 1;
                }
                threads = static_cast<int>(to_int("--threads", v));
                check_range("--threads", threads, 1, 256);
                continue;
            }
            auto it = cmds.find(tok);
            if (it == cmds.end()) throw ParseError("The following argument was not expected: " + tok);
            cmd = &it->second;
            ++i;
            for (int k = i; k < argc; ++k) {
                const std::string t = argv[k];
                if (t == "-h" || t == "--help") {
                    std::cout << kUsage;
                    return kExitOk;
                }
            }
            parse_command(*cmd, argc, argv, i, threads);
        }
        if (!cmd) throw ParseError("A subcommand is required");
        // option-level validation that CLI11 performs at parse time
        if (cmd->name == "synth") {
            check_member("--case", cmd->str("--case"), {"translate", "blob", "sphere-ellipsoid"});
        }
    } catch (const ParseError& e) {
        std::cerr << "dreg: argument-error: " << e.what() << "\n";
        return kExitArgument;
    }

    try {
        dreg::set_thread_count(threads);
        if (cmd->name == "register") return run_register(*cmd);
        if (cmd->name == "warp") return run_warp(*cmd);
        if (cmd->name == "evaluate") return run_evaluate(*cmd);
        if (cmd->name == "jacobian") return run_jacobian(*cmd);
        if (cmd->name == "synth") return run_synth(*cmd);
    } catch (const ParseError& e) {
        std::cerr << "dreg: argument-error: " << e.what() << "\n";
        return kExitArgument;
    } catch (const std::invalid_argument& e) {
        std::cerr << "dreg: argument-error: " << e.what() << "\n";
        return kExitArgument;
    } catch (const dreg::io_error& e) {
        std::cerr << "dreg: io-error: " << e.what() << "\n";
        return kExitIo;
    } catch (const dreg::numeric_error& e) {
        std::cerr << "dreg: numeric-error: " << e.what() << "\n";
        return kExitNumeric;
    } catch (const std::exception& e) {
        std::cerr << "dreg: error: " << e.what() << "\n";
        return kExitNumeric;
    }
    return kExitArgument;
}
