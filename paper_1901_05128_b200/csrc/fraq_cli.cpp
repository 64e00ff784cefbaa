// fraq_cli.cpp -- the `fraq` command line (reference: tools/fraq_main.cpp) over the B200 path.
// Subcommands weights, kernel-error, solve, convergence, bench with the reference's options,
// defaults, output files (CSV at 17 digits, meta.txt sidecar, snapshot_n<N>.csv) and exit codes
// (0 ok, 2 usage / std::invalid_argument, 1 other errors).  The reference uses CLI11 for parsing;
// this binary parses `--key value` / `--key=value` itself with the same option sets.
#include <cmath>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "fraq_bench.hpp"

namespace {

using Opts = std::map<std::string, std::string>;

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

const std::map<std::string, std::set<std::string>>& option_sets() {
    static const std::map<std::string, std::set<std::string>> sets = {
        {"weights", {"scheme", "alpha", "tau", "n", "out"}},
        {"kernel-error", {"scheme", "alpha", "tau", "np", "np1", "np2", "ns", "n-max", "out"}},
        {"solve", {"scheme", "alpha1", "alpha2", "a", "m", "grid-m", "tau", "n-steps", "t-final",
                   "init", "np", "np1", "np2", "ns", "eps-tol", "auto-kernel", "snapshot-times",
                   "out-dir", "out"}},
        {"convergence", {"scheme", "alpha1", "alpha2", "a", "m", "grid-m", "taus", "ref-tau",
                         "t-final", "init", "np", "np1", "np2", "ns", "eps-tol", "auto-kernel",
                         "out-dir"}},
        {"bench", {"scheme", "alpha1", "alpha2", "a", "m", "grid-m", "t-final", "init", "np", "np1",
                   "np2", "ns", "eps-tol", "auto-kernel", "n-list", "out"}},
    };
    return sets;
}

void usage(std::ostream& o) {
    o << "fast convolution-quadrature benchmarks for the two-state fractional Fokker-Planck "
         "system (B200)\n"
         "usage: fraq [--config FILE] <weights|kernel-error|solve|convergence|bench> [--key value]...\n";
    for (const auto& [cmd, keys] : option_sets()) {
        o << "  " << cmd << ":";
        for (const auto& k : keys) o << " --" << k;
        o << "\n";
    }
}

// argv -> (config path, subcommand, options); throws Usage on malformed command lines.
void parse_args(int argc, char** argv, std::string& config, std::string& cmd, Opts& opts) {
    int i = 1;
    auto take = [&](const std::string& arg, std::string& key, std::string& val) {
        const std::size_t eq = arg.find('=');
        key = arg.substr(2, eq == std::string::npos ? std::string::npos : eq - 2);
        if (eq != std::string::npos) {
            val = arg.substr(eq + 1);
        } else {
            if (i + 1 >= argc) throw Usage("option --" + key + " requires a value");
            val = argv[++i];
        }
    };
    for (; i < argc; ++i) {
        const std::string arg = argv[i];
        if (arg.rfind("--", 0) != 0) break;
        std::string key, val;
        take(arg, key, val);
        if (key != "config") throw Usage("unknown option --" + key);
        config = val;
    }
    if (i >= argc) throw Usage("a subcommand is required");
    cmd = argv[i++];
    const auto it = option_sets().find(cmd);
    if (it == option_sets().end()) throw Usage("unknown subcommand " + cmd);
    for (; i < argc; ++i) {
        const std::string arg = argv[i];
        if (arg.rfind("--", 0) != 0) throw Usage("unexpected argument " + arg);
        std::string key, val;
        take(arg, key, val);
        if (!it->second.count(key)) throw Usage("unknown option --" + key + " for " + cmd);
        opts[key] = val;
    }
}

std::unique_ptr<std::ofstream> open_out(const std::string& path) {
    if (path.empty() || path == "-") return nullptr;
    auto f = std::make_unique<std::ofstream>(path);
    if (!*f) throw std::runtime_error("cannot open output file: " + path);
    return f;
}

void write_meta(const std::string& dir, const fraq::ExperimentConfig& c) {
    std::ofstream m(std::filesystem::path(dir) / "meta.txt");
    using fraq::format_double;
    m << "alpha1 = " << format_double(c.alpha1) << "\nalpha2 = " << format_double(c.alpha2)
      << "\na = " << format_double(c.coupling_a) << "\ngrid-m = " << c.grid_m
      << "\nt-final = " << format_double(c.t_final) << "\nref-tau = " << format_double(c.ref_tau)
      << "\ninit = " << (c.initial == fraq::InitialData::poly_sin ? "poly_sin" : "indicator")
      << "\nnp = " << c.kernel.be_points << "\nnp1 = " << c.kernel.sbd_points_1
      << "\nnp2 = " << c.kernel.sbd_points_2 << "\nns = " << c.kernel.sbd_head
      << "\neps-tol = " << format_double(c.kernel.eps_tol)
      << "\nauto-kernel = " << (c.kernel.auto_size ? "1" : "0") << "\ntaus =";
    for (double t : c.taus) m << ' ' << format_double(t);
    m << "\nschemes =";
    for (auto s : c.schemes) m << ' ' << fraq::scheme_name(s);
    m << "\n";
}

int run(const std::string& config, const std::string& cmd, Opts opts) {
    Opts file;
    if (!config.empty()) {
        std::ifstream in(config);
        if (!in) throw std::runtime_error("cannot open config file: " + config);
        file = fraq::parse_config_text(in);
    }
    const std::string out_path = opts.count("out") ? opts["out"] : "";
    opts.erase("out");
    auto merged = [&](const std::string& k, const std::string& dflt) {
        if (auto it = opts.find(k); it != opts.end()) return it->second;
        if (auto it = file.find(k); it != file.end()) return it->second;
        return dflt;
    };
    auto num = [&](const std::string& k, const std::string& dflt) {
        return fraq::parse_fraction(merged(k, dflt));
    };
    auto cq_scheme = [&]() {
        const std::string s = merged("scheme", "be");
        if (s != "be" && s != "sbd")
            throw std::invalid_argument("scheme must be 'be' or 'sbd', got '" + s + "'");
        return s;
    };
    if (cmd == "weights") {
        const std::string s = cq_scheme();
        const double alpha = num("alpha", "0.5"), tau = num("tau", "1");
        const long n = std::lround(num("n", "10"));
        const fraq::WeightTable t =
            s == "sbd" ? fraq::sbd_weights(alpha, tau, n) : fraq::be_weights(alpha, tau, n);
        auto f = open_out(out_path);
        fraq::write_weights_csv(f ? *f : std::cout, t);
    } else if (cmd == "kernel-error") {
        const std::string s = cq_scheme();
        const double alpha = num("alpha", "0.5"), tau = num("tau", "0.001");
        const long n_max = std::lround(num("n-max", "1000"));
        fraq::KernelErrorReport rep;
        if (s == "sbd") {
            int ns = int(num("ns", "0"));
            if (ns <= 0) ns = fraq::default_sbd_head(alpha);
            rep = fraq::kernel_error_report(
                fraq::build_sbd_kernel(alpha, tau, int(num("np1", "41")), int(num("np2", "41")), ns),
                n_max);
        } else {
            rep = fraq::kernel_error_report(fraq::build_be_kernel(alpha, tau, int(num("np", "64"))),
                                            n_max);
        }
        auto f = open_out(out_path);
        fraq::write_kernel_error_csv(f ? *f : std::cout, rep);
    } else if (cmd == "solve") {
        const fraq::ExperimentConfig cfg = fraq::resolve_config(file, opts);
        const double tau = num("tau", "0");
        fraq::ProblemSpec spec;
        spec.alpha1 = cfg.alpha1;
        spec.alpha2 = cfg.alpha2;
        spec.coupling_a = cfg.coupling_a;
        spec.grid_m = cfg.grid_m;
        spec.t_final = cfg.t_final;
        spec.initial = cfg.initial;
        spec.n_steps = std::lround(cfg.t_final / (tau > 0 ? tau : cfg.t_final / 100.0));
        if (const double n = num("n-steps", "0"); n > 0) spec.n_steps = std::lround(n);
        const fraq::Scheme scheme = fraq::scheme_from_name(merged("scheme", "be"));
        std::vector<long> snaps;
        if (const std::string times = merged("snapshot-times", ""); !times.empty())
            for (double t : fraq::parse_fraction_list(times)) snaps.push_back(std::lround(t / spec.tau()));
        const std::string out_dir = merged("out-dir", ".");
        std::function<void(long, const fraq::StateField&)> observer;
        if (!snaps.empty()) {
            std::filesystem::create_directories(out_dir);
            observer = [&](long n, const fraq::StateField& f) {
                for (long s : snaps)
                    if (s == n) {
                        std::ofstream snap(std::filesystem::path(out_dir) /
                                           ("snapshot_n" + std::to_string(n) + ".csv"));
                        fraq::write_snapshot_csv(snap, spec, f);
                    }
            };
        }
        const fraq::RunResult rr = fraq::run(spec, scheme, cfg.kernel, observer);
        auto f = open_out(out_path);
        fraq::write_snapshot_csv(f ? *f : std::cout, spec, rr.final_state);
        std::cerr << "loop_seconds=" << fraq::format_double(rr.loop_seconds)
                  << " setup_seconds=" << fraq::format_double(rr.setup_seconds) << "\n";
    } else if (cmd == "convergence") {
        fraq::ExperimentConfig cfg = fraq::resolve_config(file, opts);
        cfg.validate();
        std::filesystem::create_directories(cfg.out_dir);
        const auto reports = fraq::run_convergence(cfg);
        write_meta(cfg.out_dir, cfg);
        for (const auto& rep : reports) {
            const auto path = std::filesystem::path(cfg.out_dir) /
                              ("convergence_" + fraq::scheme_name(rep.scheme) + ".csv");
            std::ofstream f(path);
            fraq::write_convergence_csv(f, rep);
            std::cout << path.string() << "\n";
        }
    } else {  // bench
        const fraq::ExperimentConfig cfg = fraq::resolve_config(file, opts);
        std::vector<long> ns;
        for (double v : fraq::parse_fraction_list(merged("n-list", "100,200,400,800,1600")))
            ns.push_back(std::lround(v));
        const auto rows = fraq::timing_sweep(cfg, ns);
        auto f = open_out(out_path);
        fraq::write_bench_csv(f ? *f : std::cout, rows);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--help" || a == "-h") {
            usage(std::cout);
            return 0;
        }
    }
    std::string config, cmd;
    Opts opts;
    try {
        parse_args(argc, argv, config, cmd, opts);
    } catch (const Usage& e) {
        std::cerr << "fraq: " << e.what() << "\n";
        usage(std::cerr);
        return 2;
    }
    try {
        return run(config, cmd, opts);
    } catch (const std::invalid_argument& e) {
        std::cerr << "fraq: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "fraq: " << e.what() << "\n";
        return 1;
    }
}
