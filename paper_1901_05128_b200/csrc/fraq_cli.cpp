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

// Options of one invocation: command line over config file over the per-subcommand default.
struct Args {
    Opts cli, file;
    std::string get(const std::string& key, const std::string& fallback) const {
        for (const Opts* src : {&cli, &file})
            if (const auto it = src->find(key); it != src->end()) return it->second;
        return fallback;
    }
    double number(const std::string& key, const std::string& fallback) const {
        return fraq::parse_fraction(get(key, fallback));
    }
    long count(const std::string& key, const std::string& fallback) const {
        return std::lround(number(key, fallback));
    }
    // the CQ family of weights / kernel-error: "be" or "sbd" only
    bool sbd_family() const {
        const std::string s = get("scheme", "be");
        if (s == "be" || s == "sbd") return s == "sbd";
        throw std::invalid_argument("scheme must be 'be' or 'sbd', got '" + s + "'");
    }
    fraq::ExperimentConfig experiment() const {
        Opts no_out(cli);
        no_out.erase("out");
        return fraq::resolve_config(file, no_out);
    }
};

// Output sink: the --out file, or stdout when absent / "-".
class Sink {
public:
    explicit Sink(const std::string& path) {
        if (path.empty() || path == "-") return;
        file_.open(path);
        if (!file_) throw std::runtime_error("cannot open output file: " + path);
    }
    std::ostream& stream() { return file_.is_open() ? static_cast<std::ostream&>(file_) : std::cout; }

private:
    std::ofstream file_;
};

// meta.txt of a convergence study: the resolved configuration, one `key = value` per line.
void write_meta(const std::string& dir, const fraq::ExperimentConfig& c) {
    using fraq::format_double;
    std::string taus, schemes;
    for (double t : c.taus) taus += " " + format_double(t);
    for (fraq::Scheme s : c.schemes) schemes += " " + fraq::scheme_name(s);
    const std::vector<std::pair<const char*, std::string>> lines = {
        {"alpha1", " " + format_double(c.alpha1)},
        {"alpha2", " " + format_double(c.alpha2)},
        {"a", " " + format_double(c.coupling_a)},
        {"grid-m", " " + std::to_string(c.grid_m)},
        {"t-final", " " + format_double(c.t_final)},
        {"ref-tau", " " + format_double(c.ref_tau)},
        {"init", c.initial == fraq::InitialData::poly_sin ? " poly_sin" : " indicator"},
        {"np", " " + std::to_string(c.kernel.be_points)},
        {"np1", " " + std::to_string(c.kernel.sbd_points_1)},
        {"np2", " " + std::to_string(c.kernel.sbd_points_2)},
        {"ns", " " + std::to_string(c.kernel.sbd_head)},
        {"eps-tol", " " + format_double(c.kernel.eps_tol)},
        {"auto-kernel", c.kernel.auto_size ? " 1" : " 0"},
        {"taus", taus},
        {"schemes", schemes},
    };
    std::ofstream meta(std::filesystem::path(dir) / "meta.txt");
    for (const auto& [key, value] : lines) meta << key << " =" << value << "\n";
}

int cmd_weights(const Args& a) {
    const bool sbd = a.sbd_family();
    const double alpha = a.number("alpha", "0.5"), tau = a.number("tau", "1");
    const long n = a.count("n", "10");
    Sink out(a.get("out", ""));
    fraq::write_weights_csv(out.stream(), sbd ? fraq::sbd_weights(alpha, tau, n)
                                              : fraq::be_weights(alpha, tau, n));
    return 0;
}

int cmd_kernel_error(const Args& a) {
    const bool sbd = a.sbd_family();
    const double alpha = a.number("alpha", "0.5"), tau = a.number("tau", "0.001");
    const long n_max = a.count("n-max", "1000");
    fraq::KernelErrorReport rep;
    if (sbd) {
        const long ns = a.count("ns", "0");
        const int head = ns > 0 ? static_cast<int>(ns) : fraq::default_sbd_head(alpha);
        rep = fraq::kernel_error_report(
            fraq::build_sbd_kernel(alpha, tau, static_cast<int>(a.count("np1", "41")),
                                   static_cast<int>(a.count("np2", "41")), head),
            n_max);
    } else {
        rep = fraq::kernel_error_report(
            fraq::build_be_kernel(alpha, tau, static_cast<int>(a.count("np", "64"))), n_max);
    }
    Sink out(a.get("out", ""));
    fraq::write_kernel_error_csv(out.stream(), rep);
    return 0;
}

int cmd_solve(const Args& a) {
    const fraq::ExperimentConfig cfg = a.experiment();
    fraq::ProblemSpec spec;
    spec.alpha1 = cfg.alpha1;
    spec.alpha2 = cfg.alpha2;
    spec.coupling_a = cfg.coupling_a;
    spec.grid_m = cfg.grid_m;
    spec.t_final = cfg.t_final;
    spec.initial = cfg.initial;
    // step count: --n-steps, else t-final / --tau, else 100 steps
    const double tau = a.number("tau", "0"), n_steps = a.number("n-steps", "0");
    spec.n_steps = n_steps > 0 ? std::lround(n_steps)
                               : (tau > 0 ? std::lround(cfg.t_final / tau) : 100L);
    const fraq::Scheme scheme = fraq::scheme_from_name(a.get("scheme", "be"));
    std::set<long> snap_levels;
    for (double t : fraq::parse_fraction_list(a.get("snapshot-times", "")))
        snap_levels.insert(std::lround(t / spec.tau()));
    const std::filesystem::path snap_dir = a.get("out-dir", ".");
    std::function<void(long, const fraq::StateField&)> observer;
    if (!snap_levels.empty()) {
        std::filesystem::create_directories(snap_dir);
        observer = [&](long n, const fraq::StateField& f) {
            if (!snap_levels.count(n)) return;
            std::ofstream snap(snap_dir / ("snapshot_n" + std::to_string(n) + ".csv"));
            fraq::write_snapshot_csv(snap, spec, f);
        };
    }
    const fraq::RunResult rr = fraq::run(spec, scheme, cfg.kernel, observer);
    Sink out(a.get("out", ""));
    fraq::write_snapshot_csv(out.stream(), spec, rr.final_state);
    std::cerr << "loop_seconds=" << fraq::format_double(rr.loop_seconds)
              << " setup_seconds=" << fraq::format_double(rr.setup_seconds) << "\n";
    return 0;
}

int cmd_convergence(const Args& a) {
    const fraq::ExperimentConfig cfg = a.experiment();
    cfg.validate();
    const std::filesystem::path dir = cfg.out_dir;
    std::filesystem::create_directories(dir);
    const std::vector<fraq::ConvergenceReport> reports = fraq::run_convergence(cfg);
    write_meta(cfg.out_dir, cfg);
    for (const fraq::ConvergenceReport& rep : reports) {
        const auto path = dir / ("convergence_" + fraq::scheme_name(rep.scheme) + ".csv");
        std::ofstream csv(path);
        fraq::write_convergence_csv(csv, rep);
        std::cout << path.string() << "\n";
    }
    return 0;
}

int cmd_bench(const Args& a) {
    const fraq::ExperimentConfig cfg = a.experiment();
    std::vector<long> counts;
    for (double v : fraq::parse_fraction_list(a.get("n-list", "100,200,400,800,1600")))
        counts.push_back(std::lround(v));
    Sink out(a.get("out", ""));
    fraq::write_bench_csv(out.stream(), fraq::timing_sweep(cfg, counts));
    return 0;
}

int run(const std::string& config, const std::string& cmd, const Opts& opts) {
    Args a;
    a.cli = opts;
    if (!config.empty()) {
        std::ifstream in(config);
        if (!in) throw std::runtime_error("cannot open config file: " + config);
        a.file = fraq::parse_config_text(in);
    }
    static const std::map<std::string, int (*)(const Args&)> table = {
        {"weights", cmd_weights},         {"kernel-error", cmd_kernel_error},
        {"solve", cmd_solve},             {"convergence", cmd_convergence},
        {"bench", cmd_bench},
    };
    return table.at(cmd)(a);
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
