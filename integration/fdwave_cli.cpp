// fdwave command line (run / verify / bench / coeff) over the reference's own
// caller code -- config.hpp, runner.hpp, io.hpp, verify.hpp, bench.hpp -- with
// the subcommands and flags of the reference CLI (proj/tools/main.cpp:206-260)
// and its exit codes (0 ok, 1 usage/config/io, 2 numerical; main.cpp:25-27).
//
// integration/Makefile builds this file twice:
//   _build/fdwave_cuda  -I include first: fdwave/kernel.hpp is the B200 drop-in,
//                       so every Solver<T> the callers build runs on the GPU;
//   _build/fdwave_cpu   the reference headers alone (OpenMP CPU Solver).
// The reference CLI itself needs CLI11, which is not vendored;
// the argument parsing here is a small hand-rolled equivalent.
//
// Caller-side addition: a config may say
// "backend": {"type": "cuda", ...}.  parse_run_config (config.hpp:262-276)
// only knows serial|parallel, so "cuda" is mapped to "parallel" before
// parsing; the drop-in Solver ignores the backend (one GPU code path).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "fdwave/bench.hpp"
#include "fdwave/config.hpp"
#include "fdwave/kernel.hpp"
#include "fdwave/runner.hpp"
#include "fdwave/stencil.hpp"
#include "fdwave/verify.hpp"

namespace {

enum Exit { kOk = 0, kUsage = 1, kNumerical = 2 };

// --name value / --flag / positionals
struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string get(const std::string& k, const std::string& dflt) const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
};

bool parse_args(int argc, char** argv, const std::vector<std::string>& flags, Args& a) {
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            const auto eq = s.find('=');
            if (eq != std::string::npos) {
                a.opt[s.substr(2, eq - 2)] = s.substr(eq + 1);
                continue;
            }
            const std::string key = s.substr(2);
            bool is_flag = false;
            for (const auto& f : flags) is_flag |= f == key;
            if (is_flag) {
                a.opt[key] = "1";
            } else {
                if (i + 1 >= argc) {
                    std::fprintf(stderr, "error: --%s needs a value\n", key.c_str());
                    return false;
                }
                a.opt[key] = argv[++i];
            }
        } else {
            a.pos.push_back(s);
        }
    }
    return true;
}

std::vector<long long> csv_ints(const std::string& s) {
    std::vector<long long> out;
    std::string tok;
    std::istringstream in(s);
    while (std::getline(in, tok, ','))
        if (!tok.empty()) out.push_back(std::stoll(tok));
    return out;
}

int do_run(const Args& a) {
    const std::string cfg_path = a.get("config", "");
    if (cfg_path.empty()) {
        std::fprintf(stderr, "error: run needs --config\n");
        return kUsage;
    }
    const std::filesystem::path out = a.get("out", "out");
    nlohmann::json j;
    try {
        std::ifstream in(cfg_path);
        if (!in) {
            std::fprintf(stderr, "error: cannot open config %s\n", cfg_path.c_str());
            return kUsage;
        }
        j = nlohmann::json::parse(in);
    } catch (const nlohmann::json::parse_error& e) {
        std::fprintf(stderr, "error: config is not valid JSON: %s\n", e.what());
        return kUsage;
    }
    if (j.contains("backend") && j["backend"].is_object() && j["backend"].value("type", "") == "cuda")
        j["backend"]["type"] = "parallel";
    fdwave::RunConfig cfg;
    try {
        cfg = fdwave::parse_run_config(j);
    } catch (const fdwave::config_error& e) {
        std::fprintf(stderr, "config error at %s\n", e.what());
        return kUsage;
    }
    if (a.has("backend")) {
        const std::string b = a.get("backend", "");
        if (b == "serial")
            cfg.backend = fdwave::Backend::Serial;
        else if (b == "parallel" || b == "cuda")
            cfg.backend = fdwave::Backend::Parallel;
        else {
            std::fprintf(stderr, "error: unknown backend %s\n", b.c_str());
            return kUsage;
        }
    }
    if (a.has("workers")) cfg.workers = std::stoi(a.get("workers", "0"));
    try {
        const auto m = fdwave::run_simulation(cfg, out, a.has("verbose"));
        std::printf("run complete: %zu steps, dt %.6e s, kernel %.3f s\n", m["n_steps"].get<std::size_t>(),
                    m["dt"].get<double>(), m["kernel_seconds"].get<double>());
        std::printf("artifacts in %s\n", out.string().c_str());
    } catch (const fdwave::instability_error& e) {
        std::fprintf(stderr, "numerical failure: %s\n", e.what());
        return kNumerical;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kUsage;
    }
    return kOk;
}

// One line per report; gates as in the reference's verify command
// (main.cpp:104-150): temporal slope within 0.2 of 2, spatial within 0.5 of
// the order for orders <= 8, analytical relative error <= 1 %, MMS error
// ratios >= 1.5 per halving.
bool report_line(const fdwave::ConvergenceReport& r, bool gated, double tol) {
    const bool pass = std::fabs(r.slope - r.nominal) <= tol;
    std::printf("%-24s slope %6.3f (nominal %.0f)  [%s]  %.1fs\n", r.label.c_str(), r.slope, r.nominal,
                gated ? (pass ? "pass" : "FAIL") : "info", r.seconds);
    return !gated || pass;
}

int do_verify(const Args& a) {
    if (a.pos.empty()) {
        std::fprintf(stderr, "error: verify needs a suite (temporal|spatial|analytical|mms)\n");
        return kUsage;
    }
    const std::string suite = a.pos[0];
    std::vector<fdwave::ConvergenceReport> reports;
    bool ok = true;
    try {
        if (suite == "analytical") {
            const auto r = fdwave::analytical_agreement_case();
            const bool pass = r.relative_error <= 0.01;
            std::printf("analytical agreement    max|diff|/peak %.5f  [%s]  %.1fs\n", r.relative_error,
                        pass ? "pass" : "FAIL", r.seconds);
            ok = pass;
        } else if (suite == "temporal") {
            reports.push_back(fdwave::temporal_convergence_study());
            ok = report_line(reports.back(), true, 0.2);
        } else if (suite == "spatial") {
            std::vector<int> orders;
            for (long long o : csv_ints(a.get("orders", "2,4,6,8"))) orders.push_back((int)o);
            for (auto& r : fdwave::spatial_convergence_study(orders)) {
                ok &= report_line(r, r.nominal <= 8.0, 0.5);
                reports.push_back(std::move(r));
            }
        } else if (suite == "mms") {
            reports.push_back(fdwave::mms_convergence_study());
            const auto& r = reports.back();
            report_line(r, false, 0.5);
            bool halving = true;
            for (std::size_t i = 1; i < r.points.size(); ++i)
                halving &= r.points[i - 1].error / r.points[i].error >= 1.5;
            std::printf("%-24s error ratios per halving >= 1.5  [%s]\n", r.label.c_str(), halving ? "pass" : "FAIL");
            ok = halving;
        } else {
            std::fprintf(stderr, "error: unknown suite \"%s\" (temporal|spatial|analytical|mms)\n", suite.c_str());
            return kUsage;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "verification failed to run: %s\n", e.what());
        return kNumerical;
    }
    const std::string csv = a.get("emit-csv", "");
    if (!csv.empty() && !reports.empty()) {
        std::ofstream f(csv);
        f << "study,resolution,error\n" << std::setprecision(12);
        for (const auto& r : reports)
            for (const auto& p : r.points) f << r.label << "," << p.resolution << "," << p.error << "\n";
    }
    return ok ? kOk : kNumerical;
}

int do_bench(const Args& a) {
    fdwave::BenchOptions o;
    o.shape.clear();
    for (long long n : csv_ints(a.get("grid", "128,128,128"))) o.shape.push_back((std::size_t)n);
    if (o.shape.size() != 2 && o.shape.size() != 3) {
        std::fprintf(stderr, "error: --grid needs 2 or 3 comma-separated extents\n");
        return kUsage;
    }
    if (a.has("orders")) {
        o.orders.clear();
        for (long long v : csv_ints(a.get("orders", ""))) o.orders.push_back((int)v);
    }
    o.steps = std::stoul(a.get("steps", "100"));
    o.repetitions = std::stoul(a.get("repetitions", "10"));
    o.workers = std::stoi(a.get("workers", "0"));
    const std::string backends = a.get("backends", "serial,parallel");
    o.run_serial = backends.find("serial") != std::string::npos;
    o.run_parallel = backends.find("parallel") != std::string::npos || backends.find("cuda") != std::string::npos;
    if (!o.run_serial && !o.run_parallel) {
        std::fprintf(stderr, "error: --backends must mention serial and/or parallel\n");
        return kUsage;
    }
    try {
        if (o.run_serial && o.run_parallel) {
            const double rel = fdwave::backend_equivalence_probe(o);
            std::printf("backend equivalence probe: max rel diff %.3e  [%s]\n", rel, rel <= 1e-12 ? "pass" : "FAIL");
            if (rel > 1e-12) return kNumerical;
        }
        const auto rows = fdwave::run_bench(o);
        std::printf("%s", fdwave::bench_markdown(rows).c_str());
        const std::string csv = a.get("emit-csv", "");
        if (!csv.empty()) std::ofstream(csv) << fdwave::bench_csv(rows);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kUsage;
    }
    return kOk;
}

int do_coeff(const Args& a) {
    try {
        const int order = std::stoi(a.get("order", "0"));
        const auto c = a.has("first") ? fdwave::first_derivative_coefficients(order)
                                      : fdwave::second_derivative_coefficients(order);
        for (double v : c) std::printf("%.17g\n", v);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kUsage;
    }
    return kOk;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s run|verify|bench|coeff [options]\n", argv[0]);
        return kUsage;
    }
    const std::string cmd = argv[1];
    Args a;
    if (!parse_args(argc, argv, {"verbose", "first"}, a)) return kUsage;
    if (cmd == "run") return do_run(a);
    if (cmd == "verify") return do_verify(a);
    if (cmd == "bench") return do_bench(a);
    if (cmd == "coeff") return do_coeff(a);
    std::fprintf(stderr, "error: unknown subcommand %s\n", cmd.c_str());
    return kUsage;
}
