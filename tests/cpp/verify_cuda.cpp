// Drives the reference's verification harness (proj/include/fdwave/verify.hpp)
// unmodified.  Built twice by oracle/Makefile:
//   verify_cuda -- -I include first, so fdwave/kernel.hpp is the drop-in and
//                  every Solver<T> in verify.hpp runs on the GPU;
//   verify_ref  -- the reference headers alone (CPU, OpenMP).
// Prints one JSON object per study; tests/test_gpu_verify.py compares the two
// and checks the reference's own acceptance gates (tools/main.cpp:123).
//
// usage: verify_{cuda,ref} [analytical] [mms] [temporal] [spatial] [quick]
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fdwave/verify.hpp"

namespace {

void print_report(const fdwave::ConvergenceReport& r) {
    std::printf("{\"study\": \"%s\", \"nominal\": %.17g, \"slope\": %.17g, \"seconds\": %.6f, \"points\": [",
                r.label.c_str(), r.nominal, r.slope, r.seconds);
    for (std::size_t i = 0; i < r.points.size(); ++i)
        std::printf("%s[%.17g, %.17g]", i ? ", " : "", r.points[i].resolution, r.points[i].error);
    std::printf("]}\n");
}

bool want(int argc, char** argv, const char* name) {
    if (argc <= 1) return true;
    for (int i = 1; i < argc; ++i)
        if (!std::strcmp(argv[i], name)) return true;
    return false;
}

}  // namespace

int main(int argc, char** argv) {
    bool quick = false;
    int n_named = 0;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "quick"))
            quick = true;
        else
            ++n_named;
    }
    const bool all = n_named == 0;
    try {
        if (all || want(argc, argv, "analytical")) {
            const fdwave::AnalyticalCasePresets p;  // the tools/main.cpp:123 gate case
            const auto r = fdwave::analytical_agreement_case(p);
            std::printf("{\"study\": \"analytical\", \"max_abs_diff\": %.17g, \"reference_peak\": %.17g, "
                        "\"relative_error\": %.17g, \"seconds\": %.6f}\n",
                        r.max_abs_diff, r.reference_peak, r.relative_error, r.seconds);
        }
        if (all || want(argc, argv, "mms")) {
            fdwave::MmsStudyPresets p;
            if (quick) {
                p.tf = 0.05;
                p.spacings = {8.0, 4.0};
            }
            print_report(fdwave::mms_convergence_study(p));
        }
        if (all || want(argc, argv, "temporal")) {
            fdwave::TemporalStudyPresets p;
            if (quick) p.tf = 0.1;
            print_report(fdwave::temporal_convergence_study(p));
        }
        if (all || want(argc, argv, "spatial")) {
            fdwave::SpatialStudyPresets p;
            if (quick) {
                p.tf = 0.1;
                p.spacings = {2.0, 1.0};
                p.reference_h = 0.5;
            }
            const std::vector<int> orders{2, 4, 8};
            for (const auto& r : fdwave::spatial_convergence_study(orders, p)) print_report(r);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "verify: %s\n", e.what());
        return 1;
    }
    return 0;
}
