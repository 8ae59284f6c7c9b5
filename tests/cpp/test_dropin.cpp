// Drop-in check: this program is written against the REFERENCE header
// volpot/summation.hpp and links integration/volpot_summation_b200.cpp in
// place of proj/src/summation.cpp (kernel.cpp/common.cpp from the reference
// tree).  Same I/O protocol as test_cpp_api.cpp; also runs direct_sum with
// the reference's coincidence exception.
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>

#include "volpot/kernel.hpp"
#include "volpot/summation.hpp"

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::ifstream in(argv[1], std::ios::binary);
    int64_t ns = 0, nt = 0;
    in.read(reinterpret_cast<char*>(&ns), 8);
    in.read(reinterpret_cast<char*>(&nt), 8);
    std::vector<volpot::Vec2> src(static_cast<size_t>(ns)), tgt(static_cast<size_t>(nt));
    std::vector<double> q(static_cast<size_t>(ns));
    in.read(reinterpret_cast<char*>(src.data()), 16 * ns);
    in.read(reinterpret_cast<char*>(q.data()), 8 * ns);
    in.read(reinterpret_cast<char*>(tgt.data()), 16 * nt);
    const volpot::Kernel k = volpot::make_kernel(volpot::KernelFamily::Laplace);
    volpot::SummationPlan plan(k, src, tgt, 1e-12);
    const std::vector<double> a = plan.apply(q);
    const std::vector<double> b = volpot::accelerated_sum(k, volpot::SourceSet{src, q}, tgt);
    int errors = 0;
    try {
        plan.apply(std::vector<double>(3, 1.0));
    } catch (const std::invalid_argument& e) {
        errors += std::string(e.what()) ==
                  "SummationPlan::apply: charge count 3 does not match source count " + std::to_string(ns);
    }
    try {
        volpot::direct_sum(k, volpot::SourceSet{{{0, 0}, {1, 1}}, {1.0, 2.0}}, {{2, 2}, {1, 1}});
    } catch (const std::invalid_argument& e) {
        errors += std::string(e.what()) == "direct_sum: target 1 coincides with source 1";
    }
    std::ofstream out(argv[2], std::ios::binary);
    out.write(reinterpret_cast<const char*>(a.data()), 8 * nt);
    out.write(reinterpret_cast<const char*>(b.data()), 8 * nt);
    out.write(reinterpret_cast<const char*>(a.data()), 8 * nt);
    std::printf("{\"levels\": %d, \"order\": %d, \"errors_ok\": %d}\n", plan.levels(),
                plan.expansion_order(), errors);
    return errors == 2 ? 0 : 1;
}
