// planner.cpp -- probe-depth planner of the sharded search (the reference's
// `equivalence` module; bound from PAPER.md:883-898).
//
// Sequential search looks at Phi entries on each side of the query key.  With
// the database dealt over `shards` uniformly at random, the number of those
// Phi entries that land on one shard is Binomial(Phi, 1/shards); a shard that
// only looks phi entries deep on a side misses some iff that count exceeds
// phi.  The bound combines the union bound over the shards of one side with
// the two sides: 1 - max(0, 1 - Phi * P[Bin > phi])^2.
#include <cmath>
#include <cstdint>

#include "../../include/hcg.h"

extern "C" {

// P[Bin(trials, p) > phi] with log-gamma terms and compensated summation
// (SPEC.md:286-292 design decision "log-gamma-based binomial terms").
double hcg_binomial_tail(uint32_t trials, double p, uint32_t phi) {
    if (!(p > 0.0 && p < 1.0)) return std::nan("");
    if (phi >= trials) return 0.0;
    const double lp = std::log(p), lq = std::log1p(-p);
    const double lgn = std::lgamma(double(trials) + 1.0);
    double sum = 0.0, comp = 0.0;
    for (uint32_t k = phi + 1; k <= trials; ++k) {
        const double lt = lgn - std::lgamma(double(k) + 1.0) - std::lgamma(double(trials - k) + 1.0) + k * lp +
                          double(trials - k) * lq;
        const double term = std::exp(lt);
        const double y = term - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum < 0.0 ? 0.0 : (sum > 1.0 ? 1.0 : sum);
}

double hcg_miss_bound(uint32_t Phi, uint32_t shards, uint32_t phi) {
    if (shards < 1 || Phi < 1) return std::nan("");
    double tail;
    if (shards == 1) tail = phi >= Phi ? 0.0 : 1.0;  // Bin(Phi, 1) == Phi
    else tail = hcg_binomial_tail(Phi, 1.0 / double(shards), phi);
    const double inner = 1.0 - double(Phi) * tail;
    const double keep = inner > 0.0 ? inner : 0.0;
    double b = 1.0 - keep * keep;
    return b < 0.0 ? 0.0 : (b > 1.0 ? 1.0 : b);
}

uint32_t hcg_plan_depth(uint32_t Phi, uint32_t shards, double target) {
    if (Phi < 1 || shards < 1) return Phi;
    for (uint32_t phi = 0; phi < Phi; ++phi)
        if (hcg_miss_bound(Phi, shards, phi) <= target) return phi;
    return Phi;
}

}  // extern "C"
