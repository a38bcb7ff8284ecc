// Compile-only check that the wrapper accepts the reference's own types:
// hc::Dataset / hc::FeatureVector (proj/include/hypercurves/vecio.hpp).
#include "hypercurves/vecio.hpp"
#include "hypercurves_b200.hpp"

hcb::NeighborList drop_in(const hc::Dataset& ds, const hc::FeatureVector& q) {
    hcb::MulticurvesIndex idx(ds, hcb::default_scheme(ds.dims, 8, 16, hcb::CurveKind::Hilbert, 0),
                              hcb::View::lifted());
    return idx.search(q, hcb::SearchParams{10, 350});
}

// The default view: the reference's float components as they are.
hcb::NeighborList drop_in_floats(const hc::Dataset& ds, const hc::FeatureVector& q) {
    hcb::MulticurvesIndex idx(ds, hcb::default_scheme(ds.dims, 8, 16, hcb::CurveKind::Hilbert, 0));
    return idx.search(q, hcb::SearchParams{10, 350});
}
