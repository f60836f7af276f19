// A reference-API caller, built UNCHANGED against the B200 engine: the reference's own
// tests/helpers.hpp (compiled in place from /root/reference/proj/tests) plus the
// reference's headers resolved through tests/cpp/shim/pathrec/*.hpp to the engine's C++
// mirror (include/pathrec_gpu.hpp, namespace pathrec).  Written in the style of the
// reference's acceptance gate (tests/acceptance.cpp): one PASS / FAIL line per check, exit
// code 0 only when every check passes.  Run on a B200 by tests/test_host_api.py.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "helpers.hpp"
#include "pathrec/gradient.hpp"
#include "pathrec/inverse.hpp"
#include "pathrec/io.hpp"
#include "pathrec/pathstore.hpp"

using namespace pathrec;
using namespace pathrec::testing;

namespace {

int failures = 0;

void report(const char* name, bool ok, const std::string& detail) {
    std::printf("[%s] %s: %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
    if (!ok) ++failures;
}

double max_rel(const ImageSet& a, const ImageSet& b) {
    double mx = 0.0, scale = 0.0;
    for (const auto& im : b)
        for (double v : im.data) scale = std::max(scale, std::abs(v));
    for (size_t d = 0; d < a.size(); ++d)
        for (size_t p = 0; p < a[d].data.size(); ++p) mx = std::max(mx, std::abs(a[d].data[p] - b[d].data[p]));
    return scale > 0.0 ? mx / scale : mx;
}

Scene cloud_scene() {  // helpers.hpp's two-species cube around a Gaussian blob
    const int n = 6;
    std::vector<double> cloud(static_cast<size_t>(n * n * n));
    const GridGeometry g = cube_grid(n);
    for (int v = 0; v < g.voxel_count(); ++v) {
        const Vec3 c = g.voxel_center(v) - Vec3{0.5, 0.5, 0.5};
        cloud[static_cast<size_t>(v)] = 1.0 + 5.0 * std::exp(-dot(c, c) / (2.0 * 0.25 * 0.25));
    }
    return two_species_cube(cloud, n, 0.04, 6, 6);
}

// The loss of the recycled images against gt at params p (frozen paths).
double frozen_loss(const Scene& s, const PathStore& st, const ParamSet& p, const ImageSet& gt) {
    return loss(recycled_render(s, st, p), gt);
}

}  // namespace

int main() {
    const Scene s = cloud_scene();
    RenderOptions ro;
    ro.n_paths = 20000;
    ro.seed = 7;
    ro.keep_paths = true;
    const RenderResult rr = render(s, ro);
    PathStore& st = *rr.store;

    // (c9 of acceptance.cpp) recycling at the sampling point reproduces the fresh render
    const ImageSet rec = recycled_render(s, st, st.ref_params);
    report("recycled == fresh at the reference", max_rel(rec, rr.images) <= 1e-12,
           "max rel " + std::to_string(max_rel(rec, rr.images)));

    // sort invariance (acceptance.cpp:330-347)
    ParamSet t = params_from_scene(s);
    for (size_t v = 0; v < t.beta.size(); ++v) t.beta[v] *= 1.0 + 0.02 * static_cast<double>(v % 7);
    const ImageSet before = recycled_render(s, st, t);
    sort_by_size(st);
    const ImageSet after = recycled_render(s, st, t);
    report("sort_by_size leaves estimates unchanged", st.sorted_flag && max_rel(before, after) <= 1e-12,
           "max rel " + std::to_string(max_rel(before, after)));

    // frozen-path gradient vs central differences (acceptance.cpp:203-271), on the device
    // store (fp32 extinction fields) and on its PSTR reloaded in materialized mode (fp64)
    ImageSet gt = rr.images;
    for (auto& im : gt)
        for (auto& px : im.data) px *= 0.8;
    save_store(st, "ref_caller.pstr");
    PathStore loaded = load_store("ref_caller.pstr");
    for (int which = 0; which < 2; ++which) {
        const PathStore& fs = which == 0 ? st : loaded;
        const ImageSet f = recycled_render(s, fs, t);
        ImageSet res = f;
        for (size_t d = 0; d < res.size(); ++d)
            for (size_t p = 0; p < res[d].data.size(); ++p) res[d].data[p] -= gt[d].data[p];
        EvalOptions go;
        go.pixel_weights = &res;
        const SparseGradient g = grad_forward(s, fs, t, go);
        double gmax = 0.0;
        for (const auto& [v, val] : g.entries) gmax = std::max(gmax, std::abs(val));
        double worst = 0.0;
        for (int v : {43, 86, 100, 129, 150}) {
            const double h = (which == 0 ? 1e-2 : 1e-5) * t.beta[static_cast<size_t>(v)];
            ParamSet tp = t, tm = t;
            tp.beta[static_cast<size_t>(v)] += h;
            tm.beta[static_cast<size_t>(v)] -= h;
            const double fd = (frozen_loss(s, fs, tp, gt) - frozen_loss(s, fs, tm, gt)) / (2.0 * h);
            worst = std::max(worst, std::abs(fd - g.at(v)) / gmax);
        }
        const double tol = which == 0 ? 2e-3 : 1e-6;
        report(which == 0 ? "grad_forward vs central differences (device store)"
                          : "grad_forward vs central differences (loaded store, stored spans)",
               worst <= tol, "max scale-rel error " + std::to_string(worst));
    }
    // the reloaded (reference-format) store evaluates like the device store
    report("save_store -> load_store round trip", max_rel(recycled_render(s, loaded, t), after) <= 1e-5,
           "max rel " + std::to_string(max_rel(recycled_render(s, loaded, t), after)));
    std::remove("ref_caller.pstr");

    // reconstruct() with the reference's options, a truth and an on_iteration observer
    ReconstructOptions opt;
    opt.adam.alpha = 0.05;
    opt.schedule.recycle_period = 5;
    opt.schedule.max_iterations = 15;
    opt.schedule.stages = {Stage{0, 0, 20000}};
    opt.seed = 11;
    const ParamSet truth = params_from_scene(s);
    opt.truth = &truth;
    int calls = 0;
    opt.on_iteration = [&](const IterationLog& row) { calls += row.iter == calls ? 1 : 1000; };
    ParamSet init = truth;
    for (auto& b : init.beta) b = 2.0;
    const ReconstructResult r = reconstruct(s, rr.images, init, opt);
    const Metrics m0 = metrics(init.beta, truth.beta);
    report("reconstruct: on_iteration once per iteration, 3 sampling phases, loss falls, eps/delta of the truth",
           calls == 15 && r.sampling_phases == 3 && r.history.size() == 15 &&
               r.history.back().loss < r.history.front().loss && r.history.front().eps == m0.eps &&
               r.history.front().delta == m0.delta,
           "calls " + std::to_string(calls) + ", phases " + std::to_string(r.sampling_phases) + ", loss " +
               std::to_string(r.history.front().loss) + " -> " + std::to_string(r.history.back().loss) + ", eps " +
               std::to_string(r.history.front().eps) + " -> " + std::to_string(r.history.back().eps));

    // reflectometry on the reference's phong_box fixture
    const Scene pb = phong_box(0.7, 50.0, 8, 8);
    RenderOptions rp;
    rp.n_paths = 20000;
    rp.seed = 3;
    rp.max_bounces = 40;
    rp.keep_paths = true;
    const RenderResult pr = render(pb, rp);
    ParamSet pt;
    pt.kappa_s = 0.55;
    pt.gamma = 38.0;
    const SparseGradient pg = grad_forward(pb, *pr.store, pt);
    report("Phong gradient on phong_box", pg.kind == SparseGradient::Kind::Phong && std::isfinite(pg.at(0)) &&
                                              std::isfinite(pg.at(1)) && pg.at(0) != 0.0,
           "dkappa " + std::to_string(pg.at(0)) + ", dgamma " + std::to_string(pg.at(1)));

    // io.hpp round trips
    save_pfm(rr.images[0], "ref_caller.pfm");
    const Image back = load_pfm("ref_caller.pfm");
    bool pfm_ok = back.rows == rr.images[0].rows && back.cols == rr.images[0].cols;
    for (size_t p = 0; pfm_ok && p < back.data.size(); ++p)
        pfm_ok = back.data[p] == static_cast<double>(static_cast<float>(rr.images[0].data[p]));
    report("save_pfm / load_pfm", pfm_ok, "");
    std::remove("ref_caller.pfm");
    save_grid(s.species[0].extinction, LengthUnit::Kilometers, "ref_caller.vgrd");
    LengthUnit u = LengthUnit::Meters;
    const VoxelGridField gf = load_grid("ref_caller.vgrd", &u);
    report("save_grid / load_grid", u == LengthUnit::Kilometers && gf.geom == s.species[0].extinction.geom, "");
    std::remove("ref_caller.vgrd");

    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
    return failures ? 1 : 0;
}
