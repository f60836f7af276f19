// C++ host-API test (run by tests/test_host_api.py on a B200).  Drives the engine only
// through include/pathrec_gpu.hpp — the reference-shaped C++ API — and checks results
// against the C restatement oracle (oracle/_build/liboracle.so, linked as the checker).
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../oracle/pathrec_oracle.h"
#include "pathrec_gpu.hpp"

using namespace pathrec_gpu;

static Scene two_species_cube(int n) {  // tests/helpers.hpp:56-79
    Scene s;
    s.bounds = {{0, 0, 0}, {1, 1, 1}};
    GridGeometry g;
    g.dims = {n, n, n};
    g.voxel_size = {1.0 / n, 1.0 / n, 1.0 / n};
    ParticleSpecies cloud, air;
    cloud.extinction.geom = air.extinction.geom = g;
    for (int v = 0; v < n * n * n; ++v) {
        cloud.extinction.values.push_back(2.0 + 0.5 * (v % 7));
        air.extinction.values.push_back(0.04);
    }
    cloud.albedo = 0.99;
    cloud.phase = PhaseFunction::henyey_greenstein(0.5);
    cloud.unknown = true;
    air.albedo = 0.912;
    air.phase = PhaseFunction::rayleigh();
    s.species = {cloud, air};
    s.light.kind = LightSource::Kind::IsotropicPoint;
    s.light.position = {0.5, 0.5, 0.5};
    Detector d;
    d.position = {0.5, 0.5, 3.0};
    d.direction = {0, 0, -1};
    d.up = {0, 1, 0};
    d.rows = d.cols = 6;
    d.fov = 0.6;
    s.detectors = {d};
    return s;
}

int main() {
    Context ctx(0);
    Scene s = two_species_cube(4);
    RenderOptions ro;
    ro.n_paths = 3000;
    ro.seed = 13;
    ro.keep_paths = true;
    RenderResult rr = render(ctx, s, ro);
    sort_by_size(*rr.store);
    if (!rr.store->sorted_flag) return 2;
    ParamSet t = params_from_scene(s);
    for (size_t v = 0; v < t.beta.size(); ++v) t.beta[v] *= 1.0 + 0.02 * (v % 7);
    ImageSet w = rr.images;
    for (auto& im : w)
        for (size_t p = 0; p < im.data.size(); ++p) im.data[p] = 1.0 + (p % 5);
    EvalOptions eo;
    eo.pixel_weights = &w;
    SparseGradient g = grad_forward(s, *rr.store, t, eo);
    ImageSet img = recycled_render(s, *rr.store, t);
    // oracle on the identical stored path set (PSTR written by the device)
    save_store(*rr.store, "host_api_test.pstr");
    orc_store* os = nullptr;
    if (orc_load_pstr("host_api_test.pstr", &os)) return 3;
    Context::Holder h(s);
    prc_gpu_params pc{t.beta.data(), t.beta.size(), 0.0, 0.0, nullptr};
    std::vector<double> oimg(36), ograd(64), wflat;
    for (auto& im : w) wflat.insert(wflat.end(), im.data.begin(), im.data.end());
    double gk, gg, mc;
    uint64_t cl;
    if (orc_evaluate(&h.desc, os, &pc, PRC_EVAL_NORMALIZE | PRC_EVAL_WANT_GRAD, wflat.data(), oimg.data(),
                     ograd.data(), &gk, &gg, &cl, &mc))
        return 4;
    double imax = 0, gmax = 0, ei = 0, eg = 0;
    for (double x : oimg) imax = std::fmax(imax, std::fabs(x));
    for (double x : ograd) gmax = std::fmax(gmax, std::fabs(x));
    for (size_t p = 0; p < 36; ++p)
        ei = std::fmax(ei, std::fabs(img[0].data[p] - oimg[p]) / std::fmax(std::fabs(oimg[p]), 1e-3 * imax));
    for (int v = 0; v < 64; ++v) eg = std::fmax(eg, std::fabs(g.at(v) - ograd[v]) / gmax);
    // self_normalize (pathstore.cpp:334-359): the mean correction factor and the images
    // divided by it, against the oracle on the same stored paths
    std::vector<double> nimg(36);
    double nmc = 0.0;
    if (orc_evaluate(&h.desc, os, &pc, PRC_EVAL_NORMALIZE | PRC_EVAL_SELF_NORMALIZE, nullptr, nimg.data(), nullptr,
                     &gk, &gg, &cl, &nmc))
        return 7;
    orc_store_free(os);
    std::printf("host api: image rel err %.3e grad rel err %.3e\n", ei, eg);
    if (!(ei <= 1e-5 && eg <= 1e-5)) return 5;
    EvalOptions sn;
    sn.self_normalize = true;
    const EvalResult nr = evaluate_store(s, *rr.store, t, sn);
    double en = 0.0;
    for (size_t p = 0; p < 36; ++p)
        en = std::fmax(en, std::fabs(nr.images[0].data[p] - nimg[p]) / std::fmax(std::fabs(nimg[p]), 1e-3 * imax));
    std::printf("host api: self_normalize mean %.6f (oracle %.6f), image rel err %.3e\n", nr.mean_correction, nmc, en);
    if (!(std::fabs(nr.mean_correction - nmc) <= 1e-6 * nmc && en <= 1e-5)) return 6;
    // reference exception behaviour
    bool threw = false;
    try {
        load_store(ctx, s, "no_such_file.pstr");
    } catch (const std::runtime_error&) {
        threw = true;
    }
    if (!threw) return 7;
    // Algorithm 2 on the device: one stage, resample every 5 iterations
    ImageSet gt = render(ctx, s, RenderOptions{20000, 99, 1, 500, -1, false}).images;
    ReconstructOptions opt;
    opt.adam.alpha = 0.05;
    opt.schedule.recycle_period = 5;
    opt.schedule.max_iterations = 12;
    opt.schedule.stages = {Stage{0, 0, 5000}};
    ParamSet init;
    init.beta.assign(64, 3.0);
    ReconstructResult res = reconstruct(ctx, s, gt, init, opt);
    std::printf("reconstruct: phases %llu loss %.3e -> %.3e\n", (unsigned long long)res.sampling_phases,
                res.history.front().loss, res.history.back().loss);
    // phases = ceil(T / N_r) (acceptance.cpp:470); finite losses; the iterate moved
    bool finite = true, moved = false;
    for (const auto& h : res.history) finite = finite && std::isfinite(h.loss);
    for (double b : res.params.beta) moved = moved || b != 3.0;
    if (res.sampling_phases != 3 || !finite || !moved) return 8;
    // the stage-scheduled loop: a coarse 4x4 stage, then the uploaded resolution
    ReconstructOptions so;
    so.adam.alpha = 0.05;
    so.schedule.recycle_period = 4;
    so.schedule.max_iterations = 12;
    so.schedule.saturation_window = 3;
    so.schedule.saturation_rel_improvement = 1.0;  // saturate as soon as the window is full
    so.schedule.stages = {Stage{4, 4, 5000}, Stage{0, 0, 5000}};
    ReconstructResult sr = reconstruct(ctx, s, gt, init, so);
    std::printf("schedule: phases %llu stages %d..%d\n", (unsigned long long)sr.sampling_phases,
                sr.history.front().stage, sr.history.back().stage);
    if (sr.sampling_phases != 3 || sr.history.size() != 12 || sr.history[3].stage != 0 || sr.history[4].stage != 1)
        return 9;
    // metrics / downsample / carve
    Metrics m = metrics({1.0, 2.0}, {1.0, 4.0});
    if (std::fabs(m.eps - 0.4) > 1e-15 || std::fabs(m.delta - 0.4) > 1e-15) return 10;
    ImageSet small = downsample_images(gt, 2, 2);
    if (small.size() != gt.size() || small[0].data.size() != 4) return 11;
    if (s.detectors.size() >= 2) {
        CarveResult cr = space_carve(ctx, s, gt, 0.0, 1.5);
        if (cr.mask.size() != 64) return 12;
    }
    std::remove("host_api_test.pstr");
    return 0;
}
