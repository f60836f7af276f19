// pathrec_gpu.hpp — C++ host API of the B200 path-recycling engine.
//
// A header-only mirror of the reference's C++ API for the hot path, so a reference
// caller switches by changing the namespace `pathrec::` -> `pathrec_gpu::`:
//
//   reference (/root/reference/proj)                    here
//   Scene, ParticleSpecies, Detector, ... scene.hpp:26-107    same value types
//   ParamSet                         transport.hpp:63-67      ParamSet
//   RenderOptions / render()         transport.hpp:154-174    RenderOptions / render()
//   PathStore / sort_by_size()       pathstore.hpp:14-28      PathStore / sort_by_size()
//   EvalOptions / EvalResult         pathstore.hpp:41-59      EvalOptions / EvalResult
//   evaluate_store()                 pathstore.hpp:64-65      evaluate_store()
//   recycled_render()                pathstore.hpp:68-69      recycled_render()
//   SparseGradient / grad_forward()  gradient.hpp:12-41       SparseGradient / grad_forward()
//   reconstruct()                    inverse.hpp:294-295      reconstruct()
//   save_store() / load_store()      pathstore.hpp:71-72      save_store() / load_store()
//
// Everything forwards through the C ABI (pathrec_gpu.h); errors come back as the
// reference's exception classes (std::invalid_argument for PRC_ERR_CONFIG/INVALID,
// std::runtime_error for IO / NUMERIC / CUDA).  `workers` is ignored: the work runs on
// the context's GPU (one process per GPU; see Context(device, rank, world, nccl_id)).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pathrec_gpu.h"

namespace pathrec_gpu {

inline void check(int rc) {
    if (rc == PRC_OK) return;
    const std::string msg = prc_gpu_last_error();
    if (rc == PRC_ERR_CONFIG || rc == PRC_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// ------------------------------------------------------------------ value types
struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
};

struct GridGeometry {  // grid.hpp:15-65
    int dims[3] = {1, 1, 1};
    Vec3 origin;
    Vec3 voxel_size{1.0, 1.0, 1.0};
    int voxel_count() const { return dims[0] * dims[1] * dims[2]; }
};

struct VoxelGridField {  // grid.hpp:68-80
    GridGeometry geom;
    std::vector<double> values;
};

struct PhaseFunction {  // phase.hpp:17-64
    enum class Kind : uint8_t { HenyeyGreenstein, Rayleigh } kind = Kind::Rayleigh;
    double g = 0.0;
    static PhaseFunction henyey_greenstein(double g) { return {Kind::HenyeyGreenstein, g}; }
    static PhaseFunction rayleigh() { return {Kind::Rayleigh, 0.0}; }
};

struct ParticleSpecies {  // scene.hpp:26-32
    std::string name;
    VoxelGridField extinction;
    double albedo = 1.0;
    PhaseFunction phase = PhaseFunction::rayleigh();
    bool unknown = false;
};

struct Detector {  // scene.hpp:34-54 (frame derived on the device side)
    Vec3 position, direction, up{0.0, 0.0, 1.0};
    int rows = 1, cols = 1;
    double fov = 1.0;
};

struct LightSource {  // scene.hpp:56-61
    enum class Kind : uint8_t { DirectionalSun, IsotropicPoint } kind = Kind::IsotropicPoint;
    Vec3 position, direction;
    double radiance = 1.0;
};

struct Brdf {  // brdf.hpp:36-63
    enum class Kind : uint8_t { Diffuse, Phong } kind = Kind::Diffuse;
    double albedo = 1.0, kappa_s = 0.0, gamma = 0.0;
    static Brdf make_diffuse(double a) { return {Kind::Diffuse, a, 0.0, 0.0}; }
    static Brdf make_phong(double k, double g) { return {Kind::Phong, 1.0, k, g}; }
};

struct Surface {  // scene.hpp:63-86
    enum class Kind : uint8_t { Sphere, Face } kind = Kind::Sphere;
    Vec3 center;
    double radius = 1.0;
    int axis = 2;
    double coord = 0.0, lo[2] = {0.0, 0.0}, hi[2] = {1.0, 1.0}, normal_sign = 1.0;
    Brdf brdf;
    bool target = false;
};

struct Scene {  // scene.hpp:88-107
    Vec3 bounds_min, bounds_max{1.0, 1.0, 1.0};
    std::vector<ParticleSpecies> species;
    std::vector<Surface> surfaces;
    LightSource light;
    std::vector<Detector> detectors;
    int unknown_species() const {
        for (size_t j = 0; j < species.size(); ++j)
            if (species[j].unknown) return (int)j;
        return -1;
    }
    int target_surface() const {
        for (size_t k = 0; k < surfaces.size(); ++k)
            if (surfaces[k].target) return (int)k;
        return -1;
    }
    size_t pixel_count() const {
        size_t n = 0;
        for (const auto& d : detectors) n += (size_t)d.rows * d.cols;
        return n;
    }
};

struct ParamSet {  // transport.hpp:63-67
    std::vector<double> beta;
    double kappa_s = 0.0, gamma = 0.0;
};

inline ParamSet params_from_scene(const Scene& s) {  // transport.cpp:119-128
    ParamSet p;
    const int u = s.unknown_species();
    if (u >= 0) p.beta = s.species[(size_t)u].extinction.values;
    const int t = s.target_surface();
    if (t >= 0 && s.surfaces[(size_t)t].brdf.kind == Brdf::Kind::Phong) {
        p.kappa_s = s.surfaces[(size_t)t].brdf.kappa_s;
        p.gamma = s.surfaces[(size_t)t].brdf.gamma;
    }
    return p;
}

struct Image {  // transport.hpp:85-98
    int rows = 0, cols = 0;
    std::vector<double> data;
};
using ImageSet = std::vector<Image>;

struct SparseGradient {  // gradient.hpp:12-23
    enum class Kind : uint8_t { Tomography, Phong } kind = Kind::Tomography;
    std::map<int, double> entries;
    double at(int v) const {
        auto it = entries.find(v);
        return it == entries.end() ? 0.0 : it->second;
    }
    void add(int v, double value) {
        if (value != 0.0) entries[v] += value;
    }
};

struct RenderOptions {  // transport.hpp:154-161
    uint64_t n_paths = 1;
    uint64_t seed = 0;
    int workers = 1;  // ignored (GPU)
    int max_bounces = 500;
    int max_scatter_events = -1;
    bool keep_paths = false;
};

struct EvalOptions {  // pathstore.hpp:41-50
    int workers = 1;  // ignored (GPU)
    bool normalize = true;
    bool want_grad = false;
    bool legacy_score = false;
    bool self_normalize = false;  // rejected (std::invalid_argument)
    const ImageSet* pixel_weights = nullptr;
    bool per_species = false;     // per-type gradients (config (c) extension)
};

struct EvalResult {  // pathstore.hpp:52-59
    ImageSet images;
    std::vector<double> grad_beta;
    double grad_kappa = 0.0, grad_gamma = 0.0;
    uint64_t clamp_events = 0;
    double mean_correction = 1.0;
};

// ------------------------------------------------------------------ context + store
class Context {
public:
    explicit Context(int device = 0) { check(prc_gpu_ctx_create(device, &ctx_)); }
    // One process per GPU joining an NCCL communicator (paths sharded by rank).
    Context(int device, int rank, int world, const void* nccl_id128) {
        check(prc_gpu_ctx_create_rank(device, rank, world, nccl_id128, &ctx_));
    }
    ~Context() { prc_gpu_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    prc_gpu_ctx* get() const { return ctx_; }

    // Uploads the scene when it differs from the one on the device.
    void use(const Scene& s) {
        Holder h(s);
        const uint64_t key = h.key();
        if (key == scene_key_) return;
        check(prc_gpu_scene_upload(ctx_, &h.desc));
        scene_key_ = key;
    }
    void set_option(const char* key, int64_t value) { check(prc_gpu_ctx_set_option(ctx_, key, value)); }

    // Scene -> prc_scene_desc (borrowed arrays) plus a content key.
    struct Holder {
        prc_scene_desc desc{};
        std::vector<prc_species_desc> sp;
        std::vector<prc_surface_desc> sf;
        std::vector<prc_detector_desc> dt;
        const Scene* s;
        static prc_vec3 v(const Vec3& a) { return {a.x, a.y, a.z}; }
        explicit Holder(const Scene& sc) : s(&sc) {
            desc.bounds_min = v(sc.bounds_min);
            desc.bounds_max = v(sc.bounds_max);
            if (!sc.species.empty()) {
                const GridGeometry& g = sc.species[0].extinction.geom;
                for (int a = 0; a < 3; ++a) desc.dims[a] = g.dims[a];
                desc.grid_origin = v(g.origin);
                desc.voxel_size = v(g.voxel_size);
            }
            for (const auto& q : sc.species)
                sp.push_back({q.extinction.values.data(), q.albedo,
                              q.phase.kind == PhaseFunction::Kind::Rayleigh ? PRC_PHASE_RAYLEIGH : PRC_PHASE_HG,
                              q.phase.g, q.unknown ? 1 : 0});
            for (const auto& q : sc.surfaces) {
                prc_surface_desc d{};
                d.kind = q.kind == Surface::Kind::Face ? PRC_SURF_FACE : PRC_SURF_SPHERE;
                d.center = v(q.center);
                d.radius = q.radius;
                d.axis = q.axis;
                d.coord = q.coord;
                d.lo[0] = q.lo[0];
                d.lo[1] = q.lo[1];
                d.hi[0] = q.hi[0];
                d.hi[1] = q.hi[1];
                d.normal_sign = q.normal_sign;
                d.brdf_kind = q.brdf.kind == Brdf::Kind::Phong ? PRC_BRDF_PHONG : PRC_BRDF_DIFFUSE;
                d.albedo = q.brdf.albedo;
                d.kappa_s = q.brdf.kappa_s;
                d.gamma = q.brdf.gamma;
                d.target = q.target ? 1 : 0;
                sf.push_back(d);
            }
            for (const auto& q : sc.detectors)
                dt.push_back({v(q.position), v(q.direction), v(q.up), q.rows, q.cols, q.fov});
            desc.n_species = (int)sp.size();
            desc.species = sp.empty() ? nullptr : sp.data();
            desc.n_surfaces = (int)sf.size();
            desc.surfaces = sf.empty() ? nullptr : sf.data();
            desc.light.kind = sc.light.kind == LightSource::Kind::DirectionalSun ? PRC_LIGHT_SUN : PRC_LIGHT_POINT;
            desc.light.position = v(sc.light.position);
            desc.light.direction = v(sc.light.direction);
            desc.light.radiance = sc.light.radiance;
            desc.n_detectors = (int)dt.size();
            desc.detectors = dt.empty() ? nullptr : dt.data();
        }
        uint64_t key() const {
            uint64_t h = 1469598103934665603ull;
            auto mix = [&](const void* p, size_t n) {
                const unsigned char* b = static_cast<const unsigned char*>(p);
                for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
            };
            mix(&desc.bounds_min, sizeof(prc_vec3) * 2 + sizeof(int) * 3 + sizeof(prc_vec3) * 2);
            mix(&desc.light, sizeof desc.light);
            for (size_t j = 0; j < sp.size(); ++j) {
                mix(&sp[j].albedo, sizeof(double));
                mix(&sp[j].phase_kind, sizeof(int));
                mix(&sp[j].g, sizeof(double));
                mix(&sp[j].unknown, sizeof(int));
                mix(s->species[j].extinction.values.data(), s->species[j].extinction.values.size() * 8);
            }
            if (!sf.empty()) mix(sf.data(), sf.size() * sizeof(prc_surface_desc));
            if (!dt.empty()) mix(dt.data(), dt.size() * sizeof(prc_detector_desc));
            return h;
        }
    };

private:
    prc_gpu_ctx* ctx_ = nullptr;
    uint64_t scene_key_ = 0;
};

// Default per-process context (LOCAL_RANK or device 0), as the reference's free functions
// have no context argument.
inline Context& default_context() {
    static thread_local std::unique_ptr<Context> c;
    if (!c) {
        const char* lr = std::getenv("LOCAL_RANK");
        c = std::make_unique<Context>(lr ? std::atoi(lr) : 0);
    }
    return *c;
}

struct PathStore {  // pathstore.hpp:14-24: a handle on the device-resident store
    std::shared_ptr<prc_gpu_store> h;
    Context* ctx = nullptr;
    prc_gpu_store_info info() const {
        prc_gpu_store_info i{};
        check(prc_gpu_store_info_get(h.get(), &i));
        return i;
    }
    bool sorted_flag() const { return info().sorted != 0; }
    std::vector<uint64_t> streams() const {  // records[i].stream in storage order
        std::vector<uint64_t> s(info().n_paths);
        check(prc_gpu_store_streams(h.get(), s.data()));
        return s;
    }
};

struct RenderResult {  // transport.hpp:165-169
    ImageSet images;
    uint64_t truncated_paths = 0;
    std::shared_ptr<PathStore> store;
};

namespace detail {
struct ParamsC {
    prc_gpu_params p{};
    explicit ParamsC(const ParamSet& ps) {
        p.beta = ps.beta.empty() ? nullptr : ps.beta.data();
        p.n_beta = ps.beta.size();
        p.kappa_s = ps.kappa_s;
        p.gamma = ps.gamma;
    }
};
inline ImageSet split(const Scene& s, const std::vector<double>& flat) {
    ImageSet out;
    size_t k = 0;
    for (const auto& d : s.detectors) {
        Image im;
        im.rows = d.rows;
        im.cols = d.cols;
        im.data.assign(flat.begin() + (long)k, flat.begin() + (long)(k + (size_t)d.rows * d.cols));
        k += (size_t)d.rows * d.cols;
        out.push_back(std::move(im));
    }
    return out;
}
inline std::vector<double> flatten(const ImageSet& im) {
    std::vector<double> f;
    for (const auto& i : im) f.insert(f.end(), i.data.begin(), i.data.end());
    return f;
}
}  // namespace detail

// transport.cpp:405-454
inline RenderResult render(Context& ctx, const Scene& scene, const RenderOptions& opt) {
    if (opt.n_paths == 0) throw std::invalid_argument("render: n_paths must be >= 1");
    ctx.use(scene);
    prc_gpu_render_opts o{opt.n_paths, opt.seed, opt.max_bounces, opt.max_scatter_events};
    std::vector<double> img(scene.pixel_count());
    uint64_t tr = 0;
    prc_gpu_store* st = nullptr;
    check(prc_gpu_render(ctx.get(), &o, nullptr, img.data(), &tr, opt.keep_paths ? &st : nullptr));
    RenderResult r;
    r.images = detail::split(scene, img);
    r.truncated_paths = tr;
    if (st) {
        r.store = std::make_shared<PathStore>();
        r.store->h = std::shared_ptr<prc_gpu_store>(st, prc_gpu_store_free);
        r.store->ctx = &ctx;
    }
    return r;
}
inline RenderResult render(const Scene& scene, const RenderOptions& opt) {
    return render(default_context(), scene, opt);
}

// pathstore.cpp:261-267
inline void sort_by_size(PathStore& store) { check(prc_gpu_sort_by_size(store.ctx->get(), store.h.get())); }

// pathstore.cpp:315-368
inline EvalResult evaluate_store(const Scene& scene, const PathStore& store, const ParamSet& t,
                                 const EvalOptions& opt) {
    Context& ctx = *store.ctx;
    ctx.use(scene);
    detail::ParamsC pc(t);
    std::vector<double> w;
    if (opt.pixel_weights) w = detail::flatten(*opt.pixel_weights);
    prc_gpu_eval_opts eo{(opt.normalize ? PRC_EVAL_NORMALIZE : 0) | (opt.want_grad ? PRC_EVAL_WANT_GRAD : 0) |
                             (opt.legacy_score ? PRC_EVAL_LEGACY_SCORE : 0) |
                             (opt.self_normalize ? PRC_EVAL_SELF_NORMALIZE : 0) |
                             (opt.per_species ? PRC_EVAL_PER_SPECIES : 0),
                         w.empty() ? nullptr : w.data()};
    std::vector<double> img(scene.pixel_count());
    const size_t V = scene.species.empty() ? 0 : (size_t)scene.species[0].extinction.geom.voxel_count();
    const size_t n_out = opt.per_species ? scene.species.size() : 1;
    const bool grad = opt.want_grad && V && (scene.unknown_species() >= 0 || opt.per_species);
    EvalResult out;
    if (grad) out.grad_beta.assign(n_out * V, 0.0);
    prc_gpu_eval_result r{img.data(), grad ? out.grad_beta.data() : nullptr, 0.0, 0.0, 0, 1.0};
    check(prc_gpu_evaluate(ctx.get(), store.h.get(), &pc.p, &eo, &r));
    out.images = detail::split(scene, img);
    out.grad_kappa = r.grad_kappa;
    out.grad_gamma = r.grad_gamma;
    out.clamp_events = r.clamp_events;
    out.mean_correction = r.mean_correction;
    return out;
}

// pathstore.cpp:370-375
inline ImageSet recycled_render(const Scene& scene, const PathStore& store, const ParamSet& t,
                                int /*workers*/ = 1) {
    return evaluate_store(scene, store, t, EvalOptions{}).images;
}

// gradient.cpp:111-128
inline SparseGradient grad_forward(const Scene& scene, const PathStore& store, const ParamSet& t,
                                   const EvalOptions& opt = {}) {
    EvalOptions e = opt;
    e.want_grad = true;
    const EvalResult r = evaluate_store(scene, store, t, e);
    SparseGradient g;
    if (scene.unknown_species() >= 0) {
        g.kind = SparseGradient::Kind::Tomography;
        for (size_t v = 0; v < r.grad_beta.size(); ++v) g.add((int)v, r.grad_beta[v]);
    } else {
        g.kind = SparseGradient::Kind::Phong;
        g.add(0, r.grad_kappa);
        g.add(1, r.grad_gamma);
    }
    return g;
}

// pathstore.cpp:410-516 (PSTR v1)
inline void save_store(const PathStore& store, const std::string& path) {
    check(prc_gpu_store_export_pstr(store.ctx->get(), store.h.get(), path.c_str()));
}
inline PathStore load_store(Context& ctx, const Scene& scene, const std::string& path) {
    ctx.use(scene);
    prc_gpu_store* st = nullptr;
    check(prc_gpu_store_import_pstr(ctx.get(), path.c_str(), &st));
    PathStore s;
    s.h = std::shared_ptr<prc_gpu_store>(st, prc_gpu_store_free);
    s.ctx = &ctx;
    return s;
}

// inverse.hpp:11-94 (single stage; resample + sort every recycle_period iterations)
struct AdamConfig {
    double alpha = 1e7, eta1 = 0.9, eta2 = 0.999, eps_guard = 1e-8;
    bool project_nonneg = true;
    std::vector<double> step_scale;
};
struct ReconstructOptions {
    AdamConfig adam;
    int recycle_period = 30;
    int max_iterations = 100;
    uint64_t n_paths = 100000;
    uint64_t seed = 0;
    int max_bounces = 500;
};
struct ReconstructResult {
    ParamSet params;
    std::vector<double> loss;
    uint64_t sampling_phases = 0;
};
inline ReconstructResult reconstruct(Context& ctx, const Scene& scene, const ImageSet& gt, const ParamSet& initial,
                                     const ReconstructOptions& opt) {
    ctx.use(scene);
    detail::ParamsC pc(initial);
    std::vector<double> g = detail::flatten(gt);
    prc_gpu_adam_config a{opt.adam.alpha, opt.adam.eta1, opt.adam.eta2, opt.adam.eps_guard,
                          opt.adam.project_nonneg ? 1 : 0,
                          opt.adam.step_scale.empty() ? nullptr : opt.adam.step_scale.data(),
                          (int)opt.adam.step_scale.size()};
    prc_gpu_reconstruct_opts ro{opt.seed, opt.n_paths, opt.max_bounces, opt.recycle_period, opt.max_iterations};
    ReconstructResult r;
    r.loss.assign((size_t)opt.max_iterations, 0.0);
    check(prc_gpu_reconstruct(ctx.get(), &pc.p, g.data(), &a, &ro, r.loss.data(), &r.sampling_phases));
    const size_t V = scene.species.empty() ? 0 : (size_t)scene.species[0].extinction.geom.voxel_count();
    if (scene.unknown_species() >= 0) r.params.beta.assign(V, 0.0);
    check(prc_gpu_opt_params(ctx.get(), r.params.beta.empty() ? nullptr : r.params.beta.data(), &r.params.kappa_s,
                             &r.params.gamma));
    return r;
}

// inverse.hpp:23-76 / inverse.cpp:154-263: the stage-scheduled loop (coarse-to-fine
// stages, saturation, eps/delta against a truth, VGRD + CSV checkpoints)
struct Stage {
    int rows = 0, cols = 0;  // <= 0 keeps the current resolution
    uint64_t n_paths = 0;
};
struct Schedule {
    int recycle_period = 30;
    int max_iterations = 100;
    std::vector<Stage> stages;
    int saturation_window = 20;
    double saturation_rel_improvement = 0.01;
    int checkpoint_every = 0;
};
struct ScheduleOptions {
    AdamConfig adam;
    Schedule schedule;
    uint64_t seed = 0;
    int max_bounces = 500;
    const ParamSet* truth = nullptr;
    std::string checkpoint_dir;
    int length_unit = 0;  // LengthUnit tag of the VGRD checkpoints
};
struct IterationLog {
    int iter = 0;
    double time_s = 0.0, loss = 0.0, eps = 0.0, delta = 0.0;
    int stage = 0;
};
struct ScheduleResult {
    ParamSet params;
    std::vector<IterationLog> history;
    uint64_t sampling_phases = 0, truncated_paths = 0;
};
inline ScheduleResult reconstruct(Context& ctx, const Scene& scene, const ImageSet& gt, const ParamSet& initial,
                                  const ScheduleOptions& opt) {
    if (opt.schedule.stages.empty()) throw std::invalid_argument("reconstruct: schedule needs at least one stage");
    ctx.use(scene);
    detail::ParamsC pc(initial);
    std::vector<double> g = detail::flatten(gt);
    prc_gpu_adam_config a{opt.adam.alpha, opt.adam.eta1, opt.adam.eta2, opt.adam.eps_guard,
                          opt.adam.project_nonneg ? 1 : 0,
                          opt.adam.step_scale.empty() ? nullptr : opt.adam.step_scale.data(),
                          (int)opt.adam.step_scale.size()};
    std::vector<prc_gpu_stage> st;
    for (const auto& x : opt.schedule.stages) st.push_back({x.rows, x.cols, x.n_paths});
    std::unique_ptr<detail::ParamsC> tc;
    if (opt.truth) tc.reset(new detail::ParamsC(*opt.truth));
    prc_gpu_schedule sch{opt.seed, opt.max_bounces, opt.schedule.recycle_period, opt.schedule.max_iterations,
                         st.data(), (int)st.size(), opt.schedule.saturation_window,
                         opt.schedule.saturation_rel_improvement, opt.schedule.checkpoint_every,
                         opt.checkpoint_dir.empty() ? nullptr : opt.checkpoint_dir.c_str(), opt.length_unit,
                         tc ? &tc->p : nullptr};
    std::vector<prc_gpu_iteration_log> h((size_t)std::max(1, opt.schedule.max_iterations));
    ScheduleResult r;
    check(prc_gpu_reconstruct_schedule(ctx.get(), &pc.p, g.data(), &a, &sch, h.data(), &r.sampling_phases,
                                       &r.truncated_paths));
    for (int t = 0; t < opt.schedule.max_iterations; ++t)
        r.history.push_back({h[t].iter, h[t].time_s, h[t].loss, h[t].eps, h[t].delta, h[t].stage});
    const size_t V = scene.species.empty() ? 0 : (size_t)scene.species[0].extinction.geom.voxel_count();
    if (scene.unknown_species() >= 0) r.params.beta.assign(V, 0.0);
    check(prc_gpu_opt_params(ctx.get(), r.params.beta.empty() ? nullptr : r.params.beta.data(), &r.params.kappa_s,
                             &r.params.gamma));
    return r;
}

// inverse.hpp:80-88 / inverse.cpp:69-101 (the occupancy test runs on the device)
struct CarveResult {
    std::vector<uint8_t> mask;
    ParamSet initial;
};
inline CarveResult space_carve(Context& ctx, const Scene& scene, const ImageSet& gt, double threshold_fraction,
                               double fill_extinction) {
    ctx.use(scene);
    std::vector<double> g = detail::flatten(gt);
    const size_t V = scene.species.empty() ? 0 : (size_t)scene.species[0].extinction.geom.voxel_count();
    CarveResult r;
    r.mask.assign(V, 0);
    r.initial.beta.assign(V, 0.0);
    check(prc_gpu_space_carve(ctx.get(), g.data(), threshold_fraction, fill_extinction, r.mask.data(),
                              r.initial.beta.data()));
    return r;
}

// inverse.hpp:97-106
struct Metrics {
    double eps = 0.0, delta = 0.0;
};
inline Metrics metrics(const std::vector<double>& estimate, const std::vector<double>& truth) {
    if (estimate.size() != truth.size()) throw std::invalid_argument("metrics: dimension mismatch");
    Metrics m;
    check(prc_gpu_metrics(estimate.data(), truth.data(), truth.size(), &m.eps, &m.delta));
    return m;
}
inline ImageSet downsample_images(const ImageSet& images, int rows, int cols) {
    std::vector<int> r, c;
    for (const auto& im : images) {
        r.push_back(im.rows);
        c.push_back(im.cols);
    }
    std::vector<double> in = detail::flatten(images), out(images.size() * (size_t)rows * cols);
    check(prc_gpu_downsample_images((int)images.size(), r.data(), c.data(), in.data(), rows, cols, out.data()));
    ImageSet o;
    for (size_t k = 0; k < images.size(); ++k) {
        Image im;
        im.rows = rows;
        im.cols = cols;
        im.data.assign(out.begin() + (long)(k * rows * cols), out.begin() + (long)((k + 1) * rows * cols));
        o.push_back(std::move(im));
    }
    return o;
}

}  // namespace pathrec_gpu
