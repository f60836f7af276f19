// pathrec_gpu.hpp — C++ host API of the B200 path-recycling engine.
//
// A header-only mirror of the reference's C++ API for the hot path (reference
// include/pathrec/*.hpp), source-compatible with it: the value types have the
// reference's members and helpers, and the free functions its signatures.  A caller of
// the reference switches by building against this header in place of the reference's
// headers (tests/cpp/shim/pathrec/*.hpp do exactly that: they define
// PATHREC_GPU_NAMESPACE as `pathrec` and include this file) and linking
// libpathrec_gpu.so.  The reference's tests/helpers.hpp compiles unchanged that way.
//
//   reference (/root/reference/proj/include/pathrec)      here
//   Vec3, Frame                   vec3.hpp:7-57           Vec3 (Frame is trace-internal)
//   GridGeometry, VoxelGridField  grid.hpp:15-80          same
//   PhaseFunction                 phase.hpp:17-64         same (eval; sampling is on the device)
//   PhongBrdf, DiffuseBrdf, Brdf  brdf.hpp:12-63          same
//   Aabb, ParticleSpecies, Detector, LightSource, Sphere, BoxFace, Surface, Scene
//                                 scene.hpp:15-107        same
//   ParamSet, Image, RenderOptions, RenderResult, render()   transport.hpp:63-174
//   PathStore, sort_by_size(), EvalOptions, EvalResult, evaluate_store(),
//   recycled_render(), save_store(), load_store()           pathstore.hpp:14-72
//   SparseGradient, grad_forward()                          gradient.hpp:12-41
//   AdamConfig, Stage, Schedule, OptState, IterationLog, ReconstructResult,
//   ReconstructOptions, loss(), adam_step(), CarveResult, space_carve(), reconstruct(),
//   Metrics, metrics(), downsample_images()                  inverse.hpp:11-106
//   load_grid/save_grid, save_pfm/load_pfm, save_pgm_preview, save_csv, load_scene
//                                 io.hpp:10-41            same (through the C ABI)
//
// What differs, by design:
// - The compute runs on a GPU context.  The reference's free functions (no context
//   argument) use a per-thread default Context on CUDA device $LOCAL_RANK (else 0);
//   every function also has an overload taking a Context& first.  `workers` is ignored.
// - PathStore is a handle on a device-resident store: `records` / `by_stream` are not
//   materialised (use save_store for the PSTR file); sorted_flag, generation, seed and
//   ref_params are kept as in the reference.  load_store(path) keeps the file's own spans
//   (PRC_IMPORT_MATERIALIZE), so evaluation reads them as the reference does.
// - Scene::finalize() normalises exactly as scene.cpp does; a finalized scene crosses the
//   ABI with prc_scene_desc::finalized set so the engine does not normalise twice.
// Errors come back as the reference's exception classes (std::invalid_argument for
// PRC_ERR_CONFIG / INVALID, std::runtime_error for IO / NUMERIC / CUDA).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pathrec.h"
#include "pathrec_gpu.h"

#ifndef PATHREC_GPU_NAMESPACE
#define PATHREC_GPU_NAMESPACE pathrec_gpu
#endif

namespace PATHREC_GPU_NAMESPACE {

inline void check(int rc, const char* (*last)() = prc_gpu_last_error) {
    if (rc == PRC_OK) return;
    const std::string msg = last();
    if (rc == PRC_ERR_CONFIG || rc == PRC_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline void check_coarse(int rc) { check(rc, prc_last_error); }

// ------------------------------------------------------------------ vec3.hpp
struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
    constexpr Vec3() = default;
    constexpr Vec3(double x_, double y_, double z_) : x(x_), y(y_), z(z_) {}
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
    Vec3 operator/(double s) const { return {x / s, y / s, z / s}; }
    Vec3 operator-() const { return {-x, -y, -z}; }
    Vec3& operator+=(const Vec3& o) {
        x += o.x;
        y += o.y;
        z += o.z;
        return *this;
    }
    bool operator==(const Vec3&) const = default;
    double norm() const { return std::sqrt(x * x + y * y + z * z); }
    Vec3 normalized() const { return *this / norm(); }
};
inline Vec3 operator*(double s, const Vec3& v) { return v * s; }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const Vec3& v) { return std::sqrt(dot(v, v)); }
inline Vec3 normalized(const Vec3& v) { return v / norm(v); }

// ------------------------------------------------------------------ grid.hpp
enum class LengthUnit : uint8_t { Meters = 0, Kilometers = 1 };

struct GridGeometry {
    std::array<int, 3> dims{1, 1, 1};
    Vec3 origin;
    Vec3 voxel_size{1.0, 1.0, 1.0};
    int voxel_count() const { return dims[0] * dims[1] * dims[2]; }
    int flat_index(int ix, int iy, int iz) const { return ix + dims[0] * (iy + dims[1] * iz); }
    Vec3 bounds_min() const { return origin; }
    Vec3 bounds_max() const {
        return {origin.x + dims[0] * voxel_size.x, origin.y + dims[1] * voxel_size.y,
                origin.z + dims[2] * voxel_size.z};
    }
    bool contains(const Vec3& p) const {
        const Vec3 lo = bounds_min(), hi = bounds_max();
        return p.x >= lo.x && p.x <= hi.x && p.y >= lo.y && p.y <= hi.y && p.z >= lo.z && p.z <= hi.z;
    }
    int voxel_of(const Vec3& p) const {  // grid.hpp:40-54
        int idx[3];
        const Vec3 rel = p - origin;
        const double r[3] = {rel.x / voxel_size.x, rel.y / voxel_size.y, rel.z / voxel_size.z};
        for (int a = 0; a < 3; ++a) {
            int i = static_cast<int>(r[a]);
            if (r[a] < 0.0) return -1;
            if (i >= dims[a]) {
                if (r[a] <= static_cast<double>(dims[a]))
                    i = dims[a] - 1;
                else
                    return -1;
            }
            idx[a] = i;
        }
        return flat_index(idx[0], idx[1], idx[2]);
    }
    Vec3 voxel_center(int flat) const {
        const int ix = flat % dims[0], iy = (flat / dims[0]) % dims[1], iz = flat / (dims[0] * dims[1]);
        return {origin.x + (ix + 0.5) * voxel_size.x, origin.y + (iy + 0.5) * voxel_size.y,
                origin.z + (iz + 0.5) * voxel_size.z};
    }
    bool operator==(const GridGeometry&) const = default;
};

struct VoxelGridField {
    GridGeometry geom;
    std::vector<double> values;
    static VoxelGridField constant(const GridGeometry& g, double value) {
        VoxelGridField f;
        f.geom = g;
        f.values.assign(static_cast<size_t>(g.voxel_count()), value);
        return f;
    }
    double at(int flat) const { return values[static_cast<size_t>(flat)]; }
};

// ------------------------------------------------------------------ phase.hpp / brdf.hpp
inline constexpr double kFourPi = 4.0 * std::numbers::pi;

class PhaseFunction {
public:
    enum class Kind : uint8_t { HenyeyGreenstein, Rayleigh };
    static PhaseFunction henyey_greenstein(double g) { return PhaseFunction(Kind::HenyeyGreenstein, g); }
    static PhaseFunction rayleigh() { return PhaseFunction(Kind::Rayleigh, 0.0); }
    Kind kind() const { return kind_; }
    double g() const { return g_; }
    double eval(double cos_theta) const {  // phase.hpp:28-33
        if (kind_ == Kind::Rayleigh) return 3.0 * (1.0 + cos_theta * cos_theta) / (16.0 * std::numbers::pi);
        const double denom = 1.0 + g_ * g_ - 2.0 * g_ * cos_theta;
        return (1.0 - g_ * g_) / (kFourPi * denom * std::sqrt(denom));
    }

private:
    PhaseFunction(Kind k, double g) : kind_(k), g_(g) {}
    Kind kind_;
    double g_;
};

struct PhongBrdf {  // brdf.hpp:12-31
    double kappa_s = 0.0;
    double gamma = 0.0;
    double eval(double cos_r) const {
        const double c = std::clamp(cos_r, 0.0, 1.0);
        return 1.0 - kappa_s + kappa_s * std::pow(c, gamma);
    }
    double d_kappa(double cos_r) const { return -1.0 + std::pow(std::clamp(cos_r, 0.0, 1.0), gamma); }
    double d_gamma(double cos_r) const {
        const double c = std::clamp(cos_r, 0.0, 1.0);
        return c <= 0.0 ? 0.0 : kappa_s * std::pow(c, gamma) * std::log(c);
    }
};
struct DiffuseBrdf {
    double albedo = 1.0;
    double eval() const { return albedo / std::numbers::pi; }
};
struct Brdf {  // brdf.hpp:40-63
    enum class Kind : uint8_t { Diffuse, Phong } kind = Kind::Diffuse;
    DiffuseBrdf diffuse;
    PhongBrdf phong;
    static Brdf make_diffuse(double albedo) {
        Brdf b;
        b.kind = Kind::Diffuse;
        b.diffuse.albedo = albedo;
        return b;
    }
    static Brdf make_phong(double kappa_s, double gamma) {
        Brdf b;
        b.kind = Kind::Phong;
        b.phong = {kappa_s, gamma};
        return b;
    }
    double eval(double cos_r) const { return kind == Kind::Phong ? phong.eval(cos_r) : diffuse.eval(); }
};

// ------------------------------------------------------------------ scene.hpp
struct Aabb {
    Vec3 min, max;
    bool contains(const Vec3& p) const {
        return p.x >= min.x && p.x <= max.x && p.y >= min.y && p.y <= max.y && p.z >= min.z && p.z <= max.z;
    }
};

struct ParticleSpecies {
    std::string name;
    VoxelGridField extinction;
    double albedo = 1.0;
    PhaseFunction phase = PhaseFunction::rayleigh();
    bool unknown = false;
};

struct Detector {
    Vec3 position;
    Vec3 direction;
    Vec3 up{0.0, 0.0, 1.0};
    int rows = 1, cols = 1;
    double fov = 1.0;
    Vec3 right_axis, up_axis;  // set by finalize()
    double half_w = 0.0, half_h = 0.0;

    void finalize() {  // scene.cpp:8-14
        direction = direction.normalized();
        right_axis = cross(direction, up).normalized();
        up_axis = cross(right_axis, direction);
        half_w = std::tan(0.5 * fov);
        half_h = half_w * static_cast<double>(rows) / static_cast<double>(cols);
    }
    int pixel_of(const Vec3& p) const {  // scene.cpp:16-28
        const Vec3 w = p - position;
        const double depth = dot(w, direction);
        if (depth <= 0.0) return -1;
        const double u = dot(w, right_axis) / depth;
        const double v = dot(w, up_axis) / depth;
        if (u < -half_w || u >= half_w || v < -half_h || v >= half_h) return -1;
        int col = static_cast<int>((u + half_w) / (2.0 * half_w) * cols);
        int row = static_cast<int>((half_h - v) / (2.0 * half_h) * rows);
        if (col >= cols) col = cols - 1;
        if (row >= rows) row = rows - 1;
        return row * cols + col;
    }
};

struct LightSource {
    enum class Kind : uint8_t { DirectionalSun, IsotropicPoint } kind = Kind::IsotropicPoint;
    Vec3 position;
    Vec3 direction;
    double radiance = 1.0;
};

struct Sphere {
    Vec3 center;
    double radius = 1.0;
};

struct BoxFace {
    int axis = 2;
    double coord = 0.0;
    double lo[2] = {0.0, 0.0};
    double hi[2] = {1.0, 1.0};
    double normal_sign = 1.0;
};

struct Surface {
    enum class Kind : uint8_t { Sphere, Face } kind = Kind::Sphere;
    Sphere sphere;
    BoxFace face;
    Brdf brdf;
    bool target = false;
    Vec3 normal_at(const Vec3& p) const {  // scene.cpp:48-55
        if (kind == Kind::Sphere) return (p - sphere.center).normalized();
        Vec3 n{0.0, 0.0, 0.0};
        if (face.axis == 0)
            n.x = face.normal_sign;
        else if (face.axis == 1)
            n.y = face.normal_sign;
        else
            n.z = face.normal_sign;
        return n;
    }
};

struct Scene {
    LengthUnit unit = LengthUnit::Meters;
    Aabb bounds{};
    std::vector<ParticleSpecies> species;
    std::vector<Surface> surfaces;
    LightSource light;
    std::vector<Detector> detectors;

    bool has_medium() const { return !species.empty(); }
    const GridGeometry* grid() const { return species.empty() ? nullptr : &species[0].extinction.geom; }
    int unknown_species() const {
        for (size_t j = 0; j < species.size(); ++j)
            if (species[j].unknown) return static_cast<int>(j);
        return -1;
    }
    int target_surface() const {
        for (size_t s = 0; s < surfaces.size(); ++s)
            if (surfaces[s].target) return static_cast<int>(s);
        return -1;
    }
    double sun_entry_area() const { return (bounds.max.x - bounds.min.x) * (bounds.max.y - bounds.min.y); }
    void finalize() {  // scene.cpp:69-75
        for (auto& d : detectors) d.finalize();
        if (light.kind == LightSource::Kind::DirectionalSun) light.direction = light.direction.normalized();
        finalized_ = true;
    }
    // extensions
    size_t pixel_count() const {
        size_t n = 0;
        for (const auto& d : detectors) n += static_cast<size_t>(d.rows) * d.cols;
        return n;
    }
    bool finalized_ = false;  // finalize() ran (see prc_scene_desc::finalized)
};

// ------------------------------------------------------------------ transport.hpp
struct ParamSet {
    std::vector<double> beta;
    double kappa_s = 0.0;
    double gamma = 0.0;
};

inline ParamSet params_from_scene(const Scene& scene) {  // transport.cpp:119-128
    ParamSet p;
    const int u = scene.unknown_species();
    if (u >= 0) p.beta = scene.species[static_cast<size_t>(u)].extinction.values;
    const int t = scene.target_surface();
    if (t >= 0) {
        p.kappa_s = scene.surfaces[static_cast<size_t>(t)].brdf.phong.kappa_s;
        p.gamma = scene.surfaces[static_cast<size_t>(t)].brdf.phong.gamma;
    }
    return p;
}

inline double species_extinction(const Scene& scene, const ParamSet& p, int j, int voxel) {
    if (scene.species[static_cast<size_t>(j)].unknown && !p.beta.empty()) return p.beta[static_cast<size_t>(voxel)];
    return scene.species[static_cast<size_t>(j)].extinction.at(voxel);
}

inline Brdf surface_brdf(const Scene& scene, const ParamSet& p, int surface) {
    const Surface& s = scene.surfaces[static_cast<size_t>(surface)];
    if (s.target) return Brdf::make_phong(p.kappa_s, p.gamma);
    return s.brdf;
}

struct Image {
    int rows = 0, cols = 0;
    std::vector<double> data;
    static Image zeros(int r, int c) {
        Image im;
        im.rows = r;
        im.cols = c;
        im.data.assign(static_cast<size_t>(r) * c, 0.0);
        return im;
    }
    double& at(int row, int col) { return data[static_cast<size_t>(row) * cols + col]; }
    double at(int row, int col) const { return data[static_cast<size_t>(row) * cols + col]; }
};
using ImageSet = std::vector<Image>;

inline double emission_prefactor(const Scene& scene) {  // transport.cpp:347-351
    if (scene.light.kind == LightSource::Kind::IsotropicPoint) return kFourPi * scene.light.radiance;
    return scene.sun_entry_area() * scene.light.radiance;
}

struct RenderOptions {
    uint64_t n_paths = 1;
    uint64_t seed = 0;
    int workers = 1;  // ignored (GPU)
    int max_bounces = 500;
    int max_scatter_events = -1;
    bool keep_paths = false;
};

// ------------------------------------------------------------------ the device context
class Context {
public:
    explicit Context(int device = 0) { check(prc_gpu_ctx_create(device, &ctx_)); }
    // One process per GPU joining an NCCL communicator (paths sharded by rank); a null
    // nccl_id with world > 1 makes a detached shard (partial sums, see pathrec_gpu.h).
    Context(int device, int rank, int world, const void* nccl_id128) {
        check(prc_gpu_ctx_create_rank(device, rank, world, nccl_id128, &ctx_));
    }
    ~Context() { prc_gpu_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    prc_gpu_ctx* get() const { return ctx_; }
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
            desc.bounds_min = v(sc.bounds.min);
            desc.bounds_max = v(sc.bounds.max);
            if (!sc.species.empty()) {
                const GridGeometry& g = sc.species[0].extinction.geom;
                for (int a = 0; a < 3; ++a) desc.dims[a] = g.dims[a];
                desc.grid_origin = v(g.origin);
                desc.voxel_size = v(g.voxel_size);
            }
            for (const auto& q : sc.species) {
                if (!(q.extinction.geom == sc.species[0].extinction.geom))
                    throw std::invalid_argument("scene: every species must share one grid geometry");
                sp.push_back({q.extinction.values.data(), q.albedo,
                              q.phase.kind() == PhaseFunction::Kind::Rayleigh ? PRC_PHASE_RAYLEIGH : PRC_PHASE_HG,
                              q.phase.g(), q.unknown ? 1 : 0});
            }
            for (const auto& q : sc.surfaces) {
                prc_surface_desc d{};
                d.kind = q.kind == Surface::Kind::Face ? PRC_SURF_FACE : PRC_SURF_SPHERE;
                d.center = v(q.sphere.center);
                d.radius = q.sphere.radius;
                d.axis = q.face.axis;
                d.coord = q.face.coord;
                d.lo[0] = q.face.lo[0];
                d.lo[1] = q.face.lo[1];
                d.hi[0] = q.face.hi[0];
                d.hi[1] = q.face.hi[1];
                d.normal_sign = q.face.normal_sign;
                d.brdf_kind = q.brdf.kind == Brdf::Kind::Phong ? PRC_BRDF_PHONG : PRC_BRDF_DIFFUSE;
                d.albedo = q.brdf.diffuse.albedo;
                d.kappa_s = q.brdf.phong.kappa_s;
                d.gamma = q.brdf.phong.gamma;
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
            desc.finalized = sc.finalized_ ? 1 : 0;
        }
        uint64_t key() const {
            uint64_t h = 1469598103934665603ull;
            auto mix = [&](const void* p, size_t n) {
                const unsigned char* b = static_cast<const unsigned char*>(p);
                for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
            };
            mix(&desc.bounds_min, sizeof(prc_vec3) * 2 + sizeof(int) * 3 + sizeof(prc_vec3) * 2);
            mix(&desc.light, sizeof desc.light);
            mix(&desc.finalized, sizeof desc.finalized);
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

    // Uploads the scene when it differs from the one on the device.
    void use(const Scene& s) {
        Holder h(s);
        const uint64_t key = h.key();
        if (have_ && key == scene_key_) return;
        check(prc_gpu_scene_upload(ctx_, &h.desc));
        scene_key_ = key;
        have_ = true;
    }

private:
    prc_gpu_ctx* ctx_ = nullptr;
    uint64_t scene_key_ = 0;
    bool have_ = false;
};

// Default per-thread context (CUDA device $LOCAL_RANK, else 0) behind the reference's
// context-free free functions.
inline Context& default_context() {
    static thread_local std::unique_ptr<Context> c;
    if (!c) {
        const char* lr = std::getenv("LOCAL_RANK");
        c = std::make_unique<Context>(lr ? std::atoi(lr) : 0);
    }
    return *c;
}

// ------------------------------------------------------------------ pathstore.hpp
// A handle on a device-resident store.  A store read by load_store(path) is imported on
// first use, when a scene is at hand (the import range-checks it against that scene).
struct PathStore {
    bool sorted_flag = false;
    uint64_t generation = 0;
    uint64_t seed = 0;
    ParamSet ref_params;

    // engine handle (extension)
    Context* ctx = nullptr;
    mutable std::shared_ptr<prc_gpu_store> h;
    mutable std::string pending_path;  // load_store(path) not yet imported
    mutable bool pending_sort = false;
    bool materialized = false;

    prc_gpu_store_info info() const {
        prc_gpu_store_info i{};
        check(prc_gpu_store_info_get(handle(), &i));
        return i;
    }
    size_t size() const { return static_cast<size_t>(info().n_paths); }
    size_t memory_bytes() const { return static_cast<size_t>(info().device_bytes); }
    std::vector<uint64_t> streams() const {  // records[i].stream in storage order
        std::vector<uint64_t> s(size());
        check(prc_gpu_store_streams(handle(), s.data()));
        return s;
    }
    // Imports a pending load_store(path) under `scene` (and applies a pending sort).
    void bind(const Scene& scene) const {
        ctx->use(scene);
        if (pending_path.empty()) return;
        prc_gpu_store* st = nullptr;
        check(prc_gpu_store_import_pstr_ex(ctx->get(), pending_path.c_str(),
                                          materialized ? PRC_IMPORT_MATERIALIZE : 0, &st));
        h = std::shared_ptr<prc_gpu_store>(st, prc_gpu_store_free);
        pending_path.clear();
        if (pending_sort) check(prc_gpu_sort_by_size(ctx->get(), h.get()));
        pending_sort = false;
    }
    prc_gpu_store* handle() const {
        if (!h) throw std::invalid_argument("PathStore: loaded store is used before any scene (evaluate it first)");
        return h.get();
    }
};

struct RenderResult {
    ImageSet images;
    uint64_t truncated_paths = 0;
    std::shared_ptr<PathStore> store;
};

struct EvalOptions {
    int workers = 1;  // ignored (GPU)
    bool normalize = true;
    bool want_grad = false;
    bool legacy_score = false;
    bool self_normalize = false;  // divide by the mean correction factor (pathstore.cpp:334-359)
    const ImageSet* pixel_weights = nullptr;
    bool per_species = false;    // extension: per-type gradients (config (c))
    bool deterministic = false;  // extension: bit-reproducible images (render() always is)
};

struct EvalResult {
    ImageSet images;
    std::vector<double> grad_beta;
    double grad_kappa = 0.0;
    double grad_gamma = 0.0;
    uint64_t clamp_events = 0;
    double mean_correction = 1.0;
};

// ------------------------------------------------------------------ gradient.hpp
struct SparseGradient {
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
inline size_t voxels(const Scene& s) { return s.species.empty() ? 0 : (size_t)s.species[0].extinction.geom.voxel_count(); }
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
        r.store->seed = opt.seed;
        r.store->ref_params = params_from_scene(scene);
    }
    return r;
}
inline RenderResult render(const Scene& scene, const RenderOptions& opt) {
    return render(default_context(), scene, opt);
}

// pathstore.cpp:261-267 (throws invalid_argument on an empty store)
inline void sort_by_size(PathStore& store) {
    if (!store.pending_path.empty()) {
        store.pending_sort = true;
    } else {
        check(prc_gpu_sort_by_size(store.ctx->get(), store.handle()));
    }
    store.sorted_flag = true;
}

// pathstore.cpp:315-368
inline EvalResult evaluate_store(const Scene& scene, const PathStore& store, const ParamSet& params_t,
                                 const EvalOptions& opt) {
    store.bind(scene);
    Context& ctx = *store.ctx;
    detail::ParamsC pc(params_t);
    std::vector<double> w;
    if (opt.pixel_weights) w = detail::flatten(*opt.pixel_weights);
    prc_gpu_eval_opts eo{(opt.normalize ? PRC_EVAL_NORMALIZE : 0) | (opt.want_grad ? PRC_EVAL_WANT_GRAD : 0) |
                             (opt.legacy_score ? PRC_EVAL_LEGACY_SCORE : 0) |
                             (opt.self_normalize ? PRC_EVAL_SELF_NORMALIZE : 0) |
                             (opt.per_species ? PRC_EVAL_PER_SPECIES : 0) |
                             (opt.deterministic ? PRC_EVAL_DETERMINISTIC : 0),
                         w.empty() ? nullptr : w.data()};
    std::vector<double> img(scene.pixel_count());
    const size_t V = detail::voxels(scene);
    const size_t n_out = opt.per_species ? scene.species.size() : 1;
    const bool grad = opt.want_grad && V && (scene.unknown_species() >= 0 || opt.per_species);
    EvalResult out;
    if (grad) out.grad_beta.assign(n_out * V, 0.0);
    prc_gpu_eval_result r{img.data(), grad ? out.grad_beta.data() : nullptr, 0.0, 0.0, 0, 1.0};
    check(prc_gpu_evaluate(ctx.get(), store.handle(), &pc.p, &eo, &r));
    out.images = detail::split(scene, img);
    out.grad_kappa = r.grad_kappa;
    out.grad_gamma = r.grad_gamma;
    out.clamp_events = r.clamp_events;
    out.mean_correction = r.mean_correction;
    return out;
}

// pathstore.cpp:370-375
inline ImageSet recycled_render(const Scene& scene, const PathStore& store, const ParamSet& params_t,
                                int workers = 1) {
    EvalOptions o;
    o.workers = workers;
    return evaluate_store(scene, store, params_t, o).images;
}

// gradient.cpp:111-128
inline SparseGradient grad_forward(const Scene& scene, const PathStore& store, const ParamSet& params_t,
                                   const EvalOptions& opt = {}) {
    EvalOptions e = opt;
    e.want_grad = true;
    const EvalResult r = evaluate_store(scene, store, params_t, e);
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
    if (!store.pending_path.empty() && !store.pending_sort) {  // never imported: the file itself
        std::FILE* in = std::fopen(store.pending_path.c_str(), "rb");
        std::FILE* out = in ? std::fopen(path.c_str(), "wb") : nullptr;
        if (!in || !out) {
            if (in) std::fclose(in);
            throw std::runtime_error("save_store: cannot open " + path);
        }
        char buf[1 << 16];
        size_t n;
        while ((n = std::fread(buf, 1, sizeof buf, in)) > 0) std::fwrite(buf, 1, n, out);
        std::fclose(in);
        std::fclose(out);
        return;
    }
    check(prc_gpu_store_set_generation(store.handle(), store.generation));
    check(prc_gpu_store_export_pstr(store.ctx->get(), store.handle(), path.c_str()));
}

// load_store(path): the reference takes no scene; the store is imported (materialized:
// the file's own spans) on the default context at its first use with a scene.
inline PathStore load_store(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("load_store: cannot open " + path);
    char magic[4] = {0, 0, 0, 0};
    uint32_t version = 0;
    uint64_t count = 0, gen = 0, seed = 0, nb = 0;
    uint8_t sorted = 0;
    bool ok = std::fread(magic, 1, 4, f) == 4 && std::fread(&version, 4, 1, f) == 1 &&
              std::fread(&count, 8, 1, f) == 1 && std::fread(&gen, 8, 1, f) == 1 && std::fread(&seed, 8, 1, f) == 1 &&
              std::fread(&sorted, 1, 1, f) == 1 && std::fread(&nb, 8, 1, f) == 1;
    PathStore s;
    if (ok && std::memcmp(magic, "PSTR", 4) == 0 && version == 1) {
        s.ref_params.beta.resize(nb);
        ok = (nb == 0 || std::fread(s.ref_params.beta.data(), 8, nb, f) == nb) &&
             std::fread(&s.ref_params.kappa_s, 8, 1, f) == 1 && std::fread(&s.ref_params.gamma, 8, 1, f) == 1;
    } else {
        ok = false;
    }
    std::fclose(f);
    if (!ok) throw std::runtime_error("load_store: bad magic, version or truncated header in " + path);
    s.sorted_flag = sorted != 0;
    s.generation = gen;
    s.seed = seed;
    s.ctx = &default_context();
    s.pending_path = path;
    s.materialized = true;
    return s;
}
// Extension: import now, under `scene`, on a given context (recomputed spans unless
// materialized).
inline PathStore load_store(Context& ctx, const Scene& scene, const std::string& path, bool materialized = false) {
    PathStore s = load_store(path);
    s.ctx = &ctx;
    s.materialized = materialized;
    s.bind(scene);
    return s;
}

// ------------------------------------------------------------------ inverse.hpp
struct AdamConfig {
    double alpha = 1e7;
    double eta1 = 0.9;
    double eta2 = 0.999;
    double eps_guard = 1e-8;
    bool project_nonneg = true;
    std::vector<double> step_scale;
};

struct Stage {
    int rows = 0, cols = 0;
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

struct OptState {
    ParamSet params;
    std::vector<double> m1, m2;
    int64_t t = 0;
    uint64_t store_generation = 0;
    ParamSet ref_params;
    std::vector<double> loss_history;
};

struct IterationLog {
    int iter = 0;
    double time_s = 0.0;
    double loss = 0.0;
    double eps = 0.0;
    double delta = 0.0;
    int stage = 0;
};

struct ReconstructResult {
    ParamSet params;
    std::vector<IterationLog> history;
    uint64_t sampling_phases = 0;
    uint64_t truncated_paths = 0;
};

struct ReconstructOptions {
    AdamConfig adam;
    Schedule schedule;
    uint64_t seed = 0;
    int workers = 1;  // ignored (GPU)
    const ParamSet* truth = nullptr;
    std::string checkpoint_dir;
    std::function<void(const IterationLog&)> on_iteration;
    int max_bounces = 500;  // extension: the trace budget of every resample
};

// inverse.cpp:11-23
inline double loss(const ImageSet& forward, const ImageSet& gt) {
    if (forward.size() != gt.size()) throw std::invalid_argument("loss: detector count mismatch");
    double acc = 0.0;
    for (size_t d = 0; d < forward.size(); ++d) {
        if (forward[d].data.size() != gt[d].data.size()) throw std::invalid_argument("loss: image shape mismatch");
        for (size_t p = 0; p < forward[d].data.size(); ++p) {
            const double r = forward[d].data[p] - gt[d].data[p];
            acc += r * r;
        }
    }
    return 0.5 * acc;
}

// inverse.cpp:41-67 on a host-held state (the device loop runs the same update in K6).
inline void adam_step(OptState& state, const SparseGradient& grad, const AdamConfig& config) {
    std::vector<double*> slots;
    if (!state.params.beta.empty()) {
        for (auto& b : state.params.beta) slots.push_back(&b);
    } else {
        slots.push_back(&state.params.kappa_s);
        slots.push_back(&state.params.gamma);
    }
    const size_t n = slots.size();
    if (state.m1.size() != n) state.m1.assign(n, 0.0);
    if (state.m2.size() != n) state.m2.assign(n, 0.0);
    ++state.t;
    const double c1 = 1.0 - std::pow(config.eta1, static_cast<double>(state.t));
    const double c2 = 1.0 - std::pow(config.eta2, static_cast<double>(state.t));
    const bool phong = state.params.beta.empty();
    for (size_t i = 0; i < n; ++i) {
        const double g = grad.at(static_cast<int>(i));
        state.m1[i] = config.eta1 * state.m1[i] + (1.0 - config.eta1) * g;
        state.m2[i] = config.eta2 * state.m2[i] + (1.0 - config.eta2) * g * g;
        const double mhat = state.m1[i] / c1;
        const double vhat = state.m2[i] / c2;
        const double scale = i < config.step_scale.size() ? config.step_scale[i] : 1.0;
        *slots[i] -= config.alpha * scale * mhat / (std::sqrt(vhat) + config.eps_guard);
        if (!phong && config.project_nonneg && *slots[i] < 0.0) *slots[i] = 0.0;
    }
    if (phong) {
        state.params.kappa_s = std::clamp(state.params.kappa_s, 0.0, 1.0);
        state.params.gamma = std::max(state.params.gamma, 0.0);
    }
}

struct CarveResult {
    std::vector<uint8_t> mask;
    ParamSet initial;
};

// inverse.cpp:69-101 (the occupancy test runs on the device)
inline CarveResult space_carve(Context& ctx, const Scene& scene, const ImageSet& gt, double threshold_fraction,
                               double fill_extinction) {
    ctx.use(scene);
    std::vector<double> g = detail::flatten(gt);
    const size_t V = detail::voxels(scene);
    CarveResult r;
    r.mask.assign(V, 0);
    r.initial.beta.assign(V, 0.0);
    check(prc_gpu_space_carve(ctx.get(), g.data(), threshold_fraction, fill_extinction, r.mask.data(),
                              r.initial.beta.data()));
    return r;
}
inline CarveResult space_carve(const Scene& scene, const ImageSet& gt, double threshold_fraction,
                               double fill_extinction) {
    return space_carve(default_context(), scene, gt, threshold_fraction, fill_extinction);
}

namespace detail {
inline void on_iteration_trampoline(const prc_gpu_iteration_log* row, void* user) {
    const auto& f = *static_cast<const std::function<void(const IterationLog&)>*>(user);
    f(IterationLog{row->iter, row->time_s, row->loss, row->eps, row->delta, row->stage});
}
}  // namespace detail

// inverse.cpp:154-263: the recycling loop on the device (resample + sort every N_r,
// stages applied at resample boundaries, saturation, eps/delta, checkpoints).
inline ReconstructResult reconstruct(Context& ctx, const Scene& scene, const ImageSet& gt, ParamSet initial,
                                     const ReconstructOptions& opt) {
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
    prc_gpu_schedule sch{};
    sch.seed = opt.seed;
    sch.max_bounces = opt.max_bounces;
    sch.recycle_period = opt.schedule.recycle_period;
    sch.max_iterations = opt.schedule.max_iterations;
    sch.stages = st.data();
    sch.n_stages = (int)st.size();
    sch.saturation_window = opt.schedule.saturation_window;
    sch.saturation_rel_improvement = opt.schedule.saturation_rel_improvement;
    sch.checkpoint_every = opt.schedule.checkpoint_every;
    sch.checkpoint_dir = opt.checkpoint_dir.empty() ? nullptr : opt.checkpoint_dir.c_str();
    sch.length_unit = (int)scene.unit;
    sch.truth = tc ? &tc->p : nullptr;
    if (opt.on_iteration) {
        sch.on_iteration = detail::on_iteration_trampoline;
        sch.user = const_cast<void*>(static_cast<const void*>(&opt.on_iteration));
    }
    std::vector<prc_gpu_iteration_log> h((size_t)std::max(1, opt.schedule.max_iterations));
    ReconstructResult r;
    check(prc_gpu_reconstruct_schedule(ctx.get(), &pc.p, g.data(), &a, &sch, h.data(), &r.sampling_phases,
                                       &r.truncated_paths));
    for (int t = 0; t < opt.schedule.max_iterations; ++t)
        r.history.push_back({h[t].iter, h[t].time_s, h[t].loss, h[t].eps, h[t].delta, h[t].stage});
    const size_t V = detail::voxels(scene);
    if (scene.unknown_species() >= 0) r.params.beta.assign(V, 0.0);
    check(prc_gpu_opt_params(ctx.get(), r.params.beta.empty() ? nullptr : r.params.beta.data(), &r.params.kappa_s,
                             &r.params.gamma));
    return r;
}
inline ReconstructResult reconstruct(const Scene& scene, const ImageSet& gt, ParamSet initial,
                                     const ReconstructOptions& opt) {
    return reconstruct(default_context(), scene, gt, std::move(initial), opt);
}

struct Metrics {
    double eps = 0.0;
    double delta = 0.0;
};

// inverse.cpp:103-114
inline Metrics metrics(const std::vector<double>& estimate, const std::vector<double>& truth) {
    if (estimate.size() != truth.size()) throw std::invalid_argument("metrics: dimension mismatch");
    Metrics m;
    check(prc_gpu_metrics(estimate.data(), truth.data(), truth.size(), &m.eps, &m.delta));
    return m;
}

// inverse.cpp:116-133
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

// ------------------------------------------------------------------ io.hpp
inline VoxelGridField load_grid(const std::string& path, LengthUnit* unit = nullptr) {
    int dims[3];
    prc_vec3 o, v;
    int u = 0;
    check(prc_gpu_load_grid(path.c_str(), dims, &o, &v, &u, nullptr, 0));
    VoxelGridField f;
    f.geom.dims = {dims[0], dims[1], dims[2]};
    f.geom.origin = {o.x, o.y, o.z};
    f.geom.voxel_size = {v.x, v.y, v.z};
    f.values.resize((size_t)dims[0] * dims[1] * dims[2]);
    check(prc_gpu_load_grid(path.c_str(), dims, &o, &v, &u, f.values.data(), f.values.size()));
    if (unit) *unit = static_cast<LengthUnit>(u);
    return f;
}

inline void save_grid(const VoxelGridField& grid, LengthUnit unit, const std::string& path) {
    const int dims[3] = {grid.geom.dims[0], grid.geom.dims[1], grid.geom.dims[2]};
    const prc_vec3 o{grid.geom.origin.x, grid.geom.origin.y, grid.geom.origin.z};
    const prc_vec3 v{grid.geom.voxel_size.x, grid.geom.voxel_size.y, grid.geom.voxel_size.z};
    check(prc_gpu_save_grid(path.c_str(), dims, &o, &v, (int)unit, grid.values.data()));
}

// The coarse C API's image writers / readers (prc_host_api.cu) for a single image.
namespace detail {
struct OneImage {  // a render result wrapper is not needed: PFM I/O is plain host code
    static void check_finite(const Image& im, const char* what) {
        size_t bad = 0, first = 0;
        for (size_t i = 0; i < im.data.size(); ++i)
            if (!std::isfinite(im.data[i])) {
                if (!bad) first = i;
                ++bad;
            }
        if (bad)
            throw std::runtime_error(std::string(what) + ": " + std::to_string(bad) +
                                     " non-finite pixel(s), first at index " + std::to_string(first));
    }
};
}  // namespace detail

// io.cpp:94-106
inline void save_pfm(const Image& image, const std::string& path) {
    detail::OneImage::check_finite(image, "save_pfm");
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("save_pfm: cannot open " + path);
    const std::string head = "Pf\n" + std::to_string(image.cols) + " " + std::to_string(image.rows) + "\n-1.0\n";
    std::fwrite(head.data(), 1, head.size(), f);
    for (int r = image.rows - 1; r >= 0; --r)
        for (int c = 0; c < image.cols; ++c) {
            const float v = static_cast<float>(image.at(r, c));
            std::fwrite(&v, sizeof v, 1, f);
        }
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) throw std::runtime_error("save_pfm: write failure on " + path);
}

// io.cpp:108-129
inline Image load_pfm(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("load_pfm: cannot open " + path);
    char magic[3] = {0, 0, 0};
    int cols = 0, rows = 0;
    double scale = 0.0;
    const int got = std::fscanf(f, "%2s %d %d %lf", magic, &cols, &rows, &scale);
    std::fgetc(f);  // single whitespace before the payload
    if (got != 4 || std::strcmp(magic, "Pf") != 0) {
        std::fclose(f);
        throw std::runtime_error("load_pfm: not a grayscale PFM: " + path);
    }
    if (cols <= 0 || rows <= 0 || scale >= 0.0) {
        std::fclose(f);
        throw std::runtime_error("load_pfm: unsupported header in " + path);
    }
    Image im = Image::zeros(rows, cols);
    bool ok = true;
    for (int r = rows - 1; r >= 0 && ok; --r)
        for (int c = 0; c < cols && ok; ++c) {
            float v = 0.0f;
            ok = std::fread(&v, sizeof v, 1, f) == 1;
            im.at(r, c) = v;
        }
    std::fclose(f);
    if (!ok) throw std::runtime_error("load_pfm: truncated payload in " + path);
    return im;
}

// io.cpp:131-145
inline void save_pgm_preview(const Image& image, const std::string& path) {
    detail::OneImage::check_finite(image, "save_pgm_preview");
    double mx = 0.0;
    for (double v : image.data) mx = std::max(mx, v);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("save_pgm_preview: cannot open " + path);
    const std::string head = "P5\n" + std::to_string(image.cols) + " " + std::to_string(image.rows) + "\n255\n";
    std::fwrite(head.data(), 1, head.size(), f);
    for (int r = 0; r < image.rows; ++r)
        for (int c = 0; c < image.cols; ++c) {
            const double t = mx > 0.0 ? std::clamp(image.at(r, c) / mx, 0.0, 1.0) : 0.0;
            std::fputc(static_cast<int>(static_cast<unsigned char>(std::lround(255.0 * std::pow(t, 1.0 / 2.2)))), f);
        }
    std::fclose(f);
}

// io.cpp:147-155
inline void save_csv(const std::vector<IterationLog>& rows, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("save_csv: cannot open " + path);
    std::fputs("iter,time_s,loss,eps,delta,stage\r\n", f);
    for (const auto& r : rows)
        std::fprintf(f, "%d,%.17g,%.17g,%.17g,%.17g,%d\r\n", r.iter, r.time_s, r.loss, r.eps, r.delta, r.stage);
    std::fclose(f);
}

// io.cpp:190-278, through prc_scene_load (the JSON loader of the coarse C API).
inline Scene load_scene(const std::string& path) {
    prc_scene* raw = nullptr;
    check_coarse(prc_scene_load(path.c_str(), &raw));
    std::unique_ptr<prc_scene, void (*)(prc_scene*)> hold(raw, prc_scene_free);
    const prc_scene_desc* d = nullptr;
    int unit = 0;
    check_coarse(prc_scene_describe(raw, &d, &unit));
    auto v3 = [](const prc_vec3& a) { return Vec3{a.x, a.y, a.z}; };
    Scene s;
    s.unit = static_cast<LengthUnit>(unit);
    s.bounds = {v3(d->bounds_min), v3(d->bounds_max)};
    GridGeometry g;
    g.dims = {d->dims[0], d->dims[1], d->dims[2]};
    g.origin = v3(d->grid_origin);
    g.voxel_size = v3(d->voxel_size);
    for (int j = 0; j < d->n_species; ++j) {
        const prc_species_desc& q = d->species[j];
        ParticleSpecies sp;
        sp.name = "species" + std::to_string(j);
        sp.extinction.geom = g;
        sp.extinction.values.assign(q.extinction, q.extinction + g.voxel_count());
        sp.albedo = q.albedo;
        sp.phase = q.phase_kind == PRC_PHASE_RAYLEIGH ? PhaseFunction::rayleigh() : PhaseFunction::henyey_greenstein(q.g);
        sp.unknown = q.unknown != 0;
        s.species.push_back(std::move(sp));
    }
    for (int k = 0; k < d->n_surfaces; ++k) {
        const prc_surface_desc& q = d->surfaces[k];
        Surface sf;
        sf.kind = q.kind == PRC_SURF_FACE ? Surface::Kind::Face : Surface::Kind::Sphere;
        sf.sphere.center = v3(q.center);
        sf.sphere.radius = q.radius;
        sf.face.axis = q.axis;
        sf.face.coord = q.coord;
        sf.face.lo[0] = q.lo[0];
        sf.face.lo[1] = q.lo[1];
        sf.face.hi[0] = q.hi[0];
        sf.face.hi[1] = q.hi[1];
        sf.face.normal_sign = q.normal_sign;
        sf.brdf = q.brdf_kind == PRC_BRDF_PHONG ? Brdf::make_phong(q.kappa_s, q.gamma) : Brdf::make_diffuse(q.albedo);
        sf.target = q.target != 0;
        s.surfaces.push_back(sf);
    }
    s.light.kind = d->light.kind == PRC_LIGHT_SUN ? LightSource::Kind::DirectionalSun : LightSource::Kind::IsotropicPoint;
    s.light.position = v3(d->light.position);
    s.light.direction = v3(d->light.direction);
    s.light.radiance = d->light.radiance;
    for (int k = 0; k < d->n_detectors; ++k) {
        const prc_detector_desc& q = d->detectors[k];
        Detector det;
        det.position = v3(q.position);
        det.direction = v3(q.direction);
        det.up = v3(q.up);
        det.rows = q.rows;
        det.cols = q.cols;
        det.fov = q.fov;
        s.detectors.push_back(det);
    }
    s.finalize();
    return s;
}

inline std::string library_version() { return prc_version(); }

}  // namespace PATHREC_GPU_NAMESPACE
