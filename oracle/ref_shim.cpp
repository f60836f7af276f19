// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline), never product.
//
// A thin extern "C" shim over the UNMODIFIED reference library (`pathrec`,
// /root/reference/proj/src/*.cpp compiled in place by oracle/Makefile).  It lets the
// Python test harness and bench.py drive the reference's own code path:
//   render (transport.cpp:405-454), sort_by_size (pathstore.cpp:261-267),
//   evaluate_store / recycled_render / grad_forward (pathstore.cpp:315-375,
//   gradient.cpp:111-128), walk_voxels (traverse.hpp:45-116), pixel_of
//   (scene.cpp:16-28), Philox4x32 (rng.hpp:11-61), save/load PSTR
//   (pathstore.cpp:410-516), reconstruct (inverse.cpp:154-263).
// The scene arrives as the product's prc_scene_desc (include/pathrec_gpu.h) so the
// same description feeds the reference, the C restatement oracle and the GPU engine.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "pathrec/gradient.hpp"
#include "pathrec/inverse.hpp"
#include "pathrec/io.hpp"
#include "pathrec/pathstore.hpp"
#include "pathrec/transport.hpp"
#include "pathrec/traverse.hpp"
#include "pathrec_gpu.h"

using namespace pathrec;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return 1;
}

Vec3 v3(const prc_vec3& v) { return {v.x, v.y, v.z}; }

Scene make_scene(const prc_scene_desc* d) {
    Scene s;
    s.bounds = {v3(d->bounds_min), v3(d->bounds_max)};
    GridGeometry g;
    g.dims = {d->dims[0], d->dims[1], d->dims[2]};
    g.origin = v3(d->grid_origin);
    g.voxel_size = v3(d->voxel_size);
    const size_t V = static_cast<size_t>(g.voxel_count());
    for (int j = 0; j < d->n_species; ++j) {
        const prc_species_desc& sd = d->species[j];
        ParticleSpecies sp;
        sp.name = "species" + std::to_string(j);
        sp.extinction.geom = g;
        sp.extinction.values.assign(sd.extinction, sd.extinction + V);
        sp.albedo = sd.albedo;
        sp.phase = sd.phase_kind == PRC_PHASE_RAYLEIGH ? PhaseFunction::rayleigh()
                                                       : PhaseFunction::henyey_greenstein(sd.g);
        sp.unknown = sd.unknown != 0;
        s.species.push_back(std::move(sp));
    }
    for (int k = 0; k < d->n_surfaces; ++k) {
        const prc_surface_desc& sd = d->surfaces[k];
        Surface sf;
        sf.kind = sd.kind == PRC_SURF_FACE ? Surface::Kind::Face : Surface::Kind::Sphere;
        sf.sphere.center = v3(sd.center);
        sf.sphere.radius = sd.radius;
        sf.face.axis = sd.axis;
        sf.face.coord = sd.coord;
        sf.face.lo[0] = sd.lo[0];
        sf.face.lo[1] = sd.lo[1];
        sf.face.hi[0] = sd.hi[0];
        sf.face.hi[1] = sd.hi[1];
        sf.face.normal_sign = sd.normal_sign;
        sf.brdf = sd.brdf_kind == PRC_BRDF_PHONG ? Brdf::make_phong(sd.kappa_s, sd.gamma)
                                                 : Brdf::make_diffuse(sd.albedo);
        sf.target = sd.target != 0;
        s.surfaces.push_back(sf);
    }
    s.light.kind = d->light.kind == PRC_LIGHT_SUN ? LightSource::Kind::DirectionalSun
                                                  : LightSource::Kind::IsotropicPoint;
    s.light.position = v3(d->light.position);
    s.light.direction = v3(d->light.direction);
    s.light.radiance = d->light.radiance;
    for (int k = 0; k < d->n_detectors; ++k) {
        const prc_detector_desc& dd = d->detectors[k];
        Detector det;
        det.position = v3(dd.position);
        det.direction = v3(dd.direction);
        det.up = v3(dd.up);
        det.rows = dd.rows;
        det.cols = dd.cols;
        det.fov = dd.fov;
        s.detectors.push_back(det);
    }
    s.finalize();
    return s;
}

ParamSet make_params(const Scene& s, const prc_gpu_params* p) {
    ParamSet out = params_from_scene(s);
    if (!p) return out;
    if (p->beta) out.beta.assign(p->beta, p->beta + p->n_beta);
    out.kappa_s = p->kappa_s;
    out.gamma = p->gamma;
    return out;
}

void bind(Scene& s, const ParamSet& p) {  // inverse.cpp:144-150 semantics
    const int u = s.unknown_species();
    if (u >= 0 && !p.beta.empty()) s.species[static_cast<size_t>(u)].extinction.values = p.beta;
    const int t = s.target_surface();
    if (t >= 0) s.surfaces[static_cast<size_t>(t)].brdf = Brdf::make_phong(p.kappa_s, p.gamma);
}

void copy_images(const ImageSet& im, double* out) {
    if (!out) return;
    size_t k = 0;
    for (const auto& i : im)
        for (double px : i.data) out[k++] = px;
}

ImageSet images_from(const Scene& s, const double* w) {
    ImageSet out;
    size_t k = 0;
    for (const auto& det : s.detectors) {
        Image im = Image::zeros(det.rows, det.cols);
        for (auto& px : im.data) px = w[k++];
        out.push_back(std::move(im));
    }
    return out;
}

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_philox(uint64_t seed, uint64_t stream, uint64_t n, uint32_t* out) {
    Philox4x32 r(seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u32();
    return 0;
}

int ref_walk(const prc_scene_desc* d, uint64_t n, const double* rays, uint32_t* counts,
             uint32_t* vox, double* len, uint64_t cap) {
    GridGeometry g;
    g.dims = {d->dims[0], d->dims[1], d->dims[2]};
    g.origin = v3(d->grid_origin);
    g.voxel_size = v3(d->voxel_size);
    uint64_t k = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const double* r = rays + 7 * i;
        Ray ray{{r[0], r[1], r[2]}, {r[3], r[4], r[5]}};
        uint32_t c = 0;
        walk_voxels(g, ray, r[6], [&](int v, double ta, double tb) {
            if (vox && k < cap) {
                vox[k] = static_cast<uint32_t>(v);
                len[k] = tb - ta;
            }
            ++k;
            ++c;
            return true;
        });
        counts[i] = c;
    }
    return 0;
}

int ref_pixel_of(const prc_scene_desc* d, int det, uint64_t n, const double* pts, int32_t* out) {
    try {
        Scene s = make_scene(d);
        for (uint64_t i = 0; i < n; ++i)
            out[i] = s.detectors[static_cast<size_t>(det)].pixel_of(
                {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* render(keep_paths) under params; optional sort; optional PSTR dump. */
int ref_render(const prc_scene_desc* d, const prc_gpu_params* params, uint64_t n, uint64_t seed,
               int max_bounces, int max_events, int workers, int sort, const char* pstr_out,
               double* images_out, uint64_t* trunc_out) {
    try {
        Scene s = make_scene(d);
        bind(s, make_params(s, params));
        RenderOptions o;
        o.n_paths = n;
        o.seed = seed;
        o.workers = workers;
        o.max_bounces = max_bounces > 0 ? max_bounces : 500;
        o.max_scatter_events = max_events;
        o.keep_paths = pstr_out != nullptr;
        RenderResult rr = render(s, o);
        copy_images(rr.images, images_out);
        if (trunc_out) *trunc_out = rr.truncated_paths;
        if (pstr_out) {
            if (sort) sort_by_size(*rr.store);
            save_store(*rr.store, pstr_out);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* load_store -> sort_by_size -> (save) ; streams in sorted storage order. */
int ref_sort_pstr(const char* in, const char* out, uint64_t* streams_out) {
    try {
        PathStore st = load_store(in);
        sort_by_size(st);
        for (size_t i = 0; i < st.records.size(); ++i) streams_out[i] = st.records[i].stream;
        if (out) save_store(st, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* evaluate_store(scene, load_store(pstr), params, opt) */
int ref_evaluate(const prc_scene_desc* d, const char* pstr, const prc_gpu_params* params,
                 int flags, const double* weights, int workers, double* images, double* grad,
                 double* gk, double* gg, uint64_t* clamps, double* mean_corr) {
    try {
        Scene s = make_scene(d);
        PathStore st = load_store(pstr);
        ParamSet t = params ? make_params(s, params) : st.ref_params;
        EvalOptions o;
        o.workers = workers;
        o.normalize = (flags & PRC_EVAL_NORMALIZE) != 0;
        o.want_grad = (flags & PRC_EVAL_WANT_GRAD) != 0;
        o.legacy_score = (flags & PRC_EVAL_LEGACY_SCORE) != 0;
        o.self_normalize = (flags & PRC_EVAL_SELF_NORMALIZE) != 0;
        ImageSet w;
        if (weights) {
            w = images_from(s, weights);
            o.pixel_weights = &w;
        }
        EvalResult r = evaluate_store(s, st, t, o);
        copy_images(r.images, images);
        if (grad)
            for (size_t v = 0; v < r.grad_beta.size(); ++v) grad[v] = r.grad_beta[v];
        if (gk) *gk = r.grad_kappa;
        if (gg) *gg = r.grad_gamma;
        if (clamps) *clamps = r.clamp_events;
        if (mean_corr) *mean_corr = r.mean_correction;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* segment_lengths (pathstore.cpp:296-313) of every record of a PSTR file, records in file
 * order, segments b = 1..B: counts[k] spans of segment k; vox/len receive them
 * concatenated.  sizes_out[0] = segments, [1] = spans (call with counts = NULL first). */
int ref_segment_lengths(const prc_scene_desc* d, const char* pstr, uint64_t* sizes_out, uint32_t* counts,
                        uint32_t* vox, double* len) {
    try {
        Scene s = make_scene(d);
        PathStore st = load_store(pstr);
        uint64_t k = 0, m = 0;
        for (const auto& rec : st.records) {
            for (const auto& seg : segment_lengths(rec, *s.grid())) {
                if (counts) counts[k] = static_cast<uint32_t>(seg.spans.size());
                for (const auto& sp : seg.spans) {
                    if (vox) {
                        vox[m] = sp.voxel;
                        len[m] = sp.length;
                    }
                    ++m;
                }
                ++k;
            }
        }
        sizes_out[0] = k;
        sizes_out[1] = m;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* CPU baseline: render(keep) + sort, then `warmup` untimed and `reps` timed recycled iterations
 * (recycled_render + residual + grad_forward) at params t with `workers` threads.
 * stats[0]=segments S, [1]=trace s, [2]=sort s, [3]=mean forward s, [4]=mean grad s,
 * [5]=events, [6]=live LE spans, [7]=live path spans, [8]=vertices. */
int ref_time_iteration(const prc_scene_desc* d, const prc_gpu_params* ref_params,
                       const prc_gpu_params* t_params, uint64_t n, uint64_t seed, int workers,
                       int warmup, int reps, double* stats) {
    try {
        Scene s = make_scene(d);
        bind(s, make_params(s, ref_params));
        RenderOptions o;
        o.n_paths = n;
        o.seed = seed;
        o.workers = workers;
        o.keep_paths = true;
        double t0 = now();
        RenderResult rr = render(s, o);
        double t1 = now();
        sort_by_size(*rr.store);
        double t2 = now();
        const PathStore& st = *rr.store;
        ParamSet t = make_params(s, t_params);
        double S = 0, E = 0, le = 0, ps = 0, V = 0;
        for (const auto& r : st.records) {
            S += r.size();
            V += static_cast<double>(r.vertices.size());
            E += static_cast<double>(r.events.size());
            le += static_cast<double>(r.le_spans.size());
            for (int b = 1; b < r.size(); ++b)
                ps += r.vertices[static_cast<size_t>(b)].span_end -
                      r.vertices[static_cast<size_t>(b)].span_begin;
        }
        ImageSet gt = rr.images;
        for (auto& im : gt)
            for (auto& px : im.data) px *= 0.9;
        double fwd = 0, grd = 0;
        for (int k = -warmup; k < reps; ++k) {
            double a = now();
            ImageSet f = recycled_render(s, st, t, workers);
            double b = now();
            ImageSet res = f;
            for (size_t i = 0; i < res.size(); ++i)
                for (size_t p = 0; p < res[i].data.size(); ++p) res[i].data[p] -= gt[i].data[p];
            EvalOptions go;
            go.workers = workers;
            go.pixel_weights = &res;
            SparseGradient g = grad_forward(s, st, t, go);
            double c = now();
            (void)g;
            if (k < 0) continue;  // untimed warm-up iterations
            fwd += b - a;
            grd += c - b;
        }
        stats[0] = S;
        stats[1] = t1 - t0;
        stats[2] = t2 - t1;
        stats[3] = fwd / reps;
        stats[4] = grd / reps;
        stats[5] = E;
        stats[6] = le;
        stats[7] = ps;
        stats[8] = V;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* reconstruct() with one stage (inverse.cpp:154-263). */
int ref_reconstruct(const prc_scene_desc* d, const prc_gpu_params* initial, const double* gt,
                    double alpha, const double* step_scale, int n_step_scale, uint64_t seed,
                    uint64_t n_paths, int recycle_period, int max_iterations, int workers,
                    double* loss_hist, double* beta_out, double* kappa_out, double* gamma_out,
                    uint64_t* phases_out) {
    try {
        Scene s = make_scene(d);
        ParamSet init = make_params(s, initial);
        ImageSet g = images_from(s, gt);
        ReconstructOptions ro;
        ro.adam.alpha = alpha;
        for (int i = 0; i < n_step_scale; ++i) ro.adam.step_scale.push_back(step_scale[i]);
        ro.schedule.recycle_period = recycle_period;
        ro.schedule.max_iterations = max_iterations;
        Stage st;
        st.n_paths = n_paths;
        ro.schedule.stages = {st};
        ro.seed = seed;
        ro.workers = workers;
        ReconstructResult r = reconstruct(s, g, init, ro);
        for (size_t i = 0; i < r.history.size(); ++i) loss_hist[i] = r.history[i].loss;
        if (beta_out)
            for (size_t v = 0; v < r.params.beta.size(); ++v) beta_out[v] = r.params.beta[v];
        if (kappa_out) *kappa_out = r.params.kappa_s;
        if (gamma_out) *gamma_out = r.params.gamma;
        if (phases_out) *phases_out = r.sampling_phases;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* adam_step (inverse.cpp:41-67) applied `steps` times with the given gradients (steps x n,
 * dense over the flattened unknowns).  phong: the unknowns are (kappa_s, gamma); else beta.
 * x_hist: steps x n unknowns after each update. */
int ref_adam(uint64_t n, const double* x0, const double* grads, int steps, double alpha, double eta1,
             double eta2, double eps, int nonneg, const double* step_scale, int n_ss, int phong,
             double* x_hist) {
    try {
        OptState st;
        if (phong) {
            st.params.kappa_s = x0[0];
            st.params.gamma = x0[1];
        } else {
            st.params.beta.assign(x0, x0 + n);
        }
        AdamConfig cfg;
        cfg.alpha = alpha;
        cfg.eta1 = eta1;
        cfg.eta2 = eta2;
        cfg.eps_guard = eps;
        cfg.project_nonneg = nonneg != 0;
        for (int i = 0; i < n_ss; ++i) cfg.step_scale.push_back(step_scale[i]);
        for (int k = 0; k < steps; ++k) {
            SparseGradient g;
            g.kind = phong ? SparseGradient::Kind::Phong : SparseGradient::Kind::Tomography;
            for (uint64_t i = 0; i < n; ++i) g.add(static_cast<int>(i), grads[k * n + i]);
            adam_step(st, g, cfg);
            for (uint64_t i = 0; i < n; ++i)
                x_hist[k * n + i] = phong ? (i == 0 ? st.params.kappa_s : st.params.gamma) : st.params.beta[i];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* loss (inverse.cpp:11-23) of images F against gt (scene's detector layout). */
int ref_loss(const prc_scene_desc* d, const double* F, const double* gt, double* out) {
    try {
        Scene s = make_scene(d);
        *out = loss(images_from(s, F), images_from(s, gt));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* reconstruct() with a stage schedule (inverse.cpp:154-263).  stages: n_stages x
 * (rows, cols) in stage_rc and n_paths in stage_n.  Per iteration: loss and stage. */
int ref_reconstruct_schedule(const prc_scene_desc* d, const prc_gpu_params* initial, const double* gt,
                             double alpha, uint64_t seed, int n_stages, const int* stage_rc,
                             const uint64_t* stage_n, int recycle_period, int max_iterations, int window,
                             double rel, int workers, double* loss_hist, int* stage_hist, uint64_t* phases_out,
                             uint64_t* truncated_out) {
    try {
        Scene s = make_scene(d);
        ParamSet init = make_params(s, initial);
        ImageSet g = images_from(s, gt);
        ReconstructOptions ro;
        ro.adam.alpha = alpha;
        ro.schedule.recycle_period = recycle_period;
        ro.schedule.max_iterations = max_iterations;
        ro.schedule.saturation_window = window;
        ro.schedule.saturation_rel_improvement = rel;
        for (int k = 0; k < n_stages; ++k) {
            Stage st;
            st.rows = stage_rc[2 * k];
            st.cols = stage_rc[2 * k + 1];
            st.n_paths = stage_n[k];
            ro.schedule.stages.push_back(st);
        }
        ro.seed = seed;
        ro.workers = workers;
        ReconstructResult r = reconstruct(s, g, init, ro);
        for (size_t i = 0; i < r.history.size(); ++i) {
            loss_hist[i] = r.history[i].loss;
            stage_hist[i] = r.history[i].stage;
        }
        *phases_out = r.sampling_phases;
        *truncated_out = r.truncated_paths;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* space_carve (inverse.cpp:69-101): mask (V bytes) and initial beta (V doubles). */
int ref_space_carve(const prc_scene_desc* d, const double* gt, double thr, double fill, uint8_t* mask,
                    double* beta) {
    try {
        Scene s = make_scene(d);
        CarveResult r = space_carve(s, images_from(s, gt), thr, fill);
        for (size_t v = 0; v < r.mask.size(); ++v) {
            mask[v] = r.mask[v];
            beta[v] = r.initial.beta[v];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* downsample_images (inverse.cpp:116-133) over n images of rows[k] x cols[k]. */
int ref_downsample(int n, const int* rows, const int* cols, const double* in, int ro, int co, double* out) {
    try {
        ImageSet im;
        size_t k = 0;
        for (int i = 0; i < n; ++i) {
            Image x = Image::zeros(rows[i], cols[i]);
            for (auto& px : x.data) px = in[k++];
            im.push_back(std::move(x));
        }
        ImageSet r = downsample_images(im, ro, co);
        size_t o = 0;
        for (const auto& x : r)
            for (double px : x.data) out[o++] = px;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* metrics (inverse.cpp:103-114). */
int ref_metrics(const double* e, const double* t, uint64_t n, double* eps, double* delta) {
    try {
        Metrics m = metrics(std::vector<double>(e, e + n), std::vector<double>(t, t + n));
        *eps = m.eps;
        *delta = m.delta;
        return 0;
    } catch (const std::exception& ex) {
        return fail(ex);
    }
}

/* save_grid (io.cpp:59-76) and save_csv (io.cpp:147-155) writers, for byte comparisons. */
int ref_save_grid(const char* path, const int* dims, const double* origin, const double* vs, int unit,
                  const double* values) {
    try {
        VoxelGridField f;
        f.geom.dims = {dims[0], dims[1], dims[2]};
        f.geom.origin = {origin[0], origin[1], origin[2]};
        f.geom.voxel_size = {vs[0], vs[1], vs[2]};
        f.values.assign(values, values + (size_t)dims[0] * dims[1] * dims[2]);
        save_grid(f, static_cast<LengthUnit>(unit), path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_save_csv(const char* path, int n, const int* iter, const double* time_s, const double* loss,
                 const double* eps, const double* delta, const int* stage) {
    try {
        std::vector<IterationLog> rows((size_t)n);
        for (int i = 0; i < n; ++i) rows[(size_t)i] = {iter[i], time_s[i], loss[i], eps[i], delta[i], stage[i]};
        save_csv(rows, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* load_scene (io.cpp:190-278) + render (transport.cpp:405-454): images of a JSON scene. */
int ref_render_json(const char* path, uint64_t n, uint64_t seed, double* images, uint64_t cap) {
    try {
        Scene s = load_scene(path);
        RenderOptions o;
        o.n_paths = n;
        o.seed = seed;
        o.workers = 1;
        RenderResult r = render(s, o);
        size_t k = 0;
        for (const auto& im : r.images)
            for (double px : im.data) {
                if (k >= cap) throw std::runtime_error("ref_render_json: capacity");
                images[k++] = px;
            }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/* save_pfm / load_pfm (io.cpp:94-129). */
int ref_save_pfm(const char* path, int rows, int cols, const double* data) {
    try {
        Image im = Image::zeros(rows, cols);
        for (size_t i = 0; i < im.data.size(); ++i) im.data[i] = data[i];
        save_pfm(im, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_load_pfm(const char* path, int* rows, int* cols, double* data, uint64_t cap) {
    try {
        Image im = load_pfm(path);
        *rows = im.rows;
        *cols = im.cols;
        if (data) {
            if (im.data.size() > cap) throw std::runtime_error("ref_load_pfm: capacity");
            for (size_t i = 0; i < im.data.size(); ++i) data[i] = im.data[i];
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
