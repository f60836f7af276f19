/*
 * pathrec_oracle.c — TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the reference
 * hot path (see pathrec_oracle.h).  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  Floating-point expressions keep
 * the reference's association order and are compiled with -ffp-contract=off (the
 * reference object code contains no FMA), so the restatement is bit-identical to the
 * reference on the same host libm; tests/test_oracle.py enforces that.
 */
#include "pathrec_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PI 3.14159265358979323846
#define FOUR_PI (4.0 * PI) /* phase.hpp:12 */
#define LOG_CLAMP 700.0    /* pathstore.cpp:18 */
#define SELF_HIT_EPS 1e-9  /* transport.cpp:14 */
#define CHUNK 4096         /* parallel.hpp:11 */

static _Thread_local char g_err[512];
static int fail(const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}
const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- vec3.hpp:8-57 */
typedef struct {
    double x, y, z;
} V3;
static V3 v3(double x, double y, double z) {
    V3 r = {x, y, z};
    return r;
}
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V3 vmul(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
static V3 vdiv(V3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }
static double vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static double vnorm(V3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
static V3 vnormalized(V3 a) { return vdiv(a, vnorm(a)); }
static V3 vcross(V3 a, V3 b) {
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vget(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static V3 from(prc_vec3 p) { return v3(p.x, p.y, p.z); }

/* Frame (vec3.hpp:41-57) */
typedef struct {
    V3 u, v, w;
} Frame;
static Frame frame_of(V3 w) {
    Frame f;
    f.w = w;
    const double sign = copysign(1.0, w.z);
    const double a = -1.0 / (sign + w.z);
    const double b = w.x * w.y * a;
    f.u = v3(1.0 + sign * w.x * w.x * a, sign * b, -sign * w.x);
    f.v = v3(b, sign + w.y * w.y * a, -w.y);
    return f;
}
static V3 frame_from_local(const Frame* f, double cos_theta, double phi) {
    double t = 1.0 - cos_theta * cos_theta;
    const double sin_theta = sqrt(t > 0.0 ? t : 0.0); /* std::max(0.0, .) */
    return vadd(vadd(vmul(f->u, sin_theta * cos(phi)), vmul(f->v, sin_theta * sin(phi))),
                vmul(f->w, cos_theta));
}

/* ---------------------------------------------------------------- rng.hpp:11-61 */
typedef struct {
    uint32_t key[2], ctr[4], block[4];
    int have;
} Rng;
static void rng_init(Rng* r, uint64_t seed, uint64_t stream) {
    r->key[0] = (uint32_t)seed;
    r->key[1] = (uint32_t)(seed >> 32);
    r->ctr[0] = 0;
    r->ctr[1] = 0;
    r->ctr[2] = (uint32_t)stream;
    r->ctr[3] = (uint32_t)(stream >> 32);
    r->have = 0;
}
static void rng_bump(Rng* r) { /* rng.hpp:42-55 */
    uint32_t c[4] = {r->ctr[0], r->ctr[1], r->ctr[2], r->ctr[3]};
    uint32_t k0 = r->key[0], k1 = r->key[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1, n3 = (uint32_t)p0;
        c[0] = n0;
        c[1] = n1;
        c[2] = n2;
        c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    if (++r->ctr[0] == 0 && ++r->ctr[1] == 0) ++r->ctr[2];
    memcpy(r->block, c, sizeof c);
}
static uint32_t rng_u32(Rng* r) { /* rng.hpp:17-23 */
    if (r->have == 0) {
        rng_bump(r);
        r->have = 4;
    }
    return r->block[4 - r->have--];
}
static double rng_double(Rng* r) { /* rng.hpp:25-31 */
    const uint64_t hi = rng_u32(r);
    const uint64_t u = (hi << 32) | rng_u32(r);
    return (double)(u >> 11) * 0x1.0p-53;
}
int orc_philox(uint64_t seed, uint64_t stream, uint64_t n, uint32_t* out) {
    Rng r;
    rng_init(&r, seed, stream);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_u32(&r);
    return 0;
}

/* --------------------------------------------------------- scene (scene.hpp/.cpp) */
typedef struct {
    V3 pos, dir, up, right, upx;
    int rows, cols;
    double hw, hh;
} Det;
typedef struct {
    const double* ext;
    double albedo;
    int kind;
    double g;
    int unknown;
} Sp;
typedef struct {
    int dims[3];
    V3 origin, vs;
} Grid;
typedef struct {
    V3 bmin, bmax;
    Grid grid;
    int has_medium;
    int n_sp;
    Sp sp[16];
    int n_surf;
    const prc_surface_desc* surf;
    prc_light_desc light;
    int n_det;
    Det* det;
    int unknown, target;
    int V;
    size_t n_pix;
    size_t* img_off;
} Scene;

static void det_finalize(Det* d, const prc_detector_desc* dd) { /* scene.cpp:8-14 */
    d->pos = from(dd->position);
    d->dir = vnormalized(from(dd->direction));
    d->up = from(dd->up);
    d->right = vnormalized(vcross(d->dir, d->up));
    d->upx = vcross(d->right, d->dir);
    d->rows = dd->rows;
    d->cols = dd->cols;
    d->hw = tan(0.5 * dd->fov);
    d->hh = d->hw * (double)dd->rows / (double)dd->cols;
}

static int pixel_of(const Det* d, V3 p) { /* scene.cpp:16-28 */
    const V3 w = vsub(p, d->pos);
    const double depth = vdot(w, d->dir);
    if (depth <= 0.0) return -1;
    const double u = vdot(w, d->right) / depth;
    const double v = vdot(w, d->upx) / depth;
    if (u < -d->hw || u >= d->hw || v < -d->hh || v >= d->hh) return -1;
    int col = (int)((u + d->hw) / (2.0 * d->hw) * d->cols);
    int row = (int)((d->hh - v) / (2.0 * d->hh) * d->rows);
    if (col >= d->cols) col = d->cols - 1;
    if (row >= d->rows) row = d->rows - 1;
    return row * d->cols + col;
}

static int scene_build(Scene* s, const prc_scene_desc* d) {
    memset(s, 0, sizeof *s);
    if (d->n_species > 16) return fail("scene: too many species");
    s->bmin = from(d->bounds_min);
    s->bmax = from(d->bounds_max);
    for (int a = 0; a < 3; ++a) s->grid.dims[a] = d->dims[a];
    s->grid.origin = from(d->grid_origin);
    s->grid.vs = from(d->voxel_size);
    s->has_medium = d->n_species > 0;
    s->V = s->has_medium ? d->dims[0] * d->dims[1] * d->dims[2] : 0;
    s->n_sp = d->n_species;
    s->unknown = -1;
    for (int j = 0; j < d->n_species; ++j) {
        s->sp[j].ext = d->species[j].extinction;
        s->sp[j].albedo = d->species[j].albedo;
        s->sp[j].kind = d->species[j].phase_kind;
        s->sp[j].g = d->species[j].g;
        s->sp[j].unknown = d->species[j].unknown;
        if (d->species[j].unknown && s->unknown < 0) s->unknown = j; /* scene.cpp:59-63 */
    }
    s->n_surf = d->n_surfaces;
    s->surf = d->surfaces;
    s->target = -1;
    for (int k = 0; k < d->n_surfaces; ++k)
        if (d->surfaces[k].target && s->target < 0) s->target = k; /* scene.cpp:65-69 */
    s->light = d->light;
    if (s->light.kind == PRC_LIGHT_SUN) { /* Scene::finalize, scene.cpp:71-74 */
        V3 dn = vnormalized(from(s->light.direction));
        s->light.direction.x = dn.x;
        s->light.direction.y = dn.y;
        s->light.direction.z = dn.z;
    }
    s->n_det = d->n_detectors;
    s->det = (Det*)calloc((size_t)(d->n_detectors > 0 ? d->n_detectors : 1), sizeof(Det));
    s->img_off = (size_t*)calloc((size_t)d->n_detectors + 1, sizeof(size_t));
    for (int k = 0; k < d->n_detectors; ++k) {
        det_finalize(&s->det[k], &d->detectors[k]);
        s->img_off[k + 1] = s->img_off[k] + (size_t)d->detectors[k].rows * d->detectors[k].cols;
    }
    s->n_pix = s->img_off[d->n_detectors];
    return 0;
}
static void scene_free(Scene* s) {
    free(s->det);
    free(s->img_off);
}

/* GridGeometry::voxel_of (grid.hpp:40-54) */
static int voxel_of(const Grid* g, V3 p) {
    int idx[3];
    const V3 rel = vsub(p, g->origin);
    const double r[3] = {rel.x / g->vs.x, rel.y / g->vs.y, rel.z / g->vs.z};
    for (int a = 0; a < 3; ++a) {
        int i = (int)r[a];
        if (r[a] < 0.0) return -1;
        if (i >= g->dims[a]) {
            if (r[a] <= (double)g->dims[a])
                i = g->dims[a] - 1;
            else
                return -1;
        }
        idx[a] = i;
    }
    return idx[0] + g->dims[0] * (idx[1] + g->dims[1] * idx[2]);
}

/* ------------------------------------------------- walk_voxels, traverse.hpp:45-116 */
typedef int (*WalkFn)(void* ctx, int v, double ta, double tb);
static void walk_voxels(const Grid* g, V3 origin, V3 dir, double max_distance, WalkFn f,
                        void* ctx) {
    if (max_distance <= 0.0) return;
    const double bmin[3] = {g->origin.x, g->origin.y, g->origin.z};
    const double bmax[3] = {g->origin.x + g->dims[0] * g->vs.x, g->origin.y + g->dims[1] * g->vs.y,
                            g->origin.z + g->dims[2] * g->vs.z}; /* grid.hpp:27-30 */
    double t0 = 0.0, t1 = max_distance;
    const double o[3] = {origin.x, origin.y, origin.z};
    const double d[3] = {dir.x, dir.y, dir.z};
    for (int a = 0; a < 3; ++a) {
        if (d[a] == 0.0) {
            if (o[a] < bmin[a] || o[a] > bmax[a]) return;
            continue;
        }
        const double inv = 1.0 / d[a];
        double ta = (bmin[a] - o[a]) * inv;
        double tb = (bmax[a] - o[a]) * inv;
        if (ta > tb) {
            double tmp = ta;
            ta = tb;
            tb = tmp;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t0 > t1) return;
    }
    if (t1 <= t0) return;
    int idx[3], step[3];
    double tmax[3], tdelta[3];
    for (int a = 0; a < 3; ++a) {
        const double vs = vget(g->vs, a);
        const double pa = o[a] + t0 * d[a];
        double r = (pa - bmin[a]) / vs;
        int i = (int)r;
        if (i < 0) i = 0;
        if (i >= g->dims[a]) i = g->dims[a] - 1;
        if (r - i == 0.0 && d[a] < 0.0 && i > 0) --i;
        idx[a] = i;
        if (d[a] > 0.0) {
            step[a] = 1;
            tdelta[a] = vs / d[a];
            tmax[a] = ((bmin[a] + (i + 1) * vs) - o[a]) / d[a];
        } else if (d[a] < 0.0) {
            step[a] = -1;
            tdelta[a] = -vs / d[a];
            tmax[a] = ((bmin[a] + i * vs) - o[a]) / d[a];
        } else {
            step[a] = 0;
            tdelta[a] = 0.0;
            tmax[a] = t1 + 1.0;
        }
    }
    double t = t0;
    while (t < t1) {
        int axis = 0;
        if (tmax[1] < tmax[axis]) axis = 1;
        if (tmax[2] < tmax[axis]) axis = 2;
        double t_next = tmax[axis];
        if (t_next > t1) t_next = t1;
        if (t_next > t) {
            const int v = idx[0] + g->dims[0] * (idx[1] + g->dims[1] * idx[2]);
            if (!f(ctx, v, t, t_next)) return;
        }
        t = tmax[axis];
        idx[axis] += step[axis];
        if (idx[axis] < 0 || idx[axis] >= g->dims[axis]) return;
        tmax[axis] += tdelta[axis];
    }
}

typedef struct {
    uint32_t* vox;
    double* len;
    uint64_t cap, k;
    uint32_t c;
} WalkOut;
static int walk_out_cb(void* p, int v, double ta, double tb) {
    WalkOut* w = (WalkOut*)p;
    if (w->vox && w->k < w->cap) {
        w->vox[w->k] = (uint32_t)v;
        w->len[w->k] = tb - ta;
    }
    w->k++;
    w->c++;
    return 1;
}
int orc_walk(const prc_scene_desc* d, uint64_t n, const double* rays, uint32_t* counts,
             uint32_t* vox, double* len, uint64_t cap) {
    Grid g;
    for (int a = 0; a < 3; ++a) g.dims[a] = d->dims[a];
    g.origin = from(d->grid_origin);
    g.vs = from(d->voxel_size);
    WalkOut w = {vox, len, cap, 0, 0};
    for (uint64_t i = 0; i < n; ++i) {
        const double* r = rays + 7 * i;
        w.c = 0;
        walk_voxels(&g, v3(r[0], r[1], r[2]), v3(r[3], r[4], r[5]), r[6], walk_out_cb, &w);
        counts[i] = w.c;
    }
    return 0;
}
int orc_pixel_of(const prc_scene_desc* d, int det, uint64_t n, const double* pts, int32_t* out) {
    Scene s;
    if (scene_build(&s, d)) return 1;
    for (uint64_t i = 0; i < n; ++i)
        out[i] = pixel_of(&s.det[det], v3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
    scene_free(&s);
    return 0;
}

/* ------------------------------------------------------- phase / brdf (phase.hpp) */
static double phase_eval(const Sp* sp, double c) { /* phase.hpp:28-33 */
    if (sp->kind == PRC_PHASE_RAYLEIGH) return 3.0 * (1.0 + c * c) / (16.0 * PI);
    const double g = sp->g;
    const double denom = 1.0 + g * g - 2.0 * g * c;
    return (1.0 - g * g) / (FOUR_PI * denom * sqrt(denom));
}
static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }
static double phase_sample_cos(const Sp* sp, double u) { /* phase.hpp:36-42, 55-60 */
    if (sp->kind == PRC_PHASE_RAYLEIGH) {
        const double q = 4.0 - 8.0 * u;
        const double disc = sqrt(q * q / 4.0 + 1.0);
        const double x = cbrt(-q / 2.0 + disc) + cbrt(-q / 2.0 - disc);
        return clampd(x, -1.0, 1.0);
    }
    const double g = sp->g;
    if (fabs(g) < 1e-9) return 2.0 * u - 1.0;
    const double s = (1.0 - g * g) / (1.0 - g + 2.0 * g * u);
    double c = (1.0 + g * g - s * s) / (2.0 * g);
    return clampd(c, -1.0, 1.0);
}
typedef struct {
    int phong;
    double albedo, kappa, gamma;
} Brdf;
static double brdf_eval(const Brdf* b, double cos_r) { /* brdf.hpp:21-24, 60-62 */
    if (!b->phong) return b->albedo / PI;
    const double c = clampd(cos_r, 0.0, 1.0);
    return 1.0 - b->kappa + b->kappa * pow(c, b->gamma);
}
static double phong_dk(const Brdf* b, double cos_r) { /* brdf.hpp:21-24 */
    const double c = clampd(cos_r, 0.0, 1.0);
    return -1.0 + pow(c, b->gamma);
}
static double phong_dg(const Brdf* b, double cos_r) { /* brdf.hpp:26-30 */
    const double c = clampd(cos_r, 0.0, 1.0);
    if (c <= 0.0) return 0.0;
    return b->kappa * pow(c, b->gamma) * log(c);
}

/* ------------------------------------------------------------------- records */
typedef struct {
    V3 pos;
    double cos_theta, cos_in, cos_out;
    uint32_t span_begin, span_end;
    int32_t voxel;
    int16_t surface;
    int8_t species;
    uint8_t kind; /* EventKind: 0 emission, 1 volume, 2 surface, 3 escape */
} Vtx;
typedef struct {
    uint32_t vertex;
    uint16_t detector;
    int32_t pixel;
    double cos_le, geom;
    uint32_t span_begin, span_end;
} Evt;
typedef struct {
    uint32_t voxel;
    double length;
} Span;
typedef struct {
    uint64_t stream;
    V3 dir0;
    int truncated;
    Vtx* v;
    uint32_t nv, cv;
    Span* sp;
    uint32_t ns, cs;
    Evt* ev;
    uint32_t ne, ce;
    Span* le;
    uint32_t nl, cl;
} Rec;
struct orc_store {
    Rec* rec;
    uint64_t n;
    uint32_t* by_stream;
    int sorted;
    uint64_t generation, seed;
    double* ref_beta;
    uint64_t n_ref_beta;
    double ref_kappa, ref_gamma;
};

#define GROW(arr, n, cap, T)                                          \
    do {                                                              \
        if ((n) >= (cap)) {                                           \
            (cap) = (cap) ? 2 * (cap) : 8;                            \
            (arr) = (T*)realloc((arr), (size_t)(cap) * sizeof(T));    \
        }                                                             \
    } while (0)

static void rec_free(Rec* r) {
    free(r->v);
    free(r->sp);
    free(r->ev);
    free(r->le);
    memset(r, 0, sizeof *r);
}
static void push_span(Span** a, uint32_t* n, uint32_t* c, uint32_t vox, double len) {
    GROW(*a, *n, *c, Span);
    (*a)[*n].voxel = vox;
    (*a)[*n].length = len;
    (*n)++;
}
static int rec_size(const Rec* r) { return (int)r->nv - 1; } /* transport.hpp:57 */

/* ------------------------------------------------------------- transport.cpp */
static double aabb_exit(V3 lo3, V3 hi3, V3 o3, V3 d3) { /* transport.cpp:16-29 */
    double t1 = INFINITY;
    const double o[3] = {o3.x, o3.y, o3.z}, d[3] = {d3.x, d3.y, d3.z};
    const double lo[3] = {lo3.x, lo3.y, lo3.z}, hi[3] = {hi3.x, hi3.y, hi3.z};
    for (int a = 0; a < 3; ++a) {
        if (d[a] > 0.0) {
            double c = (hi[a] - o[a]) / d[a];
            t1 = c < t1 ? c : t1; /* std::min(t1, c) */
        } else if (d[a] < 0.0) {
            double c = (lo[a] - o[a]) / d[a];
            t1 = c < t1 ? c : t1;
        }
    }
    return t1;
}
static int hit_sphere(const prc_surface_desc* s, V3 o, V3 d, double tmin, double tmax,
                      double* out) { /* transport.cpp:31-42 */
    const V3 oc = vsub(o, from(s->center));
    const double b = vdot(oc, d);
    const double c = vdot(oc, oc) - s->radius * s->radius;
    const double disc = b * b - c;
    if (disc < 0.0) return 0;
    const double sq = sqrt(disc);
    double t = -b - sq;
    if (t < tmin) t = -b + sq;
    if (t < tmin || t > tmax) return 0;
    *out = t;
    return 1;
}
static int hit_face(const prc_surface_desc* f, V3 o3, V3 d3, double tmin, double tmax,
                    double* out) { /* transport.cpp:44-56 */
    const double o[3] = {o3.x, o3.y, o3.z}, d[3] = {d3.x, d3.y, d3.z};
    const int a = f->axis;
    if (d[a] == 0.0) return 0;
    const double t = (f->coord - o[a]) / d[a];
    if (t < tmin || t > tmax) return 0;
    const int u = (a + 1) % 3, v = (a + 2) % 3;
    const double pu = o[u] + t * d[u];
    const double pv = o[v] + t * d[v];
    if (pu < f->lo[0] || pu > f->hi[0] || pv < f->lo[1] || pv > f->hi[1]) return 0;
    *out = t;
    return 1;
}
static int intersect_surfaces(const Scene* s, V3 o, V3 d, double tmin, double tmax, int exclude,
                              double* t_out, int* s_out) { /* transport.cpp:147-161 */
    int found = 0;
    double best = 0.0;
    int bs = -1;
    for (int k = 0; k < s->n_surf; ++k) {
        if (k == exclude) continue;
        double t;
        int hit = s->surf[k].kind == PRC_SURF_SPHERE ? hit_sphere(&s->surf[k], o, d, tmin, tmax, &t)
                                                    : hit_face(&s->surf[k], o, d, tmin, tmax, &t);
        if (hit && (!found || t < best)) {
            found = 1;
            best = t;
            bs = k;
        }
    }
    if (found) {
        if (t_out) *t_out = best;
        if (s_out) *s_out = bs;
    }
    return found;
}
static V3 normal_at(const prc_surface_desc* s, V3 p) { /* scene.cpp:50-57 */
    if (s->kind == PRC_SURF_SPHERE) return vnormalized(vsub(p, from(s->center)));
    V3 n = v3(0.0, 0.0, 0.0);
    if (s->axis == 0)
        n.x = s->normal_sign;
    else if (s->axis == 1)
        n.y = s->normal_sign;
    else
        n.z = s->normal_sign;
    return n;
}

/* Per-voxel species extinction under the evaluated parameters (transport.hpp:72-76). */
typedef struct {
    const double* sp[16];
} Ext;

typedef struct {
    const Scene* s;
    const Ext* ext;
    double tau, od;
    int scattered;
    Rec* rec;
    V3 o, d;
    /* outputs */
    double t_sc;
    int voxel;
} SegCtx;
static int seg_cb(void* p, int v, double ta, double tb) { /* transport.cpp:93-111 */
    SegCtx* c = (SegCtx*)p;
    double beta = 0.0;
    for (int j = 0; j < c->s->n_sp; ++j) beta += c->ext->sp[j][v];
    const double seg_od = beta * (tb - ta);
    if (c->tau >= 0.0 && c->od + seg_od >= c->tau && beta > 0.0) {
        const double t_sc = ta + (c->tau - c->od) / beta;
        if (c->rec) push_span(&c->rec->sp, &c->rec->ns, &c->rec->cs, (uint32_t)v, t_sc - ta);
        c->t_sc = t_sc;
        c->voxel = v;
        c->scattered = 1;
        return 0;
    }
    c->od += seg_od;
    if (c->rec) push_span(&c->rec->sp, &c->rec->ns, &c->rec->cs, (uint32_t)v, tb - ta);
    return 1;
}
enum { END_SCATTER, END_SURFACE, END_ESCAPE };
typedef struct {
    int kind;
    V3 point;
    double distance;
    int surface, voxel;
} SegEnd;
static SegEnd walk_segment(const Scene* s, const Ext* ext, V3 o, V3 d, double tau, Rec* rec,
                           int exclude) { /* transport.cpp:74-114 */
    SegEnd out;
    double t_lim = aabb_exit(s->bmin, s->bmax, o, d);
    out.kind = END_ESCAPE;
    out.surface = -1;
    out.voxel = -1;
    double th;
    int sh;
    if (intersect_surfaces(s, o, d, SELF_HIT_EPS, t_lim, exclude, &th, &sh)) {
        t_lim = th;
        out.kind = END_SURFACE;
        out.surface = sh;
    }
    out.distance = t_lim;
    out.point = vadd(o, vmul(d, t_lim));
    if (!s->has_medium) return out;
    SegCtx c = {s, ext, tau, 0.0, 0, rec, o, d, 0.0, -1};
    walk_voxels(&s->grid, o, d, t_lim, seg_cb, &c);
    if (c.scattered) {
        out.kind = END_SCATTER;
        out.distance = c.t_sc;
        out.point = vadd(o, vmul(d, c.t_sc));
        out.surface = -1;
        out.voxel = c.voxel;
    }
    return out;
}

static V3 uniform_sphere_dir(Rng* r) { /* transport.cpp:58-63 */
    const double z = 1.0 - 2.0 * rng_double(r);
    const double phi = 2.0 * PI * rng_double(r);
    double t = 1.0 - z * z;
    const double rr = sqrt(t > 0.0 ? t : 0.0);
    return v3(rr * cos(phi), rr * sin(phi), z);
}

typedef struct {
    Rec* rec;
} LeCtx;
static int le_cb(void* p, int v, double ta, double tb) {
    Rec* r = ((LeCtx*)p)->rec;
    push_span(&r->le, &r->nl, &r->cl, (uint32_t)v, tb - ta);
    return 1;
}
static void add_events(const Scene* s, Rec* rec, uint32_t vi, V3 dir_ref, int own_surface,
                       const V3* normal) { /* transport.cpp:218-254 */
    const Vtx vr = rec->v[vi];
    for (int d = 0; d < s->n_det; ++d) {
        const Det* det = &s->det[d];
        const int pixel = pixel_of(det, vr.pos);
        if (pixel < 0) continue;
        const V3 to_det = vsub(det->pos, vr.pos);
        const double r = vnorm(to_det);
        if (r <= 0.0) continue;
        const V3 w = vmul(to_det, 1.0 / r);
        double geom = 1.0 / (r * r);
        if (normal) {
            const double c_out = vdot(*normal, w);
            if (c_out <= 0.0) continue;
            geom *= c_out;
        }
        if (intersect_surfaces(s, vr.pos, w, SELF_HIT_EPS, r - SELF_HIT_EPS, own_surface, NULL,
                               NULL))
            continue;
        GROW(rec->ev, rec->ne, rec->ce, Evt);
        Evt* e = &rec->ev[rec->ne];
        e->vertex = vi;
        e->detector = (uint16_t)d;
        e->pixel = pixel;
        e->cos_le = vdot(dir_ref, w);
        e->geom = geom;
        e->span_begin = rec->nl;
        if (s->has_medium) {
            LeCtx lc = {rec};
            walk_voxels(&s->grid, vr.pos, w, r, le_cb, &lc);
        }
        rec->ev[rec->ne].span_end = rec->nl;
        rec->ne++;
    }
}

static Vtx vtx_default(void) {
    Vtx v;
    memset(&v, 0, sizeof v);
    v.cos_theta = 1.0;
    v.cos_in = 1.0;
    v.cos_out = 1.0;
    v.voxel = -1;
    v.surface = -1;
    v.species = -1;
    v.kind = 0;
    return v;
}
static void push_vtx(Rec* r, Vtx v) {
    GROW(r->v, r->nv, r->cv, Vtx);
    r->v[r->nv++] = v;
}

static int trace_path(const Scene* s, const Ext* ext, uint64_t seed, uint64_t stream,
                      int max_bounces, int max_events, Rec* rec) { /* transport.cpp:258-345 */
    Rng rng;
    rng_init(&rng, seed, stream);
    memset(rec, 0, sizeof *rec);
    rec->stream = stream;
    V3 pos, dir;
    if (s->light.kind == PRC_LIGHT_POINT) {
        pos = from(s->light.position);
        dir = uniform_sphere_dir(&rng);
    } else {
        const double u = rng_double(&rng), v = rng_double(&rng);
        pos = v3(s->bmin.x + u * (s->bmax.x - s->bmin.x), s->bmin.y + v * (s->bmax.y - s->bmin.y),
                 s->bmax.z);
        dir = from(s->light.direction);
    }
    rec->dir0 = dir;
    Vtx v0 = vtx_default();
    v0.pos = pos;
    v0.kind = 0;
    if (s->has_medium) v0.voxel = voxel_of(&s->grid, pos);
    push_vtx(rec, v0);
    int cur_surface = -1, interactions = 0;
    for (;;) {
        const double tau = s->has_medium ? -log1p(-rng_double(&rng)) : -1.0;
        const uint32_t span_begin = rec->ns;
        const SegEnd end = walk_segment(s, ext, pos, dir, tau, rec, cur_surface);
        Vtx vr = vtx_default();
        vr.pos = end.point;
        vr.span_begin = span_begin;
        vr.span_end = rec->ns;
        if (s->has_medium) vr.voxel = end.voxel >= 0 ? end.voxel : voxel_of(&s->grid, end.point);
        if (end.kind == END_ESCAPE) {
            vr.kind = 3;
            push_vtx(rec, vr);
            break;
        }
        const int budget = interactions >= max_bounces || (max_events >= 0 && interactions >= max_events);
        if (budget) {
            vr.kind = 3;
            push_vtx(rec, vr);
            rec->truncated = interactions >= max_bounces;
            break;
        }
        ++interactions;
        if (end.kind == END_SCATTER) {
            vr.kind = 1;
            const uint32_t vi = rec->nv;
            push_vtx(rec, vr);
            add_events(s, rec, vi, dir, -1, NULL);
            /* sample_direction, transport.cpp:178-202 */
            double beta[16], total = 0.0;
            for (int j = 0; j < s->n_sp; ++j) {
                const int vx = voxel_of(&s->grid, end.point);
                beta[j] = vx >= 0 ? ext->sp[j][vx] : 0.0;
                total += beta[j];
            }
            if (total <= 0.0) return fail("sample_direction: vacuum point");
            const double u = rng_double(&rng) * total;
            int j = 0;
            double acc = beta[0];
            while (j + 1 < s->n_sp && u >= acc) acc += beta[++j];
            const double c = phase_sample_cos(&s->sp[j], rng_double(&rng));
            const double phi = 2.0 * PI * rng_double(&rng);
            const Frame fr = frame_of(dir);
            const V3 nd = frame_from_local(&fr, c, phi);
            rec->v[vi].cos_theta = c;
            rec->v[vi].species = (int8_t)j;
            dir = nd;
            cur_surface = -1;
        } else {
            const int sidx = end.surface;
            V3 n = normal_at(&s->surf[sidx], end.point);
            if (vdot(n, dir) > 0.0) n = vmul(n, -1.0);
            const V3 wr = vsub(dir, vmul(n, 2.0 * vdot(dir, n)));
            vr.kind = 2;
            vr.surface = (int16_t)sidx;
            vr.cos_in = -vdot(n, dir);
            const uint32_t vi = rec->nv;
            push_vtx(rec, vr);
            add_events(s, rec, vi, wr, sidx, &n);
            const double u1 = rng_double(&rng), u2 = rng_double(&rng);
            const double cos_n = sqrt(1.0 - u1);
            const Frame fr = frame_of(n);
            dir = frame_from_local(&fr, cos_n, 2.0 * PI * u2);
            rec->v[vi].cos_out = cos_n;
            rec->v[vi].cos_theta = vdot(wr, dir);
            cur_surface = sidx;
        }
        pos = rec->v[rec->nv - 1].pos;
    }
    return 0;
}

/* --------------------------------------------------------- evaluation context */
typedef struct {
    const Scene* s;
    const double* t[16];
    const double* ref[16];
    double *bt_tot, *br_tot, *dbeta;
    Brdf brdf_t[64];
    double prefactor;
    int want_grad, legacy;
    const double* weights;
} Ctx;

static double emission_prefactor(const Scene* s) { /* transport.cpp:347-351 */
    if (s->light.kind == PRC_LIGHT_POINT) return FOUR_PI * s->light.radiance;
    return (s->bmax.x - s->bmin.x) * (s->bmax.y - s->bmin.y) * s->light.radiance;
}

static int make_ctx(Ctx* c, const Scene* s, const prc_gpu_params* t, const double* ref_beta,
                    int flags, const double* weights) { /* pathstore.cpp:41-82 */
    memset(c, 0, sizeof *c);
    c->s = s;
    c->prefactor = emission_prefactor(s);
    c->want_grad = (flags & PRC_EVAL_WANT_GRAD) != 0;
    c->legacy = (flags & PRC_EVAL_LEGACY_SCORE) != 0;
    c->weights = weights;
    for (int j = 0; j < s->n_sp; ++j) {
        const int unk = j == s->unknown;
        c->t[j] = unk && t && t->beta ? t->beta : s->sp[j].ext;
        c->ref[j] = unk && ref_beta ? ref_beta : s->sp[j].ext;
        if (t && t->species_beta && t->species_beta[j]) c->t[j] = t->species_beta[j];
    }
    if (s->has_medium) {
        const size_t V = (size_t)s->V;
        c->bt_tot = (double*)calloc(V, sizeof(double));
        c->br_tot = (double*)calloc(V, sizeof(double));
        c->dbeta = (double*)calloc(V, sizeof(double));
        for (size_t v = 0; v < V; ++v) {
            double bt = 0.0, br = 0.0;
            for (int j = 0; j < s->n_sp; ++j) {
                bt += c->t[j][v];
                br += c->ref[j][v];
            }
            c->bt_tot[v] = bt;
            c->br_tot[v] = br;
            c->dbeta[v] = bt - br;
        }
    }
    if (s->n_surf > 64) return fail("too many surfaces");
    for (int k = 0; k < s->n_surf; ++k) { /* transport.hpp:79-83 */
        const prc_surface_desc* sf = &s->surf[k];
        Brdf b;
        if (sf->target) {
            b.phong = 1;
            b.kappa = t ? t->kappa_s : sf->kappa_s;
            b.gamma = t ? t->gamma : sf->gamma;
            b.albedo = 0.0;
        } else {
            b.phong = sf->brdf_kind == PRC_BRDF_PHONG;
            b.kappa = sf->kappa_s;
            b.gamma = sf->gamma;
            b.albedo = sf->albedo;
        }
        c->brdf_t[k] = b;
    }
    return 0;
}
static void free_ctx(Ctx* c) {
    free(c->bt_tot);
    free(c->br_tot);
    free(c->dbeta);
}

static double scat_num_t(const Ctx* c, int vox, double cos_theta) { /* pathstore.cpp:84-88 */
    double num = 0.0;
    for (int j = 0; j < c->s->n_sp; ++j)
        num += c->s->sp[j].albedo * c->t[j][vox] * phase_eval(&c->s->sp[j], cos_theta);
    return num;
}
static double ext_num_ref(const Ctx* c, int vox, double cos_theta) { /* pathstore.cpp:90-94 */
    double num = 0.0;
    for (int j = 0; j < c->s->n_sp; ++j) num += c->ref[j][vox] * phase_eval(&c->s->sp[j], cos_theta);
    return num;
}
static double score_term(const Ctx* c, int vox, double cos_theta) { /* pathstore.cpp:97-105 */
    if (c->legacy) {
        const double bt = c->bt_tot[vox];
        return bt > 0.0 ? 1.0 / bt : 0.0;
    }
    const Sp* u = &c->s->sp[c->s->unknown];
    const double num = scat_num_t(c, vox, cos_theta);
    return num > 0.0 ? u->albedo * phase_eval(u, cos_theta) / num : 0.0;
}

typedef struct {
    double* images;
    double* grad;
    double gk, gg;
    uint64_t clamps;
    double sum_r;
} Partial;

static void eval_record(const Ctx* c, const Rec* rec, Partial* out, double** wbuf,
                        uint32_t* wcap) { /* pathstore.cpp:115-239 */
    const uint32_t n_events = rec->ne;
    if (n_events > *wcap) {
        *wcap = n_events;
        *wbuf = (double*)realloc(*wbuf, (size_t)n_events * sizeof(double));
    }
    double* wb = *wbuf;
    for (uint32_t i = 0; i < n_events; ++i) wb[i] = 0.0;
    const int medium = c->s->has_medium;
    const Scene* s = c->s;
    double log_prefix = 0.0;
    int dead = 0;
    uint32_t ei = 0;
    const int B = rec_size(rec);
    for (int b = 1; b <= B; ++b) {
        const Vtx* v = &rec->v[b];
        if (!dead && medium) {
            double diff = 0.0;
            for (uint32_t k = v->span_begin; k < v->span_end; ++k)
                diff += c->dbeta[rec->sp[k].voxel] * rec->sp[k].length;
            log_prefix -= diff;
        }
        while (ei < n_events && rec->ev[ei].vertex == (uint32_t)b) {
            const Evt* e = &rec->ev[ei];
            if (!dead) {
                double logval = -INFINITY;
                if (v->kind == 1) {
                    const double num = scat_num_t(c, v->voxel, e->cos_le);
                    const double den = c->br_tot[v->voxel];
                    if (num > 0.0 && den > 0.0) logval = log_prefix + log(num) - log(den);
                } else {
                    const double fr = brdf_eval(&c->brdf_t[v->surface], e->cos_le);
                    if (fr > 0.0) logval = log_prefix + log(fr);
                }
                if (logval != -INFINITY) {
                    if (medium) {
                        double od = 0.0;
                        for (uint32_t k = e->span_begin; k < e->span_end; ++k)
                            od += c->bt_tot[rec->le[k].voxel] * rec->le[k].length;
                        logval -= od;
                    }
                    if (logval > LOG_CLAMP || logval < -LOG_CLAMP) {
                        logval = clampd(logval, -LOG_CLAMP, LOG_CLAMP);
                        ++out->clamps;
                    }
                    const double val = exp(logval) * e->geom * c->prefactor;
                    out->images[s->img_off[e->detector] + (size_t)e->pixel] += val;
                    const double w =
                        c->weights ? c->weights[s->img_off[e->detector] + (size_t)e->pixel] : 1.0;
                    wb[ei] = val * w;
                }
            }
            ++ei;
        }
        if (dead || b == B) continue;
        if (v->kind == 1) {
            const double num = scat_num_t(c, v->voxel, v->cos_theta);
            const double den = ext_num_ref(c, v->voxel, v->cos_theta);
            if (num <= 0.0 || den <= 0.0) {
                dead = 1;
                continue;
            }
            log_prefix += log(num) - log(den);
        } else if (v->kind == 2) {
            const double fr = brdf_eval(&c->brdf_t[v->surface], v->cos_theta);
            if (fr <= 0.0) {
                dead = 1;
                continue;
            }
            log_prefix += log(PI * fr);
        }
    }
    if (!c->want_grad) return;
    const int unknown = s->unknown, target = s->target;
    double after = 0.0;
    uint32_t er = n_events;
    for (int b = B; b >= 1; --b) {
        const Vtx* v = &rec->v[b];
        double own = 0.0;
        while (er > 0 && rec->ev[er - 1].vertex == (uint32_t)b) {
            --er;
            const Evt* e = &rec->ev[er];
            const double w = wb[er];
            if (w == 0.0) continue;
            own += w;
            if (unknown >= 0) {
                for (uint32_t k = e->span_begin; k < e->span_end; ++k)
                    out->grad[rec->le[k].voxel] -= w * rec->le[k].length;
                if (v->kind == 1) out->grad[v->voxel] += w * score_term(c, v->voxel, e->cos_le);
            }
            if (target >= 0 && v->kind == 2 && v->surface == target) {
                const Brdf* ph = &c->brdf_t[v->surface];
                const double fr = brdf_eval(ph, e->cos_le);
                if (fr > 0.0) {
                    out->gk += w * phong_dk(ph, e->cos_le) / fr;
                    out->gg += w * phong_dg(ph, e->cos_le) / fr;
                }
            }
        }
        const double from_here = after + own;
        if (from_here != 0.0 && unknown >= 0)
            for (uint32_t k = v->span_begin; k < v->span_end; ++k)
                out->grad[rec->sp[k].voxel] -= from_here * rec->sp[k].length;
        if (after != 0.0) {
            if (v->kind == 1 && unknown >= 0)
                out->grad[v->voxel] += after * score_term(c, v->voxel, v->cos_theta);
            if (target >= 0 && v->kind == 2 && v->surface == target) {
                const Brdf* ph = &c->brdf_t[v->surface];
                const double fr = brdf_eval(ph, v->cos_theta);
                if (fr > 0.0) {
                    out->gk += after * phong_dk(ph, v->cos_theta) / fr;
                    out->gg += after * phong_dg(ph, v->cos_theta) / fr;
                }
            }
        }
        after = from_here;
    }
}

/* correction_factor (pathstore.cpp:269-294), for self_normalize. */
static double correction_factor(const Ctx* c, const Rec* p) {
    double lr = 0.0;
    const int B = rec_size(p);
    for (int b = 1; b <= B; ++b) {
        const Vtx* v = &p->v[b];
        if (c->dbeta)
            for (uint32_t k = v->span_begin; k < v->span_end; ++k)
                lr -= c->dbeta[p->sp[k].voxel] * p->sp[k].length;
        if (b == B) break;
        if (v->kind == 1) {
            double num = 0.0, num_t = 0.0;
            for (int j = 0; j < c->s->n_sp; ++j)
                num += c->ref[j][v->voxel] * phase_eval(&c->s->sp[j], v->cos_theta);
            for (int j = 0; j < c->s->n_sp; ++j)
                num_t += c->t[j][v->voxel] * phase_eval(&c->s->sp[j], v->cos_theta);
            if (num <= 0.0) return NAN;
            if (num_t <= 0.0) return 0.0;
            lr += log(num_t) - log(num);
        }
    }
    return exp(clampd(lr, -LOG_CLAMP, LOG_CLAMP));
}

static const Rec* g_sort_recs; /* qsort has no context argument */
static int cmp_by_stream(const void* a, const void* b) {
    const uint64_t sa = g_sort_recs[*(const uint32_t*)a].stream;
    const uint64_t sb = g_sort_recs[*(const uint32_t*)b].stream;
    return sa < sb ? -1 : (sa > sb ? 1 : 0);
}
static void rebuild_index(orc_store* st) { /* pathstore.cpp:243-249 */
    free(st->by_stream);
    st->by_stream = (uint32_t*)malloc((size_t)(st->n ? st->n : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < st->n; ++i) st->by_stream[i] = (uint32_t)i;
    g_sort_recs = st->rec;
    qsort(st->by_stream, st->n, sizeof(uint32_t), cmp_by_stream);
}

static int evaluate(const Scene* s, const orc_store* st, const prc_gpu_params* t, int flags,
                    const double* weights, double* images, double* grad, double* gk, double* gg,
                    uint64_t* clamps, double* mean_corr) { /* pathstore.cpp:315-368 */
    prc_gpu_params tref;
    memset(&tref, 0, sizeof tref);
    tref.beta = st->ref_beta;
    tref.n_beta = st->n_ref_beta;
    tref.kappa_s = st->ref_kappa;
    tref.gamma = st->ref_gamma;
    if (!t) t = &tref;
    Ctx c;
    if (make_ctx(&c, s, t, st->ref_beta, flags, weights)) return 1;
    const int grad_on = c.want_grad && s->unknown >= 0;
    const size_t V = (size_t)s->V;
    double* img = (double*)calloc(s->n_pix ? s->n_pix : 1, sizeof(double));
    double* g = (double*)calloc(V ? V : 1, sizeof(double));
    Partial part;
    part.images = (double*)malloc((s->n_pix ? s->n_pix : 1) * sizeof(double));
    part.grad = (double*)malloc((V ? V : 1) * sizeof(double));
    double* wbuf = NULL;
    uint32_t wcap = 0;
    double gk_tot = 0.0, gg_tot = 0.0, sum_r = 0.0;
    uint64_t cl_tot = 0;
    const uint64_t n = st->n;
    for (uint64_t b0 = 0; b0 < n; b0 += CHUNK) { /* parallel_chunks, ordered reduction */
        const uint64_t e0 = b0 + CHUNK < n ? b0 + CHUNK : n;
        memset(part.images, 0, s->n_pix * sizeof(double));
        if (grad_on) memset(part.grad, 0, V * sizeof(double));
        part.gk = part.gg = 0.0;
        part.clamps = 0;
        part.sum_r = 0.0;
        for (uint64_t pos = b0; pos < e0; ++pos) {
            const Rec* r = &st->rec[st->by_stream[pos]];
            eval_record(&c, r, &part, &wbuf, &wcap);
            if (flags & PRC_EVAL_SELF_NORMALIZE) part.sum_r += correction_factor(&c, r);
        }
        for (size_t p = 0; p < s->n_pix; ++p) img[p] += part.images[p];
        if (grad_on)
            for (size_t v = 0; v < V; ++v) g[v] += part.grad[v];
        gk_tot += part.gk;
        gg_tot += part.gg;
        cl_tot += part.clamps;
        sum_r += part.sum_r;
    }
    double scale = (flags & PRC_EVAL_NORMALIZE) && n > 0 ? 1.0 / (double)n : 1.0;
    double mc = 1.0;
    if ((flags & PRC_EVAL_SELF_NORMALIZE) && n > 0) {
        mc = sum_r / (double)n;
        if (mc > 0.0) scale /= mc;
    }
    if (scale != 1.0) {
        for (size_t p = 0; p < s->n_pix; ++p) img[p] *= scale;
        if (grad_on)
            for (size_t v = 0; v < V; ++v) g[v] *= scale;
        gk_tot *= scale;
        gg_tot *= scale;
    }
    if (images) memcpy(images, img, s->n_pix * sizeof(double));
    if (grad && grad_on) memcpy(grad, g, V * sizeof(double));
    if (gk) *gk = gk_tot;
    if (gg) *gg = gg_tot;
    if (clamps) *clamps = cl_tot;
    if (mean_corr) *mean_corr = mc;
    free(img);
    free(g);
    free(part.images);
    free(part.grad);
    free(wbuf);
    free_ctx(&c);
    return 0;
}

int orc_evaluate(const prc_scene_desc* d, const orc_store* st, const prc_gpu_params* params,
                 int flags, const double* weights, double* images, double* grad, double* gk,
                 double* gg, uint64_t* clamps, double* mean_corr) {
    Scene s;
    if (scene_build(&s, d)) return 1;
    int rc = evaluate(&s, st, params, flags, weights, images, grad, gk, gg, clamps, mean_corr);
    scene_free(&s);
    return rc;
}

/* render, transport.cpp:405-454 (with bind_params, inverse.cpp:144-150) */
int orc_render(const prc_scene_desc* d, const prc_gpu_params* params, uint64_t n, uint64_t seed,
               int max_bounces, int max_events, int keep, double* images_out,
               uint64_t* trunc_out, orc_store** store_out) {
    if (n == 0) return fail("render: n_paths must be >= 1");
    if (max_bounces <= 0) max_bounces = 500;
    Scene s;
    if (scene_build(&s, d)) return 1;
    Ext ext;
    memset(&ext, 0, sizeof ext);
    for (int j = 0; j < s.n_sp; ++j) ext.sp[j] = s.sp[j].ext;
    if (s.unknown >= 0 && params && params->beta) {
        ext.sp[s.unknown] = params->beta;
        s.sp[s.unknown].ext = params->beta;
    }
    /* target surface bound to params (bind_params); copy the surface table */
    prc_surface_desc* surf = NULL;
    if (s.n_surf > 0) {
        surf = (prc_surface_desc*)malloc((size_t)s.n_surf * sizeof *surf);
        memcpy(surf, s.surf, (size_t)s.n_surf * sizeof *surf);
        if (s.target >= 0 && params) {
            surf[s.target].brdf_kind = PRC_BRDF_PHONG;
            surf[s.target].kappa_s = params->kappa_s;
            surf[s.target].gamma = params->gamma;
        }
        s.surf = surf;
    }
    orc_store* st = (orc_store*)calloc(1, sizeof *st);
    st->n = n;
    st->seed = seed;
    st->rec = (Rec*)calloc((size_t)n, sizeof(Rec));
    if (s.unknown >= 0) { /* params_from_scene (transport.cpp:119-128) */
        st->n_ref_beta = (uint64_t)s.V;
        st->ref_beta = (double*)malloc((size_t)s.V * sizeof(double));
        memcpy(st->ref_beta, ext.sp[s.unknown], (size_t)s.V * sizeof(double));
    }
    if (s.target >= 0 && surf[s.target].brdf_kind == PRC_BRDF_PHONG) {
        st->ref_kappa = surf[s.target].kappa_s;
        st->ref_gamma = surf[s.target].gamma;
    }
    double* img = (double*)calloc(s.n_pix ? s.n_pix : 1, sizeof(double));
    double* part = (double*)malloc((s.n_pix ? s.n_pix : 1) * sizeof(double));
    uint64_t trunc = 0;
    int rc = 0;
    prc_gpu_params pref;
    memset(&pref, 0, sizeof pref);
    pref.beta = st->ref_beta;
    pref.n_beta = st->n_ref_beta;
    pref.kappa_s = st->ref_kappa;
    pref.gamma = st->ref_gamma;
    for (uint64_t b0 = 0; b0 < n && !rc; b0 += CHUNK) {
        const uint64_t e0 = b0 + CHUNK < n ? b0 + CHUNK : n;
        for (uint64_t i = b0; i < e0; ++i) {
            if (trace_path(&s, &ext, seed, i, max_bounces, max_events, &st->rec[i])) {
                rc = 1;
                break;
            }
            if (st->rec[i].truncated) ++trunc;
        }
        if (rc) break;
        /* evaluate_store(chunk, normalize = false) at the sampling parameters */
        orc_store chunk;
        memset(&chunk, 0, sizeof chunk);
        chunk.rec = st->rec + b0;
        chunk.n = e0 - b0;
        chunk.ref_beta = st->ref_beta;
        chunk.n_ref_beta = st->n_ref_beta;
        chunk.ref_kappa = st->ref_kappa;
        chunk.ref_gamma = st->ref_gamma;
        rebuild_index(&chunk);
        rc = evaluate(&s, &chunk, &pref, 0, NULL, part, NULL, NULL, NULL, NULL, NULL);
        free(chunk.by_stream);
        for (size_t p = 0; p < s.n_pix; ++p) img[p] += part[p];
    }
    if (!rc) {
        const double inv_n = 1.0 / (double)n;
        for (size_t p = 0; p < s.n_pix; ++p) img[p] *= inv_n;
        if (images_out) memcpy(images_out, img, s.n_pix * sizeof(double));
        if (trunc_out) *trunc_out = trunc;
        rebuild_index(st);
    }
    free(img);
    free(part);
    free(surf);
    scene_free(&s);
    if (rc || !keep || !store_out) {
        orc_store_free(st);
        if (store_out) *store_out = NULL;
    } else {
        *store_out = st;
    }
    return rc;
}

int orc_sort_by_size(orc_store* st) { /* pathstore.cpp:261-267: stable by B */
    if (st->n == 0) return fail("sort_by_size: empty store");
    int maxB = 0;
    for (uint64_t i = 0; i < st->n; ++i)
        if (rec_size(&st->rec[i]) > maxB) maxB = rec_size(&st->rec[i]);
    uint64_t* cnt = (uint64_t*)calloc((size_t)maxB + 2, sizeof(uint64_t));
    for (uint64_t i = 0; i < st->n; ++i) cnt[rec_size(&st->rec[i]) + 1]++;
    for (int k = 1; k <= maxB + 1; ++k) cnt[k] += cnt[k - 1];
    Rec* out = (Rec*)malloc((size_t)st->n * sizeof(Rec));
    for (uint64_t i = 0; i < st->n; ++i) out[cnt[rec_size(&st->rec[i])]++] = st->rec[i];
    free(st->rec);
    free(cnt);
    st->rec = out;
    st->sorted = 1;
    rebuild_index(st);
    return 0;
}

/* --------------------------------------------------------------- PSTR v1 I/O */
#define PUT(f, v)                                \
    do {                                         \
        __typeof__(v) _t = (v);                  \
        fwrite(&_t, sizeof _t, 1, f);            \
    } while (0)
int orc_save_pstr(const orc_store* st, const char* path) { /* pathstore.cpp:410-458 */
    FILE* f = fopen(path, "wb");
    if (!f) return fail("save_store: cannot open");
    fwrite("PSTR", 1, 4, f);
    PUT(f, (uint32_t)1);
    PUT(f, (uint64_t)st->n);
    PUT(f, (uint64_t)st->generation);
    PUT(f, (uint64_t)st->seed);
    PUT(f, (uint8_t)(st->sorted ? 1 : 0));
    PUT(f, (uint64_t)st->n_ref_beta);
    for (uint64_t i = 0; i < st->n_ref_beta; ++i) PUT(f, st->ref_beta[i]);
    PUT(f, st->ref_kappa);
    PUT(f, st->ref_gamma);
    for (uint64_t i = 0; i < st->n; ++i) {
        const Rec* r = &st->rec[i];
        PUT(f, (uint64_t)r->stream);
        PUT(f, (uint8_t)(r->truncated ? 1 : 0));
        PUT(f, r->dir0.x);
        PUT(f, r->dir0.y);
        PUT(f, r->dir0.z);
        PUT(f, (uint32_t)r->nv);
        for (uint32_t k = 0; k < r->nv; ++k) {
            const Vtx* v = &r->v[k];
            PUT(f, v->pos.x);
            PUT(f, v->pos.y);
            PUT(f, v->pos.z);
            PUT(f, v->cos_theta);
            PUT(f, v->cos_in);
            PUT(f, v->cos_out);
            PUT(f, v->span_begin);
            PUT(f, v->span_end);
            PUT(f, v->voxel);
            PUT(f, v->surface);
            PUT(f, v->species);
            PUT(f, v->kind);
        }
        PUT(f, (uint32_t)r->ns);
        for (uint32_t k = 0; k < r->ns; ++k) {
            PUT(f, r->sp[k].voxel);
            PUT(f, r->sp[k].length);
        }
        PUT(f, (uint32_t)r->ne);
        for (uint32_t k = 0; k < r->ne; ++k) {
            const Evt* e = &r->ev[k];
            PUT(f, e->vertex);
            PUT(f, e->detector);
            PUT(f, e->pixel);
            PUT(f, e->cos_le);
            PUT(f, e->geom);
            PUT(f, e->span_begin);
            PUT(f, e->span_end);
        }
        PUT(f, (uint32_t)r->nl);
        for (uint32_t k = 0; k < r->nl; ++k) {
            PUT(f, r->le[k].voxel);
            PUT(f, r->le[k].length);
        }
    }
    int bad = ferror(f);
    fclose(f);
    return bad ? fail("save_store: write failure") : 0;
}

#define GET(f, v) (fread(&(v), sizeof(v), 1, f) == 1)
int orc_load_pstr(const char* path, orc_store** out) { /* pathstore.cpp:460-516 */
    FILE* f = fopen(path, "rb");
    if (!f) return fail("load_store: cannot open");
    char magic[4];
    if (fread(magic, 1, 4, f) != 4 || memcmp(magic, "PSTR", 4) != 0) {
        fclose(f);
        return fail("load_store: bad magic at offset 0");
    }
    uint32_t version = 0;
    if (!GET(f, version)) version = 0;
    if (version != 1) {
        fclose(f);
        return fail("load_store: unsupported version");
    }
    orc_store* st = (orc_store*)calloc(1, sizeof *st);
    uint64_t count = 0, nb = 0;
    uint8_t sorted = 0;
    int ok = GET(f, count) && GET(f, st->generation) && GET(f, st->seed) && GET(f, sorted) &&
             GET(f, nb);
    st->sorted = sorted;
    st->n_ref_beta = nb;
    st->ref_beta = (double*)malloc((size_t)(nb ? nb : 1) * sizeof(double));
    for (uint64_t i = 0; ok && i < nb; ++i) ok = GET(f, st->ref_beta[i]);
    ok = ok && GET(f, st->ref_kappa) && GET(f, st->ref_gamma);
    if (!ok) {
        fclose(f);
        orc_store_free(st);
        return fail("load_store: truncated file");
    }
    st->n = count;
    st->rec = (Rec*)calloc((size_t)(count ? count : 1), sizeof(Rec));
    for (uint64_t i = 0; i < count && ok; ++i) {
        Rec* r = &st->rec[i];
        uint8_t tr = 0;
        ok = GET(f, r->stream) && GET(f, tr) && GET(f, r->dir0.x) && GET(f, r->dir0.y) &&
             GET(f, r->dir0.z) && GET(f, r->nv);
        r->truncated = tr;
        if (!ok) break;
        r->cv = r->nv;
        r->v = (Vtx*)calloc(r->nv ? r->nv : 1, sizeof(Vtx));
        for (uint32_t k = 0; k < r->nv && ok; ++k) {
            Vtx* v = &r->v[k];
            ok = GET(f, v->pos.x) && GET(f, v->pos.y) && GET(f, v->pos.z) && GET(f, v->cos_theta) &&
                 GET(f, v->cos_in) && GET(f, v->cos_out) && GET(f, v->span_begin) &&
                 GET(f, v->span_end) && GET(f, v->voxel) && GET(f, v->surface) &&
                 GET(f, v->species) && GET(f, v->kind);
        }
        ok = ok && GET(f, r->ns);
        if (!ok) break;
        r->cs = r->ns;
        r->sp = (Span*)calloc(r->ns ? r->ns : 1, sizeof(Span));
        for (uint32_t k = 0; k < r->ns && ok; ++k)
            ok = GET(f, r->sp[k].voxel) && GET(f, r->sp[k].length);
        ok = ok && GET(f, r->ne);
        if (!ok) break;
        r->ce = r->ne;
        r->ev = (Evt*)calloc(r->ne ? r->ne : 1, sizeof(Evt));
        for (uint32_t k = 0; k < r->ne && ok; ++k) {
            Evt* e = &r->ev[k];
            ok = GET(f, e->vertex) && GET(f, e->detector) && GET(f, e->pixel) && GET(f, e->cos_le) &&
                 GET(f, e->geom) && GET(f, e->span_begin) && GET(f, e->span_end);
        }
        ok = ok && GET(f, r->nl);
        if (!ok) break;
        r->cl = r->nl;
        r->le = (Span*)calloc(r->nl ? r->nl : 1, sizeof(Span));
        for (uint32_t k = 0; k < r->nl && ok; ++k)
            ok = GET(f, r->le[k].voxel) && GET(f, r->le[k].length);
    }
    fclose(f);
    if (!ok) {
        orc_store_free(st);
        return fail("load_store: truncated file");
    }
    rebuild_index(st);
    *out = st;
    return 0;
}

/* Contiguous shard [lo, hi) of the records (deep copy), for the multi-rank decomposition
 * tests: rank r of W owns records [N r / W, N (r + 1) / W). */
orc_store* orc_store_slice(const orc_store* s, uint64_t lo, uint64_t hi) {
    orc_store* o = (orc_store*)calloc(1, sizeof *o);
    o->n = hi > lo ? hi - lo : 0;
    o->rec = (Rec*)calloc((size_t)(o->n ? o->n : 1), sizeof(Rec));
    for (uint64_t i = 0; i < o->n; ++i) {
        const Rec* a = &s->rec[lo + i];
        Rec* b = &o->rec[i];
        *b = *a;
        b->v = (Vtx*)malloc((size_t)(a->nv ? a->nv : 1) * sizeof(Vtx));
        memcpy(b->v, a->v, (size_t)a->nv * sizeof(Vtx));
        b->cv = a->nv;
        b->sp = (Span*)malloc((size_t)(a->ns ? a->ns : 1) * sizeof(Span));
        memcpy(b->sp, a->sp, (size_t)a->ns * sizeof(Span));
        b->cs = a->ns;
        b->ev = (Evt*)malloc((size_t)(a->ne ? a->ne : 1) * sizeof(Evt));
        memcpy(b->ev, a->ev, (size_t)a->ne * sizeof(Evt));
        b->ce = a->ne;
        b->le = (Span*)malloc((size_t)(a->nl ? a->nl : 1) * sizeof(Span));
        memcpy(b->le, a->le, (size_t)a->nl * sizeof(Span));
        b->cl = a->nl;
    }
    o->generation = s->generation;
    o->seed = s->seed;
    o->n_ref_beta = s->n_ref_beta;
    o->ref_beta = (double*)malloc((size_t)(s->n_ref_beta ? s->n_ref_beta : 1) * sizeof(double));
    memcpy(o->ref_beta, s->ref_beta, (size_t)s->n_ref_beta * sizeof(double));
    o->ref_kappa = s->ref_kappa;
    o->ref_gamma = s->ref_gamma;
    rebuild_index(o);
    return o;
}

uint64_t orc_store_count(const orc_store* s) { return s->n; }
int orc_store_streams(const orc_store* s, uint64_t* out) {
    for (uint64_t i = 0; i < s->n; ++i) out[i] = s->rec[i].stream;
    return 0;
}
int orc_store_sizes(const orc_store* s, uint32_t* out) {
    for (uint64_t i = 0; i < s->n; ++i) out[i] = (uint32_t)rec_size(&s->rec[i]);
    return 0;
}
int orc_store_stats(const orc_store* s, double* o) {
    memset(o, 0, 7 * sizeof(double));
    for (uint64_t i = 0; i < s->n; ++i) {
        const Rec* r = &s->rec[i];
        const int B = rec_size(r);
        o[0] += B;
        o[1] += r->nv;
        o[2] += r->ne;
        o[3] += r->nl;
        for (int b = 1; b < B; ++b) o[4] += r->v[b].span_end - r->v[b].span_begin;
        o[5] += r->ns;
        o[6] += r->truncated;
    }
    return 0;
}
void orc_store_free(orc_store* s) {
    if (!s) return;
    for (uint64_t i = 0; i < s->n; ++i) rec_free(&s->rec[i]);
    free(s->rec);
    free(s->by_stream);
    free(s->ref_beta);
    free(s);
}
