// prc_wavefront.cu — event-major wavefront for the recycled iteration (default mapping).
//
// The reference evaluates one stored path at a time (eval_record, pathstore.cpp:115-239).
// Per path, ~97% of the voxel visits are local-estimation (LE) connections from the
// interaction vertices to the cameras.  On the B200 the iteration is split:
//
//   K4a k_prefix        thread per path, B-sorted store (Path Sorting): incoming-segment
//                       log-prefix at every interaction vertex -> lp[iv]
//   K4b k_le_forward    CTA per run of 128 Morton-ordered interaction vertices, camera by
//                       camera: LE transmittance, event value, image scatter, event cache
//   K5b k_le_gradient_ms<3>  same vertex order: w = value * residual, LE scatter -w*l
//                       with fp64 L2 reductions (three rays per thread in lockstep, spans
//                       in the same voxel merged in registers), vertex score terms,
//                       per-vertex weight sums own[iv]
//
// The hot walks run guard-free over the padded voxel layout (prc_device.cuh, "guard-free
// walks"): same spans as the reference walk plus a zero-beta border tail.
//   K5a k_path_gradient thread per path: suffix sums from own[iv] -> incoming-segment
//                       spans and continuation score terms
//
// All voxel indexing goes through the bit-exact fp64 DDA of prc_device.cuh.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

#include "prc_eval.cuh"

using namespace prc;

namespace {

constexpr int kWF = 256;  // vertices per CTA in the wavefront kernels
#ifndef PRC_FWD_TPB
#define PRC_FWD_TPB 128
#endif
constexpr int kFwdTPB = PRC_FWD_TPB;  // K4b: vertices per CTA (128 x 8 CTAs 379.6 ms vs 256 x 4 382.3)
#ifndef PRC_PATH_TPB
#define PRC_PATH_TPB 128
#endif
#ifndef PRC_GRAD_TPB
#define PRC_GRAD_TPB 128
#endif
constexpr int kTPB = PRC_PATH_TPB;   // thread-per-path kernels (K4a, K5a, vertex keys)
constexpr int kGradTPB = PRC_GRAD_TPB;  // K5b packets per CTA
// Occupancy (measured on B200 at 1e8 paths, config (b)).  K4b with the guarded walk: 6
// CTAs x 256 threads (40 registers) 604 ms vs 5 CTAs 613, 4 CTAs 639, 3 CTAs 714; with
// the padded, software-pipelined walk: 5 CTAs (48 registers) 449 ms vs 6 CTAs 458; with
// four steps per trip: 4 CTAs (64 registers) 411 ms vs 5 CTAs 430, 6 CTAs 876.  K5b
// packet-3 at 4 CTAs x 128 threads (128 registers) 937 ms vs 3 CTAs 977, 2 CTAs 977, 5
// CTAs 1102; packet 2 (4 CTAs) 1108, packet 4 (3 CTAs) 1132.  K4b at 64 registers in
// smaller CTAs (r15): 8 x 128 threads 379.6 ms vs 4 x 256 382.3, 2 x 512 391.4, 7 x 128 394.9.
#ifndef PRC_FWD_MINB  // -D overrides are for A/B builds (scripts/variants_lib.sh)
#define PRC_FWD_MINB 8
#endif
#ifndef PRC_GRAD1_MINB
#define PRC_GRAD1_MINB 3
#endif
#ifndef PRC_GRAD2_MINB
#define PRC_GRAD2_MINB 4
#endif
#ifndef PRC_GRAD3_MINB
#define PRC_GRAD3_MINB 4
#endif
#ifndef PRC_GRAD4_MINB
#define PRC_GRAD4_MINB 3
#endif
constexpr int kFwdMinBlocks = PRC_FWD_MINB;

inline unsigned grid_for(long long n, int tpb) {
    long long g = (n + tpb - 1) / tpb;
    return (unsigned)(g < 1 ? 1 : g);
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {  // 10 bits -> every third bit
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__device__ __forceinline__ uint32_t morton_key(const DScene& sc, V3 p) {
    const double q[3] = {(p.x - sc.bmin[0]) / (sc.bmax[0] - sc.bmin[0]),
                         (p.y - sc.bmin[1]) / (sc.bmax[1] - sc.bmin[1]),
                         (p.z - sc.bmin[2]) / (sc.bmax[2] - sc.bmin[2])};
    uint32_t c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double f = q[a] * 1024.0;
        f = f < 0.0 ? 0.0 : (f > 1023.0 ? 1023.0 : f);
        c[a] = (uint32_t)f;
    }
    return spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
}

// ------------------------------------------------------------------ vertex table
__global__ void k_vt_keys(const __grid_constant__ DScene sc, const __grid_constant__ StoreView st,
                          uint32_t* keys, uint32_t* vals, unsigned long long* iv_rec) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (long long)st.n) return;
    const int B = (int)st.B[p];
    const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
    const unsigned rs = st.stride[p];
    for (int b = 1; b < B; ++b) {
        const unsigned long long r = rb + (unsigned long long)b * rs;
        const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
        keys[iv] = morton_key(sc, mk(st.px[r], st.py[r], st.pz[r]));
        vals[iv] = (uint32_t)iv;
        iv_rec[iv] = r;
    }
}

__global__ void k_vt_gather(const __grid_constant__ StoreView st, const uint32_t* vt2iv,
                            const unsigned long long* iv_rec, long long n, double* x, double* y,
                            double* z, double* dx, double* dy, double* dz, int32_t* vox,
                            uint32_t* meta, uint32_t* iv) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t s = vt2iv[i];
    const unsigned long long r = iv_rec[s];
    x[i] = st.px[r];
    y[i] = st.py[r];
    z[i] = st.pz[r];
    dx[i] = st.dx[r];
    dy[i] = st.dy[r];
    dz[i] = st.dz[r];
    vox[i] = st.vox[r];
    meta[i] = st.meta[r];
    iv[i] = s;
}

// ------------------------------------------------------------------ K4a prefix
// Thread per path over the B-sorted store (the paper's Path Sorting mapping): the vertex
// loop is warp-uniform and record loads are coalesced.  (Measured: the segment-queue
// regeneration used by K5a is slower here, because a K4a step is only a gather + FMA.)
__device__ __forceinline__ int warp_count(bool p) { return __popc(__ballot_sync(0xffffffffu, p)); }

#ifdef PRC_PREFIX_MINB  // A/B: occupancy of K4a
#define PRC_PREFIX_LB __launch_bounds__(kTPB, PRC_PREFIX_MINB)
#else
#define PRC_PREFIX_LB __launch_bounds__(kTPB)
#endif
__global__ void PRC_PREFIX_LB k_prefix(const __grid_constant__ DScene sc,
                                                 const __grid_constant__ StoreView st,
                                                 const __grid_constant__ EvalArgs ea, double* lp) {
    const long long p = path_index(st.n);
    if (p < 0) return;
    const int B = (int)st.B[p];
    if (B < 2) return;
    const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
    const unsigned rs = st.stride[p];
    const bool med = sc.has_medium;  // without a medium the positions are not needed
    V3 xprev = med ? mk(st.px[rb], st.py[rb], st.pz[rb]) : mk(0.0, 0.0, 0.0);
    double l = 0.0;
    bool dead = false;
    for (int b = 1; b < B; ++b) {
        const unsigned long long r = rb + (unsigned long long)b * rs;
        const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
        if (dead) {
            lp[iv] = -INFINITY;
            continue;
        }
        if (sc.has_medium) {
            const V3 d = mk(st.dx[r], st.dy[r], st.dz[r]);
            l -= sc.pad_walk ? dda_optical_depth_pad(sc, xprev, d, st.tt[r], ea.db_pad)
                             : dda_optical_depth(sc, xprev, d, st.tt[r], ea.dbeta);
        }
        lp[iv] = l;
        const uint32_t m = st.meta[r];
        const uint32_t kind = meta_kind(m);
        const double ct = st.ct[r];
        if (kind == VK_VOLUME) {  // continuation, pathstore.cpp:168-184
            const int vox = st.vox[r];
            if (sc.c1_fast) {  // one species: the phase function cancels
                const double num = sc.sp[0].albedo * (double)ea.sp_t[vox];
                const double den = (double)ea.sp_ref[vox];
                if (num <= 0.0 || den <= 0.0)
                    dead = true;
                else
                    l += log(num) - log(den);
            } else {
                const double num = scat_num(sc, ea.sp_t, vox, ct);
                const double den = ext_num(sc, ea.sp_ref, vox, ct);
                if (num <= 0.0 || den <= 0.0)
                    dead = true;
                else
                    l += log(num) - log(den);
            }
        } else if (kind == VK_SURFACE) {
            if (ea.vlobe) {  // cached lobe term (EventList scenes): the same values
                const double vl = ea.vlobe[iv];
                if (meta_surface(m) == sc.target) {
                    const double fr = 1.0 - ea.phong[0] + ea.phong[0] * pow01(vl, ea.phong[1]);
                    if (fr <= 0.0)
                        dead = true;
                    else
                        l += log(PRC_PI * fr);
                } else if (vl == -INFINITY) {
                    dead = true;
                } else {
                    l += vl;
                }
            } else {
                const double fr = surf_brdf(sc, ea.phong, meta_surface(m), ct);
                if (fr <= 0.0)
                    dead = true;
                else
                    l += log(PRC_PI * fr);
            }
        }
        if (med) xprev = mk(st.px[r], st.py[r], st.pz[r]);
    }
}

// ------------------------------------------------------------------ K4b LE forward
// VertexTable::ev_f holds [j][det][i] phase values (fcache scenes), then, 8-byte aligned,
// the [det][i] cos_le of surface events (scache scenes); sized in run_forward (prc_capi.cu).
__device__ __forceinline__ double* ev_cos_of(const DScene& sc, const VertexTable& vt) {
    unsigned long long off = sc.fcache ? (unsigned long long)sc.n_species * sc.n_det * vt.n : 0ull;
    return reinterpret_cast<double*>(vt.ev_f + ((off + 1ull) & ~1ull));
}

// SC: the scene has surfaces (DScene::scache); the surface-event cache code is compiled
// only into that instance, so medium-only scenes run the code they ran before it.
template <bool SC>
__global__ void __launch_bounds__(kFwdTPB, kFwdMinBlocks) k_le_forward(const __grid_constant__ DScene sc,
                                                       const __grid_constant__ VertexTable vt,
                                                       const __grid_constant__ EvalArgs ea,
                                                       const double* __restrict__ lp) {
    const unsigned long long i = (unsigned long long)blockIdx.x * kFwdTPB + threadIdx.x;
    const bool act = i < vt.n;
    int vox = 0;
    uint32_t meta = 0;
    double lpv = -INFINITY;
    if (act) {
        vox = vt.vox[i];
        meta = vt.meta[i];
        lpv = lp[vt.iv[i]];
    }
    const uint32_t kind = meta_kind(meta);
    const int surf = meta_surface(meta);
    const bool live = act && lpv != -INFINITY;
    PRC_CHECK(sc, !(live && kind == VK_VOLUME) || (vox >= 0 && vox < sc.V), CHK_VOXEL);
    const double den = (live && kind == VK_VOLUME) ? (double)ea.br_tot[vox] : 0.0;
    // lp - log(den) is per vertex: one log per camera event instead of two (the sum is
    // re-associated, a change of ~1e-16 relative in the event value)
    const double lbase = den > 0.0 ? lpv - log(den) : 0.0;
    // Single-species volume events (DScene::c1_fast): log value = [lp - log(den) +
    // log(beta_t[vox])] + c1 with c1 = log(albedo * f(cos_le)) in fixed point.  The bracket is
    // per vertex; c1 and the pixel do not depend on beta, so after the first forward over
    // a store they come from the cache (geo_ready) and the event needs only its walk.  Both
    // paths evaluate the same expression, so a recycled image at the sampling point still
    // equals the fresh render.
    const bool c1v = sc.c1_fast && kind == VK_VOLUME;
    const bool fv = sc.fcache && kind == VK_VOLUME;  // 2..4 species: cached phase values
    const bool sv = SC && kind == VK_SURFACE;       // cached cos_le and geometry factor
    const bool fast = vt.geo_ready && (((c1v || fv) && sc.pad_walk) || sv);
    double lvol = -INFINITY;
    if (c1v && live && den > 0.0) {
        const double bt = (double)ea.sp_t[vox];
        if (bt > 0.0) lvol = lbase + log(bt);
    }
    // Cached surface events without a medium: when |lp| < 300 and 1e-100 <= f_r <= 1e100 the
    // log value stays inside the clamp range, so exp(lp + log f_r) is taken as e^lp * f_r
    // (one exp per vertex instead of a log and an exp per event; ~1e-16 relative)
    const double elp = (sv && live && fast && !sc.has_medium && fabs(lpv) < 300.0) ? exp(lpv) : 0.0;
    unsigned clamps = 0;
    for (int k = 0; k < sc.n_det; ++k) {
        const unsigned long long e = (unsigned long long)k * vt.n + i;
        // vertex position re-read per camera (L1 hits) instead of being kept live across
        // the DDA: frees registers for the walk's loop invariants
        const V3 x = mk(vt.x[i], vt.y[i], vt.z[i]);
        int pix = -1;
        int32_t q = INT32_MIN;
        V3 w;
        double r = 0.0, geom = 0.0, logval = -INFINITY, direct = 0.0;
        if (fast) {
            if (sv) {
                if (live) {
                    pix = vt.ev_pix[e];
                    if (pix >= 0) {
                        const double fr = surf_brdf(sc, ea.phong, surf, ev_cos_of(sc, vt)[e]);
                        if (fr > 0.0) {
                            if (elp != 0.0 && fr >= 1e-100 && fr <= 1e100) {
                                direct = elp * fr;
                                geom = (double)__int_as_float(vt.ev_c1[e]);
                            } else {
                                logval = lpv + log(fr);
                            }
                        }
                    }
                }
            } else if (c1v) {
                if (lvol != -INFINITY) {
                    pix = vt.ev_pix[e];
                    q = vt.ev_c1[e];
                    if (pix >= 0 && q != INT32_MIN) logval = lvol + c1_dequant(sc, q);
                }
            } else if (live && den > 0.0) {
                pix = vt.ev_pix[e];
                if (pix >= 0) {
                    double num = 0.0;  // scat_num with the cached phase values
                    for (int j = 0; j < sc.n_species; ++j)
                        num += sc.sp[j].albedo * (double)ea.sp_t[(long long)j * sc.V + vox] *
                               (double)vt.ev_f[((unsigned long long)j * sc.n_det + k) * vt.n + i];
                    if (num > 0.0) logval = lbase + log(num);
                }
            }
            if (logval != -INFINITY) {
                // w, r and geom exactly as event_geometry (the walk's indexing is bit-exact);
                // a cached surface event needs the ray only for the LE walk
                double inv_r = 0.0;
                if (!sv || sc.has_medium) {
                    const V3 to_det = ld3(sc.det[k].pos) - x;
                    r = norm3(to_det);
                    inv_r = 1.0 / r;
                    w = to_det * inv_r;
                }
                // 1/r^2 as (1/r)^2: one division per event instead of two (~1e-16 relative
                // in the event value; the walk's indexing does not depend on it)
                geom = sv ? (double)__int_as_float(vt.ev_c1[e]) : inv_r * inv_r;
            }
        } else if (act && (live || !vt.geo_ready)) {
            const DDet& D = sc.det[k];
            pix = pixel_of(D, x);
            double cos_le;
            if (pix >= 0 &&
                event_geometry(sc, D, x, mk(vt.dx[i], vt.dy[i], vt.dz[i]), kind, surf, w, r, geom, cos_le)) {
                if (c1v) {
                    q = c1_quant(sc, log(sc.sp[0].albedo * phase_eval(sc.sp[0], cos_le)));
                    if (lvol != -INFINITY && q != INT32_MIN) logval = lvol + c1_dequant(sc, q);
                } else if (fv) {
                    double num = 0.0;  // scat_num with f32-rounded phase values (as the cache)
                    for (int j = 0; j < sc.n_species; ++j) {
                        const float fj = (float)phase_eval(sc.sp[j], cos_le);
                        if (!vt.geo_ready) vt.ev_f[((unsigned long long)j * sc.n_det + k) * vt.n + i] = fj;
                        num += sc.sp[j].albedo * (double)ea.sp_t[(long long)j * sc.V + vox] * (double)fj;
                    }
                    if (live && num > 0.0 && den > 0.0) logval = lbase + log(num);
                } else if (kind == VK_VOLUME) {
                    if (live) {
                        const double num = scat_num(sc, ea.sp_t, vox, cos_le);
                        if (num > 0.0 && den > 0.0) logval = lbase + log(num);
                    }
                } else {
                    if (sv) {  // cached for later passes; both passes use the f32 geometry factor
                        geom = (double)(float)geom;
                        q = __float_as_int((float)geom);
                        if (!vt.geo_ready) ev_cos_of(sc, vt)[e] = cos_le;
                    }
                    if (live) {
                        const double fr = surf_brdf(sc, ea.phong, surf, cos_le);
                        if (fr > 0.0) logval = lpv + log(fr);
                    }
                }
            } else {
                pix = -1;
            }
        }
        float val = 0.0f;
        if (SC && direct != 0.0) {
            const double contrib = direct * geom * sc.prefactor;
            val = (float)contrib;
            if (contrib != 0.0) image_add(sc, ea, sc.det[k].img_off + pix, contrib);
        } else if (logval != -INFINITY) {
            if (sc.has_medium) {
                logval -= sc.pad_walk ? dda_optical_depth_pad(sc, x, w, r, ea.bt_pad)
                                      : dda_optical_depth(sc, x, w, r, ea.bt_tot);
            }
            if (logval > PRC_LOG_CLAMP || logval < -PRC_LOG_CLAMP) {
                logval = clampd(logval, -PRC_LOG_CLAMP, PRC_LOG_CLAMP);
                ++clamps;
            }
            const double contrib = exp(logval) * geom * sc.prefactor;
            val = (float)contrib;
            if (contrib != 0.0) image_add(sc, ea, sc.det[k].img_off + pix, contrib);
        }
        if (act) {
            vt.ev_val[e] = val;
            if (!vt.geo_ready) {  // the event geometry, cached for later forwards over this store
                vt.ev_pix[e] = pix;
                vt.ev_c1[e] = q;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) clamps += __shfl_down_sync(0xffffffffu, clamps, o);
    if ((threadIdx.x & 31) == 0 && clamps) atomicAdd(ea.clamps, (unsigned long long)clamps);
}

// ------------------------------------------------------------------ K5b LE gradient
__device__ __forceinline__ double score_j(const DScene& sc, const EvalArgs& ea, int j, int vox,
                                          double c, double num) {
    // score_term, pathstore.cpp:97-105, for species j (legacy: 1 / beta_t_tot)
    if (ea.legacy) {
        const double bt = (double)ea.bt_tot[vox];
        return bt > 0.0 ? 1.0 / bt : 0.0;
    }
    return num > 0.0 ? sc.sp[j].albedo * phase_eval(sc.sp[j], c) / num : 0.0;
}

// The gradient passes' event geometry: surface events of DScene::scache scenes take cos_le
// from the per-store cache K4b wrote (and w, r as event_geometry computes them); the rest
// recompute it.  Only events with a value reach here, so the visibility test has passed.
template <bool SC>
__device__ __forceinline__ void grad_event_geometry(const DScene& sc, const VertexTable& vt, const EvalArgs& ea,
                                                    int k, unsigned long long i, V3 x, V3 d, uint32_t kind,
                                                    int surf, V3& w, double& r, double& cos_le) {
    if (SC && vt.geo_ready && kind == VK_SURFACE) {
        if (ea.do_beta) {  // the LE walk's ray
            const V3 to_det = ld3(sc.det[k].pos) - x;
            r = norm3(to_det);
            w = to_det * (1.0 / r);
        }
        cos_le = ev_cos_of(sc, vt)[(unsigned long long)k * vt.n + i];
        return;
    }
    double geom;
    event_geometry(sc, sc.det[k], x, d, kind, surf, w, r, geom, cos_le);
}

// One LE ray per thread, one fp64 L2 reduction per voxel visit (packet = 1).  Lane
// spreading: within each chunk of 32*spread vertices, lane l of warp w takes vertex
// l*spread + w, so one RED instruction touches 32 distinct Morton neighbourhoods instead
// of (at high vertex density) one voxel 32 times.
__global__ void __launch_bounds__(kWF, PRC_GRAD1_MINB) k_le_gradient(const __grid_constant__ DScene sc,
                                                        const __grid_constant__ VertexTable vt,
                                                        const __grid_constant__ EvalArgs ea,
                                                        double* __restrict__ own, int spread) {
    const unsigned long long g = (unsigned long long)blockIdx.x * kWF + threadIdx.x;
    unsigned long long i = g;
    if (spread > 1) {
        const unsigned long long chunk = 32ull * (unsigned long long)spread;
        const unsigned long long c0 = (g / chunk) * chunk;
        if (c0 + chunk <= vt.n) i = c0 + (g % 32ull) * spread + ((g / 32ull) % spread);
    }
    const bool act = i < vt.n;
    int vox = 0;
    uint32_t meta = 0;
    if (act) {
        vox = vt.vox[i];
        meta = vt.meta[i];
    }
    const uint32_t kind = meta_kind(meta);
    const int surf = meta_surface(meta);
    const bool on_target = sc.target >= 0 && kind == VK_SURFACE && surf == sc.target;
    const bool single = !ea.per_species;
    double own_acc = 0.0, acc = 0.0, gk = 0.0, gg = 0.0;
    for (int k = 0; k < sc.n_det; ++k) {
        double w = 0.0;
        if (act) {
            const int pix = vt.ev_pix[(unsigned long long)k * vt.n + i];
            if (pix >= 0) {
                const double val = (double)vt.ev_val[(unsigned long long)k * vt.n + i];
                PRC_CHECK(sc, pix >= 0 && sc.det[k].img_off + pix < sc.n_pix, CHK_PIXEL);
                w = ea.weights ? val * ea.weights[sc.det[k].img_off + pix] : val;
            }
        }
        if (w == 0.0) continue;  // pathstore.cpp:197-198
        own_acc += w;
        const V3 x = mk(vt.x[i], vt.y[i], vt.z[i]);
        V3 wd;
        double r, cos_le;
        grad_event_geometry<true>(sc, vt, ea, k, i, x, mk(vt.dx[i], vt.dy[i], vt.dz[i]), kind, surf, wd, r, cos_le);
        if (ea.do_beta) {
            const double cf = -w;
            if (sc.pad_walk) {
                dda_scatter_pad(sc, x, wd, r, ea.g_pad, cf);
            } else {
                double* gs = ea.g_span;
                dda_walk(sc, x, wd, r, [&](int v, double ta, double tb) {
                    atomicAdd(gs + v, cf * (tb - ta));
                    return true;
                });
            }
            if (kind == VK_VOLUME) {
                const double num = ea.legacy ? 0.0 : scat_num(sc, ea.sp_t, vox, cos_le);
                if (single) {
                    acc += w * score_j(sc, ea, sc.unknown, vox, cos_le, num);
                } else {
                    for (int j = 0; j < sc.n_species; ++j)
                        atomicAdd(ea.g_vert + (long long)j * sc.V + vox, w * score_j(sc, ea, j, vox, cos_le, num));
                }
            }
        }
        if (on_target) phong_scores(ea.phong, cos_le, w, gk, gg);
    }
    if (act) {
        own[vt.iv[i]] = own_acc;
        if (single && acc != 0.0) atomicAdd(ea.g_vert + vox, acc);
    }
    if (sc.target >= 0) cta_add2<kWF>(gk, gg, ea.g_phong);
}

// ------------------------------------------------------------------ K5b, lockstep packets
// One ray of a lockstep packet over the padded gradient table.  The voxel is carried as a
// pointer into the table, so a span's RED takes its address straight from loop-carried
// state: no address arithmetic per RED, and no fresh address registers whose reuse must
// wait for the RED to read them (the LSU reads a RED's operands late when reductions
// queue, and the next write to those registers stalls on the long scoreboard: r11 source
// counters put 17.5% of K5b's stall samples on one such write).  Measured at 1e8 paths:
// 1289 -> 1286 ms per iteration, i.e. the RED rate, not the stall, bounds K5b.
struct PRay {
    double t, t1, tx, ty, tz, dx, dy, dz, cf;
    double* p;
    int sx, oy, oz;
    bool alive;

    __device__ __forceinline__ void dead(double* g) {
        t = t1 = tx = ty = tz = dx = dy = dz = cf = 0.0;
        p = g;
        sx = oy = oz = 0;
        alive = false;
    }
    __device__ __forceinline__ void from(const DdaState& S, double* g, double c) {
        t = S.t; t1 = S.t1; tx = S.tx; ty = S.ty; tz = S.tz; dx = S.dx; dy = S.dy; dz = S.dz;
        cf = c;
        p = g + S.v;
        sx = S.sx; oy = S.oy; oz = S.oz;
        alive = S.alive;
    }
    // One iteration of traverse.hpp:100-115 on the padded layout (dda_step_pad): returns
    // whether the span [t, min(tmax, t1)] is emitted, its contribution cf * length and
    // its table address.  A ray that is no longer alive keeps stepping and emits nothing.
    __device__ __forceinline__ bool step(double& x, double*& a) {
        int off;
        const double tm = dda_advance(tx, ty, tz, dx, dy, dz, sx, oy, oz, off);
        const bool last = tm >= t1;
        const double tn = last ? t1 : tm;
        const bool e = alive && tn > t;
        x = cf * (tn - t);
        a = p;
        t = tm;
        p += off;
        alive = alive && !last;
        return e;
    }
};

// fp64 reduction x into *a when e, as one predicated RED.
__device__ __forceinline__ void red_add_p(bool e, double* a, double x) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %0, 0;\n\t"
        "@p red.global.add.f64 [%1], %2;\n\t"
        "}" ::"r"((int)e),
        "l"(a), "d"(x)
        : "memory");
}

// One thread walks the LE rays of M consecutive Morton-ordered vertices (a packet: at
// high vertex density they share a voxel) to the same camera in lockstep, one DDA step
// per ray per iteration.  Spans that land in the same voxel at the same iteration are
// summed in registers before a single fp64 L2 reduction, so the number of REDs falls
// (~0.39 per voxel visit for M = 3 at 1e8 paths: the reference DDA on the bench geometry
// gives 0.53 / 0.39 / 0.31 for M = 2 / 3 / 4 vertices in a 0.3-voxel cube), while `spread` keeps the 32 lanes of a
// warp on distinct packets far apart in Morton order (no same-address RED conflicts).
// F = 1: the common scene class of the recycling loop (one species with the fixed-point
// event term, no surfaces, the default score, one gradient): every interaction vertex is a
// volume scatter whose score term is 1 / beta_t, so an event needs only its position, the
// camera and its cached value -- no incoming direction, phase function or surface tests.
// F = 2: 2..4 species without surfaces (config (c)): the score terms come from the phase
// values K4b cached, so again no direction or cos_le is needed.
template <int M, bool SC, int F = 0>
__global__ void __launch_bounds__(kGradTPB, M == 2 ? PRC_GRAD2_MINB : (M == 3 ? PRC_GRAD3_MINB : PRC_GRAD4_MINB)) k_le_gradient_ms(const __grid_constant__ DScene sc,
                                                        const __grid_constant__ VertexTable vt,
                                                        const __grid_constant__ EvalArgs ea,
                                                        double* __restrict__ own, int spread) {
    const unsigned long long n_pk = (vt.n + M - 1) / M;
    const unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pk = g;
    if (spread > 1) {
        const unsigned long long chunk = 32ull * (unsigned long long)spread;
        const unsigned long long c0 = (g / chunk) * chunk;
        if (c0 + chunk <= n_pk) pk = c0 + (g % 32ull) * spread + ((g / 32ull) % spread);
    }
    const bool single = !ea.per_species;
    double own_acc[M], acc[M];
#pragma unroll
    for (int r = 0; r < M; ++r) own_acc[r] = acc[r] = 0.0;
    // F = 2 with per-type gradients: each packet slot's per-species vertex scores summed over
    // the cameras in shared memory (thread-private rows), one reduction per (vertex,
    // species) after the camera loop instead of one per event (config (c))
    double* accj = nullptr;
    if constexpr (F == 2) {
        __shared__ double s_accj[kGradTPB * M * kFCacheMax];
        accj = s_accj + threadIdx.x * (M * kFCacheMax);
#pragma unroll
        for (int q = 0; q < M * kFCacheMax; ++q) accj[q] = 0.0;
    }
    double gk = 0.0, gg = 0.0;
    for (int k = 0; k < sc.n_det; ++k) {
        DdaState S[M];
        double cf[M];
#pragma unroll
        for (int r = 0; r < M; ++r) {
            S[r] = DdaState{};  // dead: the branch-free step advances it harmlessly
            cf[r] = 0.0;
            const unsigned long long i = pk * M + r;
            if (pk >= n_pk || i >= vt.n) continue;
            const int pix = vt.ev_pix[(unsigned long long)k * vt.n + i];
            if (pix < 0) continue;
            const double val = (double)vt.ev_val[(unsigned long long)k * vt.n + i];
            PRC_CHECK(sc, sc.det[k].img_off + pix < sc.n_pix, CHK_PIXEL);
            const double w = ea.weights ? val * ea.weights[sc.det[k].img_off + pix] : val;
            if (w == 0.0) continue;
            own_acc[r] += w;
            const V3 x = mk(vt.x[i], vt.y[i], vt.z[i]);
            if constexpr (F != 0) {  // event_geometry's connection (transport.cpp:226-229), nothing else
                const V3 to_det = ld3(sc.det[k].pos) - x;
                const double rr = norm3(to_det);
                S[r].template init<true>(sc, x, to_det * (1.0 / rr), rr);
                cf[r] = -w;
                const int vox = vt.vox[i];
                PRC_CHECK(sc, vox >= 0 && vox < sc.V, CHK_VOXEL);
                if constexpr (F == 1) {
                    const double bt = (double)ea.sp_t[vox];
                    if (bt > 0.0) acc[r] += w / bt;  // score_term = 1 / beta_t (pathstore.cpp:97-105)
                } else {  // score_term (pathstore.cpp:97-105) from the cached phase values
                    float fj[kFCacheMax];
                    double num = 0.0;
                    for (int j = 0; j < sc.n_species; ++j) {
                        fj[j] = vt.ev_f[((unsigned long long)j * sc.n_det + k) * vt.n + i];
                        num += sc.sp[j].albedo * (double)ea.sp_t[(long long)j * sc.V + vox] * (double)fj[j];
                    }
                    if (num > 0.0) {
                        if (single)
                            acc[r] += w * (sc.sp[sc.unknown].albedo * (double)fj[sc.unknown] / num);
                        else
                            for (int j = 0; j < sc.n_species; ++j)
                                accj[r * kFCacheMax + j] += w * (sc.sp[j].albedo * (double)fj[j] / num);
                    }
                }
                continue;
            }
            const V3 d = mk(vt.dx[i], vt.dy[i], vt.dz[i]);
            const uint32_t meta = vt.meta[i];
            const uint32_t kind = meta_kind(meta);
            const int surf = meta_surface(meta);
            V3 wd;
            double rr, cos_le;
            grad_event_geometry<SC>(sc, vt, ea, k, i, x, d, kind, surf, wd, rr, cos_le);
            if (ea.do_beta) {
                S[r].template init<true>(sc, x, wd, rr);  // packets run on the padded layout only
                cf[r] = -w;
                if (kind == VK_VOLUME) {
                    const int vox = vt.vox[i];
                    if (single && sc.c1_fast && !ea.legacy) {
                        // one species: albedo f / (albedo beta_t f) = 1 / beta_t (score_term,
                        // pathstore.cpp:97-105), no phase-function evaluations per event
                        const double bt = (double)ea.sp_t[vox];
                        if (bt > 0.0) acc[r] += w / bt;
                        continue;
                    }
                    if (sc.fcache && !ea.legacy) {
                        // score_term (pathstore.cpp:97-105) from the phase values K4b cached
                        float fj[kFCacheMax];
                        double num = 0.0;
                        for (int j = 0; j < sc.n_species; ++j) {
                            fj[j] = vt.ev_f[((unsigned long long)j * sc.n_det + k) * vt.n + i];
                            num += sc.sp[j].albedo * (double)ea.sp_t[(long long)j * sc.V + vox] * (double)fj[j];
                        }
                        if (num > 0.0) {
                            if (single)
                                acc[r] += w * (sc.sp[sc.unknown].albedo * (double)fj[sc.unknown] / num);
                            else
                                for (int j = 0; j < sc.n_species; ++j)
                                    atomicAdd(ea.g_vert + (long long)j * sc.V + vox,
                                              w * (sc.sp[j].albedo * (double)fj[j] / num));
                        }
                        continue;
                    }
                    const double num = ea.legacy ? 0.0 : scat_num(sc, ea.sp_t, vox, cos_le);
                    if (single) {
                        acc[r] += w * score_j(sc, ea, sc.unknown, vox, cos_le, num);
                    } else {
                        for (int j = 0; j < sc.n_species; ++j)
                            atomicAdd(ea.g_vert + (long long)j * sc.V + vox,
                                      w * score_j(sc, ea, j, vox, cos_le, num));
                    }
                }
            }
            if (sc.target >= 0 && kind == VK_SURFACE && surf == sc.target)
                phong_scores(ea.phong, cos_le, w, gk, gg);
        }
        double* g = ea.g_pad;
        if (ea.g_pad_copies > 1) g += (long long)(blockIdx.x % ea.g_pad_copies) * ea.g_pad_stride;
        if (M == 2) {  // hand-scheduled pair
            while (S[0].alive || S[1].alive) {
                double l0, l1;
                const int v0 = dda_step_pad(S[0], l0);
                const int v1 = dda_step_pad(S[1], l1);
                const double x1 = cf[1] * l1;
                const bool same = v0 >= 0 && v0 == v1;
                RED_ADD_IF(sc, g, ea.g_pad_stride, v0, cf[0] * l0 + (same ? x1 : 0.0));
                RED_ADD_IF(sc, g, ea.g_pad_stride, same ? -1 : v1, x1);
            }
        } else if (M == 3) {  // hand-scheduled triple (the default packet)
            PRay R0, R1, R2;
            if (S[0].alive) R0.from(S[0], g, cf[0]); else R0.dead(g);
            if (S[1].alive) R1.from(S[1], g, cf[1]); else R1.dead(g);
            if (S[2].alive) R2.from(S[2], g, cf[2]); else R2.dead(g);
            auto pstep3 = [&]() {
                double x0, x1, x2;
                double *a0, *a1, *a2;
                bool e0 = R0.step(x0, a0);
                bool e1 = R1.step(x1, a1);
                bool e2 = R2.step(x2, a2);
#ifdef PRC_CHECKED
                {
                    const double* hi = g + ea.g_pad_stride;
                    const bool b0 = e0 && !(a0 >= g && a0 < hi), b1 = e1 && !(a1 >= g && a1 < hi),
                               b2 = e2 && !(a2 >= g && a2 < hi);
                    PRC_CHECK(sc, !b0 && !b1 && !b2, CHK_PAD_RED);
                    e0 = e0 && !b0;
                    e1 = e1 && !b1;
                    e2 = e2 && !b2;
                }
#endif
                // same voxel <=> same address; launch_le_gradient runs this packet only on
                // padded tables below 2^29 voxels (4 GB), so the low 32 bits decide
                const uint32_t l0 = (uint32_t)(uintptr_t)a0, l1 = (uint32_t)(uintptr_t)a1,
                               l2 = (uint32_t)(uintptr_t)a2;
                const bool s10 = e0 && e1 && l1 == l0;
                const bool s20 = e0 && e2 && l2 == l0;
                const bool s21 = e1 && e2 && l2 == l1 && !s20;
                red_add_p(e0, a0, x0 + (s10 ? x1 : 0.0) + (s20 ? x2 : 0.0));
                red_add_p(e1 && !s10, a1, x1 + (s21 ? x2 : 0.0));
                red_add_p(e2 && !s20 && !s21, a2, x2);
            };
            while (R0.alive || R1.alive || R2.alive) pstep3();  // (two steps per trip: same time)
        } else if (M == 4) {  // hand-scheduled quad
            while (S[0].alive || S[1].alive || S[2].alive || S[3].alive) {
                double l0, l1, l2, l3;
                const int v0 = dda_step_pad(S[0], l0);
                const int v1 = dda_step_pad(S[1], l1);
                const int v2 = dda_step_pad(S[2], l2);
                const int v3 = dda_step_pad(S[3], l3);
                const double x1 = cf[1] * l1, x2 = cf[2] * l2, x3 = cf[3] * l3;
                const bool s10 = v1 == v0, s20 = v2 == v0, s30 = v3 == v0;
                const bool s21 = v2 == v1 && !s20, s31 = v3 == v1 && !s30;
                const bool s32 = v3 == v2 && !s30 && !s31;
                RED_ADD_IF(sc, g, ea.g_pad_stride, v0, cf[0] * l0 + (s10 ? x1 : 0.0) + (s20 ? x2 : 0.0) + (s30 ? x3 : 0.0));
                RED_ADD_IF(sc, g, ea.g_pad_stride, s10 ? -1 : v1, x1 + (s21 ? x2 : 0.0) + (s31 ? x3 : 0.0));
                RED_ADD_IF(sc, g, ea.g_pad_stride, (s20 || s21) ? -1 : v2, x2 + (s32 ? x3 : 0.0));
                RED_ADD_IF(sc, g, ea.g_pad_stride, (s30 || s31 || s32) ? -1 : v3, x3);
            }
        } else {
            bool any = false;
#pragma unroll
            for (int r = 0; r < M; ++r) any |= S[r].alive;
            while (any) {
                int v[M];
                double val[M];
#pragma unroll
                for (int r = 0; r < M; ++r) {
                    double l;
                    v[r] = dda_step_pad(S[r], l);
                    val[r] = cf[r] * l;
                }
#pragma unroll
                for (int r = 1; r < M; ++r) {  // merge equal voxels into the first occurrence
                    bool merged = false;
#pragma unroll
                    for (int q = 0; q < r; ++q) {
                        if (!merged && v[r] >= 0 && v[q] == v[r]) {
                            val[q] += val[r];
                            merged = true;
                        }
                    }
                    if (merged) v[r] = -1;
                }
                any = false;
#pragma unroll
                for (int r = 0; r < M; ++r) {
                    RED_ADD_IF(sc, g, ea.g_pad_stride, v[r], val[r]);
                    any |= S[r].alive;
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < M; ++r) {
        const unsigned long long i = pk * M + r;
        if (pk >= n_pk || i >= vt.n) continue;
        own[vt.iv[i]] = own_acc[r];
        if (single && acc[r] != 0.0) atomicAdd(ea.g_vert + vt.vox[i], acc[r]);
        if constexpr (F == 2) {
            if (!single) {
                const int vox = vt.vox[i];
                for (int j = 0; j < sc.n_species; ++j) {
                    const double a = accj[r * kFCacheMax + j];
                    if (a != 0.0) atomicAdd(ea.g_vert + (long long)j * sc.V + vox, a);
                }
            }
        }
    }
    if constexpr (F == 0) {  // F != 0: scenes without surfaces (launch_le_gradient)
        if (sc.target >= 0) cta_add2<kGradTPB>(gk, gg, ea.g_phong);
    }
}

// K5a without a beta gradient (no medium, or no unknown species and no per-type
// gradients): of pathstore.cpp:213-237 only the target surface's continuation Phong
// scores remain -- no spans to scatter, so no regeneration and none of k_path_gradient's
// walk state.  The same arithmetic in the same order as k_path_gradient.
__global__ void __launch_bounds__(kTPB) k_path_scores(const __grid_constant__ DScene sc,
                                                      const __grid_constant__ StoreView st,
                                                      const __grid_constant__ EvalArgs ea,
                                                      const double* __restrict__ own) {
    const long long p = path_index(st.n);
    const int B = p >= 0 ? (int)st.B[p] : 0;
    double gk = 0.0, gg = 0.0;
    if (B >= 2) {
        const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
        const unsigned rs = st.stride[p];
        double W = 0.0;
        bool any = false;
        for (int b = 1; b < B; ++b) {
            const double o = own[ib + (unsigned long long)(b - 1) * rs];
            W += o;
            any |= o != 0.0;
        }
        double prefix = 0.0;
        for (int b = 1; b < B && any; ++b) {
            const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
            const double prefix_next = prefix + own[iv];
            const double after = W - prefix_next;
            if (after != 0.0) {
                const unsigned long long r = rb + (unsigned long long)b * rs;
                const uint32_t m = st.meta[r];
                if (meta_kind(m) == VK_SURFACE && meta_surface(m) == sc.target) {
                    if (ea.vlobe)
                        phong_scores_lc(ea.phong, ea.vlobe[iv], after, gk, gg);
                    else
                        phong_scores(ea.phong, st.ct[r], after, gk, gg);
                }
            }
            prefix = prefix_next;
        }
    }
    cta_add2<kTPB>(gk, gg, ea.g_phong);
}

// ------------------------------------------------------------------ K5a path suffix
// Thread per path (B-sorted).  Segment lengths (in voxels) are exponentially distributed,
// so a warp walking "segment b of every lane" in lockstep idles most lanes.  Instead every
// lane owns the queue of its path's segments: lanes step their current segment while at
// least half the warp (or every lane that still has work) is walking, then all idle lanes
// set up their next segment together (work regeneration; set-up cost is paid in batches).
// from_here = W - prefix (suffix sums of pathstore.cpp:219-237 from own[iv]) weights the
// incoming segment's spans; continuation score terms use after = W - prefix_next.
template <bool PAD>
// K5a occupancy (r15b, 1e8 paths): 6 CTAs x 128 (80 registers, with 112-138 B of spills
// per thread accepted: prc_wavefront.ptxas.txt) 49.3 ms vs 5 CTAs (95 registers, no bound)
// 53.2, 8 CTAs 53.0
#ifndef PRC_PATHG_MINB
#define PRC_PATHG_MINB 6
#endif
#define PRC_PATHG_LB __launch_bounds__(kTPB, PRC_PATHG_MINB)
__global__ void PRC_PATHG_LB k_path_gradient(const __grid_constant__ DScene sc,
                                                        const __grid_constant__ StoreView st,
                                                        const __grid_constant__ EvalArgs ea,
                                                        const double* __restrict__ own) {
    const long long p = path_index(st.n);
    const int B = p >= 0 ? (int)st.B[p] : 0;
    unsigned long long rb = 0, ib = 0;
    unsigned rs = 0;
    double W = 0.0;
    bool any = false;
    if (B >= 2) {
        rb = st.rec_base[p];
        ib = st.iv_base[p];
        rs = st.stride[p];
        for (int b = 1; b < B; ++b) {
            const double o = own[ib + (unsigned long long)(b - 1) * rs];
            W += o;
            any |= o != 0.0;
        }
    }
    const bool walk = ea.do_beta;  // segment spans only with a beta gradient: positions needed
    V3 xprev = any && walk ? mk(st.px[rb], st.py[rb], st.pz[rb]) : mk(0, 0, 0);
    int b = 1;
    bool done = !any;
    double prefix = 0.0, cf = 0.0, gk = 0.0, gg = 0.0;
    DdaState S{};  // dead until the first segment is set up
    const int nx = sc.dims[0], ny = sc.dims[1], nz = sc.dims[2];
    double* g = PAD ? ea.g_pad : ea.g_span;
    for (;;) {
        while (!done && !S.alive) {
            if (b >= B) {
                done = true;
                break;
            }
            const unsigned long long r = rb + (unsigned long long)b * rs;
            const double o = own[ib + (unsigned long long)(b - 1) * rs];
            const double from_here = W - prefix;
            const double prefix_next = prefix + o;
            const double after = W - prefix_next;
            if (after != 0.0) {
                const uint32_t m = st.meta[r];
                const uint32_t kind = meta_kind(m);
                if (kind == VK_VOLUME && ea.do_beta) vertex_scores(sc, ea, st.vox[r], st.ct[r], after);
                if (sc.target >= 0 && kind == VK_SURFACE && meta_surface(m) == sc.target) {
                    if (ea.vlobe)
                        phong_scores_lc(ea.phong, ea.vlobe[ib + (unsigned long long)(b - 1) * rs], after, gk, gg);
                    else
                        phong_scores(ea.phong, st.ct[r], after, gk, gg);
                }
            }
            if (from_here != 0.0 && ea.do_beta) {
                S.init<PAD>(sc, xprev, mk(st.dx[r], st.dy[r], st.dz[r]), st.tt[r]);
                cf = -from_here;
            }
            prefix = prefix_next;
            if (walk) xprev = mk(st.px[r], st.py[r], st.pz[r]);
            ++b;
        }
        const int walking = warp_count(S.alive);
        if (walking == 0 && warp_count(!done) == 0) break;
        const int target = min(16, warp_count(!done));
        do {  // 4 steps between warp votes
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double len;
                const int v = PAD ? dda_step_pad(S, len) : (S.alive ? dda_step_len<false>(S, nx, ny, nz, len) : -1);
                RED_ADD_IF(sc, g, PAD ? ea.g_pad_stride : sc.V, v, cf * len);
            }
        } while (warp_count(S.alive) >= target && target > 0);
    }
    if (sc.target >= 0) cta_add2<kTPB>(gk, gg, ea.g_phong);
}

// ------------------------------------------------------------------ padded layout
__global__ void k_pad_tables(const __grid_constant__ DScene sc, const float* __restrict__ bt,
                             const float* __restrict__ db, double* __restrict__ bt_pad, double* __restrict__ db_pad) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= sc.V) return;
    const int nx = sc.dims[0], ny = sc.dims[1];
    const int ix = (int)(v % nx), iy = (int)((v / nx) % ny), iz = (int)(v / ((long long)nx * ny));
    const long long pv = (ix + 1) + (long long)sc.pnx * (iy + 1) + (long long)sc.pnxny * (iz + 1);
    bt_pad[pv] = (double)bt[v];
    db_pad[pv] = (double)db[v];
}

__global__ void k_unpad_add(const __grid_constant__ DScene sc, const double* __restrict__ g_pad,
                            int copies, long long stride, double* __restrict__ g_span) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= sc.V) return;
    const int nx = sc.dims[0], ny = sc.dims[1];
    const int ix = (int)(v % nx), iy = (int)((v / nx) % ny), iz = (int)(v / ((long long)nx * ny));
    const long long pv = (ix + 1) + (long long)sc.pnx * (iy + 1) + (long long)sc.pnxny * (iz + 1);
    double acc = g_pad[pv];
    for (int r = 1; r < copies; ++r) acc += g_pad[(long long)r * stride + pv];
    g_span[v] += acc;
}

// ------------------------------------------------------------------ self-normalisation
// correction_factor (pathstore.cpp:269-294) of every path, summed (EvalOptions::
// self_normalize, pathstore.cpp:334-359): lr = -sum over ALL segments (the escape segment
// included) of the dbeta optical depth, plus log(ext_t) - log(ext_ref) at every volume
// vertex before the last; exp(clamp(lr)), or 0 when ext_t vanishes.  The segments are
// re-walked with the bit-exact DDA over the padded dbeta table (or the unpadded one).
// *err: a vertex with zero reference extinction (the reference throws).
__global__ void __launch_bounds__(kTPB) k_correction(const __grid_constant__ DScene sc,
                                                     const __grid_constant__ StoreView st,
                                                     const __grid_constant__ EvalArgs ea,
                                                     double* __restrict__ sum, int* __restrict__ err,
                                                     double* __restrict__ per_path) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double c = 0.0;
    if (p < (long long)st.n) {
        const int B = (int)st.B[p];
        const unsigned long long rb = st.rec_base[p];
        const unsigned rs = st.stride[p];
        V3 xprev = mk(st.px[rb], st.py[rb], st.pz[rb]);
        double lr = 0.0;
        bool zero = false;
        for (int b = 1; b <= B; ++b) {
            const unsigned long long r = rb + (unsigned long long)b * rs;
            if (sc.has_medium) {
                const V3 d = mk(st.dx[r], st.dy[r], st.dz[r]);
                lr -= sc.pad_walk ? dda_optical_depth_pad(sc, xprev, d, st.tt[r], ea.db_pad)
                                  : dda_optical_depth(sc, xprev, d, st.tt[r], ea.dbeta);
            }
            if (b == B) break;
            const uint32_t m = st.meta[r];
            if (meta_kind(m) == VK_VOLUME) {
                const int vox = st.vox[r];
                const double ct = st.ct[r];
                const double num = ext_num(sc, ea.sp_ref, vox, ct);
                const double num_t = ext_num(sc, ea.sp_t, vox, ct);
                if (num <= 0.0) {
                    atomicExch(err, 1);
                    zero = true;
                    break;
                }
                if (num_t <= 0.0) {
                    zero = true;
                    break;
                }
                lr += log(num_t) - log(num);
            }
            xprev = mk(st.px[r], st.py[r], st.pz[r]);
        }
        c = zero ? 0.0 : exp(clampd(lr, -PRC_LOG_CLAMP, PRC_LOG_CLAMP));
        if (per_path) per_path[p] = c;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c != 0.0) atomicAdd(sum, c);
}

// ------------------------------------------------------------------ event list (no medium)
// Scenes without a medium have only surface interaction vertices and no LE walks; K4b over
// the dense [det][i] cache is then bound by the latency of one cache load per (vertex,
// camera) slot, most of which hold no event (config (d): 14%).  The event list keeps the
// events only (prc_kernels.cuh, EventList).
__global__ void k_evc_count(const __grid_constant__ DScene sc, const __grid_constant__ VertexTable vt,
                            unsigned long long* __restrict__ cnt) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= vt.n) return;
    if (meta_kind(vt.meta[i]) != VK_SURFACE) return;
    unsigned c = 0;
    for (int k = 0; k < sc.n_det; ++k) c += vt.ev_pix[(unsigned long long)k * vt.n + i] >= 0 ? 1u : 0u;
    cnt[vt.iv[i]] = c;
}

__global__ void k_evc_fill(const __grid_constant__ DScene sc, const __grid_constant__ VertexTable vt,
                           const unsigned long long* __restrict__ off, uint32_t* __restrict__ ev_iv,
                           int32_t* __restrict__ ev_px, double* __restrict__ ev_lobe, float* __restrict__ ev_geom,
                           uint8_t* __restrict__ ev_surf) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= vt.n) return;
    const uint32_t m = vt.meta[i];
    if (meta_kind(m) != VK_SURFACE) return;
    const uint32_t iv = vt.iv[i];
    unsigned long long o = off[iv];
    const double* cosv = ev_cos_of(sc, vt);
    const int sf = meta_surface(m);
    const DSurf& f = sc.surf[sf];
    for (int k = 0; k < sc.n_det; ++k) {
        const unsigned long long e = (unsigned long long)k * vt.n + i;
        const int pix = vt.ev_pix[e];
        if (pix < 0) continue;
        ev_iv[o] = iv;
        ev_px[o] = (int32_t)(sc.det[k].img_off + pix);
        ev_lobe[o] = sf == sc.target ? log(clampd(cosv[e], 0.0, 1.0))
                              : brdf_eval(f.brdf_kind, f.albedo, f.kappa, f.gamma, cosv[e]);
        ev_geom[o] = __int_as_float(vt.ev_c1[e]);
        ev_surf[o] = (uint8_t)sf;
        ++o;
    }
}

// EvalArgs::vlobe (thread per path): the continuation lobe term of every surface vertex,
// computed as K4a / K5a compute it.
__global__ void k_vlobe(const __grid_constant__ DScene sc, const __grid_constant__ StoreView st,
                        double* __restrict__ vlobe) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (long long)st.n) return;
    const int B = (int)st.B[p];
    const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
    const unsigned rs = st.stride[p];
    for (int b = 1; b < B; ++b) {
        const unsigned long long r = rb + (unsigned long long)b * rs;
        const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
        const uint32_t m = st.meta[r];
        double v = 0.0;
        if (meta_kind(m) == VK_SURFACE) {
            const int sf = meta_surface(m);
            const double ct = st.ct[r];
            if (sf == sc.target) {
                v = log(clampd(ct, 0.0, 1.0));
            } else {
                const DSurf& f = sc.surf[sf];
                const double fr = brdf_eval(f.brdf_kind, f.albedo, f.kappa, f.gamma, ct);
                v = fr <= 0.0 ? -INFINITY : log(PRC_PI * fr);
            }
        }
        vlobe[iv] = v;
    }
}

// K4b' and K5b' take kEvcEPT events per thread, kEvcTPB apart, and issue all their loads
// before the first use: a single event per thread keeps too few bytes in flight to cover
// the two dependent round trips (event -> lp[iv]) at the HBM rate.
constexpr int kEvcTPB = 256;
constexpr int kEvcEPT = 4;

// K4b' (thread per event): k_le_forward<true>'s cached surface event without a medium,
// the same operations on the same values (pathstore.cpp:133-166).
__global__ void __launch_bounds__(kEvcTPB) k_evc_forward(const __grid_constant__ DScene sc,
                                                         const __grid_constant__ EventList el,
                                                         const __grid_constant__ EvalArgs ea,
                                                         const double* __restrict__ lp) {
    const unsigned long long base = (unsigned long long)blockIdx.x * (kEvcTPB * kEvcEPT) + threadIdx.x;
    uint32_t iv[kEvcEPT];
    int px[kEvcEPT], sf[kEvcEPT];
    double lobe[kEvcEPT], lpv[kEvcEPT];
    float geom[kEvcEPT];
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        const unsigned long long j = base + (unsigned long long)k * kEvcTPB;
        iv[k] = 0xffffffffu;
        px[k] = sf[k] = 0;
        lobe[k] = 0.0;
        geom[k] = 0.0f;
        if (j < el.n) {
            iv[k] = el.iv[j];
            px[k] = el.px[j];
            sf[k] = el.surf[j];
            lobe[k] = el.lobe[j];
            geom[k] = el.geom[j];
        }
    }
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        PRC_CHECK(sc, iv[k] == 0xffffffffu || iv[k] < el.n_iv, CHK_SLOT);
        lpv[k] = iv[k] != 0xffffffffu ? lp[iv[k]] : -INFINITY;
    }
    unsigned clamps = 0;
    const double kap = ea.phong[0], gam = ea.phong[1];
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        const unsigned long long j = base + (unsigned long long)k * kEvcTPB;
        if (j >= el.n) break;
        float val = 0.0f;
        if (lpv[k] != -INFINITY) {
            // surf_brdf from the cached lobe term: the same operations on the same values
            const double fr = sf[k] == sc.target ? 1.0 - kap + kap * pow01(lobe[k], gam) : lobe[k];
            if (fr > 0.0) {
                PRC_CHECK(sc, px[k] >= 0 && px[k] < sc.n_pix, CHK_PIXEL);
                const double elp = fabs(lpv[k]) < 300.0 ? exp(lpv[k]) : 0.0;
                double contrib;
                if (elp != 0.0 && fr >= 1e-100 && fr <= 1e100) {
                    const double direct = elp * fr;
                    contrib = direct * (double)geom[k] * sc.prefactor;
                } else {
                    double logval = lpv[k] + log(fr);
                    if (logval > PRC_LOG_CLAMP || logval < -PRC_LOG_CLAMP) {
                        logval = clampd(logval, -PRC_LOG_CLAMP, PRC_LOG_CLAMP);
                        ++clamps;
                    }
                    contrib = exp(logval) * (double)geom[k] * sc.prefactor;
                }
                val = (float)contrib;
                if (contrib != 0.0) image_add(sc, ea, px[k], contrib);
            }
        }
        el.val[j] = val;
    }
    for (int o = 16; o > 0; o >>= 1) clamps += __shfl_down_sync(0xffffffffu, clamps, o);
    if ((threadIdx.x & 31) == 0 && clamps) atomicAdd(ea.clamps, (unsigned long long)clamps);
}

// K5b' (thread per event): w = value * residual (pathstore.cpp:196-212; no medium, so no
// LE spans), the target surface's Phong scores, and the per-vertex weight sums own[iv]
// (own zeroed by the caller) by a segmented warp scan over the iv-ordered events: a
// vertex's events are contiguous, so at most two partial sums (a warp boundary) reach
// own[iv], and 0 + a + b is order-free.  The Phong scores leave with one reduction per CTA.
__global__ void __launch_bounds__(kEvcTPB) k_evc_gradient(const __grid_constant__ DScene sc,
                                                          const __grid_constant__ EventList el,
                                                          const __grid_constant__ EvalArgs ea,
                                                          double* __restrict__ own) {
    const int lane = threadIdx.x & 31;
    double gk = 0.0, gg = 0.0;
    for (unsigned long long c0 = (unsigned long long)blockIdx.x * (kEvcTPB * kEvcEPT); c0 < el.n;
         c0 += (unsigned long long)gridDim.x * (kEvcTPB * kEvcEPT)) {
    const unsigned long long base = c0 + threadIdx.x;
    uint32_t iv[kEvcEPT];
    int px[kEvcEPT];
    bool tg[kEvcEPT];
    double val[kEvcEPT], wt[kEvcEPT];
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        const unsigned long long j = base + (unsigned long long)k * kEvcTPB;
        iv[k] = 0xffffffffu;
        px[k] = 0;
        tg[k] = false;
        val[k] = 0.0;
        if (j < el.n) {
            iv[k] = el.iv[j];
            px[k] = el.px[j];
            tg[k] = sc.target >= 0 && el.surf[j] == sc.target;
            val[k] = (double)el.val[j];
        }
    }
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        PRC_CHECK(sc, iv[k] == 0xffffffffu || (px[k] >= 0 && px[k] < sc.n_pix), CHK_PIXEL);
        wt[k] = ea.weights && iv[k] != 0xffffffffu ? ea.weights[px[k]] : 1.0;
    }
#pragma unroll
    for (int k = 0; k < kEvcEPT; ++k) {
        const unsigned long long j = base + (unsigned long long)k * kEvcTPB;
        const double w = ea.weights ? val[k] * wt[k] : val[k];
        if (tg[k] && w != 0.0) phong_scores_lc(ea.phong, el.lobe[j], w, gk, gg);
        double sum = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double o = __shfl_up_sync(0xffffffffu, sum, d);
            const uint32_t oiv = __shfl_up_sync(0xffffffffu, iv[k], d);
            if (lane >= d && oiv == iv[k]) sum += o;
        }
        const uint32_t niv = __shfl_down_sync(0xffffffffu, iv[k], 1);
        if (iv[k] != 0xffffffffu && (lane == 31 || niv != iv[k]) && sum != 0.0) {
            PRC_CHECK(sc, iv[k] < el.n_iv, CHK_SLOT);
            atomicAdd(own + iv[k], sum);
        }
    }
    }
    if (sc.target >= 0) cta_add2<kEvcTPB>(gk, gg, ea.g_phong);
}

}  // namespace

#define LAUNCH_DONE()              \
    do {                           \
        if (launches) ++*launches; \
        return cudaGetLastError(); \
    } while (0)

cudaError_t launch_vt_keys(const DScene& sc, const StoreView& st, uint32_t* keys, uint32_t* vals,
                           unsigned long long* iv_rec, cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_vt_keys<<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, keys, vals, iv_rec);
    LAUNCH_DONE();
}

cudaError_t sort_pairs_u32(const uint32_t* ki, uint32_t* ko, const uint32_t* vi, uint32_t* vo,
                           long long n, void** tmp, size_t* tmp_bytes, cudaStream_t s) {
    size_t need = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, need, ki, ko, vi, vo, (int64_t)n, 0, 30, s);
    if (e != cudaSuccess) return e;
    if (need > *tmp_bytes) {
        if (*tmp) cudaFree(*tmp);
        e = prc_malloc_retry(tmp, need);
        if (e != cudaSuccess) {
            *tmp = nullptr;
            *tmp_bytes = 0;
            return e;
        }
        *tmp_bytes = need;
    }
    return cub::DeviceRadixSort::SortPairs(*tmp, need, ki, ko, vi, vo, (int64_t)n, 0, 30, s);
}

cudaError_t launch_vt_gather(const StoreView& st, const uint32_t* vt2iv, const unsigned long long* iv_rec,
                             long long n, double* x, double* y, double* z, double* dx, double* dy,
                             double* dz, int32_t* vox, uint32_t* meta, uint32_t* iv, cudaStream_t s,
                             unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_vt_gather<<<grid_for(n, 256), 256, 0, s>>>(st, vt2iv, iv_rec, n, x, y, z, dx, dy, dz, vox, meta, iv);
    LAUNCH_DONE();
}

cudaError_t launch_prefix(const DScene& sc, const StoreView& st, const EvalArgs& ea, double* lp,
                          cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_prefix<<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, ea, lp);
    LAUNCH_DONE();
}

cudaError_t launch_le_forward(const DScene& sc, const VertexTable& vt, const EvalArgs& ea,
                              const double* lp, cudaStream_t s, unsigned long long* launches) {
    if (vt.n == 0) return cudaSuccess;
    if (sc.scache)
        k_le_forward<true><<<grid_for((long long)vt.n, kFwdTPB), kFwdTPB, 0, s>>>(sc, vt, ea, lp);
    else
        k_le_forward<false><<<grid_for((long long)vt.n, kFwdTPB), kFwdTPB, 0, s>>>(sc, vt, ea, lp);
    LAUNCH_DONE();
}

cudaError_t launch_le_gradient(const DScene& sc, const VertexTable& vt, const EvalArgs& ea, double* own,
                               int spread, int packet, cudaStream_t s, unsigned long long* launches) {
    if (vt.n == 0) return cudaSuccess;
    // the packet-3 merge compares the low 32 bits of table addresses: exact below 2^29
    // padded voxels (4 GB per copy); larger tables take packet 2 (int voxel compares)
    if (packet == 3 && (long long)sc.pnxny * (long long)(sc.dims[2] + 2) >= (1ll << 29)) packet = 2;
    if (packet > 1) {
        const long long n_pk = ((long long)vt.n + packet - 1) / packet;
        // the specialised set-ups (F, above): scenes without surfaces, default score
        const bool plain = !sc.scache && sc.n_surf == 0 && sc.target < 0 && !ea.legacy && ea.do_beta;
        const int F = plain && sc.c1_fast && !ea.per_species ? 1 : (plain && sc.fcache && vt.geo_ready ? 2 : 0);
        if (packet == 2)
            (sc.scache ? k_le_gradient_ms<2, true>
                       : F == 1 ? k_le_gradient_ms<2, false, 1> : F == 2 ? k_le_gradient_ms<2, false, 2> : k_le_gradient_ms<2, false>)
                <<<grid_for(n_pk, kGradTPB), kGradTPB, 0, s>>>(sc, vt, ea, own, spread);
        else if (packet == 3)
            (sc.scache ? k_le_gradient_ms<3, true>
                       : F == 1 ? k_le_gradient_ms<3, false, 1> : F == 2 ? k_le_gradient_ms<3, false, 2> : k_le_gradient_ms<3, false>)
                <<<grid_for(n_pk, kGradTPB), kGradTPB, 0, s>>>(sc, vt, ea, own, spread);
        else
            (sc.scache ? k_le_gradient_ms<4, true>
                       : F == 1 ? k_le_gradient_ms<4, false, 1> : F == 2 ? k_le_gradient_ms<4, false, 2> : k_le_gradient_ms<4, false>)
                <<<grid_for(n_pk, kGradTPB), kGradTPB, 0, s>>>(sc, vt, ea, own, spread);
        LAUNCH_DONE();
    }
    k_le_gradient<<<grid_for((long long)vt.n, kWF), kWF, 0, s>>>(sc, vt, ea, own, spread);
    LAUNCH_DONE();
}

cudaError_t launch_correction(const DScene& sc, const StoreView& st, const EvalArgs& ea, double* sum, int* err,
                              double* per_path, cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_correction<<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, ea, sum, err, per_path);
    LAUNCH_DONE();
}

cudaError_t launch_evc_count(const DScene& sc, const VertexTable& vt, unsigned long long* cnt, cudaStream_t s,
                             unsigned long long* launches) {
    if (vt.n == 0) return cudaSuccess;
    k_evc_count<<<grid_for((long long)vt.n, 256), 256, 0, s>>>(sc, vt, cnt);
    LAUNCH_DONE();
}

cudaError_t launch_evc_fill(const DScene& sc, const VertexTable& vt, const unsigned long long* off, uint32_t* iv,
                            int32_t* px, double* lobe, float* geom, uint8_t* surf, cudaStream_t s,
                            unsigned long long* launches) {
    if (vt.n == 0) return cudaSuccess;
    k_evc_fill<<<grid_for((long long)vt.n, 256), 256, 0, s>>>(sc, vt, off, iv, px, lobe, geom, surf);
    LAUNCH_DONE();
}

cudaError_t launch_vlobe(const DScene& sc, const StoreView& st, double* vlobe, cudaStream_t s,
                         unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_vlobe<<<grid_for((long long)st.n, 128), 128, 0, s>>>(sc, st, vlobe);
    LAUNCH_DONE();
}

// K5b' runs persistent: 4 resident CTAs per SM (56 registers) stride over the events, so
// no CTA retires waiting for its reductions to drain (r2 at config (d): 1.55 -> 1.12 ms
// against one CTA per 1024 events; K4b' the other way round, 1.015 vs 1.045 ms).
unsigned evc_blocks(unsigned long long n) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)std::min<long long>(grid_for((long long)n, kEvcTPB * kEvcEPT), 4ll * std::max(sms, 1));
}

cudaError_t launch_evc_forward(const DScene& sc, const EventList& el, const EvalArgs& ea, const double* lp,
                               cudaStream_t s, unsigned long long* launches) {
    if (el.n == 0) return cudaSuccess;
    k_evc_forward<<<grid_for((long long)el.n, kEvcTPB * kEvcEPT), kEvcTPB, 0, s>>>(sc, el, ea, lp);
    LAUNCH_DONE();
}

cudaError_t launch_evc_gradient(const DScene& sc, const EventList& el, const EvalArgs& ea, double* own,
                                cudaStream_t s, unsigned long long* launches) {
    if (el.n_iv == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(own, 0, el.n_iv * sizeof(double), s);
    if (e != cudaSuccess) return e;
    if (el.n == 0) return cudaSuccess;
    k_evc_gradient<<<evc_blocks(el.n), kEvcTPB, 0, s>>>(sc, el, ea, own);
    LAUNCH_DONE();
}

cudaError_t launch_path_gradient(const DScene& sc, const StoreView& st, const EvalArgs& ea,
                                 const double* own, cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    if (!ea.do_beta) {  // only the target surface's Phong scores
        if (sc.target < 0) return cudaSuccess;
        k_path_scores<<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, ea, own);
        LAUNCH_DONE();
    }
    if (sc.pad_walk)
        k_path_gradient<true><<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, ea, own);
    else
        k_path_gradient<false><<<grid_for((long long)st.n, kTPB), kTPB, 0, s>>>(sc, st, ea, own);
    LAUNCH_DONE();
}

cudaError_t launch_pad_tables(const DScene& sc, const float* bt_tot, const float* dbeta, double* bt_pad,
                              double* db_pad, cudaStream_t s, unsigned long long* launches) {
    if (sc.V == 0) return cudaSuccess;
    k_pad_tables<<<grid_for(sc.V, 256), 256, 0, s>>>(sc, bt_tot, dbeta, bt_pad, db_pad);
    LAUNCH_DONE();
}

cudaError_t launch_unpad_add(const DScene& sc, const double* g_pad, int copies, long long stride,
                             double* g_span, cudaStream_t s, unsigned long long* launches) {
    if (sc.V == 0) return cudaSuccess;
    k_unpad_add<<<grid_for(sc.V, 256), 256, 0, s>>>(sc, g_pad, copies, stride, g_span);
    LAUNCH_DONE();
}
