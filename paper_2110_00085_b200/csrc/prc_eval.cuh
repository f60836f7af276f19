// prc_eval.cuh — device helpers shared by the per-path and the event-major kernels:
// local-estimation geometry (add_events, transport.cpp:218-254), the scattering
// numerators of eval_record (pathstore.cpp:84-105) and the gradient score terms.
#pragma once
#include "prc_kernels.cuh"

namespace prc {

// image[idx] += v for a contribution v >= 0 (EvalArgs::img_mode).  Mode 2 adds the 128-bit
// fixed-point value floor(v / quantum) as (hi, lo) u64 words: the lo atomic returns the old
// word, so every wrap-around carries into hi exactly once and the final pair is the exact
// sum in any order of the additions.
__device__ __forceinline__ void image_add(const DScene& sc, const EvalArgs& ea, long long idx, double v) {
    PRC_CHECK(sc, idx >= 0 && idx < sc.n_pix, CHK_PIXEL);
#ifdef PRC_CHECKED
    if (idx < 0 || idx >= sc.n_pix) return;
#endif
    if (ea.img_mode == 0) {
        atomicAdd(ea.images + idx, v);
    } else if (ea.img_mode == 1) {
        atomicMax(ea.img_max, (unsigned long long)__double_as_longlong(v));  // v >= 0: bits order as values
    } else {
        const double x = v * ea.img_inv_quantum;  // a power of two: exact
        const double h = floor(x * 0x1p-64);
        const unsigned long long hi = (unsigned long long)h;
        const unsigned long long lo = (unsigned long long)(x - h * 0x1p64);
        unsigned long long* cell = ea.img_fx + 2 * idx;
        const unsigned long long old = atomicAdd(cell, lo);
        atomicAdd(cell + 1, hi + (old + lo < old ? 1ull : 0ull));
    }
}

__device__ __forceinline__ double scat_num(const DScene& sc, const float* sp, int vox, double c) {
    double num = 0.0;  // scat_num_t, pathstore.cpp:84-88
    for (int j = 0; j < sc.n_species; ++j)
        num += sc.sp[j].albedo * (double)sp[(long long)j * sc.V + vox] * phase_eval(sc.sp[j], c);
    return num;
}
// Fixed-point event term of single-species scenes (DScene::c1_fast): c1 = log(albedo * f)
// -> q with c1 ~ c1_mid + q * c1_iq; INT32_MIN when albedo * f == 0 (no event).
__device__ __forceinline__ int32_t c1_quant(const DScene& sc, double c1) {
    if (!(c1 > -INFINITY)) return INT32_MIN;
    const double q = rint((c1 - sc.c1_mid) * sc.c1_q);
    return (int32_t)fmin(fmax(q, -2147483000.0), 2147483000.0);
}
__device__ __forceinline__ double c1_dequant(const DScene& sc, int32_t q) {
    return sc.c1_mid + (double)q * sc.c1_iq;
}
__device__ __forceinline__ double ext_num(const DScene& sc, const float* sp, int vox, double c) {
    double num = 0.0;  // ext_num_ref, pathstore.cpp:90-94
    for (int j = 0; j < sc.n_species; ++j)
        num += (double)sp[(long long)j * sc.V + vox] * phase_eval(sc.sp[j], c);
    return num;
}
__device__ __forceinline__ double surf_brdf(const DScene& sc, const double* phong, int s, double c) {
    const DSurf& f = sc.surf[s];
    if (f.target) return brdf_eval(1, 0.0, phong[0], phong[1], c);
    return brdf_eval(f.brdf_kind, f.albedo, f.kappa, f.gamma, c);
}

// Local-estimation connection geometry (add_events, transport.cpp:218-254): the
// connection direction w, distance r, 1/r^2 (x departure cosine at surfaces), the
// visibility test against the surfaces and the lobe cosine.  Recomputed bit-exactly
// from the stored vertex and incoming direction, so events are never stored.
__device__ __forceinline__ bool event_geometry(const DScene& sc, const DDet& D, V3 x, V3 din,
                                               uint32_t kind, int surf, V3& w, double& r,
                                               double& geom, double& cos_le) {
    const V3 to_det = ld3(D.pos) - x;
    r = norm3(to_det);
    if (r <= 0.0) return false;
    w = to_det * (1.0 / r);
    geom = 1.0 / (r * r);
    V3 dir_ref = din;
    int own = -1;
    if (kind == VK_SURFACE) {
        V3 n = normal_at(sc.surf[surf], x);
        if (dot3(n, din) > 0.0) n = n * -1.0;
        const double c_out = dot3(n, w);
        if (c_out <= 0.0) return false;
        geom *= c_out;
        dir_ref = din - n * (2.0 * dot3(din, n));
        own = surf;
    }
    if (sc.n_surf > 0) {
        double th;
        if (intersect_surfaces(sc, x, w, PRC_SELF_HIT_EPS, r - PRC_SELF_HIT_EPS, own, th) >= 0)
            return false;
    }
    cos_le = dot3(dir_ref, w);
    return true;
}

struct Rec {
    V3 x, d;
    double t, ct;
    int vox;
    uint32_t meta;
};
__device__ __forceinline__ Rec load_rec(const StoreView& st, unsigned long long r) {
    Rec o;
    o.x = mk(st.px[r], st.py[r], st.pz[r]);
    o.d = mk(st.dx[r], st.dy[r], st.dz[r]);
    o.t = st.tt[r];
    o.ct = st.ct[r];
    o.vox = st.vox[r];
    o.meta = st.meta[r];
    return o;
}

// Longest-processing-time first: the store is sorted by ascending B, so thread ids are
// mapped back to front and the longest paths are scheduled in the first wave.
__device__ __forceinline__ long long path_index(unsigned long long n) {
    const unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    return g < n ? (long long)(n - 1 - g) : -1;
}



__device__ __forceinline__ void vertex_scores(const DScene& sc, const EvalArgs& ea, int vox,
                                              double c, double wgt) {
    // score_term, pathstore.cpp:97-105 (per species j when per_species is set)
    if (ea.legacy) {
        const double bt = (double)ea.bt_tot[vox];
        const double s = bt > 0.0 ? 1.0 / bt : 0.0;
        if (s == 0.0) return;
        const int n_out = ea.per_species ? sc.n_species : 1;
        for (int j = 0; j < n_out; ++j) atomicAdd(ea.g_vert + (long long)j * sc.V + vox, wgt * s);
        return;
    }
    if (sc.c1_fast && !ea.per_species) {  // one species: albedo f / (albedo beta_t f) = 1 / beta_t
        const double bt = (double)ea.sp_t[vox];
        if (bt > 0.0) atomicAdd(ea.g_vert + vox, wgt / bt);
        return;
    }
    const double num = scat_num(sc, ea.sp_t, vox, c);
    if (!(num > 0.0)) return;
    if (ea.per_species) {
        for (int j = 0; j < sc.n_species; ++j)
            atomicAdd(ea.g_vert + (long long)j * sc.V + vox,
                      wgt * (sc.sp[j].albedo * phase_eval(sc.sp[j], c) / num));
    } else {
        const DSpecies& u = sc.sp[sc.unknown];
        atomicAdd(ea.g_vert + vox, wgt * (u.albedo * phase_eval(u, c) / num));
    }
}

// d_kappa / d_gamma of the Phong lobe over f_r (brdf.hpp:21-30) from lc = log(clamp(c, 0, 1)).
__device__ __forceinline__ void phong_scores_lc(const double* phong, double lc, double wgt, double& gk,
                                                double& gg) {
    const double kap = phong[0], gam = phong[1];
    const double pw = pow01(lc, gam);
    const double fr = 1.0 - kap + kap * pw;
    if (fr > 0.0) {
        gk += wgt * (-1.0 + pw) / fr;
        gg += wgt * (lc == -INFINITY ? 0.0 : kap * pw * lc) / fr;
    }
}
// Adds (a, b) over the CTA into dst[0], dst[1]: warp shuffles, then one pair of fp64
// reductions per CTA (per-warp reductions into two addresses serialise at L2).  Every
// thread of the CTA must call it.
template <int TPB>
__device__ __forceinline__ void cta_add2(double a, double b, double* dst) {
    __shared__ double sa[TPB / 32], sb[TPB / 32];
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sa[threadIdx.x >> 5] = a;
        sb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int r = 0; r < TPB / 32; ++r) {
            x += sa[r];
            y += sb[r];
        }
        if (x != 0.0 || y != 0.0) {
            atomicAdd(dst, x);
            atomicAdd(dst + 1, y);
        }
    }
}

__device__ __forceinline__ void phong_scores(const double* phong, double c, double wgt, double& gk,
                                             double& gg) {  // brdf.hpp:21-30
    phong_scores_lc(phong, log(clampd(c, 0.0, 1.0)), wgt, gk, gg);
}


}  // namespace prc
