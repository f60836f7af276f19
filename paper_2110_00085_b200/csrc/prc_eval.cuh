// prc_eval.cuh — device helpers shared by the per-path and the event-major kernels:
// local-estimation geometry (add_events, transport.cpp:218-254), the scattering
// numerators of eval_record (pathstore.cpp:84-105) and the gradient score terms.
#pragma once
#include "prc_kernels.cuh"

namespace prc {

__device__ __forceinline__ double scat_num(const DScene& sc, const float* sp, int vox, double c) {
    double num = 0.0;  // scat_num_t, pathstore.cpp:84-88
    for (int j = 0; j < sc.n_species; ++j)
        num += sc.sp[j].albedo * (double)sp[(long long)j * sc.V + vox] * phase_eval(sc.sp[j], c);
    return num;
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

__device__ __forceinline__ void phong_scores(const double* phong, double c, double wgt, double& gk,
                                             double& gg) {  // brdf.hpp:21-30
    const double kap = phong[0], gam = phong[1];
    const double cc = clampd(c, 0.0, 1.0);
    const double pw = pow(cc, gam);
    const double fr = 1.0 - kap + kap * pw;
    if (fr > 0.0) {
        gk += wgt * (-1.0 + pw) / fr;
        gg += wgt * (cc <= 0.0 ? 0.0 : kap * pw * log(cc)) / fr;
    }
}


// ---------------------------------------------------------------- warp-aggregated RED
// Lanes of a warp in the event-major wavefront walk near-parallel rays from nearby
// vertices, so at a given DDA iteration several lanes often sit in the same voxel.
// agg_red() groups the lanes that are executing it together by key
// (__match_any_sync) and sums each group exactly: every contribution is encoded in
// fixed point against a warp-uniform scale 2^(56-E) (|x| < 2^56, so up to 32 of them
// fit an int64) and split into three 21-bit limbs reduced with __reduce_add_sync
// (REDUX).  One lane per group then issues a single fp64 reduction to L2.  Singleton
// groups take the direct path with the unquantised value.
struct WarpScale {
    double scale, inv;  // 2^(56-E), 2^(E-56) with |every contribution| < 2^E
};

// Warp-uniform scale from each lane's bound |x| <= bound (call with all 32 lanes).
__device__ __forceinline__ WarpScale warp_scale(double bound) {
    double m = bound;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    int e = 0;
    if (m > 0.0) frexp(m, &e);  // m < 2^e
    WarpScale w;
    w.scale = ldexp(1.0, 56 - e);
    w.inv = ldexp(1.0, e - 56);
    return w;
}

__device__ __forceinline__ void agg_red(double* base, unsigned key, double x, const WarpScale& ws) {
    const unsigned act = __activemask();
    const unsigned grp = __match_any_sync(act, key);
    if ((grp & (grp - 1)) == 0) {  // singleton
        atomicAdd(base + key, x);
        return;
    }
    const long long q = __double2ll_rn(x * ws.scale);
    const unsigned l0 = (unsigned)q & 0x1fffffu;
    const unsigned l1 = (unsigned)(q >> 21) & 0x1fffffu;
    const int l2 = (int)(q >> 42);
    const unsigned s0 = __reduce_add_sync(grp, l0);
    const unsigned s1 = __reduce_add_sync(grp, l1);
    const int s2 = __reduce_add_sync(grp, l2);
    if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) {
        const long long tot = ((long long)s2 << 42) + ((long long)s1 << 21) + (long long)s0;
        atomicAdd(base + key, (double)tot * ws.inv);
    }
}

// Run-based variant: only lanes adjacent in lane order with equal keys are combined
// (Morton ordering puts vertices of one voxel in consecutive lanes, and their rays to
// one camera advance through the same voxels).  Runs are found with one shuffle and a
// ballot; no MATCH instruction.
__device__ __forceinline__ void run_red(double* base, unsigned key, double x, const WarpScale& ws) {
    const unsigned act = __activemask();
    const int lane = threadIdx.x & 31;
    const unsigned prev = __shfl_up_sync(act, key, 1);
    const unsigned below = act & ((1u << lane) - 1u);                 // active lanes below me
    const bool prev_act = lane > 0 && ((act >> (lane - 1)) & 1u);
    const bool head = !(prev_act && prev == key);
    const unsigned heads = __ballot_sync(act, head);
    // run = [my head, next head) restricted to active lanes
    const unsigned hb = heads & (below | (1u << lane));                // heads at or below me
    const int my_head = 31 - __clz(hb);
    const unsigned above = heads & ~((2u << lane) - 1u);               // heads strictly above me
    const unsigned end_mask = above ? ((1u << (__ffs(above) - 1)) - 1u) : 0xffffffffu;
    const unsigned run = act & end_mask & ~((1u << my_head) - 1u);
    if ((run & (run - 1)) == 0) {  // singleton run
        atomicAdd(base + key, x);
        return;
    }
    const long long q = __double2ll_rn(x * ws.scale);
    const unsigned s0 = __reduce_add_sync(run, (unsigned)q & 0x1fffffu);
    const unsigned s1 = __reduce_add_sync(run, (unsigned)(q >> 21) & 0x1fffffu);
    const int s2 = __reduce_add_sync(run, (int)(q >> 42));
    if (lane == my_head) {
        const long long tot = ((long long)s2 << 42) + ((long long)s1 << 21) + (long long)s0;
        atomicAdd(base + key, (double)tot * ws.inv);
    }
}

}  // namespace prc
