// prc_materialized.cu — evaluation of imported PSTR stores over their STORED spans.
//
// The recycling kernels (prc_wavefront.cu) never store voxel spans: every pass re-walks
// segments and local-estimation rays with the bit-exact DDA.  A store written by the
// reference (save_store, pathstore.cpp:410-453) carries no per-vertex directions, only
// positions, so the re-walk there runs along chord directions whose last bits differ from
// the sampled ones.  The materialized mode instead keeps the file's own segment spans,
// events and LE spans on the device and evaluates them exactly as eval_record reads them
// (pathstore.cpp:115-238): the same voxel ids, the same f64 span lengths, fp64 fields and
// accumulation.  It is the parity / interchange path for reference-written stores, not the
// throughput path (thread per path, stored spans streamed from HBM).
#include "prc_eval.cuh"

using namespace prc;

namespace {

constexpr int kMatTPB = 128;

inline unsigned mat_grid(long long n) {
    const long long g = (n + kMatTPB - 1) / kMatTPB;
    return (unsigned)(g < 1 ? 1 : g);
}

// make_context, pathstore.cpp:63-80: species sums in species order, fp64.
__global__ void k_mat_prep(int n_species, long long V, const __grid_constant__ MatCtx m) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    double bt = 0.0, br = 0.0;
    for (int j = 0; j < n_species; ++j) {
        bt += m.t[j][v];
        br += m.ref[(long long)j * V + v];
    }
    m.bt_tot[v] = bt;
    m.br_tot[v] = br;
    m.dbeta[v] = bt - br;
}

// scat_num_t / ext_num_ref (pathstore.cpp:84-94) over the fp64 species values.
__device__ __forceinline__ double mat_scat_num_t(const DScene& sc, const MatCtx& m, int vox, double c) {
    double num = 0.0;
    for (int j = 0; j < sc.n_species; ++j) num += sc.sp[j].albedo * m.t[j][vox] * phase_eval(sc.sp[j], c);
    return num;
}
__device__ __forceinline__ double mat_ext_num_ref(const DScene& sc, const MatCtx& m, int vox, double c) {
    double num = 0.0;
    for (int j = 0; j < sc.n_species; ++j) num += m.ref[(long long)j * sc.V + vox] * phase_eval(sc.sp[j], c);
    return num;
}

// grad[voxel] += wgt * score_term(voxel, c) (pathstore.cpp:97-105, 209-211, 227-229); with
// per_species every species' own score term.
__device__ __forceinline__ void mat_vertex_score(const DScene& sc, const MatCtx& m, const EvalArgs& ea, int vox,
                                                 double c, double wgt) {
    const int n_out = ea.per_species ? sc.n_species : 1;
    if (ea.legacy) {
        const double bt = m.bt_tot[vox];
        const double s = bt > 0.0 ? 1.0 / bt : 0.0;
        for (int j = 0; j < n_out; ++j) atomicAdd(ea.g_vert + (long long)j * sc.V + vox, wgt * s);
        return;
    }
    const double num = mat_scat_num_t(sc, m, vox, c);
    if (!(num > 0.0)) return;
    if (ea.per_species) {
        for (int j = 0; j < sc.n_species; ++j)
            atomicAdd(ea.g_vert + (long long)j * sc.V + vox, wgt * (sc.sp[j].albedo * phase_eval(sc.sp[j], c) / num));
    } else {
        const DSpecies& u = sc.sp[sc.unknown];
        atomicAdd(ea.g_vert + vox, wgt * (u.albedo * phase_eval(u, c) / num));
    }
}

// eval_record forward, pathstore.cpp:115-185.
__global__ void __launch_bounds__(kMatTPB) k_mat_forward(const __grid_constant__ DScene sc,
                                                         const __grid_constant__ MatView mv,
                                                         const __grid_constant__ MatCtx m,
                                                         const __grid_constant__ EvalArgs ea) {
    const unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= mv.n) return;
    const unsigned long long r = mv.rec[p];
    const unsigned long long v0 = mv.v_base[r], s0 = mv.s_base[r], l0 = mv.l_base[r];
    const unsigned long long e1 = mv.e_base[r + 1];
    const int B = (int)(mv.v_base[r + 1] - v0) - 1;
    const bool medium = sc.has_medium != 0;
    double log_prefix = 0.0;
    bool dead = false;
    unsigned long long ei = mv.e_base[r];
    unsigned long long clamps = 0;
    for (int b = 1; b <= B; ++b) {
        const unsigned long long vi = v0 + (unsigned long long)b;
        const uint32_t meta = mv.v_meta[vi];
        const uint32_t kind = meta_kind(meta);
        const int vox = mv.v_vox[vi];
        const int surf = meta_surface(meta);
        if (!dead && medium) {
            double diff = 0.0;
            for (uint32_t s = mv.v_sb[vi]; s < mv.v_se[vi]; ++s)
                diff += m.dbeta[mv.s_vox[s0 + s]] * mv.s_len[s0 + s];
            log_prefix -= diff;
        }
        while (ei < e1 && mv.e_vert[ei] == (uint32_t)b) {
            double val = 0.0;
            if (!dead) {
                const double c = mv.e_cos[ei];
                double logval = -INFINITY;
                if (kind == VK_VOLUME) {
                    const double num = mat_scat_num_t(sc, m, vox, c);
                    const double den = m.br_tot[vox];
                    if (num > 0.0 && den > 0.0) logval = log_prefix + log(num) - log(den);
                } else {
                    const double fr = surf_brdf(sc, ea.phong, surf, c);
                    if (fr > 0.0) logval = log_prefix + log(fr);
                }
                if (logval != -INFINITY) {
                    if (medium) {
                        double od = 0.0;
                        for (uint32_t s = mv.e_sb[ei]; s < mv.e_se[ei]; ++s)
                            od += m.bt_tot[mv.l_vox[l0 + s]] * mv.l_len[l0 + s];
                        logval -= od;
                    }
                    if (logval > PRC_LOG_CLAMP || logval < -PRC_LOG_CLAMP) {
                        logval = clampd(logval, -PRC_LOG_CLAMP, PRC_LOG_CLAMP);
                        ++clamps;
                    }
                    val = exp(logval) * mv.e_geom[ei] * sc.prefactor;
                    image_add(sc, ea, sc.det[mv.e_det[ei]].img_off + mv.e_pix[ei], val);
                }
            }
            mv.e_val[ei] = val;
            ++ei;
        }
        if (dead || b == B) continue;
        if (kind == VK_VOLUME) {
            const double c = mv.v_ct[vi];
            const double num = mat_scat_num_t(sc, m, vox, c);
            const double den = mat_ext_num_ref(sc, m, vox, c);
            if (num <= 0.0 || den <= 0.0) {
                dead = true;
                continue;
            }
            log_prefix += log(num) - log(den);
        } else if (kind == VK_SURFACE) {
            const double fr = surf_brdf(sc, ea.phong, surf, mv.v_ct[vi]);
            if (fr <= 0.0) {
                dead = true;
                continue;
            }
            log_prefix += log(PRC_PI * fr);
        }
    }
    if (clamps) atomicAdd(ea.clamps, clamps);
}

// eval_record reverse pass with suffix sums, pathstore.cpp:187-238.
__global__ void __launch_bounds__(kMatTPB) k_mat_gradient(const __grid_constant__ DScene sc,
                                                          const __grid_constant__ MatView mv,
                                                          const __grid_constant__ MatCtx m,
                                                          const __grid_constant__ EvalArgs ea) {
    const unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= mv.n) return;
    const unsigned long long r = mv.rec[p];
    const unsigned long long v0 = mv.v_base[r], s0 = mv.s_base[r], l0 = mv.l_base[r];
    const unsigned long long e0 = mv.e_base[r];
    const int B = (int)(mv.v_base[r + 1] - v0) - 1;
    double after = 0.0, gk = 0.0, gg = 0.0;
    unsigned long long er = mv.e_base[r + 1];
    for (int b = B; b >= 1; --b) {
        const unsigned long long vi = v0 + (unsigned long long)b;
        const uint32_t meta = mv.v_meta[vi];
        const uint32_t kind = meta_kind(meta);
        const int vox = mv.v_vox[vi];
        const int surf = meta_surface(meta);
        const bool target = sc.target >= 0 && kind == VK_SURFACE && surf == sc.target;
        double own = 0.0;
        while (er > e0 && mv.e_vert[er - 1] == (uint32_t)b) {
            --er;
            const double wt = ea.weights ? ea.weights[sc.det[mv.e_det[er]].img_off + mv.e_pix[er]] : 1.0;
            const double w = mv.e_val[er] * wt;
            if (w == 0.0) continue;
            own += w;
            if (ea.do_beta) {
                for (uint32_t s = mv.e_sb[er]; s < mv.e_se[er]; ++s)
                    atomicAdd(ea.g_span + mv.l_vox[l0 + s], -(w * mv.l_len[l0 + s]));
                if (kind == VK_VOLUME) mat_vertex_score(sc, m, ea, vox, mv.e_cos[er], w);
            }
            if (target) phong_scores(ea.phong, mv.e_cos[er], w, gk, gg);
        }
        const double from_here = after + own;
        if (from_here != 0.0 && ea.do_beta)
            for (uint32_t s = mv.v_sb[vi]; s < mv.v_se[vi]; ++s)
                atomicAdd(ea.g_span + mv.s_vox[s0 + s], -(from_here * mv.s_len[s0 + s]));
        if (after != 0.0) {
            if (kind == VK_VOLUME && ea.do_beta) mat_vertex_score(sc, m, ea, vox, mv.v_ct[vi], after);
            if (target) phong_scores(ea.phong, mv.v_ct[vi], after, gk, gg);
        }
        after = from_here;
    }
    if (gk != 0.0 || gg != 0.0) {
        atomicAdd(ea.g_phong, gk);
        atomicAdd(ea.g_phong + 1, gg);
    }
}

// correction_factor (pathstore.cpp:269-294) of every path over its stored spans, summed:
// lr = -sum over all segments' spans (the escape segment included) of dbeta l, plus
// log(ext_t) - log(ext_ref) at every volume vertex before the last; the path's factor is
// exp(clamp(lr)), or 0 when ext_t vanishes.  *err: a vertex with zero reference
// extinction (the reference throws).
__global__ void __launch_bounds__(kMatTPB) k_mat_correction(const __grid_constant__ DScene sc,
                                                            const __grid_constant__ MatView mv,
                                                            const __grid_constant__ MatCtx m,
                                                            double* __restrict__ sum, int* __restrict__ err,
                                                            double* __restrict__ per_path) {
    const unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    double c = 0.0;
    if (p < mv.n) {
        const unsigned long long r = mv.rec[p];
        const unsigned long long v0 = mv.v_base[r], s0 = mv.s_base[r];
        const int B = (int)(mv.v_base[r + 1] - v0) - 1;
        double lr = 0.0;
        bool zero = false;
        for (int b = 1; b <= B; ++b) {
            const unsigned long long vi = v0 + (unsigned long long)b;
            if (sc.has_medium)
                for (uint32_t k = mv.v_sb[vi]; k < mv.v_se[vi]; ++k)
                    lr -= m.dbeta[mv.s_vox[s0 + k]] * mv.s_len[s0 + k];
            if (b == B) break;
            if (meta_kind(mv.v_meta[vi]) == VK_VOLUME) {
                const int vox = mv.v_vox[vi];
                const double ct = mv.v_ct[vi];
                const double num = mat_ext_num_ref(sc, m, vox, ct);
                double num_t = 0.0;
                for (int j = 0; j < sc.n_species; ++j) num_t += m.t[j][vox] * phase_eval(sc.sp[j], ct);
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
        }
        c = zero ? 0.0 : exp(clampd(lr, -PRC_LOG_CLAMP, PRC_LOG_CLAMP));
        if (per_path) per_path[p] = c;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c != 0.0) atomicAdd(sum, c);
}

__global__ void k_gather_u64(const uint32_t* __restrict__ perm, long long n,
                             const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}

}  // namespace

#define MAT_LAUNCH_DONE()                  \
    do {                                   \
        if (launches) ++*launches;         \
        return cudaGetLastError();         \
    } while (0)

cudaError_t launch_mat_prep(int n_species, long long V, const MatCtx& m, cudaStream_t s,
                            unsigned long long* launches) {
    if (V == 0) return cudaSuccess;
    k_mat_prep<<<mat_grid(V), kMatTPB, 0, s>>>(n_species, V, m);
    MAT_LAUNCH_DONE();
}

cudaError_t launch_mat_forward(const DScene& sc, const MatView& mv, const MatCtx& m, const EvalArgs& ea,
                               cudaStream_t s, unsigned long long* launches) {
    if (mv.n == 0) return cudaSuccess;
    k_mat_forward<<<mat_grid((long long)mv.n), kMatTPB, 0, s>>>(sc, mv, m, ea);
    MAT_LAUNCH_DONE();
}

cudaError_t launch_mat_gradient(const DScene& sc, const MatView& mv, const MatCtx& m, const EvalArgs& ea,
                                cudaStream_t s, unsigned long long* launches) {
    if (mv.n == 0) return cudaSuccess;
    k_mat_gradient<<<mat_grid((long long)mv.n), kMatTPB, 0, s>>>(sc, mv, m, ea);
    MAT_LAUNCH_DONE();
}

cudaError_t launch_mat_correction(const DScene& sc, const MatView& mv, const MatCtx& m, double* sum, int* err,
                                  double* per_path, cudaStream_t s, unsigned long long* launches) {
    if (mv.n == 0) return cudaSuccess;
    k_mat_correction<<<mat_grid((long long)mv.n), kMatTPB, 0, s>>>(sc, mv, m, sum, err, per_path);
    MAT_LAUNCH_DONE();
}

cudaError_t launch_gather_u64(const uint32_t* perm, long long n, const unsigned long long* src,
                              unsigned long long* dst, cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_gather_u64<<<mat_grid(n), kMatTPB, 0, s>>>(perm, n, src, dst);
    MAT_LAUNCH_DONE();
}
