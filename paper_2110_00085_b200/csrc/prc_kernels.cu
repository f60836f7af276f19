// prc_kernels.cu — sm_100a kernels of the path-recycling hot loop.
//
//   K1 k_trace<WRITE>     path generation (transport.cpp:258-345)        thread per path
//   K2 k_sort_*           stable counting sort by B (pathstore.cpp:261-267)
//   K3 k_prep*            per-voxel context (pathstore.cpp:41-82)         thread per voxel
//   K4 k_forward          recycled forward (pathstore.cpp:121-185)        thread per path
//   K5 k_gradient         fused gradient (pathstore.cpp:187-238)          thread per path
//   K6 k_loss / k_adam    loss, residual, ADAM (inverse.cpp:11-67, 239-247)
//
// Thread-per-path over a B-sorted, bucket-major store is the paper's Path Sorting
// mapping (§5.3): the 32 lanes of a warp hold paths of identical size B, so the
// vertex loop is warp-uniform and every record field is a single coalesced load.
// Voxel spans are never stored: each pass re-walks segments and local-estimation (LE)
// rays with the bit-exact fp64 DDA of prc_device.cuh.
#include <algorithm>

#include "prc_eval.cuh"

using namespace prc;

namespace {

constexpr int kTPB = 128;

inline unsigned grid_for(long long n, int tpb = kTPB) {
    long long g = (n + tpb - 1) / tpb;
    return (unsigned)(g < 1 ? 1 : g);
}

// ------------------------------------------------------------------ scan / max (resample path)
constexpr int kScanTPB = 512;
constexpr int kScanIPT = 8;
constexpr int kScanChunk = kScanTPB * kScanIPT;

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* sw) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sw[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kScanTPB / 32; ++i) t += sw[i];
    return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kScanTPB) k_chunk_sum(const unsigned long long* __restrict__ in, long long n,
                                                        unsigned long long* __restrict__ sums) {
    __shared__ unsigned long long sw[kScanTPB / 32];
    const long long base = (long long)blockIdx.x * kScanChunk;
    unsigned long long v = 0;
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
        const long long i = base + (long long)k * kScanTPB + threadIdx.x;
        if (i < n) v += in[i];
    }
    const unsigned long long t = block_sum_u64(v, sw);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

// out may alias in: a CTA reads its chunk into shared memory before writing it.
__global__ void __launch_bounds__(kScanTPB) k_chunk_scan(const unsigned long long* in, long long n,
                                                         const unsigned long long* __restrict__ offs,
                                                         unsigned long long* out) {
    __shared__ unsigned long long sm[kScanChunk];
    __shared__ unsigned long long sw[kScanTPB / 32];
    const long long base = (long long)blockIdx.x * kScanChunk;
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
        const int j = k * kScanTPB + threadIdx.x;
        const long long i = base + j;
        sm[j] = i < n ? in[i] : 0ull;
    }
    __syncthreads();
    // each thread owns kScanIPT consecutive elements
    unsigned long long local[kScanIPT], tot = 0;
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
        local[k] = tot;
        tot += sm[threadIdx.x * kScanIPT + k];
    }
    // exclusive scan of the thread totals: warp scan, then the warp totals
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long inc = tot;
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = lane < kScanTPB / 32 ? sw[lane] : 0ull;
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        if (lane < kScanTPB / 32) sw[lane] = x;  // inclusive warp-total prefix
    }
    __syncthreads();
    const unsigned long long off = (offs ? offs[blockIdx.x] : 0ull) + (w > 0 ? sw[w - 1] : 0ull) + (inc - tot);
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) sm[threadIdx.x * kScanIPT + k] = off + local[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
        const int j = k * kScanTPB + threadIdx.x;
        const long long i = base + j;
        if (i < n) out[i] = sm[j];
    }
}

__global__ void k_max_u32(const uint32_t* __restrict__ in, long long n, uint32_t* out) {
    uint32_t m = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        m = max(m, in[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// exclusive scan of in[0, n) into out, chunk sums in tmp (then the next level's after them)
cudaError_t scan_levels(const unsigned long long* in, unsigned long long* out, long long n,
                        unsigned long long* tmp, cudaStream_t s) {
    const long long chunks = (n + kScanChunk - 1) / kScanChunk;
    if (chunks == 1) {
        k_chunk_scan<<<1, kScanTPB, 0, s>>>(in, n, nullptr, out);
        return cudaGetLastError();
    }
    k_chunk_sum<<<(unsigned)chunks, kScanTPB, 0, s>>>(in, n, tmp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = scan_levels(tmp, tmp, chunks, tmp + chunks, s);  // chunk offsets, in place
    if (e != cudaSuccess) return e;
    k_chunk_scan<<<(unsigned)chunks, kScanTPB, 0, s>>>(in, n, tmp, out);
    return cudaGetLastError();
}

// ============================================================================ K1 trace
template <bool WRITE>
__device__ __forceinline__ void trace_one(const DScene& sc, const TraceArgs& a, unsigned long long p) {
    Philox rng;
    rng.init(a.seed, a.stream_base + p);
    V3 pos, dir;
    if (sc.light_kind == 1) {  // uniform_sphere_dir, transport.cpp:58-63
        pos = ld3(sc.light_pos);
        const double z = 1.0 - 2.0 * rng.uniform();
        const double phi = 2.0 * PRC_PI * rng.uniform();
        double q = 1.0 - z * z;
        const double r = sqrt(q > 0.0 ? q : 0.0);
        dir = mk(r * cos(phi), r * sin(phi), z);
    } else {
        const double u = rng.uniform();
        const double v = rng.uniform();
        pos = mk(sc.bmin[0] + u * (sc.bmax[0] - sc.bmin[0]), sc.bmin[1] + v * (sc.bmax[1] - sc.bmin[1]),
                 sc.bmax[2]);
        dir = ld3(sc.light_dir);
    }
    unsigned long long w = 0;
    if (WRITE) {
        w = a.off[p];
        a.rec.px[w] = pos.x;
        a.rec.py[w] = pos.y;
        a.rec.pz[w] = pos.z;
        a.rec.dx[w] = dir.x;
        a.rec.dy[w] = dir.y;
        a.rec.dz[w] = dir.z;
        a.rec.tt[w] = 0.0;
        a.rec.ct[w] = 1.0;
        a.rec.vox[w] = sc.has_medium ? voxel_of(sc, pos) : -1;
        a.rec.meta[w] = make_meta(VK_EMISSION, -1, -1);
        ++w;
    }
    uint32_t nv = 1;
    int cur_surface = -1, interactions = 0;
    uint8_t truncated = 0;
    for (;;) {
        const double tau = sc.has_medium ? -log1p(-rng.uniform()) : -1.0;
        // walk_segment, transport.cpp:74-114
        double t_lim = INFINITY;  // aabb_exit, transport.cpp:16-29
        {
            const double o[3] = {pos.x, pos.y, pos.z}, d[3] = {dir.x, dir.y, dir.z};
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                if (d[ax] > 0.0) {
                    const double c = (sc.bmax[ax] - o[ax]) / d[ax];
                    t_lim = c < t_lim ? c : t_lim;
                } else if (d[ax] < 0.0) {
                    const double c = (sc.bmin[ax] - o[ax]) / d[ax];
                    t_lim = c < t_lim ? c : t_lim;
                }
            }
        }
        uint32_t kind = VK_ESCAPE;
        int surf = -1;
        if (sc.n_surf > 0) {
            double th;
            const int s = intersect_surfaces(sc, pos, dir, PRC_SELF_HIT_EPS, t_lim, cur_surface, th);
            if (s >= 0) {
                t_lim = th;
                kind = VK_SURFACE;
                surf = s;
            }
        }
        double dist = t_lim;
        V3 point = pos + dir * t_lim;
        int svox = -1;
        if (sc.has_medium) {
            double od = 0.0;
            const double* bt = a.beta_tot;
            dda_walk(sc, pos, dir, t_lim, [&](int v, double ta, double tb) {
                const double beta = bt[v];
                const double seg_od = beta * (tb - ta);
                if (tau >= 0.0 && od + seg_od >= tau && beta > 0.0) {
                    const double t_sc = ta + (tau - od) / beta;
                    kind = VK_VOLUME;
                    dist = t_sc;
                    point = pos + dir * t_sc;
                    surf = -1;
                    svox = v;
                    return false;
                }
                od += seg_od;
                return true;
            });
        }
        const int vox = sc.has_medium ? (svox >= 0 ? svox : voxel_of(sc, point)) : -1;
        const bool escape = kind == VK_ESCAPE;
        const bool budget = !escape && (interactions >= a.max_bounces ||
                                        (a.max_events >= 0 && interactions >= a.max_events));
        if (escape || budget) {
            if (budget) truncated = interactions >= a.max_bounces ? 1 : 0;
            if (WRITE) {
                a.rec.px[w] = point.x;
                a.rec.py[w] = point.y;
                a.rec.pz[w] = point.z;
                a.rec.dx[w] = dir.x;
                a.rec.dy[w] = dir.y;
                a.rec.dz[w] = dir.z;
                a.rec.tt[w] = dist;
                a.rec.ct[w] = 1.0;
                a.rec.vox[w] = vox;
                a.rec.meta[w] = make_meta(VK_ESCAPE, -1, -1);
            }
            ++nv;
            break;
        }
        ++interactions;
        double cos_theta;
        int species = -1;
        V3 ndir;
        if (kind == VK_VOLUME) {  // sample_direction, transport.cpp:178-202
            const int vx = voxel_of(sc, point);
            double beta[PRC_MAX_SPECIES];
            double total = 0.0;
            for (int j = 0; j < sc.n_species; ++j) {
                beta[j] = vx >= 0 ? a.sp_beta[(long long)j * sc.V + vx] : 0.0;
                total += beta[j];
            }
            if (total <= 0.0) {
                atomicExch(a.err, 1);
                if (!WRITE) a.B[p] = nv;
                return;
            }
            const double u = rng.uniform() * total;
            int j = 0;
            double acc = beta[0];
            while (j + 1 < sc.n_species && u >= acc) acc += beta[++j];
            const double c = phase_sample_cos(sc.sp[j], rng.uniform());
            const double phi = 2.0 * PRC_PI * rng.uniform();
            ndir = frame_from_local(dir, c, phi);
            cos_theta = c;
            species = j;
            cur_surface = -1;
        } else {  // surface bounce, transport.cpp:322-341
            V3 n = normal_at(sc.surf[surf], point);
            if (dot3(n, dir) > 0.0) n = n * -1.0;
            const V3 wr = dir - n * (2.0 * dot3(dir, n));
            const double u1 = rng.uniform();
            const double u2 = rng.uniform();
            const double cos_n = sqrt(1.0 - u1);
            ndir = frame_from_local(n, cos_n, 2.0 * PRC_PI * u2);
            cos_theta = dot3(wr, ndir);
            cur_surface = surf;
        }
        if (WRITE) {
            a.rec.px[w] = point.x;
            a.rec.py[w] = point.y;
            a.rec.pz[w] = point.z;
            a.rec.dx[w] = dir.x;
            a.rec.dy[w] = dir.y;
            a.rec.dz[w] = dir.z;
            a.rec.tt[w] = dist;
            a.rec.ct[w] = cos_theta;
            a.rec.vox[w] = vox;
            a.rec.meta[w] = make_meta(kind, species, kind == VK_SURFACE ? surf : -1);
            ++w;
        }
        ++nv;
        dir = ndir;
        pos = point;
    }
    if (!WRITE) {
        a.B[p] = nv - 1;
        a.trunc[p] = truncated;
    }
}

// Path regeneration: a CTA owns `chunk` consecutive paths and every thread takes the next
// untraced one as soon as its current path ends, so a lane whose path escaped early does
// not idle until the longest path of its warp is done (path lengths B vary from 1 to ~50).
// A path's trace depends only on its Philox stream, so the results do not depend on which
// thread traces it.  Measured (r2, trace of one store, 8 paths per thread vs 1): (b) 1e8
// paths 783 -> 740 ms, (e) 713 -> 679 ms at 3e7, (d) 32.9 -> 29.8 ms; at 1e6 paths (a)
// 4.9 -> 6.3 ms (too few CTAs), so small stores keep one path per thread.
template <bool WRITE>
__global__ void __launch_bounds__(kTPB) k_trace(const __grid_constant__ DScene sc,
                                                const __grid_constant__ TraceArgs a, unsigned chunk) {
    __shared__ unsigned next;
    if (threadIdx.x == 0) next = 0;
    __syncthreads();
    const unsigned long long base = (unsigned long long)blockIdx.x * chunk;
    for (;;) {
        const unsigned k = atomicAdd(&next, 1u);
        const unsigned long long p = base + k;
        if (k >= chunk || p >= a.n) break;
        trace_one<WRITE>(sc, a, p);
    }
}

// ============================================================================ K3 prep
struct SrcPtrs {
    const double* p[PRC_MAX_SPECIES];
};

__global__ void k_prep_ref(int n_species, long long V, SrcPtrs src, double* br64, float* sp_ref,
                           float* br, double* beta_tot64) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    double s = 0.0;
    for (int j = 0; j < n_species; ++j) {
        const double b = src.p[j][v];
        sp_ref[(long long)j * V + v] = (float)b;
        s += b;
    }
    br64[v] = s;
    br[v] = (float)s;
    if (beta_tot64) beta_tot64[v] = s;
}

__global__ void k_prep(int n_species, long long V, SrcPtrs src, const double* br64, float* sp_t,
                       float* bt, float* dbeta) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    double s = 0.0;
    for (int j = 0; j < n_species; ++j) {
        const double b = src.p[j][v];
        sp_t[(long long)j * V + v] = (float)b;
        s += b;
    }
    bt[v] = (float)s;
    dbeta[v] = (float)(s - br64[v]);
}

__global__ void k_set_species(int n_species, long long V, int unknown, const double* scene_sp,
                              const double* beta_u, double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n_species * V) return;
    const int j = (int)(i / V);
    out[i] = (j == unknown && beta_u) ? beta_u[i - (long long)j * V] : scene_sp[i];
}

// ============================================================================ K4 forward
__global__ void __launch_bounds__(kTPB) k_forward(const __grid_constant__ DScene sc,
                                                  const __grid_constant__ StoreView st,
                                                  const __grid_constant__ EvalArgs ea) {
    const long long p = path_index(st.n);
    unsigned clamps = 0;
    if (p >= 0) {
        const int B = (int)st.B[p];
        if (B >= 2) {
            const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
            const unsigned rs = st.stride[p];
            V3 xprev = mk(st.px[rb], st.py[rb], st.pz[rb]);
            double lp = 0.0;
            bool dead = false;
            for (int b = 1; b < B; ++b) {
                const Rec R = load_rec(st, rb + (unsigned long long)b * rs);
                const uint32_t kind = meta_kind(R.meta);
                const int surf = meta_surface(R.meta);
                if (!dead && sc.has_medium) {  // log-prefix of the incoming segment
                    double diff = 0.0;
                    const float* db = ea.dbeta;
                    dda_walk(sc, xprev, R.d, R.t, [&](int v, double ta, double tb) {
                        diff = fma((double)__ldg(db + v), tb - ta, diff);
                        return true;
                    });
                    lp -= diff;
                }
                const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
                for (int k = 0; k < sc.n_det; ++k) {
                    float val = 0.0f;
                    int pix = -1;
                    if (!dead) {
                        const DDet& D = sc.det[k];
                        pix = pixel_of(D, R.x);
                        V3 w;
                        double r, geom, cos_le;
                        if (pix >= 0 && event_geometry(sc, D, R.x, R.d, kind, surf, w, r, geom, cos_le)) {
                            double logval = -INFINITY;
                            if (kind == VK_VOLUME) {
                                const double num = scat_num(sc, ea.sp_t, R.vox, cos_le);
                                const double den = (double)ea.br_tot[R.vox];
                                if (num > 0.0 && den > 0.0) logval = lp + log(num) - log(den);
                            } else {
                                const double fr = surf_brdf(sc, ea.phong, surf, cos_le);
                                if (fr > 0.0) logval = lp + log(fr);
                            }
                            if (logval != -INFINITY) {
                                if (sc.has_medium) {
                                    double od = 0.0;
                                    const float* bt = ea.bt_tot;
                                    dda_walk(sc, R.x, w, r, [&](int v, double ta, double tb) {
                                        od = fma((double)__ldg(bt + v), tb - ta, od);
                                        return true;
                                    });
                                    logval -= od;
                                }
                                if (logval > PRC_LOG_CLAMP || logval < -PRC_LOG_CLAMP) {
                                    logval = clampd(logval, -PRC_LOG_CLAMP, PRC_LOG_CLAMP);
                                    ++clamps;
                                }
                                const double v = exp(logval) * geom * sc.prefactor;
                                image_add(sc, ea, D.img_off + pix, v);
                                val = (float)v;
                            }
                        } else {
                            pix = -1;
                        }
                    }
                    st.ev_val[(unsigned long long)k * st.n_iv + iv] = val;
                    st.ev_pix[(unsigned long long)k * st.n_iv + iv] = pix;
                }
                if (!dead) {  // continuation factor at vertex b
                    if (kind == VK_VOLUME) {
                        const double num = scat_num(sc, ea.sp_t, R.vox, R.ct);
                        const double den = ext_num(sc, ea.sp_ref, R.vox, R.ct);
                        if (num <= 0.0 || den <= 0.0)
                            dead = true;
                        else
                            lp += log(num) - log(den);
                    } else if (kind == VK_SURFACE) {
                        const double fr = surf_brdf(sc, ea.phong, surf, R.ct);
                        if (fr <= 0.0)
                            dead = true;
                        else
                            lp += log(PRC_PI * fr);
                    }
                }
                xprev = R.x;
            }
        }
    }
    // warp-aggregate the clamp counter
    for (int o = 16; o > 0; o >>= 1) clamps += __shfl_down_sync(0xffffffffu, clamps, o);
    if ((threadIdx.x & 31) == 0 && clamps) atomicAdd(ea.clamps, (unsigned long long)clamps);
}

// ============================================================================ K5 gradient
__device__ __forceinline__ double event_weight(const StoreView& st, const EvalArgs& ea,
                                               const DScene& sc, int k, unsigned long long iv,
                                               int& pix) {
    pix = st.ev_pix[(unsigned long long)k * st.n_iv + iv];
    if (pix < 0) return 0.0;
    const double val = (double)st.ev_val[(unsigned long long)k * st.n_iv + iv];
    return ea.weights ? val * ea.weights[sc.det[k].img_off + pix] : val;
}

__global__ void __launch_bounds__(kTPB) k_gradient(const __grid_constant__ DScene sc,
                                                   const __grid_constant__ StoreView st,
                                                   const __grid_constant__ EvalArgs ea) {
    const long long p = path_index(st.n);
    double gk = 0.0, gg = 0.0;
    if (p >= 0) {
        const int B = (int)st.B[p];
        if (B >= 2) {
            const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
            const unsigned rs = st.stride[p];
            // pass A: total event weight of the path (suffix sums are W - prefix)
            double W = 0.0;
            bool any = false;
            for (int b = 1; b < B; ++b) {
                const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
                double own = 0.0;
                for (int k = 0; k < sc.n_det; ++k) {
                    int pix;
                    const double w = event_weight(st, ea, sc, k, iv, pix);
                    if (w != 0.0) {
                        own += w;
                        any = true;
                    }
                }
                W += own;
            }
            if (any) {
                V3 xprev = mk(st.px[rb], st.py[rb], st.pz[rb]);
                double prefix = 0.0;
                for (int b = 1; b < B; ++b) {
                    const Rec R = load_rec(st, rb + (unsigned long long)b * rs);
                    const uint32_t kind = meta_kind(R.meta);
                    const int surf = meta_surface(R.meta);
                    const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
                    double own = 0.0;
                    for (int k = 0; k < sc.n_det; ++k) {
                        int pix;
                        const double w = event_weight(st, ea, sc, k, iv, pix);
                        if (w != 0.0) own += w;
                    }
                    const double from_here = W - prefix;
                    const double prefix_next = prefix + own;
                    const double after = W - prefix_next;
                    if (from_here != 0.0 && ea.do_beta) {  // incoming segment spans
                        const double cf = -from_here;
                        double* g = ea.g_span;
                        dda_walk(sc, xprev, R.d, R.t, [&](int v, double ta, double tb) {
                            atomicAdd(g + v, cf * (tb - ta));
                            return true;
                        });
                    }
                    const bool on_target = sc.target >= 0 && kind == VK_SURFACE && surf == sc.target;
                    for (int k = 0; k < sc.n_det; ++k) {
                        int pix;
                        const double w = event_weight(st, ea, sc, k, iv, pix);
                        if (w == 0.0) continue;
                        V3 wd;
                        double r, geom, cos_le;
                        event_geometry(sc, sc.det[k], R.x, R.d, kind, surf, wd, r, geom, cos_le);
                        if (ea.do_beta) {
                            const double cf = -w;
                            double* g = ea.g_span;
                            dda_walk(sc, R.x, wd, r, [&](int v, double ta, double tb) {
                                atomicAdd(g + v, cf * (tb - ta));
                                return true;
                            });
                            if (kind == VK_VOLUME) vertex_scores(sc, ea, R.vox, cos_le, w);
                        }
                        if (on_target) phong_scores(ea.phong, cos_le, w, gk, gg);
                    }
                    if (after != 0.0) {
                        if (kind == VK_VOLUME && ea.do_beta) vertex_scores(sc, ea, R.vox, R.ct, after);
                        if (on_target) phong_scores(ea.phong, R.ct, after, gk, gg);
                    }
                    prefix = prefix_next;
                    xprev = R.x;
                }
            }
        }
    }
    if (sc.target >= 0) {
        for (int o = 16; o > 0; o >>= 1) {
            gk += __shfl_down_sync(0xffffffffu, gk, o);
            gg += __shfl_down_sync(0xffffffffu, gg, o);
        }
        if ((threadIdx.x & 31) == 0 && (gk != 0.0 || gg != 0.0)) {
            atomicAdd(ea.g_phong, gk);
            atomicAdd(ea.g_phong + 1, gg);
        }
    }
}

// ============================================================================ K6 & utils
__global__ void k_scale(double* x, long long n, double s) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] *= s;
}

__global__ void k_combine(const double* gs, const double* gv, int n_out, long long V, double s,
                          double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)n_out * V) return;
    const long long v = i % V;
    out[i] = (gs[v] + gv[i]) * s;
}

__global__ void k_loss_residual(const double* F, const double* gt, long long n, double* res,
                                double* loss) {  // inverse.cpp:11-23, 239-242
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    if (i < n) {
        const double r = F[i] - gt[i];
        res[i] = r;
        acc = r * r;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(loss, 0.5 * acc);
}

// mode 0: tomography (project beta >= 0 when requested); 1: Phong (kappa in [0,1],
// gamma >= 0).  adam_step, inverse.cpp:41-67.
__global__ void k_adam(double* x, double* m1, double* m2, const double* g, long long n, double alpha,
                       double eta1, double eta2, double eps, double c1, double c2,
                       const double* step_scale, int n_ss, int mode) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double gi = g[i];
    m1[i] = eta1 * m1[i] + (1.0 - eta1) * gi;
    m2[i] = eta2 * m2[i] + (1.0 - eta2) * gi * gi;
    const double mhat = m1[i] / c1;
    const double vhat = m2[i] / c2;
    const double scale = i < n_ss ? step_scale[i] : 1.0;
    double xi = x[i] - alpha * scale * mhat / (sqrt(vhat) + eps);
    if (mode == 0 && xi < 0.0) xi = 0.0;  // project_nonneg
    if (mode == 1) xi = i == 0 ? clampd(xi, 0.0, 1.0) : (xi > 0.0 ? xi : 0.0);
    x[i] = xi;
}

__global__ void k_size_terms(const uint32_t* B, long long n, unsigned long long* rt,
                             unsigned long long* it) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t b = B[i];
    rt[i] = (unsigned long long)b + 1ull;
    it[i] = b >= 2 ? (unsigned long long)(b - 1) : 0ull;
}

__global__ void k_path_major(const unsigned long long* ro, const unsigned long long* io, long long n,
                             unsigned long long* rb, uint32_t* stride, unsigned long long* ib) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    rb[i] = ro[i];
    stride[i] = 1u;
    ib[i] = io[i];
}

// ============================================================================ K2 sort
// Pass 1: per-tile histogram of B (bin-major output so one exclusive scan yields the
// stable destination base of every (bin, tile)).
__global__ void k_sort_hist(const uint32_t* B, long long n, int nb, int tile,
                            unsigned long long* th) {
    extern __shared__ unsigned int h[];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const long long t0 = (long long)blockIdx.x * tile;
    const long long t1 = t0 + tile < n ? t0 + tile : n;
    for (long long i = t0 + threadIdx.x; i < t1; i += blockDim.x) atomicAdd(&h[B[i]], 1u);
    __syncthreads();
    const long long n_tiles = gridDim.x;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) th[(long long)i * n_tiles + blockIdx.x] = h[i];
}

// Pass 2: one warp walks its tile in order; equal keys within a 32-element chunk are
// ranked with __match_any_sync, so the permutation is exactly std::stable_sort's.
__global__ void __launch_bounds__(32) k_sort_rank(const uint32_t* B, long long n, int nb, int tile,
                                                  const unsigned long long* toff, uint32_t* perm) {
    extern __shared__ unsigned long long run[];
    const long long n_tiles = gridDim.x;
    const int lane = threadIdx.x;
    for (int i = lane; i < nb; i += 32) run[i] = toff[(long long)i * n_tiles + blockIdx.x];
    __syncwarp();
    const long long t0 = (long long)blockIdx.x * tile;
    const long long t1 = t0 + tile < n ? t0 + tile : n;
    const unsigned lt = (1u << lane) - 1u;
    for (long long c = t0; c < t1; c += 32) {
        const long long i = c + lane;
        const bool act = i < t1;
        const uint32_t key = act ? B[i] : 0xffffffffu;
        const unsigned mask = __match_any_sync(0xffffffffu, key);
        const unsigned rank = __popc(mask & lt);
        unsigned long long base = 0;
        if (act) base = run[key];
        __syncwarp();
        if (act) {
            perm[base + rank] = (uint32_t)i;
            if (rank == 0) run[key] = base + (unsigned long long)__popc(mask);
        }
        __syncwarp();
    }
}

__global__ void k_bucket_layout(const uint32_t* perm, const uint32_t* B_old,
                                const unsigned long long* s_old, const uint8_t* tr_old, long long n,
                                const unsigned long long* bstart, const unsigned long long* brec,
                                const unsigned long long* biv, uint32_t* B_new,
                                unsigned long long* s_new, uint8_t* tr_new, unsigned long long* rb,
                                uint32_t* stride, unsigned long long* ib) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t src = perm[i];
    const uint32_t k = B_old[src];
    B_new[i] = k;
    s_new[i] = s_old[src];
    tr_new[i] = tr_old[src];
    const unsigned long long j = (unsigned long long)i - bstart[k];
    stride[i] = (uint32_t)(bstart[k + 1] - bstart[k]);
    rb[i] = brec[k] + j;
    ib[i] = biv[k] + j;
}

// Stream ids of a fresh shard (stream_base + i) and the truncated-path count, on the
// device: at 1e8 paths the host versions moved 800 MB up and 100 MB down per resample.
__global__ void k_iota_u64(unsigned long long* out, long long n, unsigned long long base) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = base + (unsigned long long)i;
}

__global__ void k_count_nonzero_u8(const uint8_t* x, long long n, unsigned long long* count) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned c = __popc(__ballot_sync(0xffffffffu, i < n && x[i] != 0));
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

// One record field at a time (sort_by_size's re-layout): the transient is one field
// (<= 8 B per record) instead of a second copy of all records (72 B per record), so a
// store can fill ~85% of HBM and still be sorted.  Fields move as raw bits.
template <class T>
__global__ void k_gather_field(const __grid_constant__ StoreView o, const uint32_t* perm, long long n,
                               const unsigned long long* rbn, const uint32_t* sn,
                               const T* __restrict__ src, T* __restrict__ dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = perm[i];
    const int B = (int)o.B[p];
    const unsigned long long ob = o.rec_base[p], nb = rbn[i];
    const unsigned os = o.stride[p], ns = sn[i];
    for (int b = 0; b <= B; ++b) dst[nb + (unsigned long long)b * ns] = src[ob + (unsigned long long)b * os];
}

// ============================================================================ diagnostics
__global__ void k_philox(unsigned long long seed, unsigned long long stream, unsigned long long n,
                         uint32_t* out) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    Philox r;
    r.init(seed, stream);
    for (unsigned long long i = 0; i < n; ++i) out[i] = r.u32();
}

template <bool PAD>
__global__ void k_walk(const __grid_constant__ DScene sc, const double* rays, long long n,
                       uint32_t* counts, const unsigned long long* off, uint32_t* vox,
                       double* len) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = rays + 7 * i;
    uint32_t c = 0;
    unsigned long long w = off ? off[i] : 0;
    auto f = [&](int v, double ta, double tb) {
        if (off) {
            vox[w] = (uint32_t)v;
            len[w] = tb - ta;
            ++w;
        }
        ++c;
        return true;
    };
    if (PAD)
        dda_walk_pad(sc, mk(r[0], r[1], r[2]), mk(r[3], r[4], r[5]), r[6], f);
    else
        dda_walk(sc, mk(r[0], r[1], r[2]), mk(r[3], r[4], r[5]), r[6], f);
    if (!off) counts[i] = c;
}

// space_carve (inverse.cpp:69-101): voxel centre (grid.hpp:56-62, same operation order)
// projected into every detector; occupied when every view sees it above the threshold.
__global__ void k_space_carve(const __grid_constant__ DScene sc, const double* __restrict__ gt,
                              const double* __restrict__ thr, double fill, uint8_t* mask, double* beta) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= sc.V) return;
    const int nx = sc.dims[0], ny = sc.dims[1];
    const int ix = (int)(v % nx), iy = (int)((v / nx) % ny), iz = (int)(v / ((long long)nx * ny));
    const V3 c = mk(sc.gorg[0] + ((double)ix + 0.5) * sc.vs[0], sc.gorg[1] + ((double)iy + 0.5) * sc.vs[1],
                    sc.gorg[2] + ((double)iz + 0.5) * sc.vs[2]);
    bool occupied = true;
    for (int k = 0; k < sc.n_det && occupied; ++k) {
        const int pixel = pixel_of(sc.det[k], c);
        occupied = pixel >= 0 && gt[sc.det[k].img_off + pixel] > thr[k];
    }
    if (mask) mask[v] = occupied ? 1 : 0;
    if (beta) beta[v] = occupied ? fill : 0.0;
}

__global__ void k_pixel_of(const __grid_constant__ DScene sc, int det, const double* pts, long long n,
                           int32_t* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = pixel_of(sc.det[det], mk(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]));
}

__global__ void k_events(const __grid_constant__ DScene sc, const __grid_constant__ StoreView st,
                         int32_t* pix_out, double* cos_out, double* geom_out, double* ray_out) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= (long long)st.n) return;
    const int B = (int)st.B[p];
    const unsigned long long rb = st.rec_base[p], ib = st.iv_base[p];
    const unsigned rs = st.stride[p];
    for (int b = 1; b < B; ++b) {
        const Rec R = load_rec(st, rb + (unsigned long long)b * rs);
        const unsigned long long iv = ib + (unsigned long long)(b - 1) * rs;
        for (int k = 0; k < sc.n_det; ++k) {
            const unsigned long long slot = (unsigned long long)k * st.n_iv + iv;
            int pix = pixel_of(sc.det[k], R.x);
            V3 w = mk(0, 0, 0);
            double r = 0, geom = 0, cos_le = 0;
            if (pix >= 0 &&
                !event_geometry(sc, sc.det[k], R.x, R.d, meta_kind(R.meta), meta_surface(R.meta), w, r,
                                geom, cos_le))
                pix = -1;
            pix_out[slot] = pix;
            cos_out[slot] = cos_le;
            geom_out[slot] = geom;
            ray_out[4 * slot + 0] = w.x;
            ray_out[4 * slot + 1] = w.y;
            ray_out[4 * slot + 2] = w.z;
            ray_out[4 * slot + 3] = r;
        }
    }
}

__global__ void __launch_bounds__(kTPB) k_stats(const __grid_constant__ DScene sc,
                                                const __grid_constant__ StoreView st,
                                                unsigned long long* out) {
    const long long p = path_index(st.n);
    unsigned long long ev = 0, live = 0, le = 0, all = 0;
    if (p >= 0) {
        const int B = (int)st.B[p];
        const unsigned long long rb = st.rec_base[p];
        const unsigned rs = st.stride[p];
        V3 xprev = mk(st.px[rb], st.py[rb], st.pz[rb]);
        for (int b = 1; b <= B; ++b) {
            const Rec R = load_rec(st, rb + (unsigned long long)b * rs);
            unsigned long long c = 0;
            if (sc.has_medium)
                dda_walk(sc, xprev, R.d, R.t, [&](int, double, double) {
                    ++c;
                    return true;
                });
            all += c;
            if (b < B) {
                live += c;
                for (int k = 0; k < sc.n_det; ++k) {
                    const DDet& D = sc.det[k];
                    if (pixel_of(D, R.x) < 0) continue;
                    V3 w;
                    double r, geom, cos_le;
                    if (!event_geometry(sc, D, R.x, R.d, meta_kind(R.meta), meta_surface(R.meta), w, r,
                                        geom, cos_le))
                        continue;
                    ++ev;
                    if (sc.has_medium)
                        dda_walk(sc, R.x, w, r, [&](int, double, double) {
                            ++le;
                            return true;
                        });
                }
            }
            xprev = R.x;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        ev += __shfl_down_sync(0xffffffffu, ev, o);
        live += __shfl_down_sync(0xffffffffu, live, o);
        le += __shfl_down_sync(0xffffffffu, le, o);
        all += __shfl_down_sync(0xffffffffu, all, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, ev);
        atomicAdd(out + 1, live);
        atomicAdd(out + 2, le);
        atomicAdd(out + 3, all);
    }
}

}  // namespace

// ============================================================================ launchers
#define LAUNCH_DONE()                      \
    do {                                   \
        if (launches) ++*launches;         \
        return cudaGetLastError();         \
    } while (0)

cudaError_t launch_trace(const DScene& sc, const TraceArgs& a, bool write, cudaStream_t s,
                         unsigned long long* launches) {
    if (a.n == 0) return cudaSuccess;
    const unsigned chunk = a.n >= 5000000ull ? kTPB * 8u : (unsigned)kTPB;  // paths per CTA
    if (write)
        k_trace<true><<<grid_for((long long)a.n, (int)chunk), kTPB, 0, s>>>(sc, a, chunk);
    else
        k_trace<false><<<grid_for((long long)a.n, (int)chunk), kTPB, 0, s>>>(sc, a, chunk);
    LAUNCH_DONE();
}

cudaError_t launch_prep_ref(int n_species, long long V, const double* const* src_ref, double* br64,
                            float* sp_ref, float* br, double* beta_tot64, cudaStream_t s,
                            unsigned long long* launches) {
    if (V == 0) return cudaSuccess;
    SrcPtrs sp{};
    for (int j = 0; j < n_species; ++j) sp.p[j] = src_ref[j];
    k_prep_ref<<<grid_for(V, 256), 256, 0, s>>>(n_species, V, sp, br64, sp_ref, br, beta_tot64);
    LAUNCH_DONE();
}

cudaError_t launch_prep(int n_species, long long V, const double* const* src_t, const double* br64,
                        float* sp_t, float* bt, float* dbeta, cudaStream_t s,
                        unsigned long long* launches) {
    if (V == 0) return cudaSuccess;
    SrcPtrs sp{};
    for (int j = 0; j < n_species; ++j) sp.p[j] = src_t[j];
    k_prep<<<grid_for(V, 256), 256, 0, s>>>(n_species, V, sp, br64, sp_t, bt, dbeta);
    LAUNCH_DONE();
}

cudaError_t launch_set_species(int n_species, long long V, int unknown, const double* scene_sp,
                               const double* beta_u, double* out, cudaStream_t s,
                               unsigned long long* launches) {
    if (V == 0 || n_species == 0) return cudaSuccess;
    k_set_species<<<grid_for((long long)n_species * V, 256), 256, 0, s>>>(n_species, V, unknown,
                                                                           scene_sp, beta_u, out);
    LAUNCH_DONE();
}

cudaError_t launch_forward(const DScene& sc, const StoreView& st, const EvalArgs& ea, cudaStream_t s,
                           unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_forward<<<grid_for((long long)st.n), kTPB, 0, s>>>(sc, st, ea);
    LAUNCH_DONE();
}

cudaError_t launch_gradient(const DScene& sc, const StoreView& st, const EvalArgs& ea,
                            cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_gradient<<<grid_for((long long)st.n), kTPB, 0, s>>>(sc, st, ea);
    LAUNCH_DONE();
}

cudaError_t launch_scale(double* x, long long n, double scale, cudaStream_t s,
                         unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_scale<<<grid_for(n, 256), 256, 0, s>>>(x, n, scale);
    LAUNCH_DONE();
}

namespace {
__global__ void k_fx_limbs(const unsigned long long* __restrict__ fx, long long n, unsigned long long* __restrict__ l) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long lo = fx[2 * i], hi = fx[2 * i + 1];
    const unsigned long long m = (1ull << 43) - 1;
    l[3 * i] = lo & m;
    l[3 * i + 1] = ((lo >> 43) | (hi << 21)) & m;
    l[3 * i + 2] = hi >> 22;
}
__global__ void k_limbs_images(const unsigned long long* __restrict__ l, long long n, double quantum,
                               double* __restrict__ img) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    img[i] = (((double)l[3 * i + 2] * 0x1p86 + (double)l[3 * i + 1] * 0x1p43) + (double)l[3 * i]) * quantum;
}
}  // namespace

cudaError_t launch_fixed_to_limbs(const unsigned long long* fx, long long n, unsigned long long* limbs,
                                  cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_fx_limbs<<<grid_for(n, 256), 256, 0, s>>>(fx, n, limbs);
    LAUNCH_DONE();
}

cudaError_t launch_limbs_to_images(const unsigned long long* limbs, long long n, double quantum, double* images,
                                   cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_limbs_images<<<grid_for(n, 256), 256, 0, s>>>(limbs, n, quantum, images);
    LAUNCH_DONE();
}

cudaError_t launch_combine_grad(const double* gs, const double* gv, int n_out, long long V,
                                double scale, double* out, cudaStream_t s,
                                unsigned long long* launches) {
    if (V == 0) return cudaSuccess;
    k_combine<<<grid_for((long long)n_out * V, 256), 256, 0, s>>>(gs, gv, n_out, V, scale, out);
    LAUNCH_DONE();
}

cudaError_t launch_loss_residual(const double* F, const double* gt, long long n, double* res,
                                 double* loss, cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_loss_residual<<<grid_for(n, 256), 256, 0, s>>>(F, gt, n, res, loss);
    LAUNCH_DONE();
}

cudaError_t launch_adam(double* x, double* m1, double* m2, const double* g, long long n, double alpha,
                        double eta1, double eta2, double eps, double c1, double c2,
                        const double* step_scale, int n_ss, int mode, cudaStream_t s,
                        unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_adam<<<grid_for(n, 256), 256, 0, s>>>(x, m1, m2, g, n, alpha, eta1, eta2, eps, c1, c2,
                                             step_scale, n_ss, mode);
    LAUNCH_DONE();
}

// Exclusive u64 scan, reduce-then-scan: a CTA of kScanTPB threads owns a chunk of
// kScanChunk elements.  Pass 1 writes the chunk sums, the chunk sums are scanned in place
// by the same routine (one more level per 4096x), pass 2 scans each chunk in shared memory
// from its chunk offset.  Used on the resample path (trace offsets, the sort's tile
// histograms, the event list), 1e8-element scans take ~0.1 ms.
cudaError_t scan_u64(const unsigned long long* in, unsigned long long* out, long long n, void** tmp,
                     size_t* tmp_bytes, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    // chunk-sum arrays of every level, in tmp
    size_t need = 0;
    for (long long m = n; m > 1;) {
        m = (m + kScanChunk - 1) / kScanChunk;
        need += (size_t)m * sizeof(unsigned long long);
        if (m == 1) break;
    }
    need = need > 0 ? need : sizeof(unsigned long long);
    if (need > *tmp_bytes) {
        if (*tmp) cudaFree(*tmp);
        cudaError_t e = prc_malloc_retry(tmp, need);
        if (e != cudaSuccess) {
            *tmp = nullptr;
            *tmp_bytes = 0;
            return e;
        }
        *tmp_bytes = need;
    }
    return scan_levels(in, out, n, static_cast<unsigned long long*>(*tmp), s);
}

cudaError_t reduce_max_u32(const uint32_t* in, long long n, uint32_t* out_dev, void** tmp,
                           size_t* tmp_bytes, cudaStream_t s) {
    (void)tmp;
    (void)tmp_bytes;
    cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || n <= 0) return e;
    const long long blocks = std::min<long long>((n + 1023) / 1024, 4096);
    k_max_u32<<<(unsigned)blocks, 256, 0, s>>>(in, n, out_dev);
    return cudaGetLastError();
}

cudaError_t launch_size_terms(const uint32_t* B, long long n, unsigned long long* rt,
                              unsigned long long* it, cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_size_terms<<<grid_for(n, 256), 256, 0, s>>>(B, n, rt, it);
    LAUNCH_DONE();
}

cudaError_t launch_path_major_layout(const unsigned long long* ro, const unsigned long long* io,
                                     long long n, unsigned long long* rb, uint32_t* stride,
                                     unsigned long long* ib, cudaStream_t s,
                                     unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_path_major<<<grid_for(n, 256), 256, 0, s>>>(ro, io, n, rb, stride, ib);
    LAUNCH_DONE();
}

cudaError_t launch_sort_hist(const uint32_t* B, long long n, int nb, int tile,
                             unsigned long long* th, cudaStream_t s, unsigned long long* launches) {
    const long long n_tiles = (n + tile - 1) / tile;
    k_sort_hist<<<(unsigned)n_tiles, 256, (size_t)nb * sizeof(unsigned), s>>>(B, n, nb, tile, th);
    LAUNCH_DONE();
}

cudaError_t launch_sort_rank(const uint32_t* B, long long n, int nb, int tile,
                             const unsigned long long* toff, uint32_t* perm, cudaStream_t s,
                             unsigned long long* launches) {
    const long long n_tiles = (n + tile - 1) / tile;
    const size_t smem = (size_t)nb * sizeof(unsigned long long);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_sort_rank, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_sort_rank<<<(unsigned)n_tiles, 32, smem, s>>>(B, n, nb, tile, toff, perm);
    LAUNCH_DONE();
}

cudaError_t launch_bucket_layout(const uint32_t* perm, const uint32_t* B_old,
                                 const unsigned long long* s_old, const uint8_t* tr_old, long long n,
                                 const unsigned long long* bstart, const unsigned long long* brec,
                                 const unsigned long long* biv, uint32_t* B_new,
                                 unsigned long long* s_new, uint8_t* tr_new, unsigned long long* rb,
                                 uint32_t* stride, unsigned long long* ib, cudaStream_t s,
                                 unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_bucket_layout<<<grid_for(n, 256), 256, 0, s>>>(perm, B_old, s_old, tr_old, n, bstart, brec, biv,
                                                      B_new, s_new, tr_new, rb, stride, ib);
    LAUNCH_DONE();
}

cudaError_t launch_iota_u64(unsigned long long* out, long long n, unsigned long long base, cudaStream_t s,
                            unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_iota_u64<<<grid_for(n, 256), 256, 0, s>>>(out, n, base);
    LAUNCH_DONE();
}

cudaError_t launch_count_nonzero_u8(const uint8_t* x, long long n, unsigned long long* count, cudaStream_t s,
                                    unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_count_nonzero_u8<<<grid_for(n, 256), 256, 0, s>>>(x, n, count);
    LAUNCH_DONE();
}

cudaError_t launch_gather_field(const StoreView& o, const uint32_t* perm, long long n,
                                const unsigned long long* rbn, const uint32_t* sn, const void* src,
                                void* dst, int elem_bytes, cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    if (elem_bytes == 8)
        k_gather_field<unsigned long long><<<grid_for(n, 128), 128, 0, s>>>(
            o, perm, n, rbn, sn, (const unsigned long long*)src, (unsigned long long*)dst);
    else
        k_gather_field<uint32_t><<<grid_for(n, 128), 128, 0, s>>>(o, perm, n, rbn, sn, (const uint32_t*)src,
                                                                  (uint32_t*)dst);
    LAUNCH_DONE();
}

cudaError_t launch_philox(unsigned long long seed, unsigned long long stream, unsigned long long n,
                          uint32_t* out, cudaStream_t s, unsigned long long* launches) {
    k_philox<<<1, 1, 0, s>>>(seed, stream, n, out);
    LAUNCH_DONE();
}

cudaError_t launch_walk(const DScene& sc, const double* rays, long long n, uint32_t* counts,
                        const unsigned long long* off, uint32_t* vox, double* len, cudaStream_t s,
                        unsigned long long* launches, bool pad) {
    if (n == 0) return cudaSuccess;
    if (pad)
        k_walk<true><<<grid_for(n), kTPB, 0, s>>>(sc, rays, n, counts, off, vox, len);
    else
        k_walk<false><<<grid_for(n), kTPB, 0, s>>>(sc, rays, n, counts, off, vox, len);
    LAUNCH_DONE();
}

cudaError_t launch_space_carve(const DScene& sc, const double* gt, const double* thr, double fill, uint8_t* mask,
                               double* beta, cudaStream_t s, unsigned long long* launches) {
    if (sc.V == 0) return cudaSuccess;
    k_space_carve<<<grid_for(sc.V), kTPB, 0, s>>>(sc, gt, thr, fill, mask, beta);
    LAUNCH_DONE();
}

cudaError_t launch_pixel_of(const DScene& sc, int det, const double* pts, long long n, int32_t* out,
                            cudaStream_t s, unsigned long long* launches) {
    if (n == 0) return cudaSuccess;
    k_pixel_of<<<grid_for(n), kTPB, 0, s>>>(sc, det, pts, n, out);
    LAUNCH_DONE();
}

cudaError_t launch_stats(const DScene& sc, const StoreView& st, unsigned long long* out,
                         cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_stats<<<grid_for((long long)st.n), kTPB, 0, s>>>(sc, st, out);
    LAUNCH_DONE();
}

cudaError_t launch_events(const DScene& sc, const StoreView& st, int32_t* pix, double* cos_le,
                          double* geom, double* ray, cudaStream_t s, unsigned long long* launches) {
    if (st.n == 0) return cudaSuccess;
    k_events<<<grid_for((long long)st.n), kTPB, 0, s>>>(sc, st, pix, cos_le, geom, ray);
    LAUNCH_DONE();
}
