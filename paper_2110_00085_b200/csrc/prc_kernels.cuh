// prc_kernels.cuh — kernel argument blocks and host-side launchers (prc_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "prc_device.cuh"

// Device path store in structure-of-arrays form.  Record (p, b) = vertex b of the path
// in storage position p lives at rec_base[p] + b * stride[p]; its event-cache slot
// (interaction vertices b = 1..B-1) at iv_base[p] + (b - 1) * stride[p].  After the
// trace the layout is path-major (stride 1); after sort_by_size it is bucket-major
// (paths of equal B interleaved, stride = bucket population) so that a warp of 32
// consecutive sorted paths reads each field of vertex b with one coalesced request.
struct StoreView {
    unsigned long long n;
    const uint32_t* B;
    const unsigned long long* rec_base;
    const uint32_t* stride;
    const unsigned long long* iv_base;
    const double *px, *py, *pz, *dx, *dy, *dz, *tt, *ct;
    const int32_t* vox;
    const uint32_t* meta;
    unsigned long long n_iv;
    float* ev_val;    // [det][iv]: cached event value (K4 -> K5)
    int32_t* ev_pix;  // [det][iv]: pixel, -1 when no event
};

// Interaction vertices (b = 1..B-1 of every path) in Morton order of their position:
// the unit of the event-major wavefront.  A CTA takes a contiguous run of vertices and
// walks the cameras one after another, so a warp's 32 local-estimation rays start within
// a voxel or two of each other and run to the same camera (coherent DDA trip counts,
// L1-resident beta gathers, overlapping voxel sets for the gradient scatter).
struct VertexTable {
    unsigned long long n;
    const double *x, *y, *z, *dx, *dy, *dz;
    const int32_t* vox;
    const uint32_t* meta;
    const uint32_t* iv;  // interaction-vertex slot (path-layout index) of entry i
    float* ev_val;       // [det][i] cached event value (K4b -> K5b), 0 when no event
    int32_t* ev_pix;     // [det][i] pixel, -1 when no event (geometric: dead vertices keep theirs)
    // Beta-independent part of a single-species volume event's value (K4b): c1 =
    // log(albedo * phase(cos_le)) in fixed point (DScene::c1_fast; INT32_MIN = no event).
    // Written with ev_pix by the first forward over a store, read by later ones
    // (geo_ready), which then skip pixel_of, the visibility tests, the phase function and
    // its log.
    int32_t* ev_c1;      // [det][i]
    // Scenes with DScene::fcache: the phase values f_j(cos_le) of every species as f32,
    // [j][det][i]; written and read like ev_c1 (both passes use the rounded values).
    // Scenes with DScene::scache: each surface event's cos_le as f64, [det][i], stored in
    // the same buffer after the phase values (ev_cos_of); its geometry factor (f32) is kept
    // in ev_c1, unused by surface events otherwise.  (One buffer keeps the kernel parameter
    // layout of medium-only scenes unchanged.)
    float* ev_f;
    int geo_ready;
};

struct RecordsOut {
    double *px, *py, *pz, *dx, *dy, *dz, *tt, *ct;
    int32_t* vox;
    uint32_t* meta;
};

struct EvalArgs {
    const float* sp_t;    // n_species x V, extinction under the evaluated parameters
    const float* sp_ref;  // n_species x V, extinction the paths were sampled under
    const float* bt_tot;  // V
    const float* br_tot;  // V
    const float* dbeta;   // V: bt_tot - br_tot (computed in fp64, stored fp32)
    const double* phong;  // [kappa_s, gamma] bound to the target surface
    double* images;       // raw (un-normalised) pixel sums
    unsigned long long* clamps;
    const double* weights;  // pixel weights (residuals), NULL = 1
    double* g_span;         // V: transmittance part of dL/dbeta, shared by all species
    double* g_vert;         // n_vert_out x V: vertex score parts
    double* g_phong;        // [d kappa, d gamma]
    // padded layout (DScene::pad_walk): bt_tot / dbeta with a zero border, and the
    // padded accumulator of the LE + path span gradient (folded into g_span by k_unpad_add)
    const double* bt_pad;  // fp64: the walk's FMA takes it without an F2F conversion
    const double* db_pad;
    double* g_pad;
    // K5b reduces into g_pad_copies copies of the padded gradient, g_pad_stride apart (CTA b
    // into copy b mod copies): same-address reductions from many SMs spread over more L2
    // lines.  Measured at 1e8 paths (config (b)): K5b 784 -> 718 ms with 2 copies, 697 with 4,
    // 694 with 8; at 256^3 (config (e)) 1973 -> 1808 (2) -> 1728 ms (4).  Default 8 (r13:
    // 670 -> 663 ms at 128^3).  k_unpad_add sums the copies; K5a uses copy 0.
    long long g_pad_stride;
    int g_pad_copies;
    int per_species, legacy, do_beta;
    // Image accumulation (image_add, prc_eval.cuh): 0 fp64 reductions into `images`
    // (default); 1 the largest contribution's bits into *img_max (first pass of a
    // deterministic evaluation); 2 exact 128-bit fixed-point sums into img_fx (two u64 per
    // pixel, quantum 1 / img_inv_quantum), independent of the order of the additions, so the
    // image is bit-reproducible (render() is, transport.hpp:171-173).
    int img_mode;
    unsigned long long* img_max;
    unsigned long long* img_fx;
    double img_inv_quantum;
    // Scenes on the event list (no medium): per interaction-vertex slot, the surface
    // vertex's continuation lobe term -- the target surface's lc = log(clamp(cos, 0, 1)),
    // any other surface's log(pi f_r(cos)) (-inf: f_r <= 0); NULL elsewhere.  K4a / K5a
    // then skip the fixed surfaces' BRDF and logs (the same values, cached).
    const double* vlobe;
};

struct TraceArgs {
    const double* beta_tot;  // V, fp64 total extinction (sampling point)
    const double* sp_beta;   // n_species x V, fp64
    unsigned long long seed, stream_base, n;
    int max_bounces, max_events;
    uint32_t* B;
    uint8_t* trunc;
    int* err;
    const unsigned long long* off;  // write pass: record offset of each path
    RecordsOut rec;
};

// cudaMalloc that, when the device is out of memory, first hands the engine's cached
// blocks (prc_capi.cu, BlockCache) back to the driver and retries.
cudaError_t prc_malloc_retry(void** p, size_t bytes);

// ---- launchers (return cudaError_t); `launches` counts kernels issued -------------
// Padded layout: bt_pad/db_pad interiors <- bt_tot/dbeta (borders stay zero), and
// g_span += interior of g_pad (all copies).
cudaError_t launch_pad_tables(const DScene& sc, const float* bt_tot, const float* dbeta, double* bt_pad,
                              double* db_pad, cudaStream_t s, unsigned long long* launches);
cudaError_t launch_unpad_add(const DScene& sc, const double* g_pad, int copies, long long stride,
                             double* g_span, cudaStream_t s,
                             unsigned long long* launches);
cudaError_t launch_trace(const DScene& sc, const TraceArgs& a, bool write, cudaStream_t s,
                         unsigned long long* launches);
cudaError_t launch_prep(int n_species, long long V, const double* const* src_t,
                        const double* br_tot64, float* sp_t, float* bt_tot, float* dbeta,
                        cudaStream_t s, unsigned long long* launches);
cudaError_t launch_prep_ref(int n_species, long long V, const double* const* src_ref,
                            double* br_tot64, float* sp_ref, float* br_tot, double* beta_tot64,
                            cudaStream_t s, unsigned long long* launches);
cudaError_t launch_forward(const DScene& sc, const StoreView& st, const EvalArgs& ea,
                           cudaStream_t s, unsigned long long* launches);
cudaError_t launch_gradient(const DScene& sc, const StoreView& st, const EvalArgs& ea,
                            cudaStream_t s, unsigned long long* launches);
cudaError_t launch_scale(double* x, long long n, double scale, cudaStream_t s,
                         unsigned long long* launches);
// Deterministic images (EvalArgs::img_mode 2): the 128-bit sums (hi, lo) split into three
// 43-bit limbs (so ranks can add them with an integer allreduce without losing carries),
// then images[p] = ((l2 * 2^86 + l1 * 2^43) + l0) * quantum.
cudaError_t launch_fixed_to_limbs(const unsigned long long* fx, long long n, unsigned long long* limbs,
                                  cudaStream_t s, unsigned long long* launches);
cudaError_t launch_limbs_to_images(const unsigned long long* limbs, long long n, double quantum, double* images,
                                   cudaStream_t s, unsigned long long* launches);
cudaError_t launch_combine_grad(const double* g_span, const double* g_vert, int n_out, long long V,
                                double scale, double* out, cudaStream_t s,
                                unsigned long long* launches);
cudaError_t launch_loss_residual(const double* F, const double* gt, long long n, double* residual,
                                 double* loss, cudaStream_t s, unsigned long long* launches);
cudaError_t launch_adam(double* x, double* m1, double* m2, const double* g, long long n,
                        double alpha, double eta1, double eta2, double eps, double c1, double c2,
                        const double* step_scale, int n_step_scale, int mode, cudaStream_t s,
                        unsigned long long* launches);
cudaError_t launch_set_species(int n_species, long long V, int unknown, const double* scene_sp,
                               const double* beta_unknown, double* out, cudaStream_t s,
                               unsigned long long* launches);

// Exclusive scan of n uint64 values (CUB).  tmp is grown as needed.
cudaError_t scan_u64(const unsigned long long* in, unsigned long long* out, long long n,
                     void** tmp, size_t* tmp_bytes, cudaStream_t s);
cudaError_t launch_size_terms(const uint32_t* B, long long n, unsigned long long* rec_terms,
                              unsigned long long* iv_terms, cudaStream_t s,
                              unsigned long long* launches);
cudaError_t launch_path_major_layout(const unsigned long long* rec_off,
                                     const unsigned long long* iv_off, long long n,
                                     unsigned long long* rec_base, uint32_t* stride,
                                     unsigned long long* iv_base, cudaStream_t s,
                                     unsigned long long* launches);
cudaError_t reduce_max_u32(const uint32_t* in, long long n, uint32_t* out_dev, void** tmp,
                           size_t* tmp_bytes, cudaStream_t s);

// ---- K2 stable counting sort by B ------------------------------------------------
// tile_hist: nb * n_tiles counters (bin-major).  perm[dest] = source position.
cudaError_t launch_sort_hist(const uint32_t* B, long long n, int nb, int tile,
                             unsigned long long* tile_hist, cudaStream_t s,
                             unsigned long long* launches);
cudaError_t launch_sort_rank(const uint32_t* B, long long n, int nb, int tile,
                             const unsigned long long* tile_off, uint32_t* perm,
                             cudaStream_t s, unsigned long long* launches);
// Builds the bucket-major layout of sorted path i from the bucket table.
cudaError_t launch_bucket_layout(const uint32_t* perm, const uint32_t* B_old,
                                 const unsigned long long* stream_old, const uint8_t* trunc_old,
                                 long long n, const unsigned long long* bucket_start,
                                 const unsigned long long* bucket_rec,
                                 const unsigned long long* bucket_iv, uint32_t* B_new,
                                 unsigned long long* stream_new, uint8_t* trunc_new,
                                 unsigned long long* rec_base, uint32_t* stride,
                                 unsigned long long* iv_base, cudaStream_t s,
                                 unsigned long long* launches);
cudaError_t launch_iota_u64(unsigned long long* out, long long n, unsigned long long base, cudaStream_t s,
                            unsigned long long* launches);
// count += number of nonzero bytes in x[0, n)
cudaError_t launch_count_nonzero_u8(const uint8_t* x, long long n, unsigned long long* count, cudaStream_t s,
                                    unsigned long long* launches);
cudaError_t launch_gather_field(const StoreView& old_st, const uint32_t* perm, long long n,
                                const unsigned long long* rec_base_new, const uint32_t* stride_new,
                                const void* src, void* dst, int elem_bytes, cudaStream_t s,
                                unsigned long long* launches);

// ---- event-major wavefront (default mapping) -------------------------------------
// Vertex-table construction: Morton keys + iv -> record map, CUB radix sort, gather.
cudaError_t launch_vt_keys(const DScene& sc, const StoreView& st, uint32_t* keys,
                           uint32_t* iv_values, unsigned long long* iv_rec, cudaStream_t s,
                           unsigned long long* launches);
cudaError_t sort_pairs_u32(const uint32_t* keys_in, uint32_t* keys_out, const uint32_t* vals_in,
                           uint32_t* vals_out, long long n, void** tmp, size_t* tmp_bytes,
                           cudaStream_t s);
cudaError_t launch_vt_gather(const StoreView& st, const uint32_t* vt2iv,
                             const unsigned long long* iv_rec, long long n, double* x, double* y,
                             double* z, double* dx, double* dy, double* dz, int32_t* vox,
                             uint32_t* meta, uint32_t* iv, cudaStream_t s,
                             unsigned long long* launches);
// K4a: per-path log-prefix at every interaction vertex (lp[iv], -inf when dead).
cudaError_t launch_prefix(const DScene& sc, const StoreView& st, const EvalArgs& ea, double* lp,
                          cudaStream_t s, unsigned long long* launches);
// K4b: per-event LE forward over the vertex table.
cudaError_t launch_le_forward(const DScene& sc, const VertexTable& vt, const EvalArgs& ea,
                              const double* lp, cudaStream_t s, unsigned long long* launches);
// K5b: per-event LE gradient scatter (fp64 L2 reductions; `packet` rays per thread in
// lockstep with in-register voxel merging, lanes `spread` packets apart) and the
// per-vertex event-weight sums own[iv].
cudaError_t launch_le_gradient(const DScene& sc, const VertexTable& vt, const EvalArgs& ea,
                               double* own, int spread, int packet, cudaStream_t s,
                               unsigned long long* launches);
// Event list of a scene without a medium (reflectometry, config (d)): no LE walks, so an
// event is a BRDF evaluation, one image reduction and its weight -- and most (vertex,
// camera) slots of the dense [det][i] cache hold no event (a surface point faces few
// cameras).  Built once per store geometry from that cache, in interaction-vertex order
// (events of one vertex contiguous, cameras ascending): the log-prefix gathers of K4b'
// and the weight sums of K5b' run along lp / own.
struct EventList {
    unsigned long long n, n_iv;
    const unsigned long long* off;  // [n_iv + 1]: events of slot iv are [off[iv], off[iv + 1])
    const uint32_t* iv;             // interaction-vertex slot of the event
    const int32_t* px;              // image index img_off[det] + pixel
    // the target surface's events: lc = log(clamp(cos_le, 0, 1)) (pow01); other surfaces
    // (fixed BRDF): the BRDF value f_r(cos_le) itself
    const double* lobe;
    const float* geom;              // cached f32 geometry factor
    const uint8_t* surf;            // surface id
    float* val;                     // event value, K4b' -> K5b'
};
// cnt[iv] = events of slot iv (cnt zeroed by the caller, n_iv + 1 entries).
cudaError_t launch_evc_count(const DScene& sc, const VertexTable& vt, unsigned long long* cnt, cudaStream_t s,
                             unsigned long long* launches);
cudaError_t launch_evc_fill(const DScene& sc, const VertexTable& vt, const unsigned long long* off, uint32_t* iv,
                            int32_t* px, double* lobe, float* geom, uint8_t* surf, cudaStream_t s,
                            unsigned long long* launches);
// EvalArgs::vlobe of every interaction vertex of the store (thread per path).
cudaError_t launch_vlobe(const DScene& sc, const StoreView& st, double* vlobe, cudaStream_t s,
                         unsigned long long* launches);
// K4b' and K5b' (thread per event) over the event list.
cudaError_t launch_evc_forward(const DScene& sc, const EventList& el, const EvalArgs& ea, const double* lp,
                               cudaStream_t s, unsigned long long* launches);
cudaError_t launch_evc_gradient(const DScene& sc, const EventList& el, const EvalArgs& ea, double* own,
                                cudaStream_t s, unsigned long long* launches);
// Sum over the store of correction_factor (pathstore.cpp:269-294) under the current
// context (EvalOptions::self_normalize), and each path's factor into per_path[storage
// position] when per_path is not NULL; *err set on a zero reference extinction.
cudaError_t launch_correction(const DScene& sc, const StoreView& st, const EvalArgs& ea, double* sum, int* err,
                              double* per_path, cudaStream_t s, unsigned long long* launches);
// K5a: per-path suffix pass (segment spans, continuation scores) from own[iv].
cudaError_t launch_path_gradient(const DScene& sc, const StoreView& st, const EvalArgs& ea,
                                 const double* own, cudaStream_t s, unsigned long long* launches);

// ---- diagnostics / export ----------------------------------------------------------
cudaError_t launch_philox(unsigned long long seed, unsigned long long stream,
                          unsigned long long n, uint32_t* out, cudaStream_t s,
                          unsigned long long* launches);
cudaError_t launch_walk(const DScene& sc, const double* rays, long long n, uint32_t* counts,
                        const unsigned long long* offsets, uint32_t* vox, double* len,
                        cudaStream_t s, unsigned long long* launches, bool pad = false);
// thr[k] = threshold_fraction * max of view k (host-computed, as inverse.cpp:76-80)
cudaError_t launch_space_carve(const DScene& sc, const double* gt, const double* thr, double fill, uint8_t* mask,
                               double* beta, cudaStream_t s, unsigned long long* launches);
cudaError_t launch_pixel_of(const DScene& sc, int det, const double* pts, long long n,
                            int32_t* out, cudaStream_t s, unsigned long long* launches);
// Per (interaction vertex, detector) event materialisation: valid, pixel, cos_le,
// geom and the LE ray (origin is the vertex; w xyz, r) — slot layout as the cache.
// Counting pass: out[0] events, [1] live path spans, [2] LE spans, [3] all path spans.
cudaError_t launch_stats(const DScene& sc, const StoreView& st, unsigned long long* out,
                         cudaStream_t s, unsigned long long* launches);
cudaError_t launch_events(const DScene& sc, const StoreView& st, int32_t* pix, double* cos_le,
                          double* geom, double* ray_w, cudaStream_t s,
                          unsigned long long* launches);

// ---- materialized evaluation of imported PSTR stores (prc_materialized.cu) ----------
// The reference's own path records as loaded by load_store (pathstore.cpp:455-516):
// stored segment spans, events and LE spans, evaluated exactly as eval_record
// (pathstore.cpp:115-238) reads them, in fp64.  Record arrays are in file order; the
// storage position p of the (possibly sorted) store holds record rec[p].
struct MatView {
    unsigned long long n;                 // paths in this shard
    const unsigned long long* rec;        // [n] record index of storage position p
    const unsigned long long* v_base;     // [n_rec + 1] first vertex of record r
    const unsigned long long* s_base;     // [n_rec] first segment span of record r
    const unsigned long long* e_base;     // [n_rec + 1] first event of record r
    const unsigned long long* l_base;     // [n_rec] first LE span of record r
    const uint32_t* v_meta;               // kind | species << 8 | surface << 16
    const int32_t* v_vox;
    const double* v_ct;                   // cos_theta
    const uint32_t *v_sb, *v_se;          // span range, relative to s_base[r]
    const uint32_t* s_vox;
    const double* s_len;
    const uint32_t* e_vert;               // vertex b of the event
    const int32_t* e_det;
    const int32_t* e_pix;
    const double *e_cos, *e_geom;
    const uint32_t *e_sb, *e_se;          // LE span range, relative to l_base[r]
    const uint32_t* l_vox;
    const double* l_len;
    double* e_val;                        // [events] forward value (K4 -> K5; wbuf / weight)
};

// Per-voxel fp64 context of make_context (pathstore.cpp:54-81): beta_t_tot, beta_ref_tot
// and dbeta from the evaluated species values src_t and the store's reference values
// ref (n_species x V, fp64).
struct MatCtx {
    const double* t[PRC_MAX_SPECIES];
    const double* ref;     // n_species x V
    double* bt_tot;        // V
    double* br_tot;        // V
    double* dbeta;         // V
};
cudaError_t launch_mat_prep(int n_species, long long V, const MatCtx& m, cudaStream_t s,
                            unsigned long long* launches);
// Forward (pathstore.cpp:115-185) or reverse (pathstore.cpp:187-238) over every path.
cudaError_t launch_mat_forward(const DScene& sc, const MatView& mv, const MatCtx& m, const EvalArgs& ea,
                               cudaStream_t s, unsigned long long* launches);
cudaError_t launch_mat_gradient(const DScene& sc, const MatView& mv, const MatCtx& m, const EvalArgs& ea,
                                cudaStream_t s, unsigned long long* launches);
// correction_factor over the stored spans, summed into *sum (self_normalize)
cudaError_t launch_mat_correction(const DScene& sc, const MatView& mv, const MatCtx& m, double* sum, int* err,
                                  double* per_path, cudaStream_t s, unsigned long long* launches);
// dst[i] = src[perm[i]]
cudaError_t launch_gather_u64(const uint32_t* perm, long long n, const unsigned long long* src,
                              unsigned long long* dst, cudaStream_t s, unsigned long long* launches);

// ---- NVLS multicast reduction fused into the K4 / K5 epilogues (prc_nvls.cu) -------
// out[e] += scale * (span(e) + g_vert[e]) on every rank, e < n_out * V: span(e) sums the
// padded gradient copies at voxel e mod V (g_pad non-null) or reads g_span[e mod V]; a
// plain buffer (images) passes only g_span.
struct NvlsFold {
    const double* g_pad;
    int copies;
    long long stride;
    const double* g_span;
    const double* g_vert;
    int n_out;
    long long V;
    int nx, ny, pnx, pnxny;
    double scale;
    double* mc;  // set by nvls_fold
};
__device__ __forceinline__ double fold_value(const NvlsFold& a, long long e) {
    const long long v = e % a.V;
    double s = 0.0;
    if (a.g_pad) {  // k_unpad_add's sum over the copies
        const int ix = (int)(v % a.nx), iy = (int)((v / a.nx) % a.ny), iz = (int)(v / ((long long)a.nx * a.ny));
        const long long pv = (ix + 1) + (long long)a.pnx * (iy + 1) + (long long)a.pnxny * (iz + 1);
        s = a.g_pad[pv];
        for (int c = 1; c < a.copies; ++c) s += a.g_pad[(long long)c * a.stride + pv];
    } else if (a.g_span) {
        s = a.g_span[v];
    }
    if (a.g_vert) s += a.g_vert[e];
    return s;
}
struct NvlsState;
#include <string>
typedef struct ncclComm* ncclComm_t;
// The multicast buffer of n doubles: an NCCL symmetric window with NVLS multimem (world >= 2)
// or a CUDA multicast object on this device alone (world == 1); `emulate` (world == 1) folds
// into a plain buffer with atomics instead, to validate the fold where no multicast exists.
// nullptr + err when the system offers no multicast.
NvlsState* nvls_create(ncclComm_t comm, int world, int device, size_t n_doubles, bool emulate, std::string* err);
void nvls_destroy(NvlsState* s);
double* nvls_local(NvlsState* s);
size_t nvls_capacity(const NvlsState* s);
// Zeroes this rank's copy of [offset, offset + n_out V) and adds every rank's fold into it.
cudaError_t nvls_fold(NvlsState* s, NvlsFold a, size_t offset, cudaStream_t q, unsigned long long* launches);
