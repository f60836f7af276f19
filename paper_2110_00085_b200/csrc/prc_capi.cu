// prc_capi.cu — host runtime and C ABI (include/pathrec_gpu.h) of the B200 engine.
//
// The context owns one CUDA device, one stream, the finalized scene and (for
// world > 1) an NCCL communicator; a path store is a device-resident SoA shard of
// contiguous stream ids [stream_base, stream_base + n).  Reference counterparts:
// render (transport.cpp:405-454), sort_by_size (pathstore.cpp:261-267),
// evaluate_store (pathstore.cpp:315-368), grad_forward (gradient.cpp:111-128),
// reconstruct / adam_step / loss (inverse.cpp:11-67, 154-263), PSTR v1
// (pathstore.cpp:410-516), C-ABI conventions (capi.cpp:17-32).
#include <nccl.h>

#include <algorithm>
#include <set>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pathrec_gpu.h"
#include "prc_kernels.cuh"

#define PRC_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_last_error;

struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t _e = (x);                                                            \
        if (_e != cudaSuccess)                                                           \
            throw Err(PRC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));    \
    } while (0)
#define NK(x)                                                                            \
    do {                                                                                 \
        ncclResult_t _r = (x);                                                           \
        if (_r != ncclSuccess)                                                           \
            throw Err(PRC_ERR_CUDA, std::string(#x) + ": " + ncclGetErrorString(_r));    \
    } while (0)

// Process-wide cache of freed device blocks of >= 1 MB.  The loop frees one path-store
// generation and allocates the next, of nearly the same sizes, every recycle period
// (inverse.cpp:175-204); reusing the blocks skips the driver's unmap / map of tens of GB,
// whose cost varied 10x with what ran on the device before.  A free synchronizes the
// device first, as cudaFree does, so a cached block is idle when it is handed out again.
// Blocks are reused for requests of 7/8 of their size or more; a failed cudaMalloc
// releases the device's cached blocks and retries; contexts release them when destroyed.
struct BlockCache {
    struct Blk {
        void* p;
        size_t bytes;
        int dev;
    };
    std::mutex mu;
    std::vector<Blk> blocks;
};
BlockCache& block_cache() {
    static BlockCache* c = new BlockCache;  // never destroyed: frees may run at process exit
    return *c;
}
constexpr size_t kCacheMin = size_t(1) << 20;

void cache_release(int dev) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    std::vector<BlockCache::Blk> keep;
    for (const auto& b : c.blocks) {
        if (dev >= 0 && b.dev != dev) {
            keep.push_back(b);
            continue;
        }
        cudaSetDevice(b.dev);
        cudaFree(b.p);
    }
    cudaSetDevice(cur);
    c.blocks.swap(keep);
}

// Returns a block of at least `bytes`; *cap receives its size.
void* cache_alloc(size_t bytes, size_t* cap) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (bytes >= kCacheMin) {
        BlockCache& c = block_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        size_t best = c.blocks.size();
        for (size_t i = 0; i < c.blocks.size(); ++i) {
            const auto& b = c.blocks[i];
            if (b.dev == dev && b.bytes >= bytes && b.bytes - b.bytes / 8 <= bytes &&
                (best == c.blocks.size() || b.bytes < c.blocks[best].bytes))
                best = i;
        }
        if (best != c.blocks.size()) {
            void* p = c.blocks[best].p;
            *cap = c.blocks[best].bytes;
            c.blocks.erase(c.blocks.begin() + (long)best);
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        cache_release(dev);
        CK(cudaMalloc(&p, bytes));
    }
    *cap = bytes;
    return p;
}

void cache_free(void* p, size_t cap) {
    if (!p) return;
    if (cap < kCacheMin) {
        cudaFree(p);
        return;
    }
    cudaPointerAttributes a{};
    int dev = 0;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess)
        dev = a.device;
    else
        cudaGetDevice(&dev);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    cudaSetDevice(cur);
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.blocks.push_back({p, cap, dev});
}

}  // namespace

cudaError_t prc_malloc_retry(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaErrorMemoryAllocation) return e;
    cudaGetLastError();
    int dev = 0;
    cudaGetDevice(&dev);
    cache_release(dev);
    return cudaMalloc(p, bytes);
}

namespace {

template <class T>
struct DBuf {  // owning device buffer (BlockCache)
    T* p = nullptr;
    size_t n = 0, cap = 0;  // elements, block bytes
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { reset(); }
    void reset() {
        if (p) cache_free(p, cap);
        p = nullptr;
        n = cap = 0;
    }
    void alloc(size_t count) {
        if (count == n && p) return;
        reset();
        if (count == 0) return;
        p = static_cast<T*>(cache_alloc(count * sizeof(T), &cap));
        n = count;
    }
    void grow(size_t count) {
        if (count > n) alloc(count);
    }
    size_t bytes() const { return n * sizeof(T); }
    void swap(DBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(cap, o.cap);
    }
};

// --------------------------------------------------------------- host fp64 vector ops
// Same operation order as vec3.hpp (compiled with -ffp-contract=off).
struct H3 {
    double x, y, z;
};
H3 h3(const prc_vec3& v) { return {v.x, v.y, v.z}; }
H3 hsub(H3 a, H3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double hdot(H3 a, H3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
double hnorm(H3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
H3 hnormalized(H3 a) {
    const double n = hnorm(a);
    return {a.x / n, a.y / n, a.z / n};
}
H3 hcross(H3 a, H3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
void put3(double* d, H3 v) {
    d[0] = v.x;
    d[1] = v.y;
    d[2] = v.z;
}

}  // namespace

struct prc_gpu_store;

struct prc_gpu_ctx {
    std::recursive_mutex mu;  // serialises the calls on this context (begin())
    int device = 0, rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    unsigned long long launches = 0;
    int mode = 0;        // 0: event-major wavefront (default), 1: fused thread-per-path
    bool timed_sub = false, timed_grad = false;  // sub-phase events recorded this call
    int spread = 0;      // K5b lane spreading factor; 0: by vertex density (auto_spread)
    int opt_per_species = 0;  // opt_step computes per-type gradients of every species
    int packet = 3;      // K5b rays per thread walked in lockstep (measured best: 3)
    bool evc_enable = true;  // event list for scenes without a medium (option "events")
    bool pad_ok = false, pad_enable = true;  // guard-free padded walks valid / allowed
    // scene
    bool have_scene = false;
    DScene dsc{};
    long long V = 0, n_pix = 0;
    std::vector<double> host_sp;  // n_species x V (scene values)
    DBuf<double> scene_sp;        // device copy
    std::vector<prc_surface_desc> surfaces;
    std::vector<prc_detector_desc> det_desc;  // as uploaded (stage schedules re-finalize)
    bool det_finalized = false;               // prc_scene_desc::finalized of the upload
    double scene_kappa = 0.0, scene_gamma = 0.0;
    // evaluation scratch
    DBuf<float> sp_t, bt_tot, dbeta;
    DBuf<double> bt_pad, db_pad, g_pad;  // padded layout (pad_walk)
    DBuf<double> param_beta, species_t, trace_sp, images, weights, g_span, g_vert, g_out, phong,
        g_phong, loss;
    DBuf<unsigned long long> clamps, u64tmp_a, u64tmp_b, n_trunc;
    DBuf<unsigned long long> img_max, img_fx, img_limbs;  // deterministic images (image_pass)
    const double* grad_res = nullptr;  // combined, reduced gradient of the last run_gradient
    // NVLS multicast reduction (option "nvls", prc_nvls.cu): [0, n_pix) images, then the
    // n_species x V gradient
    bool nvls_enable = false, nvls_emulate = false;
    NvlsState* nvls = nullptr;
    DBuf<uint32_t> u32tmp;
    DBuf<int> err;
    DBuf<double> selfn;  // self-normalisation sum (mean_correction)
    DBuf<unsigned> check;  // DScene::check (checked builds record range violations here)
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    // device-resident optimizer (Algorithm 2)
    bool opt_ready = false;
    int opt_mode = 0;  // 0 tomography, 1 Phong
    DBuf<double> opt_x, opt_m1, opt_m2, opt_gt, opt_step_scale;
    long long opt_n = 0;
    int64_t opt_t = 0;
    prc_gpu_adam_config adam{};
    int n_step_scale = 0;
    // forward-reuse cache: grad_forward right after recycled_render at the same point
    // (inverse.cpp:205, 246) reuses the stored forward instead of recomputing K3/K4
    unsigned long long fwd_gen = 0;
    // bumped whenever cameras, scene or options change: invalidates every store's cached
    // event geometry (prc_gpu_store::geo_key)
    unsigned long long geo_gen = 1;
    // bumped by every scene upload: a store whose reference-side tables (br_tot64, sp_ref,
    // br_tot) were built under another upload rebuilds them before use (store_for_scene)
    unsigned long long scene_gen = 0;
    unsigned long long last_fwd_gen = ~0ull, last_fwd_key = 0;
    const prc_gpu_store* last_fwd_store = nullptr;
    unsigned long long last_fwd_clamps = 0;
    // timing
    cudaEvent_t ev[9] = {};  // [0..5] phases, [6] after K4a, [7] before K5a, [8] spare
    cudaEvent_t timer[2] = {};
    double last_ms[8] = {};
    std::set<prc_gpu_store*> stores;  // live stores made by this context (orphaned on destroy)
    int g_pad_copies = 1;  // see EvalArgs::g_pad_copies
    int grad_copies_max = 0;  // option "grad_copies" (applied at scene upload); 0: 8 while <= 2 GB
    ~prc_gpu_ctx() {
        if (cub_tmp) cudaFree(cub_tmp);
        for (auto& e : timer)
            if (e) cudaEventDestroy(e);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        nvls_destroy(nvls);
        if (comm) ncclCommDestroy(comm);
        if (stream) cudaStreamDestroy(stream);
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    void check_scene() const {
        if (!have_scene) throw Err(PRC_ERR_INVALID, "no scene uploaded");
    }
    void allreduce(double* buf, size_t count) {
        if (comm && count > 0)
            NK(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, comm, stream));
    }
    void allreduce_u64(unsigned long long* buf, size_t count) {
        if (comm && count > 0)
            NK(ncclAllReduce(buf, buf, count, ncclUint64, ncclSum, comm, stream));
    }
};

struct prc_gpu_store {
    prc_gpu_ctx* ctx = nullptr;  // null once the context is destroyed (the store stays freeable)
    int device = 0;
    unsigned long long n = 0, n_global = 0, stream_base = 0, seed = 0, generation = 0;
    bool sorted = false;
    int max_B = 0;
    DBuf<uint32_t> B, stride;
    DBuf<unsigned long long> stream, rec_base, iv_base;
    DBuf<uint8_t> trunc;
    DBuf<double> px, py, pz, dx, dy, dz, tt, ct;
    DBuf<int32_t> vox;
    DBuf<uint32_t> meta;
    unsigned long long n_rec = 0, n_iv = 0;
    DBuf<float> ev_val;    // event cache: [det][iv] (path mode) or [det][vt] (wavefront)
    DBuf<int32_t> ev_pix;
    DBuf<int32_t> ev_c1;   // wavefront: beta-independent event term (VertexTable::ev_c1)
    DBuf<float> ev_f;      // wavefront, 2..4 species: phase values (VertexTable::ev_f)
    unsigned long long geo_key = 0;  // == ctx geo_gen while ev_pix / ev_c1 hold the geometry
    DBuf<double> lp, own;  // per interaction vertex: log-prefix (K4a), weight sum (K5b)
    // event list of scenes without a medium (EventList, prc_kernels.cuh); valid while
    // evc_key == geo_key == ctx geo_gen
    unsigned long long evc_key = 0, n_evc = 0;
    bool evc_vals = false;  // the last forward's event values are in evc_val (K4b')
    DBuf<unsigned long long> evc_off;
    DBuf<uint32_t> evc_iv;
    DBuf<int32_t> evc_px;
    DBuf<double> evc_lobe;
    DBuf<float> evc_geom, evc_val;
    DBuf<uint8_t> evc_surf;
    DBuf<double> evc_vlobe;  // EvalArgs::vlobe, per interaction-vertex slot
    bool vt_ready = false; // Morton-ordered vertex table (wavefront mapping)
    DBuf<double> vt_x, vt_y, vt_z, vt_dx, vt_dy, vt_dz;
    DBuf<int32_t> vt_vox;
    DBuf<uint32_t> vt_meta, vt_iv;
    DBuf<double> br_tot64;
    DBuf<float> sp_ref, br_tot;
    std::vector<double> ref_beta;
    double ref_kappa = 0.0, ref_gamma = 0.0;
    unsigned long long segments = 0, truncated = 0;
    // scene the store was built or last re-bound under (store_for_scene)
    unsigned long long scene_gen = 0;
    int dims[3] = {0, 0, 0};
    int n_species = 0;
    // Materialized imports (prc_gpu_store_import_pstr_ex with PRC_IMPORT_MATERIALIZE): the
    // file's own spans / events on the device (MatView, prc_materialized.cu) and its raw
    // record bytes on the host (export writes them back verbatim).
    bool mat = false;
    std::vector<char> mat_bytes;
    std::vector<size_t> mat_off;  // record r = mat_bytes[mat_off[r], mat_off[r + 1])
    DBuf<unsigned long long> m_rec, m_vbase, m_sbase, m_ebase, m_lbase;
    DBuf<uint32_t> m_vmeta, m_vsb, m_vse, m_svox, m_evert, m_esb, m_ese, m_lvox;
    DBuf<int32_t> m_vvox, m_edet, m_epix;
    DBuf<double> m_vct, m_slen, m_ecos, m_egeom, m_llen, m_eval;
    DBuf<double> m_ref64, m_bt, m_br, m_db;  // fp64 context of make_context
    unsigned long long m_events = 0;
    MatCtx m_ctx{};

    prc_gpu_store() = default;
    explicit prc_gpu_store(prc_gpu_ctx* c) : ctx(c), device(c->device) { c->stores.insert(this); }
    prc_gpu_store(const prc_gpu_store&) = delete;
    prc_gpu_store& operator=(const prc_gpu_store&) = delete;
    ~prc_gpu_store() {
        if (ctx) ctx->stores.erase(this);
    }

    StoreView view() {
        StoreView v{};
        v.n = n;
        v.B = B.p;
        v.rec_base = rec_base.p;
        v.stride = stride.p;
        v.iv_base = iv_base.p;
        v.px = px.p;
        v.py = py.p;
        v.pz = pz.p;
        v.dx = dx.p;
        v.dy = dy.p;
        v.dz = dz.p;
        v.tt = tt.p;
        v.ct = ct.p;
        v.vox = vox.p;
        v.meta = meta.p;
        v.n_iv = n_iv;
        v.ev_val = ev_val.p;
        v.ev_pix = ev_pix.p;
        return v;
    }
    void alloc_records(unsigned long long nr) {
        n_rec = nr;
        px.alloc(nr);
        py.alloc(nr);
        pz.alloc(nr);
        dx.alloc(nr);
        dy.alloc(nr);
        dz.alloc(nr);
        tt.alloc(nr);
        ct.alloc(nr);
        vox.alloc(nr);
        meta.alloc(nr);
    }
    RecordsOut rec_out() {
        return RecordsOut{px.p, py.p, pz.p, dx.p, dy.p, dz.p, tt.p, ct.p, vox.p, meta.p};
    }
    MatView mat_view() {
        MatView v{};
        v.n = n;
        v.rec = m_rec.p;
        v.v_base = m_vbase.p;
        v.s_base = m_sbase.p;
        v.e_base = m_ebase.p;
        v.l_base = m_lbase.p;
        v.v_meta = m_vmeta.p;
        v.v_vox = m_vvox.p;
        v.v_ct = m_vct.p;
        v.v_sb = m_vsb.p;
        v.v_se = m_vse.p;
        v.s_vox = m_svox.p;
        v.s_len = m_slen.p;
        v.e_vert = m_evert.p;
        v.e_det = m_edet.p;
        v.e_pix = m_epix.p;
        v.e_cos = m_ecos.p;
        v.e_geom = m_egeom.p;
        v.e_sb = m_esb.p;
        v.e_se = m_ese.p;
        v.l_vox = m_lvox.p;
        v.l_len = m_llen.p;
        v.e_val = m_eval.p;
        return v;
    }
    unsigned long long mat_device_bytes() const {
        return m_rec.bytes() + m_vbase.bytes() + m_sbase.bytes() + m_ebase.bytes() + m_lbase.bytes() +
               m_vmeta.bytes() + m_vsb.bytes() + m_vse.bytes() + m_svox.bytes() + m_evert.bytes() + m_esb.bytes() +
               m_ese.bytes() + m_lvox.bytes() + m_vvox.bytes() + m_edet.bytes() + m_epix.bytes() + m_vct.bytes() +
               m_slen.bytes() + m_ecos.bytes() + m_egeom.bytes() + m_llen.bytes() + m_eval.bytes() +
               m_ref64.bytes() + m_bt.bytes() + m_br.bytes() + m_db.bytes();
    }
    unsigned long long device_bytes() const {
        return mat_device_bytes() + B.bytes() + stride.bytes() + stream.bytes() + rec_base.bytes() + iv_base.bytes() +
               trunc.bytes() + px.bytes() * 8 + vox.bytes() + meta.bytes() + ev_val.bytes() +
               ev_pix.bytes() + ev_c1.bytes() + ev_f.bytes() + br_tot64.bytes() + sp_ref.bytes() + br_tot.bytes() + lp.bytes() +
               own.bytes() + vt_x.bytes() * 6 + vt_vox.bytes() + vt_meta.bytes() + vt_iv.bytes() + evc_off.bytes() +
               evc_iv.bytes() + evc_px.bytes() + evc_lobe.bytes() + evc_geom.bytes() + evc_val.bytes() + evc_surf.bytes() + evc_vlobe.bytes();
    }
};

namespace {

// Contiguous stream range [lo, hi) of rank r among w: floor(N r / w) ..
// floor(N (r + 1) / w), exact in 128-bit arithmetic; the ranges of all ranks partition
// [0, N) and differ in size by at most one.
void shard_range(unsigned long long N, int r, int w, unsigned long long* lo, unsigned long long* hi) {
    *lo = (unsigned long long)((unsigned __int128)N * (unsigned)r / (unsigned)w);
    *hi = (unsigned long long)((unsigned __int128)N * (unsigned)(r + 1) / (unsigned)w);
}

int fail(int code, const std::string& m) {
    g_last_error = m;
    return code;
}

int classify(const std::exception& e) {
    if (auto* x = dynamic_cast<const Err*>(&e)) return x->code;
    if (dynamic_cast<const std::bad_alloc*>(&e)) return PRC_ERR_CUDA;
    return PRC_ERR_CONFIG;
}

#define ABI_TRY try {
#define ABI_CATCH                               \
    }                                           \
    catch (const std::exception& e) {           \
        return fail(classify(e), e.what());     \
    }                                           \
    return PRC_OK;

// Every entry point on a context holds its lock for the call: calls on one context are
// serialised, distinct contexts are independent (SURVEY §8(b) threading; the reference's
// OptState is single-owner).
std::unique_lock<std::recursive_mutex> begin(prc_gpu_ctx* c) {
    std::unique_lock<std::recursive_mutex> lk(c->mu);
    CK(cudaSetDevice(c->device));
    return lk;
}

// ----------------------------------------------------------------------- scene upload
// Detector::finalize (scene.cpp:8-14) for every detector, at the resolution of the
// descriptor or rows[k] x cols[k] when given; assigns image offsets, returns n_pix.
long long finalize_detectors(DScene& s, const prc_detector_desc* dd, int n, const int* rows, const int* cols,
                             bool finalized) {
    long long off = 0;
    for (int k = 0; k < n; ++k) {
        const prc_detector_desc& q = dd[k];
        const int nr = rows ? rows[k] : q.rows, nc = cols ? cols[k] : q.cols;
        if (nr <= 0 || nc <= 0) throw Err(PRC_ERR_CONFIG, "detector: non-positive pixel grid");
        DDet& t = s.det[k];
        // a finalized scene (Scene::finalize ran on the host) carries the unit direction
        const H3 dir = finalized ? h3(q.direction) : hnormalized(h3(q.direction));
        const H3 right = hnormalized(hcross(dir, h3(q.up)));
        const H3 up = hcross(right, dir);
        put3(t.pos, h3(q.position));
        put3(t.dir, dir);
        put3(t.right, right);
        put3(t.up, up);
        t.hw = std::tan(0.5 * q.fov);
        t.hh = t.hw * static_cast<double>(nr) / static_cast<double>(nc);
        t.rows = nr;
        t.cols = nc;
        t.img_off = off;
        off += (long long)nr * nc;
    }
    s.n_pix = off;
    return off;
}

void nvls_setup(prc_gpu_ctx* c);

void upload_scene(prc_gpu_ctx* c, const prc_scene_desc* d) {
    ++c->scene_gen;
    ++c->geo_gen;  // cameras / species / surfaces may change: cached event geometry is stale
    ++c->fwd_gen;  // and so is a cached forward (grad_forward after recycled_render)
    if (d->n_species < 0 || d->n_species > PRC_MAX_SPECIES)
        throw Err(PRC_ERR_CONFIG, "scene: species count outside 0..16");
    if (d->n_surfaces < 0 || d->n_surfaces > PRC_MAX_SURF)
        throw Err(PRC_ERR_CONFIG, "scene: at most 64 surfaces supported");
    if (d->n_detectors < 1 || d->n_detectors > PRC_MAX_DET)
        throw Err(PRC_ERR_CONFIG, "scene: detector count outside 1..64");
    DScene s{};
    s.bmin[0] = d->bounds_min.x;
    s.bmin[1] = d->bounds_min.y;
    s.bmin[2] = d->bounds_min.z;
    s.bmax[0] = d->bounds_max.x;
    s.bmax[1] = d->bounds_max.y;
    s.bmax[2] = d->bounds_max.z;
    s.has_medium = d->n_species > 0;
    s.n_species = d->n_species;
    long long V = 0;
    if (s.has_medium) {
        for (int a = 0; a < 3; ++a) {
            if (d->dims[a] <= 0) throw Err(PRC_ERR_CONFIG, "scene: grid dims must be positive");
            s.dims[a] = d->dims[a];
        }
        s.gorg[0] = d->grid_origin.x;
        s.gorg[1] = d->grid_origin.y;
        s.gorg[2] = d->grid_origin.z;
        s.vs[0] = d->voxel_size.x;
        s.vs[1] = d->voxel_size.y;
        s.vs[2] = d->voxel_size.z;
        for (int a = 0; a < 3; ++a) s.gmax[a] = s.gorg[a] + s.dims[a] * s.vs[a];  // grid.hpp:27-30
        V = (long long)s.dims[0] * s.dims[1] * s.dims[2];
    }
    s.V = V;
    s.dda_packed = s.has_medium && s.dims[0] <= 512 && s.dims[1] <= 512 && s.dims[2] <= 512 ? 1 : 0;
    s.unknown = -1;
    std::vector<double> sp((size_t)d->n_species * (size_t)V);
    for (int j = 0; j < d->n_species; ++j) {
        const prc_species_desc& q = d->species[j];
        if (!q.extinction) throw Err(PRC_ERR_CONFIG, "scene: species extinction is null");
        std::memcpy(sp.data() + (size_t)j * V, q.extinction, (size_t)V * sizeof(double));
        s.sp[j].albedo = q.albedo;
        s.sp[j].g = q.g;
        s.sp[j].kind = q.phase_kind == PRC_PHASE_RAYLEIGH ? 1 : 0;
        s.sp[j].unknown = q.unknown;
        if (q.unknown) {
            if (s.unknown >= 0) throw Err(PRC_ERR_CONFIG, "more than one unknown species");
            s.unknown = j;
        }
        if (s.sp[j].kind == 0 && std::abs(q.g) >= 1.0) throw Err(PRC_ERR_CONFIG, "|g| must be < 1");
    }
    s.n_surf = d->n_surfaces;
    s.target = -1;
    c->scene_kappa = c->scene_gamma = 0.0;
    for (int k = 0; k < d->n_surfaces; ++k) {
        const prc_surface_desc& q = d->surfaces[k];
        DSurf& f = s.surf[k];
        f.kind = q.kind == PRC_SURF_FACE ? 1 : 0;
        f.axis = q.axis;
        f.brdf_kind = q.brdf_kind == PRC_BRDF_PHONG ? 1 : 0;
        f.target = q.target;
        put3(f.c, h3(q.center));
        f.radius = q.radius;
        f.coord = q.coord;
        f.lo[0] = q.lo[0];
        f.lo[1] = q.lo[1];
        f.hi[0] = q.hi[0];
        f.hi[1] = q.hi[1];
        f.normal_sign = q.normal_sign;
        f.albedo = q.albedo;
        f.kappa = q.kappa_s;
        f.gamma = q.gamma;
        if (f.kind == 1 && (q.axis < 0 || q.axis > 2)) throw Err(PRC_ERR_CONFIG, "face axis outside 0..2");
        if (q.target) {
            if (s.target >= 0) throw Err(PRC_ERR_CONFIG, "more than one target surface");
            if (f.brdf_kind != 1) throw Err(PRC_ERR_CONFIG, "target surface must carry a Phong lobe");
            s.target = k;
            c->scene_kappa = q.kappa_s;
            c->scene_gamma = q.gamma;
        }
    }
    s.light_kind = d->light.kind == PRC_LIGHT_SUN ? 0 : 1;
    put3(s.light_pos, h3(d->light.position));
    H3 ld = h3(d->light.direction);
    if (s.light_kind == 0 && !d->finalized) ld = hnormalized(ld);  // Scene::finalize, scene.cpp:71-74
    put3(s.light_dir, ld);
    s.radiance = d->light.radiance;
    // emission_prefactor, transport.cpp:347-351
    s.prefactor = s.light_kind == 1 ? PRC_FOUR_PI * s.radiance
                                    : (s.bmax[0] - s.bmin[0]) * (s.bmax[1] - s.bmin[1]) * s.radiance;
    s.n_det = d->n_detectors;
    c->det_finalized = d->finalized != 0;
    const long long off = finalize_detectors(s, d->detectors, d->n_detectors, nullptr, nullptr, c->det_finalized);
    s.n_pix = off;
    // Fixed-point event term of single-species scenes (DScene::c1_fast): the range of
    // log(albedo * f) over cos in [-1, 1], from the phase function's extremes.
    s.c1_fast = 0;
    if (s.n_species == 1 && s.sp[0].albedo > 0.0) {
        const DSpecies& sp = s.sp[0];
        double fmin, fmax;
        if (sp.kind == 1) {
            fmin = 3.0 / (16.0 * PRC_PI);
            fmax = 6.0 / (16.0 * PRC_PI);
        } else {
            const double g = std::fabs(sp.g);
            fmin = (1.0 - g * g) / (4.0 * PRC_PI * std::pow(1.0 + g, 3.0));
            fmax = (1.0 - g * g) / (4.0 * PRC_PI * std::pow(1.0 - g, 3.0));
        }
        const double lo = std::log(sp.albedo * fmin), hi = std::log(sp.albedo * fmax);
        const double h = 0.5 * (hi - lo) + 1.0;  // + margin for cos_le rounding past +-1
        if (std::isfinite(lo) && std::isfinite(hi) && h < 64.0) {
            s.c1_fast = 1;
            s.c1_mid = 0.5 * (lo + hi);
            s.c1_q = std::ldexp(1.0, (int)std::floor(std::log2(1073741824.0 / h)));
            s.c1_iq = 1.0 / s.c1_q;
        }
    }
    s.fcache = s.n_species >= 2 && s.n_species <= kFCacheMax ? 1 : 0;
    s.scache = s.n_surf > 0 ? 1 : 0;
    // Guard-free walks over the padded layout (prc_device.cuh, dda_walk_pad): exact when
    // the rounding of the tmax sums (~512 ulp of a distance <= 4R) stays far below a voxel.
    if (s.has_medium) {
        double R = 0.0, vmin = std::min(s.vs[0], std::min(s.vs[1], s.vs[2]));
        for (int a = 0; a < 3; ++a)
            R = std::max({R, std::fabs(s.bmin[a]), std::fabs(s.bmax[a]), std::fabs(s.gorg[a]), std::fabs(s.gmax[a]),
                          std::fabs(s.light_pos[a])});
        const long long vpad = (long long)(s.dims[0] + 2) * (s.dims[1] + 2) * (s.dims[2] + 2);
        c->pad_ok = vpad < (1ll << 31) && vmin > 0.0 && 4.0 * R < 1e9 * vmin;
        s.vs_pow2 = 1;
        for (int a = 0; a < 3; ++a) {
            int e = 0;
            const double m = std::frexp(s.vs[a], &e);
            if (!(m == 0.5 && e >= -59 && e <= 21)) s.vs_pow2 = 0;
            s.inv_vs[a] = 1.0 / s.vs[a];
        }
        s.pad_walk = c->pad_ok && c->pad_enable ? 1 : 0;
        s.pnx = s.dims[0] + 2;
        s.pnxny = (s.dims[0] + 2) * (s.dims[1] + 2);
        s.vpad = (long long)s.pnxny * (long long)(s.dims[2] + 2);
    }
    if (!c->check.p) {
        c->check.alloc(1);
        CK(cudaMemset(c->check.p, 0, sizeof(unsigned)));
    }
    s.check = c->check.p;
    c->dsc = s;
    c->V = V;
    c->n_pix = off;
    c->host_sp.swap(sp);
    c->surfaces.assign(d->surfaces, d->surfaces + d->n_surfaces);
    c->det_desc.assign(d->detectors, d->detectors + d->n_detectors);
    c->scene_sp.alloc(c->host_sp.size());
    if (!c->host_sp.empty())
        CK(cudaMemcpy(c->scene_sp.p, c->host_sp.data(), c->host_sp.size() * sizeof(double),
                      cudaMemcpyHostToDevice));
    const size_t nsV = (size_t)std::max(1, d->n_species) * (size_t)std::max<long long>(V, 1);
    c->sp_t.alloc(nsV);
    c->bt_tot.alloc((size_t)std::max<long long>(V, 1));
    c->dbeta.alloc((size_t)std::max<long long>(V, 1));
    c->param_beta.alloc((size_t)std::max<long long>(V, 1));
    c->species_t.alloc(nsV);
    c->trace_sp.alloc(nsV);
    c->images.alloc((size_t)off);
    c->weights.alloc((size_t)off);
    c->g_span.alloc((size_t)std::max<long long>(V, 1));
    {
        const size_t vpad = c->pad_ok ? (size_t)s.pnxny * (size_t)(s.dims[2] + 2) : 1;
        c->bt_pad.alloc(vpad);
        c->db_pad.alloc(vpad);
        // copies of the padded gradient for K5b (EvalArgs::g_pad_copies): 8 while they take
        // at most 2 GB (K5b at 1e8 paths: 784 -> 697 ms with 4 copies at 128^3, 670 -> 663 with
        // 8; 1973 -> 1728 ms with 4 at 256^3, where one copy alone exceeds L2), and up to 32
        // while they fit in 64 MB of L2 (small grids, where reductions into the same lines
        // queue: config (a), 32^3, K5b 2.42 -> 2.28 ms with 32 copies); an explicit
        // "grad_copies" option is taken as given
        const size_t l2_copies = vpad > 0 ? (size_t(64) << 20) / (vpad * 8) : 1;
        c->g_pad_copies = !(c->pad_ok && vpad > 0) ? 1
                          : c->grad_copies_max > 0
                              ? c->grad_copies_max
                              : (int)std::max<size_t>(1, std::min<size_t>(std::max<size_t>(8, std::min<size_t>(32, l2_copies)),
                                                                          (size_t(2) << 30) / (vpad * 8)));
        c->g_pad.alloc(vpad * (size_t)c->g_pad_copies);
        CK(cudaMemset(c->bt_pad.p, 0, c->bt_pad.bytes()));  // borders stay zero
        CK(cudaMemset(c->db_pad.p, 0, c->db_pad.bytes()));
    }
    c->g_vert.alloc(nsV);
    c->g_out.alloc(nsV);
    c->phong.alloc(2);
    c->g_phong.alloc(2);
    c->loss.alloc(1);
    c->clamps.alloc(1);
    c->n_trunc.alloc(1);
    c->err.alloc(1);
    c->have_scene = true;
    c->opt_ready = false;
    nvls_setup(c);
}

// (Re)creates the NVLS multicast buffer for the current images and gradient sizes
// (collective over the ranks when world > 1: every rank uploads the same scene).
void nvls_setup(prc_gpu_ctx* c) {
    const size_t need = (size_t)c->n_pix + (size_t)std::max(1, c->dsc.n_species) * (size_t)std::max<long long>(c->V, 1);
    if (!c->nvls_enable) {
        nvls_destroy(c->nvls);
        c->nvls = nullptr;
        return;
    }
    if (c->nvls && nvls_capacity(c->nvls) >= need) return;
    nvls_destroy(c->nvls);
    c->nvls = nullptr;
    std::string err;
    c->nvls = nvls_create(c->comm, c->comm ? c->world : 1, c->device, need, c->nvls_emulate, &err);
    if (!c->nvls) throw Err(PRC_ERR_CUDA, "nvls: " + err);
}

// Species source pointers + Phong values for the evaluated parameters.
struct Resolved {
    const double* src[PRC_MAX_SPECIES] = {};
    double kappa = 0.0, gamma = 0.0;
};

Resolved resolve_params(prc_gpu_ctx* c, const prc_gpu_params* p, const prc_gpu_store* ref_store) {
    Resolved r;
    const DScene& s = c->dsc;
    for (int j = 0; j < s.n_species; ++j) r.src[j] = c->scene_sp.p + (size_t)j * c->V;
    r.kappa = c->scene_kappa;
    r.gamma = c->scene_gamma;
    if (!p) {
        if (ref_store) {  // evaluate at the store's sampling parameters
            if (s.unknown >= 0 && !ref_store->ref_beta.empty()) {
                CK(cudaMemcpyAsync(c->param_beta.p, ref_store->ref_beta.data(),
                                   (size_t)c->V * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                r.src[s.unknown] = c->param_beta.p;
            }
            r.kappa = ref_store->ref_kappa;
            r.gamma = ref_store->ref_gamma;
        }
        return r;
    }
    if (p->beta && s.unknown >= 0) {
        if ((long long)p->n_beta != c->V) throw Err(PRC_ERR_CONFIG, "params: beta size != voxel count");
        CK(cudaMemcpyAsync(c->param_beta.p, p->beta, (size_t)c->V * sizeof(double),
                           cudaMemcpyHostToDevice, c->stream));
        r.src[s.unknown] = c->param_beta.p;
    }
    if (p->species_beta) {
        for (int j = 0; j < s.n_species; ++j) {
            if (!p->species_beta[j]) continue;
            double* dst = c->species_t.p + (size_t)j * c->V;
            CK(cudaMemcpyAsync(dst, p->species_beta[j], (size_t)c->V * sizeof(double),
                               cudaMemcpyHostToDevice, c->stream));
            r.src[j] = dst;
        }
    }
    if (s.target >= 0) {
        r.kappa = p->kappa_s;
        r.gamma = p->gamma;
    }
    return r;
}

// Stamps a store with the current scene (trace / import).
void stamp_store(prc_gpu_ctx* c, prc_gpu_store* st) {
    st->scene_gen = c->scene_gen;
    for (int a = 0; a < 3; ++a) st->dims[a] = c->dsc.dims[a];
    st->n_species = c->dsc.n_species;
}

// fp64 reference species values of a materialized store (make_context's ref side,
// pathstore.cpp:54-61): the scene's values, the unknown species' from ref_params.beta.
void mat_ref_tables(prc_gpu_ctx* c, prc_gpu_store* st) {
    const DScene& s = c->dsc;
    const long long V = c->V;
    const size_t nsV = (size_t)std::max(1, s.n_species) * (size_t)std::max<long long>(V, 1);
    st->m_ref64.alloc(nsV);
    st->m_bt.alloc((size_t)std::max<long long>(V, 1));
    st->m_br.alloc((size_t)std::max<long long>(V, 1));
    st->m_db.alloc((size_t)std::max<long long>(V, 1));
    if (s.n_species > 0 && V > 0) {
        CK(cudaMemcpyAsync(st->m_ref64.p, c->scene_sp.p, (size_t)s.n_species * V * 8, cudaMemcpyDeviceToDevice,
                           c->stream));
        if (s.unknown >= 0 && !st->ref_beta.empty())
            CK(cudaMemcpyAsync(st->m_ref64.p + (size_t)s.unknown * V, st->ref_beta.data(), (size_t)V * 8,
                               cudaMemcpyHostToDevice, c->stream));
    }
    c->sync();
}

// Reference-side tables of a store for the scene on the device.  make_context
// (pathstore.cpp:41-82) rebuilds the reference side from the current scene and the
// store's ref_params on every call; the store caches it per scene upload.  A store built
// under another grid cannot be evaluated (its voxel ids index that grid).
void store_for_scene(prc_gpu_ctx* c, prc_gpu_store* st) {
    const DScene& s = c->dsc;
    if (st->n_species != s.n_species || st->dims[0] != s.dims[0] || st->dims[1] != s.dims[1] ||
        st->dims[2] != s.dims[2])
        throw Err(PRC_ERR_INVALID, "the store was built for a different grid or species set than the uploaded scene");
    if (st->scene_gen == c->scene_gen) return;
    const long long V = c->V;
    const double* src[PRC_MAX_SPECIES] = {};
    for (int j = 0; j < s.n_species; ++j) src[j] = c->scene_sp.p + (size_t)j * V;
    if (s.unknown >= 0 && !st->ref_beta.empty()) {
        if ((long long)st->ref_beta.size() != V) throw Err(PRC_ERR_INVALID, "store reference beta size != voxel count");
        c->trace_sp.grow((size_t)V);
        CK(cudaMemcpyAsync(c->trace_sp.p, st->ref_beta.data(), (size_t)V * 8, cudaMemcpyHostToDevice, c->stream));
        src[s.unknown] = c->trace_sp.p;
    }
    CK(launch_prep_ref(s.n_species, V, src, st->br_tot64.p, st->sp_ref.p, st->br_tot.p, nullptr, c->stream,
                       &c->launches));
    c->sync();
    if (st->mat) mat_ref_tables(c, st);
    st->scene_gen = c->scene_gen;
}

// 64-bit content hash of the evaluated parameters (forward-reuse key).
unsigned long long mix64(unsigned long long h, unsigned long long x) {
    h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    return h * 0xff51afd7ed558ccdull;
}
unsigned long long hash_doubles(unsigned long long h, const double* p, size_t n) {
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(p);
    unsigned long long a = h, b = h ^ 0x632be59bd9b4e019ull;
    size_t i = 0;
    for (; i + 1 < n; i += 2) {
        a = (a ^ w[i]) * 0x9E3779B97F4A7C15ull;
        b = (b ^ w[i + 1]) * 0xC2B2AE3D27D4EB4Full;
    }
    if (i < n) a = (a ^ w[i]) * 0x9E3779B97F4A7C15ull;
    return mix64(a, b);
}
unsigned long long params_key(const prc_gpu_ctx* c, const prc_gpu_params* p, const prc_gpu_store* st,
                              int flags) {
    unsigned long long h = mix64(0x1234567ull, (unsigned long long)(uintptr_t)st);
    h = mix64(h, (unsigned long long)c->mode);
    h = mix64(h, (unsigned long long)(flags & (PRC_EVAL_NORMALIZE | PRC_EVAL_DETERMINISTIC)));
    if (!p) return mix64(h, 0xabcdefull);
    double kg[2] = {p->kappa_s, p->gamma};
    h = hash_doubles(h, kg, 2);
    if (p->beta) h = hash_doubles(mix64(h, p->n_beta), p->beta, (size_t)p->n_beta);
    if (p->species_beta)
        for (int j = 0; j < c->dsc.n_species; ++j)
            h = p->species_beta[j] ? hash_doubles(mix64(h, 100 + j), p->species_beta[j], (size_t)c->V)
                                   : mix64(h, 200 + j);
    return h;
}

// ----------------------------------------------------------------------- K3 + K4 + K5
struct EvalRun {
    bool want_grad = false, per_species = false, legacy = false, normalize = true;
    bool deterministic = false;  // bit-reproducible image (two passes, image_pass)
    double grad_scale = 1.0;     // scale of the combined gradient (1 / N with normalize)
    const double* weights = nullptr;  // device
};

// Vertex table of the event-major wavefront: interaction vertices in Morton order of
// their position (built once per store layout; geometry only, so valid for any beta).
void ensure_vertex_table(prc_gpu_ctx* c, prc_gpu_store* st) {
    if (st->vt_ready) return;
    st->geo_key = 0;  // the event cache indexes the vertex table
    const long long n = (long long)st->n_iv;
    cudaStream_t q = c->stream;
    const size_t nn = (size_t)std::max<long long>(n, 1);
    st->vt_x.alloc(nn);
    st->vt_y.alloc(nn);
    st->vt_z.alloc(nn);
    st->vt_dx.alloc(nn);
    st->vt_dy.alloc(nn);
    st->vt_dz.alloc(nn);
    st->vt_vox.alloc(nn);
    st->vt_meta.alloc(nn);
    st->vt_iv.alloc(nn);
    if (n > 0) {
        DBuf<uint32_t> keys, keys_s, vals, vals_s;
        DBuf<unsigned long long> iv_rec;
        keys.alloc(nn);
        keys_s.alloc(nn);
        vals.alloc(nn);
        vals_s.alloc(nn);
        iv_rec.alloc(nn);
        CK(launch_vt_keys(c->dsc, st->view(), keys.p, vals.p, iv_rec.p, q, &c->launches));
        CK(sort_pairs_u32(keys.p, keys_s.p, vals.p, vals_s.p, n, &c->cub_tmp, &c->cub_bytes, q));
        CK(launch_vt_gather(st->view(), vals_s.p, iv_rec.p, n, st->vt_x.p, st->vt_y.p, st->vt_z.p,
                            st->vt_dx.p, st->vt_dy.p, st->vt_dz.p, st->vt_vox.p, st->vt_meta.p,
                            st->vt_iv.p, q, &c->launches));
        c->sync();
    }
    st->vt_ready = true;
}

VertexTable vertex_table(prc_gpu_store* st) {
    VertexTable v{};
    v.n = st->n_iv;
    v.x = st->vt_x.p;
    v.y = st->vt_y.p;
    v.z = st->vt_z.p;
    v.dx = st->vt_dx.p;
    v.dy = st->vt_dy.p;
    v.dz = st->vt_dz.p;
    v.vox = st->vt_vox.p;
    v.meta = st->vt_meta.p;
    v.iv = st->vt_iv.p;
    v.ev_val = st->ev_val.p;
    v.ev_pix = st->ev_pix.p;
    v.ev_c1 = st->ev_c1.p;
    v.ev_f = st->ev_f.p;
    v.geo_ready = st->geo_key == st->ctx->geo_gen ? 1 : 0;
    return v;
}

// Scenes without a medium evaluate over the event list (EventList): surface events only,
// int32 image indices, at most 255 surfaces.
bool evc_applies(const prc_gpu_ctx* c) {
    const DScene& s = c->dsc;
    return c->evc_enable && c->mode == 0 && !s.has_medium && s.scache && s.n_surf <= 255 &&
           c->n_pix < (1ll << 31);
}

bool evc_ready(const prc_gpu_ctx* c, const prc_gpu_store* st) {
    return evc_applies(c) && st->geo_key == c->geo_gen && st->evc_key == c->geo_gen;
}

EventList event_list(prc_gpu_store* st) {
    EventList el{};
    el.n = st->n_evc;
    el.n_iv = st->n_iv;
    el.off = st->evc_off.p;
    el.iv = st->evc_iv.p;
    el.px = st->evc_px.p;
    el.lobe = st->evc_lobe.p;
    el.geom = st->evc_geom.p;
    el.surf = st->evc_surf.p;
    el.val = st->evc_val.p;
    return el;
}

// (Re)builds the event list from the dense cache a forward over the store just wrote.
// Called after every dense pass: whatever invalidated the list (a new geometry
// generation, a re-sorted store with its rebuilt vertex table) also sent this forward
// down the dense path.
void build_event_list(prc_gpu_ctx* c, prc_gpu_store* st) {
    st->evc_key = 0;
    if (!evc_applies(c) || st->geo_key != c->geo_gen) return;
    cudaStream_t q = c->stream;
    const size_t niv = (size_t)st->n_iv;
    st->evc_off.grow(niv + 1);
    DBuf<unsigned long long> cnt;
    cnt.alloc(niv + 1);
    CK(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), q));
    const VertexTable vt = vertex_table(st);
    CK(launch_evc_count(c->dsc, vt, cnt.p, q, &c->launches));
    CK(scan_u64(cnt.p, st->evc_off.p, (long long)niv + 1, &c->cub_tmp, &c->cub_bytes, q));
    unsigned long long n = 0;
    CK(cudaMemcpyAsync(&n, st->evc_off.p + niv, 8, cudaMemcpyDeviceToHost, q));
    c->sync();
    const size_t nn = (size_t)std::max<unsigned long long>(n, 1);
    st->evc_iv.grow(nn);
    st->evc_px.grow(nn);
    st->evc_lobe.grow(nn);
    st->evc_geom.grow(nn);
    st->evc_val.grow(nn);
    st->evc_surf.grow(nn);
    CK(launch_evc_fill(c->dsc, vt, st->evc_off.p, st->evc_iv.p, st->evc_px.p, st->evc_lobe.p, st->evc_geom.p,
                       st->evc_surf.p, q, &c->launches));
    st->evc_vlobe.grow(std::max<size_t>(niv, 1));
    CK(launch_vlobe(c->dsc, st->view(), st->evc_vlobe.p, q, &c->launches));
    st->n_evc = n;
    st->evc_key = c->geo_gen;
}

EvalArgs eval_args(prc_gpu_ctx* c, prc_gpu_store* st, const EvalRun& er, const double* phong_dev) {
    const DScene& s = c->dsc;
    EvalArgs ea{};
    ea.sp_t = c->sp_t.p;
    ea.sp_ref = st->sp_ref.p;
    ea.bt_tot = c->bt_tot.p;
    ea.br_tot = st->br_tot.p;
    ea.dbeta = c->dbeta.p;
    ea.phong = phong_dev;
    ea.images = c->images.p;
    ea.clamps = c->clamps.p;
    ea.weights = er.weights;
    ea.g_span = c->g_span.p;
    ea.bt_pad = c->bt_pad.p;
    ea.db_pad = c->db_pad.p;
    ea.g_pad = c->g_pad.p;
    ea.g_pad_copies = c->g_pad_copies;
    ea.g_pad_stride = (long long)(c->g_pad.n / (size_t)std::max(1, c->g_pad_copies));
    ea.g_vert = c->g_vert.p;
    ea.g_phong = c->g_phong.p;
    ea.per_species = er.per_species ? 1 : 0;
    ea.legacy = er.legacy ? 1 : 0;
    ea.do_beta = s.has_medium && (s.unknown >= 0 || er.per_species) ? 1 : 0;
    ea.vlobe = evc_ready(c, st) ? st->evc_vlobe.p : nullptr;
    return ea;
}

// Runs the image-producing kernel `launch` and all-reduces the raw images.  Deterministic
// runs take two passes: the first finds the largest contribution (EvalArgs::img_mode 1), the
// second adds exact 128-bit fixed-point values with a quantum 2^-101 of it (img_mode 2), so
// the image does not depend on the order of the atomic additions, nor on how paths are
// spread over ranks (render() is bit-reproducible under any worker count in the reference,
// transport.hpp:171-173).  Contributions below the quantum (< 2^-101 of the largest) are
// dropped.
template <class F>
void image_pass(prc_gpu_ctx* c, EvalArgs& ea, const EvalRun& er, F&& launch) {
    cudaStream_t q = c->stream;
    if (!er.deterministic) {
        ea.img_mode = 0;
        launch(ea);
        CK(cudaEventRecord(c->ev[2], q));
        if (c->nvls) {  // the images' cross-rank sum by multimem reductions (prc_nvls.cu)
            NvlsFold a{};
            a.g_span = c->images.p;
            a.n_out = 1;
            a.V = c->n_pix;
            a.nx = a.ny = a.pnx = a.pnxny = 1;
            a.scale = 1.0;
            CK(nvls_fold(c->nvls, a, 0, q, &c->launches));
            CK(cudaMemcpyAsync(c->images.p, nvls_local(c->nvls), (size_t)c->n_pix * 8, cudaMemcpyDeviceToDevice, q));
        } else {
            c->allreduce(c->images.p, (size_t)c->n_pix);
        }
        return;
    }
    const size_t n = (size_t)c->n_pix;
    c->img_max.grow(1);
    c->img_fx.grow(std::max<size_t>(2 * n, 1));
    c->img_limbs.grow(std::max<size_t>(3 * n, 1));
    CK(cudaMemsetAsync(c->img_max.p, 0, 8, q));
    ea.img_mode = 1;
    ea.img_max = c->img_max.p;
    launch(ea);
    if (c->comm) NK(ncclAllReduce(c->img_max.p, c->img_max.p, 1, ncclUint64, ncclMax, c->comm, q));
    unsigned long long bits = 0;
    CK(cudaMemcpyAsync(&bits, c->img_max.p, 8, cudaMemcpyDeviceToHost, q));
    c->sync();
    double vmax;
    std::memcpy(&vmax, &bits, 8);
    CK(cudaMemsetAsync(c->img_fx.p, 0, c->img_fx.bytes(), q));
    CK(cudaMemsetAsync(c->clamps.p, 0, sizeof(unsigned long long), q));  // the first pass counted them
    int e = 0;
    std::frexp(vmax, &e);  // vmax < 2^e: every term of the second pass is below 2^101
    ea.img_mode = 2;
    ea.img_fx = c->img_fx.p;
    ea.img_inv_quantum = std::ldexp(1.0, std::min(1023, 101 - e));
    const double quantum = std::ldexp(1.0, std::max(-1074, e - 101));
    if (vmax > 0.0) launch(ea);
    CK(cudaEventRecord(c->ev[2], q));
    CK(launch_fixed_to_limbs(c->img_fx.p, (long long)n, c->img_limbs.p, q, &c->launches));
    if (c->comm) NK(ncclAllReduce(c->img_limbs.p, c->img_limbs.p, 3 * n, ncclUint64, ncclSum, c->comm, q));
    CK(launch_limbs_to_images(c->img_limbs.p, (long long)n, quantum, c->images.p, q, &c->launches));
    ea.img_mode = 0;
}

// K3 prep + K4 forward (+ image allreduce).  Raw pixel sums land in c->images.
// Events [0]..[3] bracket prep / forward / allreduce.
void run_forward(prc_gpu_ctx* c, prc_gpu_store* st, const Resolved& r, const EvalRun& er,
                 const double*& phong_dev, EvalArgs& ea) {
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    CK(cudaEventRecord(c->ev[0], q));
    CK(launch_prep(s.n_species, c->V, r.src, st->br_tot64.p, c->sp_t.p, c->bt_tot.p, c->dbeta.p, q,
                   &c->launches));
    if (c->mode == 0 && s.pad_walk)
        CK(launch_pad_tables(s, c->bt_tot.p, c->dbeta.p, c->bt_pad.p, c->db_pad.p, q, &c->launches));
    if (!phong_dev) {
        const double ph[2] = {r.kappa, r.gamma};
        CK(cudaMemcpyAsync(c->phong.p, ph, sizeof ph, cudaMemcpyHostToDevice, q));
        phong_dev = c->phong.p;
    }
    if (st->mat) {  // stored spans (prc_materialized.cu)
        for (int j = 0; j < PRC_MAX_SPECIES; ++j) st->m_ctx.t[j] = r.src[j];
        st->m_ctx.ref = st->m_ref64.p;
        st->m_ctx.bt_tot = st->m_bt.p;
        st->m_ctx.br_tot = st->m_br.p;
        st->m_ctx.dbeta = st->m_db.p;
        CK(launch_mat_prep(s.n_species, c->V, st->m_ctx, q, &c->launches));
        ++c->fwd_gen;
        CK(cudaMemsetAsync(c->images.p, 0, c->images.bytes(), q));
        CK(cudaMemsetAsync(c->clamps.p, 0, sizeof(unsigned long long), q));
        CK(cudaMemsetAsync(st->m_eval.p, 0, st->m_eval.bytes(), q));
        ea = eval_args(c, st, er, phong_dev);
        c->timed_sub = c->timed_grad = false;
        CK(cudaEventRecord(c->ev[1], q));
        image_pass(c, ea, er, [&](const EvalArgs& a) {
            CK(launch_mat_forward(s, st->mat_view(), st->m_ctx, a, q, &c->launches));
        });
        c->allreduce_u64(c->clamps.p, 1);
        CK(cudaEventRecord(c->ev[3], q));
        return;
    }
    const size_t slots = (size_t)s.n_det * (size_t)std::max<unsigned long long>(st->n_iv, 1);
    // ev_f: phase values [j][det][i] (fcache), then 8-byte aligned the surface events' f64
    // cos_le [det][i] (scache); ev_cos_of in prc_wavefront.cu
    const size_t fslots = std::max<size_t>(
        1, ((s.fcache ? (size_t)s.n_species * slots : 0) + 1) / 2 * 2 + (s.scache ? 2 * slots : 0));
    if (st->ev_val.n < slots || st->ev_pix.n < slots ||
        (c->mode == 0 && (st->ev_c1.n < slots || st->ev_f.n < fslots)))
        st->geo_key = 0;
    st->ev_val.grow(slots);
    st->ev_pix.grow(slots);
    if (c->mode == 0) {
        st->ev_c1.grow(slots);
        st->ev_f.grow(fslots);
    }
    st->lp.grow((size_t)std::max<unsigned long long>(st->n_iv, 1));
    st->own.grow((size_t)std::max<unsigned long long>(st->n_iv, 1));
    ++c->fwd_gen;  // invalidates any cached forward
    if (c->mode == 0) ensure_vertex_table(c, st);
    CK(cudaMemsetAsync(c->images.p, 0, c->images.bytes(), q));
    CK(cudaMemsetAsync(c->clamps.p, 0, sizeof(unsigned long long), q));
    ea = eval_args(c, st, er, phong_dev);
    c->timed_sub = c->mode == 0;
    c->timed_grad = false;
    CK(cudaEventRecord(c->ev[1], q));
    if (c->mode == 0) {
        CK(launch_prefix(s, st->view(), ea, st->lp.p, q, &c->launches));
        CK(cudaEventRecord(c->ev[6], q));
        if (evc_ready(c, st)) {
            image_pass(c, ea, er, [&](const EvalArgs& a) {
                CK(launch_evc_forward(s, event_list(st), a, st->lp.p, q, &c->launches));
            });
            st->evc_vals = true;
        } else {
            image_pass(c, ea, er, [&](const EvalArgs& a) {
                CK(launch_le_forward(s, vertex_table(st), a, st->lp.p, q, &c->launches));
                st->geo_key = c->geo_gen;  // K4b wrote the event geometry (stream-ordered for later launches)
            });
            st->evc_vals = false;  // this pass's event values are in the dense cache
            build_event_list(c, st);  // later forwards over the store take the event list
        }
    } else {
        st->geo_key = 0;  // the per-path kernels reuse ev_pix in path layout
        image_pass(c, ea, er, [&](const EvalArgs& a) { CK(launch_forward(s, st->view(), a, q, &c->launches)); });
    }
    c->allreduce_u64(c->clamps.p, 1);
    CK(cudaEventRecord(c->ev[3], q));
}

// K5b lane spreading.  Lanes far apart in Morton order avoid same-voxel reductions in one
// RED instruction; lanes close together walk coherent rays.  The contention scale is the
// interaction vertices per voxel d per gradient copy C.  Round 2, K5b ms at spread
// 4 / 16 / 32 / 64: (b) 1e8 paths at 128^3 (d = 150, C = 8) 672 / 603 / 602 / 607, (c)
// (d = 151) - / 714 / 704 / 705; 5e7 paths (d = 75) 322 / 302 / 307 / -; 3e7 paths (d = 45)
// 188 / 185 / 189 / -; 2.5e7 (d = 37) 157 / 155 / - / -; 1e7 paths (d = 15) 64.5 / 67.3 /
// - / 74.0; (e) 256^3 (d = 23, C = 8) 1499 / 1524 / 1584 / 1658; (a) 32^3 (d = 96, C = 32)
// 2.28 / 2.39 / 2.47 / 2.52.
int auto_spread(const prc_gpu_ctx* c, const prc_gpu_store* st) {
    if (c->spread > 0) return c->spread;
    const double d = (double)st->n_iv / (double)std::max<long long>(c->V, 1);
    const double q = d / (double)std::max(1, c->g_pad_copies);
    return q >= 15.0 ? 32 : q >= 4.0 ? 16 : 4;
}

// K5 gradient with weights ea.weights, then its reduction over ranks and the combination
// grad_j = scale (g_span + g_vert[j]) (n_out species slices) into c->grad_res.  Event [4]
// after K5.  With NVLS (option "nvls") one fold kernel does the padded-copy sum, the
// combination and the cross-rank sum through multimem reductions (prc_nvls.cu); otherwise
// k_unpad_add, ncclAllReduce of g_span and g_vert, and k_combine.
void run_gradient(prc_gpu_ctx* c, prc_gpu_store* st, const EvalArgs& ea, int n_out, double scale) {
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    CK(cudaMemsetAsync(c->g_span.p, 0, c->g_span.bytes(), q));
    CK(cudaMemsetAsync(c->g_vert.p, 0, c->g_vert.bytes(), q));
    CK(cudaMemsetAsync(c->g_phong.p, 0, 2 * sizeof(double), q));
    if (st->mat) {
        CK(launch_mat_gradient(s, st->mat_view(), st->m_ctx, ea, q, &c->launches));
    } else if (c->mode == 0) {
        if (s.pad_walk) CK(cudaMemsetAsync(c->g_pad.p, 0, c->g_pad.bytes(), q));
        // lane spreading only de-conflicts the LE-span reductions; without them (no medium,
        // or no beta gradient) lanes take consecutive vertices so the event loads coalesce
        if (evc_ready(c, st) && st->evc_vals)
            CK(launch_evc_gradient(s, event_list(st), ea, st->own.p, q, &c->launches));
        else
            CK(launch_le_gradient(s, vertex_table(st), ea, st->own.p, ea.do_beta ? auto_spread(c, st) : 1,
                                  s.pad_walk ? c->packet : 1, q, &c->launches));
        CK(cudaEventRecord(c->ev[7], q));
        c->timed_grad = true;
        CK(launch_path_gradient(s, st->view(), ea, st->own.p, q, &c->launches));
    } else {
        CK(launch_gradient(s, st->view(), ea, q, &c->launches));
    }
    const bool padded = !st->mat && c->mode == 0 && s.pad_walk;
    CK(cudaEventRecord(c->ev[4], q));
    c->grad_res = nullptr;
    if (ea.do_beta && c->nvls) {
        NvlsFold a{};
        if (padded) {
            a.g_pad = c->g_pad.p;
            a.copies = c->g_pad_copies;
            a.stride = ea.g_pad_stride;
        } else {
            a.g_span = c->g_span.p;
        }
        a.g_vert = c->g_vert.p;
        a.n_out = n_out;
        a.V = c->V;
        a.nx = s.dims[0];
        a.ny = s.dims[1];
        a.pnx = s.pnx;
        a.pnxny = s.pnxny;
        a.scale = scale;
        CK(nvls_fold(c->nvls, a, (size_t)c->n_pix, q, &c->launches));
        c->grad_res = nvls_local(c->nvls) + c->n_pix;
    } else if (ea.do_beta) {
        if (padded) CK(launch_unpad_add(s, c->g_pad.p, c->g_pad_copies, ea.g_pad_stride, c->g_span.p, q, &c->launches));
        c->allreduce(c->g_span.p, c->g_span.n);
        c->allreduce(c->g_vert.p, c->g_vert.n);
        CK(launch_combine_grad(c->g_span.p, c->g_vert.p, n_out, c->V, scale, c->g_out.p, q, &c->launches));
        c->grad_res = c->g_out.p;
    }
    c->allreduce(c->g_phong.p, 2);
}

// Runs K3 prep, K4 forward (+ image allreduce) and optionally K5 (+ grad allreduce).
// Leaves raw sums in c->images / c->g_span / c->g_vert / c->g_phong; returns clamps.
unsigned long long run_eval(prc_gpu_ctx* c, prc_gpu_store* st, const Resolved& r, const EvalRun& er,
                            const double* phong_dev) {
    cudaStream_t q = c->stream;
    EvalArgs ea;
    run_forward(c, st, r, er, phong_dev, ea);
    if (er.want_grad)
        run_gradient(c, st, ea, er.per_species ? c->dsc.n_species : 1, er.grad_scale);
    else
        CK(cudaEventRecord(c->ev[4], q));
    unsigned long long cl = 0;
    CK(cudaMemcpyAsync(&cl, c->clamps.p, sizeof cl, cudaMemcpyDeviceToHost, q));
    return cl;
}

void record_timings(prc_gpu_ctx* c) {
    c->sync();
    float ms;
    const int pairs[5][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}};
    for (int i = 0; i < 5; ++i) {
        CK(cudaEventElapsedTime(&ms, c->ev[pairs[i][0]], c->ev[pairs[i][1]]));
        c->last_ms[i] = ms;
    }
    CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]));
    c->last_ms[5] = ms;
    c->last_ms[6] = c->last_ms[7] = 0.0;
    if (c->mode == 0 && c->timed_sub) {
        CK(cudaEventElapsedTime(&ms, c->ev[1], c->ev[6]));
        c->last_ms[6] = ms;
        if (c->timed_grad) {
            CK(cudaEventElapsedTime(&ms, c->ev[7], c->ev[4]));
            c->last_ms[7] = ms;
        }
    }
}

// ----------------------------------------------------------------------- K1 trace
// Builds a path-major store for this rank's shard, sampled under species values
// `sp_dev` (n_species x V, fp64, device) and Phong values (kappa, gamma).
std::unique_ptr<prc_gpu_store> trace_store(prc_gpu_ctx* c, const prc_gpu_render_opts* o,
                                           const double* sp_dev, double kappa, double gamma,
                                           const double* ref_beta_host_or_dev, bool ref_on_dev) {
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    auto st = std::make_unique<prc_gpu_store>(c);
    stamp_store(c, st.get());
    const unsigned long long N = o->n_paths;
    st->n_global = N;
    unsigned long long end = 0;
    shard_range(N, c->rank, c->world, &st->stream_base, &end);
    st->n = end - st->stream_base;
    st->seed = o->seed;
    st->ref_kappa = kappa;
    st->ref_gamma = gamma;
    const long long V = c->V;
    // reference context of the store (make_context's ref side, pathstore.cpp:54-81)
    st->br_tot64.alloc((size_t)std::max<long long>(V, 1));
    st->sp_ref.alloc((size_t)std::max(1, s.n_species) * (size_t)std::max<long long>(V, 1));
    st->br_tot.alloc((size_t)std::max<long long>(V, 1));
    const double* src[PRC_MAX_SPECIES] = {};
    for (int j = 0; j < s.n_species; ++j) src[j] = sp_dev + (size_t)j * V;
    CK(launch_prep_ref(s.n_species, V, src, st->br_tot64.p, st->sp_ref.p, st->br_tot.p, nullptr, q,
                       &c->launches));
    if (s.unknown >= 0) {
        st->ref_beta.resize((size_t)V);
        CK(cudaMemcpyAsync(st->ref_beta.data(), ref_beta_host_or_dev ? ref_beta_host_or_dev
                                                                      : sp_dev + (size_t)s.unknown * V,
                           (size_t)V * sizeof(double),
                           ref_on_dev || !ref_beta_host_or_dev ? cudaMemcpyDeviceToHost
                                                               : cudaMemcpyHostToHost,
                           q));
    }
    const unsigned long long n = st->n;
    st->B.alloc(std::max<unsigned long long>(n, 1));
    st->trunc.alloc(std::max<unsigned long long>(n, 1));
    st->stream.alloc(std::max<unsigned long long>(n, 1));
    // stream ids of a fresh shard are stream_base + i
    CK(launch_iota_u64(st->stream.p, (long long)n, st->stream_base, q, &c->launches));
    TraceArgs a{};
    a.beta_tot = st->br_tot64.p;
    a.sp_beta = sp_dev;
    a.seed = o->seed;
    a.stream_base = st->stream_base;
    a.n = n;
    a.max_bounces = o->max_bounces > 0 ? o->max_bounces : 500;
    a.max_events = o->max_scatter_events;
    a.B = st->B.p;
    a.trunc = st->trunc.p;
    a.err = c->err.p;
    CK(cudaMemsetAsync(c->err.p, 0, sizeof(int), q));
    CK(launch_trace(s, a, false, q, &c->launches));
    // offsets: exclusive scans of (B + 1) and (B - 1)+
    c->u64tmp_a.grow(std::max<unsigned long long>(n, 1) * 2);
    c->u64tmp_b.grow(std::max<unsigned long long>(n, 1) * 2);
    unsigned long long* rt = c->u64tmp_a.p;
    unsigned long long* it = c->u64tmp_a.p + std::max<unsigned long long>(n, 1);
    st->rec_base.alloc(std::max<unsigned long long>(n, 1));
    st->iv_base.alloc(std::max<unsigned long long>(n, 1));
    st->stride.alloc(std::max<unsigned long long>(n, 1));
    CK(launch_size_terms(st->B.p, (long long)n, rt, it, q, &c->launches));
    CK(scan_u64(rt, c->u64tmp_b.p, (long long)n, &c->cub_tmp, &c->cub_bytes, q));
    CK(scan_u64(it, c->u64tmp_b.p + std::max<unsigned long long>(n, 1), (long long)n, &c->cub_tmp,
                &c->cub_bytes, q));
    CK(launch_path_major_layout(c->u64tmp_b.p, c->u64tmp_b.p + std::max<unsigned long long>(n, 1),
                                (long long)n, st->rec_base.p, st->stride.p, st->iv_base.p, q,
                                &c->launches));
    int errf = 0;
    CK(cudaMemcpyAsync(&errf, c->err.p, sizeof errf, cudaMemcpyDeviceToHost, q));
    unsigned long long last[4] = {0, 0, 0, 0};
    uint32_t lastB = 0;
    if (n) {
        CK(cudaMemcpyAsync(&last[0], c->u64tmp_b.p + (n - 1), sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, q));
        CK(cudaMemcpyAsync(&last[1], c->u64tmp_b.p + std::max<unsigned long long>(n, 1) + (n - 1),
                           sizeof(unsigned long long), cudaMemcpyDeviceToHost, q));
        CK(cudaMemcpyAsync(&lastB, st->B.p + (n - 1), sizeof lastB, cudaMemcpyDeviceToHost, q));
    }
    c->u32tmp.grow(1);
    uint32_t maxB = 0;
    if (n) {
        CK(reduce_max_u32(st->B.p, (long long)n, c->u32tmp.p, &c->cub_tmp, &c->cub_bytes, q));
        CK(cudaMemcpyAsync(&maxB, c->u32tmp.p, sizeof maxB, cudaMemcpyDeviceToHost, q));
    }
    c->sync();
    if (errf) throw Err(PRC_ERR_CONFIG, "sample_direction: vacuum point");
    st->max_B = (int)maxB;
    st->n_rec = n ? last[0] + lastB + 1 : 0;
    st->n_iv = n ? last[1] + (lastB >= 2 ? lastB - 1 : 0) : 0;
    st->segments = st->n_rec - n;
    st->alloc_records(std::max<unsigned long long>(st->n_rec, 1));
    a.off = st->rec_base.p;
    a.rec = st->rec_out();
    CK(launch_trace(s, a, true, q, &c->launches));
    // truncated count
    {
        CK(cudaMemsetAsync(c->u64tmp_a.p, 0, sizeof(unsigned long long), q));
        CK(launch_count_nonzero_u8(st->trunc.p, (long long)n, c->u64tmp_a.p, q, &c->launches));
        unsigned long long cnt = 0;
        CK(cudaMemcpyAsync(&cnt, c->u64tmp_a.p, sizeof cnt, cudaMemcpyDeviceToHost, q));
        c->sync();
        st->truncated = cnt;
    }
    return st;
}

// ----------------------------------------------------------------------- K2 sort
void sort_store(prc_gpu_ctx* c, prc_gpu_store* st) {
    if (st->n_global == 0 || (st->n == 0 && c->world == 1))
        throw Err(PRC_ERR_CONFIG, "sort_by_size: empty store");
    const long long n = (long long)st->n;
    if (n == 0) {
        st->sorted = true;
        return;
    }
    cudaStream_t q = c->stream;
    const int nb = st->max_B + 1;
    const int tile = 4096;
    const long long n_tiles = (n + tile - 1) / tile;
    DBuf<unsigned long long> th, toff;
    th.alloc((size_t)nb * n_tiles);
    toff.alloc((size_t)nb * n_tiles);
    CK(launch_sort_hist(st->B.p, n, nb, tile, th.p, q, &c->launches));
    CK(scan_u64(th.p, toff.p, (long long)nb * n_tiles, &c->cub_tmp, &c->cub_bytes, q));
    DBuf<uint32_t> perm;
    perm.alloc((size_t)n);
    CK(launch_sort_rank(st->B.p, n, nb, tile, toff.p, perm.p, q, &c->launches));
    // bucket table: start of bin k = toff[k * n_tiles] (one strided copy of column 0)
    std::vector<unsigned long long> bstart(nb + 1), brec(nb + 1), biv(nb + 1);
    CK(cudaMemcpy2DAsync(bstart.data(), sizeof(unsigned long long), toff.p,
                         (size_t)n_tiles * sizeof(unsigned long long), sizeof(unsigned long long), (size_t)nb,
                         cudaMemcpyDeviceToHost, q));
    c->sync();
    bstart[nb] = (unsigned long long)n;
    unsigned long long R = 0, I = 0;
    for (int k = 0; k <= nb; ++k) {
        brec[k] = R;
        biv[k] = I;
        if (k < nb) {
            const unsigned long long cnt = bstart[k + 1] - bstart[k];
            R += cnt * (unsigned long long)(k + 1);
            I += cnt * (unsigned long long)(k >= 2 ? k - 1 : 0);
        }
    }
    DBuf<unsigned long long> d_bstart, d_brec, d_biv;
    d_bstart.alloc(nb + 1);
    d_brec.alloc(nb + 1);
    d_biv.alloc(nb + 1);
    CK(cudaMemcpyAsync(d_bstart.p, bstart.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, q));
    CK(cudaMemcpyAsync(d_brec.p, brec.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, q));
    CK(cudaMemcpyAsync(d_biv.p, biv.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, q));
    auto ns = std::make_unique<prc_gpu_store>();
    ns->B.alloc((size_t)n);
    ns->stream.alloc((size_t)n);
    ns->trunc.alloc((size_t)n);
    ns->rec_base.alloc((size_t)n);
    ns->stride.alloc((size_t)n);
    ns->iv_base.alloc((size_t)n);
    CK(launch_bucket_layout(perm.p, st->B.p, st->stream.p, st->trunc.p, n, d_bstart.p, d_brec.p,
                            d_biv.p, ns->B.p, ns->stream.p, ns->trunc.p, ns->rec_base.p,
                            ns->stride.p, ns->iv_base.p, q, &c->launches));
    // re-layout one record field at a time through one spare field buffer (8 B per record,
    // not a second store): an 8-byte field is gathered into the spare, which then takes the
    // old field's place; the two 4-byte fields are gathered into the spare's halves and
    // copied back
    const StoreView old_view = st->view();
    DBuf<double> spare;
    spare.alloc(st->n_rec);
    for (DBuf<double>* f : {&st->px, &st->py, &st->pz, &st->dx, &st->dy, &st->dz, &st->tt, &st->ct}) {
        CK(launch_gather_field(old_view, perm.p, n, ns->rec_base.p, ns->stride.p, f->p, spare.p, 8, q,
                               &c->launches));
        f->swap(spare);
    }
    uint32_t* half0 = reinterpret_cast<uint32_t*>(spare.p);
    uint32_t* half1 = half0 + st->n_rec;
    CK(launch_gather_field(old_view, perm.p, n, ns->rec_base.p, ns->stride.p, st->vox.p, half0, 4, q,
                           &c->launches));
    CK(launch_gather_field(old_view, perm.p, n, ns->rec_base.p, ns->stride.p, st->meta.p, half1, 4, q,
                           &c->launches));
    CK(cudaMemcpyAsync(st->vox.p, half0, st->n_rec * 4, cudaMemcpyDeviceToDevice, q));
    CK(cudaMemcpyAsync(st->meta.p, half1, st->n_rec * 4, cudaMemcpyDeviceToDevice, q));
    if (st->mat) {  // storage position -> file record of a materialized store
        DBuf<unsigned long long> nr;
        nr.alloc((size_t)n);
        CK(launch_gather_u64(perm.p, n, st->m_rec.p, nr.p, q, &c->launches));
        c->sync();
        st->m_rec.swap(nr);
    }
    c->sync();
    st->B.swap(ns->B);
    st->stream.swap(ns->stream);
    st->trunc.swap(ns->trunc);
    st->rec_base.swap(ns->rec_base);
    st->stride.swap(ns->stride);
    st->iv_base.swap(ns->iv_base);
    st->sorted = true;
    st->vt_ready = false;  // vertex table indexes the old layout
    ++c->fwd_gen;          // the event cache indexes the old layout too
}

// ----------------------------------------------------------------------- PSTR I/O
template <class T>
void put(std::ofstream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <class T>
T get(std::ifstream& is) {
    T v{};
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
}

template <class T>
std::vector<T> d2h(const DBuf<T>& b, size_t n, cudaStream_t q) {
    std::vector<T> h(n);
    if (n) CK(cudaMemcpyAsync(h.data(), b.p, n * sizeof(T), cudaMemcpyDeviceToHost, q));
    return h;
}

// save_store of a materialized store: the header from the store, then the file's own
// record bytes in storage order (so a sorted store writes what sort_by_size + save_store
// of the reference writes, pathstore.cpp:261-267, 410-453).
void export_materialized(prc_gpu_ctx* c, prc_gpu_store* st, const std::string& path) {
    std::vector<unsigned long long> rec(st->n);
    if (st->n) CK(cudaMemcpyAsync(rec.data(), st->m_rec.p, st->n * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Err(PRC_ERR_IO, "save_store: cannot open " + path);
    os.write("PSTR", 4);
    put<uint32_t>(os, 1u);
    put<uint64_t>(os, st->n);
    put<uint64_t>(os, st->generation);
    put<uint64_t>(os, st->seed);
    put<uint8_t>(os, st->sorted ? 1 : 0);
    put<uint64_t>(os, st->ref_beta.size());
    for (double b : st->ref_beta) put<double>(os, b);
    put<double>(os, st->ref_kappa);
    put<double>(os, st->ref_gamma);
    for (unsigned long long r : rec)
        os.write(st->mat_bytes.data() + st->mat_off[r], (std::streamsize)(st->mat_off[r + 1] - st->mat_off[r]));
    if (!os) throw Err(PRC_ERR_IO, "save_store: write failure on " + path);
}

void export_pstr(prc_gpu_ctx* c, prc_gpu_store* st, const std::string& path) {
    if (st->mat) return export_materialized(c, st, path);
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    const unsigned long long n = st->n;
    auto B = d2h(st->B, n, q);
    auto streams = d2h(st->stream, n, q);
    auto trunc = d2h(st->trunc, n, q);
    auto rb = d2h(st->rec_base, n, q);
    auto rs = d2h(st->stride, n, q);
    auto ib = d2h(st->iv_base, n, q);
    auto px = d2h(st->px, st->n_rec, q), py = d2h(st->py, st->n_rec, q), pz = d2h(st->pz, st->n_rec, q);
    auto dx = d2h(st->dx, st->n_rec, q), dy = d2h(st->dy, st->n_rec, q), dz = d2h(st->dz, st->n_rec, q);
    auto tt = d2h(st->tt, st->n_rec, q), ct = d2h(st->ct, st->n_rec, q);
    auto vox = d2h(st->vox, st->n_rec, q);
    auto meta = d2h(st->meta, st->n_rec, q);
    // events on the device
    const size_t slots = (size_t)s.n_det * (size_t)std::max<unsigned long long>(st->n_iv, 1);
    DBuf<int32_t> epix;
    DBuf<double> ecos, egeom, eray;
    epix.alloc(slots);
    ecos.alloc(slots);
    egeom.alloc(slots);
    eray.alloc(4 * slots);
    CK(launch_events(s, st->view(), epix.p, ecos.p, egeom.p, eray.p, q, &c->launches));
    auto hpix = d2h(epix, slots, q);
    auto hcos = d2h(ecos, slots, q);
    auto hgeom = d2h(egeom, slots, q);
    auto hray = d2h(eray, 4 * slots, q);
    c->sync();
    // rays: every segment b = 1..B and every event's LE connection
    std::vector<double> rays;
    auto rec = [&](unsigned long long p, int b) { return rb[p] + (unsigned long long)b * rs[p]; };
    for (unsigned long long p = 0; p < n; ++p) {
        for (int b = 1; b <= (int)B[p]; ++b) {
            const auto r0 = rec(p, b - 1), r1 = rec(p, b);
            rays.insert(rays.end(), {px[r0], py[r0], pz[r0], dx[r1], dy[r1], dz[r1], tt[r1]});
        }
        for (int b = 1; b < (int)B[p]; ++b) {
            const auto r1 = rec(p, b);
            const unsigned long long iv = ib[p] + (unsigned long long)(b - 1) * rs[p];
            for (int k = 0; k < s.n_det; ++k) {
                const size_t slot = (size_t)k * st->n_iv + iv;
                if (hpix[slot] < 0) continue;
                rays.insert(rays.end(), {px[r1], py[r1], pz[r1], hray[4 * slot], hray[4 * slot + 1],
                                         hray[4 * slot + 2], hray[4 * slot + 3]});
            }
        }
    }
    const long long nr = (long long)(rays.size() / 7);
    std::vector<uint32_t> counts(nr), svox;
    std::vector<double> slen;
    std::vector<unsigned long long> offs(nr + 1, 0);
    if (s.has_medium && nr > 0) {
        DBuf<double> drays;
        DBuf<uint32_t> dcounts, dvox;
        DBuf<unsigned long long> doff;
        DBuf<double> dlen;
        drays.alloc(rays.size());
        dcounts.alloc(nr);
        CK(cudaMemcpyAsync(drays.p, rays.data(), rays.size() * 8, cudaMemcpyHostToDevice, q));
        CK(launch_walk(s, drays.p, nr, dcounts.p, nullptr, nullptr, nullptr, q, &c->launches));
        counts = d2h(dcounts, nr, q);
        c->sync();
        for (long long i = 0; i < nr; ++i) offs[i + 1] = offs[i] + counts[i];
        const unsigned long long tot = offs[nr];
        doff.alloc(nr);
        dvox.alloc(std::max<unsigned long long>(tot, 1));
        dlen.alloc(std::max<unsigned long long>(tot, 1));
        CK(cudaMemcpyAsync(doff.p, offs.data(), nr * 8, cudaMemcpyHostToDevice, q));
        CK(launch_walk(s, drays.p, nr, dcounts.p, doff.p, dvox.p, dlen.p, q, &c->launches));
        svox = d2h(dvox, tot, q);
        slen = d2h(dlen, tot, q);
        c->sync();
    }
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Err(PRC_ERR_IO, "save_store: cannot open " + path);
    os.write("PSTR", 4);
    put<uint32_t>(os, 1u);
    put<uint64_t>(os, n);
    put<uint64_t>(os, st->generation);
    put<uint64_t>(os, st->seed);
    put<uint8_t>(os, st->sorted ? 1 : 0);
    put<uint64_t>(os, st->ref_beta.size());
    for (double b : st->ref_beta) put<double>(os, b);
    put<double>(os, st->ref_kappa);
    put<double>(os, st->ref_gamma);
    long long ray = 0;
    for (unsigned long long p = 0; p < n; ++p) {
        const int Bp = (int)B[p];
        put<uint64_t>(os, streams[p]);
        put<uint8_t>(os, trunc[p]);
        const auto r0 = rec(p, 0);
        put<double>(os, dx[r0]);
        put<double>(os, dy[r0]);
        put<double>(os, dz[r0]);
        put<uint32_t>(os, (uint32_t)(Bp + 1));
        uint32_t span_pos = 0;
        const long long seg_ray0 = ray;
        for (int b = 0; b <= Bp; ++b) {
            const auto r = rec(p, b);
            const uint32_t m = meta[r];
            const uint32_t kind = m & 0xffu;
            double cos_in = 1.0, cos_out = 1.0;
            if (kind == VK_SURFACE) {  // facing normal; cos_out from the continuation direction
                const prc_surface_desc& sf = c->surfaces[(int)(int16_t)(m >> 16)];
                H3 x{px[r], py[r], pz[r]}, din{dx[r], dy[r], dz[r]}, nn;
                if (sf.kind == PRC_SURF_SPHERE)
                    nn = hnormalized(hsub(x, h3(sf.center)));
                else
                    nn = {sf.axis == 0 ? sf.normal_sign : 0.0, sf.axis == 1 ? sf.normal_sign : 0.0,
                          sf.axis == 2 ? sf.normal_sign : 0.0};
                if (hdot(nn, din) > 0.0) nn = {-nn.x, -nn.y, -nn.z};
                cos_in = -hdot(nn, din);
                if (b < Bp) {
                    const auto rn = rec(p, b + 1);
                    cos_out = hdot(nn, H3{dx[rn], dy[rn], dz[rn]});
                }
            }
            uint32_t sb = 0, se = 0;
            if (b >= 1) {
                sb = span_pos;
                span_pos += s.has_medium ? counts[seg_ray0 + (b - 1)] : 0;
                se = span_pos;
            }
            put<double>(os, px[r]);
            put<double>(os, py[r]);
            put<double>(os, pz[r]);
            put<double>(os, ct[r]);
            put<double>(os, cos_in);
            put<double>(os, cos_out);
            put<uint32_t>(os, sb);
            put<uint32_t>(os, se);
            put<int32_t>(os, vox[r]);
            put<int16_t>(os, (int16_t)(m >> 16));
            put<int8_t>(os, (int8_t)((m >> 8) & 0xffu));
            put<uint8_t>(os, (uint8_t)kind);
        }
        put<uint32_t>(os, span_pos);
        for (int b = 1; b <= Bp; ++b) {
            const long long rr = seg_ray0 + (b - 1);
            if (!s.has_medium) continue;
            for (unsigned long long k = offs[rr]; k < offs[rr + 1]; ++k) {
                put<uint32_t>(os, svox[k]);
                put<double>(os, slen[k]);
            }
        }
        ray += Bp;
        // events
        uint32_t ne = 0;
        for (int b = 1; b < Bp; ++b) {
            const unsigned long long iv = ib[p] + (unsigned long long)(b - 1) * rs[p];
            for (int k = 0; k < s.n_det; ++k) ne += hpix[(size_t)k * st->n_iv + iv] >= 0 ? 1 : 0;
        }
        put<uint32_t>(os, ne);
        const long long le_ray0 = ray;
        uint32_t le_pos = 0;
        long long er = le_ray0;
        for (int b = 1; b < Bp; ++b) {
            const unsigned long long iv = ib[p] + (unsigned long long)(b - 1) * rs[p];
            for (int k = 0; k < s.n_det; ++k) {
                const size_t slot = (size_t)k * st->n_iv + iv;
                if (hpix[slot] < 0) continue;
                const uint32_t cnt = s.has_medium ? counts[er] : 0;
                put<uint32_t>(os, (uint32_t)b);
                put<uint16_t>(os, (uint16_t)k);
                put<int32_t>(os, hpix[slot]);
                put<double>(os, hcos[slot]);
                put<double>(os, hgeom[slot]);
                put<uint32_t>(os, le_pos);
                put<uint32_t>(os, le_pos + cnt);
                le_pos += cnt;
                ++er;
            }
        }
        put<uint32_t>(os, le_pos);
        for (long long rr = le_ray0; rr < er; ++rr) {
            if (!s.has_medium) continue;
            for (unsigned long long k = offs[rr]; k < offs[rr + 1]; ++k) {
                put<uint32_t>(os, svox[k]);
                put<double>(os, slen[k]);
            }
        }
        ray = er;
    }
    if (!os) throw Err(PRC_ERR_IO, "save_store: write failure on " + path);
}

// Host arrays of the stored spans / events of a materialized import (MatView).
struct MatHost {
    std::vector<unsigned long long> vbase{0}, sbase, ebase{0}, lbase;
    std::vector<uint32_t> vmeta, vsb, vse, svox, evert, esb, ese, lvox;
    std::vector<int32_t> vvox, edet, epix;
    std::vector<double> vct, slen, ecos, egeom, llen;
};

std::unique_ptr<prc_gpu_store> import_pstr(prc_gpu_ctx* c, const std::string& path, bool materialize) {
    const DScene& s = c->dsc;
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Err(PRC_ERR_IO, "load_store: cannot open " + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "PSTR", 4) != 0)
        throw Err(PRC_ERR_IO, "load_store: bad magic at offset 0 in " + path);
    if (get<uint32_t>(is) != 1) throw Err(PRC_ERR_IO, "load_store: unsupported version");
    auto st = std::make_unique<prc_gpu_store>(c);
    stamp_store(c, st.get());
    const uint64_t count = get<uint64_t>(is);
    st->generation = get<uint64_t>(is);
    st->seed = get<uint64_t>(is);
    st->sorted = get<uint8_t>(is) != 0;
    const uint64_t nb = get<uint64_t>(is);
    st->ref_beta.resize(nb);
    for (auto& b : st->ref_beta) b = get<double>(is);
    st->ref_kappa = get<double>(is);
    st->ref_gamma = get<double>(is);
    if (!is) throw Err(PRC_ERR_IO, "load_store: truncated file " + path);
    if (s.unknown >= 0 && !st->ref_beta.empty() && (long long)nb != c->V)
        throw Err(PRC_ERR_CONFIG, "load_store: reference beta size != voxel count");
    // this rank's slice of the records
    unsigned long long lo = 0, hi = 0;
    shard_range(count, c->rank, c->world, &lo, &hi);
    st->n_global = count;
    st->stream_base = lo;
    st->n = hi - lo;
    std::vector<uint32_t> B;
    std::vector<unsigned long long> streams, rb, ib;
    std::vector<uint8_t> trunc;
    std::vector<double> px, py, pz, dx, dy, dz, tt, ct;
    std::vector<int32_t> vox;
    std::vector<uint32_t> meta;
    unsigned long long n_iv = 0;
    int maxB = 0;
    MatHost mh;
    st->mat = materialize;
    if (materialize) st->mat_off.push_back(0);
    for (uint64_t i = 0; i < count; ++i) {
        const std::streampos rec_start = is.tellg();
        const uint64_t stream = get<uint64_t>(is);
        const uint8_t tr = get<uint8_t>(is);
        H3 d0{get<double>(is), get<double>(is), get<double>(is)};
        const uint32_t nv = get<uint32_t>(is);
        if (!is || nv == 0) throw Err(PRC_ERR_IO, "load_store: truncated file " + path);
        const bool mine = i >= lo && i < hi;
        H3 prev{0, 0, 0}, pdir = d0;
        if (mine) {
            B.push_back(nv - 1);
            streams.push_back(stream);
            trunc.push_back(tr);
            rb.push_back(px.size());
            ib.push_back(n_iv);
            n_iv += nv >= 3 ? nv - 2 : 0;
            maxB = std::max(maxB, (int)nv - 1);
        }
        const bool keep = materialize && mine;
        for (uint32_t k = 0; k < nv; ++k) {
            H3 x{get<double>(is), get<double>(is), get<double>(is)};
            const double cth = get<double>(is);
            (void)get<double>(is);  // cos_in (not on the recycling path)
            (void)get<double>(is);  // cos_out
            const uint32_t vsb = get<uint32_t>(is);
            const uint32_t vse = get<uint32_t>(is);
            const int32_t vx = get<int32_t>(is);
            const int16_t sf = get<int16_t>(is);
            const int8_t spc = get<int8_t>(is);
            const uint8_t kind = get<uint8_t>(is);
            if (!mine) continue;
            // the kernels index the grid with stored voxel ids: range-check them
            if (vx < -1 || (long long)vx >= c->V || (kind == VK_VOLUME && vx < 0))
                throw Err(PRC_ERR_IO, "load_store: vertex voxel index outside the uploaded grid in " + path);
            // incoming direction: dir0 for the first segment, the chord direction after,
            // formed as the reference's segment_lengths does, d * (1.0 / len)
            // (pathstore.cpp:300-311), so the re-walk is that function's walk bit for bit
            H3 d = d0;
            double t = 0.0;
            if (k >= 1) {
                const H3 ch = hsub(x, prev);
                t = hnorm(ch);
                if (k >= 2) {
                    const double inv = 1.0 / t;
                    d = t > 0.0 ? H3{ch.x * inv, ch.y * inv, ch.z * inv} : pdir;
                }
            }
            px.push_back(x.x);
            py.push_back(x.y);
            pz.push_back(x.z);
            dx.push_back(d.x);
            dy.push_back(d.y);
            dz.push_back(d.z);
            tt.push_back(t);
            ct.push_back(cth);
            vox.push_back(vx);
            meta.push_back((uint32_t)(kind & 0xffu) | ((uint32_t)(uint8_t)spc << 8) |
                           ((uint32_t)(uint16_t)sf << 16));
            if (keep) {
                mh.vmeta.push_back(meta.back());
                mh.vvox.push_back(vx);
                mh.vct.push_back(cth);
                mh.vsb.push_back(vsb);
                mh.vse.push_back(vse);
            }
            prev = x;
            pdir = d;
        }
        if (!keep) {  // spans, events and LE spans are recomputed on the device: skip them
            uint32_t ns = get<uint32_t>(is);
            is.seekg((std::streamoff)ns * 12, std::ios::cur);
            uint32_t ne = get<uint32_t>(is);
            is.seekg((std::streamoff)ne * 34, std::ios::cur);
            uint32_t nl = get<uint32_t>(is);
            is.seekg((std::streamoff)nl * 12, std::ios::cur);
            if (!is) throw Err(PRC_ERR_IO, "load_store: truncated file " + path);
            continue;
        }
        // materialized: the stored spans and events as eval_record reads them, range-checked
        // against the uploaded scene (pathstore.cpp:455-516 reads them unchecked)
        auto bad = [&](const char* what) {
            return Err(PRC_ERR_IO, std::string("load_store: ") + what + " in record " + std::to_string(i) + " of " + path);
        };
        const uint32_t ns = get<uint32_t>(is);
        mh.sbase.push_back(mh.svox.size());
        for (uint32_t k = 0; k < ns; ++k) {
            const uint32_t v = get<uint32_t>(is);
            const double l = get<double>(is);
            if ((long long)v >= c->V) throw bad("span voxel outside the uploaded grid");
            mh.svox.push_back(v);
            mh.slen.push_back(l);
        }
        for (uint32_t k = 0; k < nv; ++k) {
            const size_t vi = mh.vsb.size() - nv + k;
            if (mh.vsb[vi] > mh.vse[vi] || mh.vse[vi] > ns) throw bad("vertex span range outside the record");
        }
        const uint32_t ne = get<uint32_t>(is);
        std::vector<uint32_t> ese_tmp;
        for (uint32_t k = 0; k < ne; ++k) {
            const uint32_t vb = get<uint32_t>(is);
            const uint16_t det = get<uint16_t>(is);
            const int32_t pix = get<int32_t>(is);
            const double cl = get<double>(is);
            const double gm = get<double>(is);
            const uint32_t eb = get<uint32_t>(is);
            const uint32_t ee = get<uint32_t>(is);
            if (vb >= nv) throw bad("event vertex outside the path");
            if (det >= s.n_det || pix < 0 || (long long)pix >= (long long)s.det[det].rows * s.det[det].cols)
                throw bad("event detector / pixel outside the uploaded cameras");
            if (eb > ee) throw bad("event span range reversed");
            mh.evert.push_back(vb);
            mh.edet.push_back(det);
            mh.epix.push_back(pix);
            mh.ecos.push_back(cl);
            mh.egeom.push_back(gm);
            mh.esb.push_back(eb);
            mh.ese.push_back(ee);
            ese_tmp.push_back(ee);
        }
        mh.ebase.push_back(mh.evert.size());
        const uint32_t nl = get<uint32_t>(is);
        for (uint32_t e : ese_tmp)
            if (e > nl) throw bad("event span range outside the record");
        mh.lbase.push_back(mh.lvox.size());
        for (uint32_t k = 0; k < nl; ++k) {
            const uint32_t v = get<uint32_t>(is);
            const double l = get<double>(is);
            if ((long long)v >= c->V) throw bad("LE span voxel outside the uploaded grid");
            mh.lvox.push_back(v);
            mh.llen.push_back(l);
        }
        mh.vbase.push_back(mh.vmeta.size());
        if (!is) throw Err(PRC_ERR_IO, "load_store: truncated file " + path);
        // raw record bytes for a verbatim export
        const std::streampos rec_end = is.tellg();
        const size_t len = (size_t)(rec_end - rec_start);
        const size_t at = st->mat_bytes.size();
        st->mat_bytes.resize(at + len);
        is.seekg(rec_start);
        is.read(st->mat_bytes.data() + at, (std::streamsize)len);
        st->mat_off.push_back(st->mat_bytes.size());
        if (!is) throw Err(PRC_ERR_IO, "load_store: truncated file " + path);
    }
    cudaStream_t q = c->stream;
    const unsigned long long n = st->n;
    st->max_B = maxB;
    st->n_iv = n_iv;
    st->n_rec = px.size();
    st->segments = st->n_rec - n;
    for (auto t : trunc) st->truncated += t;
    auto up = [&](auto& dst, const auto& src) {
        using T = typename std::decay_t<decltype(src)>::value_type;
        dst.alloc(std::max<size_t>(src.size(), 1));
        if (!src.empty())
            CK(cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, q));
    };
    std::vector<uint32_t> stride(n, 1u);
    up(st->B, B);
    up(st->stream, streams);
    up(st->trunc, trunc);
    up(st->rec_base, rb);
    up(st->iv_base, ib);
    up(st->stride, stride);
    up(st->px, px);
    up(st->py, py);
    up(st->pz, pz);
    up(st->dx, dx);
    up(st->dy, dy);
    up(st->dz, dz);
    up(st->tt, tt);
    up(st->ct, ct);
    up(st->vox, vox);
    up(st->meta, meta);
    // reference-side context from the stored ref params
    const long long V = c->V;
    st->br_tot64.alloc((size_t)std::max<long long>(V, 1));
    st->sp_ref.alloc((size_t)std::max(1, s.n_species) * (size_t)std::max<long long>(V, 1));
    st->br_tot.alloc((size_t)std::max<long long>(V, 1));
    const double* src[PRC_MAX_SPECIES] = {};
    for (int j = 0; j < s.n_species; ++j) src[j] = c->scene_sp.p + (size_t)j * V;
    if (s.unknown >= 0 && !st->ref_beta.empty()) {
        c->trace_sp.grow((size_t)V);
        CK(cudaMemcpyAsync(c->trace_sp.p, st->ref_beta.data(), (size_t)V * 8, cudaMemcpyHostToDevice, q));
        src[s.unknown] = c->trace_sp.p;
    }
    CK(launch_prep_ref(s.n_species, V, src, st->br_tot64.p, st->sp_ref.p, st->br_tot.p, nullptr, q,
                       &c->launches));
    c->sync();
    if (materialize) {
        std::vector<unsigned long long> rec(n);
        for (unsigned long long k = 0; k < n; ++k) rec[k] = k;
        up(st->m_rec, rec);
        up(st->m_vbase, mh.vbase);
        up(st->m_sbase, mh.sbase);
        up(st->m_ebase, mh.ebase);
        up(st->m_lbase, mh.lbase);
        up(st->m_vmeta, mh.vmeta);
        up(st->m_vvox, mh.vvox);
        up(st->m_vct, mh.vct);
        up(st->m_vsb, mh.vsb);
        up(st->m_vse, mh.vse);
        up(st->m_svox, mh.svox);
        up(st->m_slen, mh.slen);
        up(st->m_evert, mh.evert);
        up(st->m_edet, mh.edet);
        up(st->m_epix, mh.epix);
        up(st->m_ecos, mh.ecos);
        up(st->m_egeom, mh.egeom);
        up(st->m_esb, mh.esb);
        up(st->m_ese, mh.ese);
        up(st->m_lvox, mh.lvox);
        up(st->m_llen, mh.llen);
        st->m_events = mh.evert.size();
        st->m_eval.alloc(std::max<size_t>(mh.evert.size(), 1));
        mat_ref_tables(c, st.get());
    }
    return st;
}

void copy_out(prc_gpu_ctx* c, double* host, const double* dev, size_t n) {
    if (host && n) CK(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

}  // namespace

// =============================================================================== C ABI
PRC_EXPORT const char* prc_gpu_version(void) { return "pathrec-b200 0.1 (sm_100a)"; }
PRC_EXPORT const char* prc_gpu_last_error(void) { return g_last_error.c_str(); }

static int ctx_init(prc_gpu_ctx* c, int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Err(PRC_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) throw Err(PRC_ERR_INVALID, "device index out of range");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw Err(PRC_ERR_CUDA, "pathrec-b200 requires an sm_100 (B200) device");
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& ev : c->ev) CK(cudaEventCreate(&ev));
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_ctx_create(int device, prc_gpu_ctx** out) {
    if (!out) return fail(PRC_ERR_INVALID, "prc_gpu_ctx_create: null argument");
    ABI_TRY
    auto c = std::make_unique<prc_gpu_ctx>();
    ctx_init(c.get(), device);
    *out = c.release();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_nccl_unique_id(void* out128) {
    if (!out128) return fail(PRC_ERR_INVALID, "prc_gpu_nccl_unique_id: null argument");
    ABI_TRY
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof id);
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_shard_range(uint64_t n, int rank, int world, uint64_t* lo, uint64_t* hi) {
    if (!lo || !hi) return fail(PRC_ERR_INVALID, "prc_gpu_shard_range: null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(PRC_ERR_INVALID, "rank/world out of range");
    unsigned long long a, b;
    shard_range(n, rank, world, &a, &b);
    *lo = a;
    *hi = b;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_ctx_create_rank(int device, int rank, int world, const void* nccl_id,
                                       prc_gpu_ctx** out) {
    if (!out) return fail(PRC_ERR_INVALID, "prc_gpu_ctx_create_rank: null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(PRC_ERR_INVALID, "rank/world out of range");
    ABI_TRY
    auto c = std::make_unique<prc_gpu_ctx>();
    ctx_init(c.get(), device);
    c->rank = rank;
    c->world = world;
    if (nccl_id) {  // world 1 with an id builds a 1-rank communicator (exercises NCCL)
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        NK(ncclCommInitRank(&c->comm, world, id, rank));
    }
    *out = c.release();
    ABI_CATCH
}

PRC_EXPORT void prc_gpu_ctx_destroy(prc_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (prc_gpu_store* st : ctx->stores) st->ctx = nullptr;  // still freeable by the caller
    const int dev = ctx->device;
    delete ctx;
    cache_release(dev);
}

PRC_EXPORT int prc_gpu_ctx_set_option(prc_gpu_ctx* ctx, const char* key, int64_t value) {
    if (!ctx || !key) return fail(PRC_ERR_INVALID, "prc_gpu_ctx_set_option: null argument");
    const std::string k(key);
    if (k == "mode") {
        if (value != 0 && value != 1) return fail(PRC_ERR_CONFIG, "mode must be 0 (wavefront) or 1 (path)");
        ctx->mode = (int)value;
    } else if (k == "spread") {  // 0: by vertex density
        if (value < 0 || value > 4096) return fail(PRC_ERR_CONFIG, "spread must be in 0..4096");
        ctx->spread = (int)value;
    } else if (k == "per_species") {
        ctx->opt_per_species = value ? 1 : 0;
    } else if (k == "packet") {
        if (value < 1 || value > 4) return fail(PRC_ERR_CONFIG, "packet must be in 1..4");
        ctx->packet = (int)value;
    } else if (k == "grad_copies") {
        if (value < 0 || value > 64) return fail(PRC_ERR_CONFIG, "grad_copies must be in 0..64");
        ctx->grad_copies_max = (int)value;
    } else if (k == "nvls") {  // applied at the next scene upload; 2: fold without multicast (1 rank)
        if (value < 0 || value > 2) return fail(PRC_ERR_CONFIG, "nvls must be 0, 1 or 2");
        ctx->nvls_enable = value != 0;
        ctx->nvls_emulate = value == 2;
    } else if (k == "events") {
        ctx->evc_enable = value != 0;
    } else if (k == "pad") {
        ctx->pad_enable = value != 0;
        ctx->dsc.pad_walk = ctx->pad_ok && ctx->pad_enable ? 1 : 0;
    } else {
        return fail(PRC_ERR_CONFIG, "unknown option " + k);
    }
    ++ctx->fwd_gen;  // a cached forward was computed under the old options
    ++ctx->geo_gen;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_release_cached_memory(void) {
    cache_release(-1);
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_ctx_rank(const prc_gpu_ctx* ctx, int* rank, int* world) {
    if (!ctx || !rank || !world) return fail(PRC_ERR_INVALID, "prc_gpu_ctx_rank: null argument");
    *rank = ctx->rank;
    *world = ctx->world;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_scene_upload(prc_gpu_ctx* ctx, const prc_scene_desc* scene) {
    if (!ctx || !scene) return fail(PRC_ERR_INVALID, "prc_gpu_scene_upload: null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    upload_scene(ctx, scene);
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_scene_voxel_count(const prc_gpu_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return fail(PRC_ERR_INVALID, "null argument");
    *out = (uint64_t)ctx->V;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_scene_pixel_count(const prc_gpu_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return fail(PRC_ERR_INVALID, "null argument");
    *out = (uint64_t)ctx->n_pix;
    return PRC_OK;
}

// Sum of a per-rank counter over the communicator (exact below 2^53).
static uint64_t global_count(prc_gpu_ctx* ctx, uint64_t local) {
    double t = (double)local;
    if (ctx->comm) {
        CK(cudaMemcpy(ctx->loss.p, &t, 8, cudaMemcpyHostToDevice));
        ctx->allreduce(ctx->loss.p, 1);
        ctx->sync();
        CK(cudaMemcpy(&t, ctx->loss.p, 8, cudaMemcpyDeviceToHost));
    }
    return (uint64_t)t;
}

PRC_EXPORT int prc_gpu_render(prc_gpu_ctx* ctx, const prc_gpu_render_opts* opts,
                              const prc_gpu_params* params, double* images_out,
                              uint64_t* truncated_out, prc_gpu_store** store_out) {
    if (!ctx || !opts) return fail(PRC_ERR_INVALID, "prc_gpu_render: null argument");
    if (opts->n_paths == 0) return fail(PRC_ERR_CONFIG, "prc_gpu_render: n_paths must be >= 1");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    const DScene& s = ctx->dsc;
    // bind_params: sampling species values (inverse.cpp:144-150)
    Resolved r = resolve_params(ctx, params, nullptr);
    const double* beta_u = (s.unknown >= 0 && params && params->beta) ? ctx->param_beta.p : nullptr;
    CK(launch_set_species(s.n_species, ctx->V, s.unknown, ctx->scene_sp.p, beta_u, ctx->trace_sp.p,
                          ctx->stream, &ctx->launches));
    if (params && params->species_beta)
        for (int j = 0; j < s.n_species; ++j)
            if (params->species_beta[j])
                CK(cudaMemcpyAsync(ctx->trace_sp.p + (size_t)j * ctx->V, r.src[j],
                                   (size_t)ctx->V * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    auto st = trace_store(ctx, opts, ctx->trace_sp.p, r.kappa, r.gamma, nullptr, true);
    if (!images_out) {  // nobody reads the fresh image: trace only (the resample of reconstruct)
        ctx->sync();
        if (truncated_out) *truncated_out = global_count(ctx, st->truncated);
        if (store_out) *store_out = st.release();
        return PRC_OK;
    }
    // fresh evaluation at the sampling point (render's evaluate_store, transport.cpp:432-435)
    Resolved rr;
    for (int j = 0; j < s.n_species; ++j) rr.src[j] = ctx->trace_sp.p + (size_t)j * ctx->V;
    rr.kappa = r.kappa;
    rr.gamma = r.gamma;
    EvalRun er;
    er.deterministic = true;  // render() is bit-reproducible (transport.hpp:171-173)
    run_eval(ctx, st.get(), rr, er, nullptr);
    CK(launch_scale(ctx->images.p, ctx->n_pix, 1.0 / (double)opts->n_paths, ctx->stream, &ctx->launches));
    copy_out(ctx, images_out, ctx->images.p, (size_t)ctx->n_pix);
    ctx->sync();
    if (truncated_out) *truncated_out = global_count(ctx, st->truncated);
    if (store_out) *store_out = st.release();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_sort_by_size(prc_gpu_ctx* ctx, prc_gpu_store* store) {
    if (!ctx || !store) return fail(PRC_ERR_INVALID, "prc_gpu_sort_by_size: null argument");
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_sort_by_size: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    sort_store(ctx, store);
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_info_get(const prc_gpu_store* st, prc_gpu_store_info* o) {
    if (!st || !o) return fail(PRC_ERR_INVALID, "prc_gpu_store_info_get: null argument");
    o->n_paths = st->n;
    o->n_paths_global = st->n_global;
    o->stream_base = st->stream_base;
    o->segments = st->segments;
    o->vertices = st->n_rec;
    o->interaction_vertices = st->n_iv;
    o->truncated = st->truncated;
    o->seed = st->seed;
    o->generation = st->generation;
    o->sorted = st->sorted ? 1 : 0;
    o->max_size = st->max_B;
    o->device_bytes = st->device_bytes();
    o->materialized = st->mat ? 1 : 0;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_store_streams(const prc_gpu_store* st, uint64_t* out) {
    if (!st || !out) return fail(PRC_ERR_INVALID, "prc_gpu_store_streams: null argument");
    if (!st->ctx) return fail(PRC_ERR_INVALID, "prc_gpu_store_streams: the store's context was destroyed");
    ABI_TRY
    auto _lk = begin(st->ctx);
    if (st->n) CK(cudaMemcpy(out, st->stream.p, st->n * 8, cudaMemcpyDeviceToHost));
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_sizes(const prc_gpu_store* st, uint32_t* out) {
    if (!st || !out) return fail(PRC_ERR_INVALID, "prc_gpu_store_sizes: null argument");
    if (!st->ctx) return fail(PRC_ERR_INVALID, "prc_gpu_store_sizes: the store's context was destroyed");
    ABI_TRY
    auto _lk = begin(st->ctx);
    if (st->n) CK(cudaMemcpy(out, st->B.p, st->n * 4, cudaMemcpyDeviceToHost));
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_export_pstr(prc_gpu_ctx* ctx, const prc_gpu_store* store,
                                         const char* path) {
    if (!ctx || !store || !path) return fail(PRC_ERR_INVALID, "prc_gpu_store_export_pstr: null argument");
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_store_export_pstr: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    store_for_scene(ctx, const_cast<prc_gpu_store*>(store));
    export_pstr(ctx, const_cast<prc_gpu_store*>(store), path);
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_import_pstr(prc_gpu_ctx* ctx, const char* path, prc_gpu_store** out) {
    if (!ctx || !path || !out) return fail(PRC_ERR_INVALID, "prc_gpu_store_import_pstr: null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    *out = import_pstr(ctx, path, false).release();
    ++ctx->fwd_gen;
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_import_pstr_ex(prc_gpu_ctx* ctx, const char* path, int flags, prc_gpu_store** out) {
    if (!ctx || !path || !out) return fail(PRC_ERR_INVALID, "prc_gpu_store_import_pstr_ex: null argument");
    if (flags & ~PRC_IMPORT_MATERIALIZE) return fail(PRC_ERR_CONFIG, "prc_gpu_store_import_pstr_ex: unknown flags");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    *out = import_pstr(ctx, path, (flags & PRC_IMPORT_MATERIALIZE) != 0).release();
    ++ctx->fwd_gen;
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_set_generation(prc_gpu_store* st, uint64_t g) {
    if (!st) return fail(PRC_ERR_INVALID, "null store");
    st->generation = g;
    return PRC_OK;
}

PRC_EXPORT void prc_gpu_store_free(prc_gpu_store* st) {
    if (!st) return;
    cudaSetDevice(st->device);
    if (st->ctx) ++st->ctx->fwd_gen;  // a later store may reuse this address
    delete st;
}

static double mean_correction(prc_gpu_ctx* c, prc_gpu_store* st, const EvalRun& er, double* per_path = nullptr);

PRC_EXPORT int prc_gpu_evaluate(prc_gpu_ctx* ctx, const prc_gpu_store* store,
                                const prc_gpu_params* params, const prc_gpu_eval_opts* opts,
                                prc_gpu_eval_result* res) {
    if (!ctx || !store || !res) return fail(PRC_ERR_INVALID, "prc_gpu_evaluate: null argument");
    const int flags = opts ? opts->flags : PRC_EVAL_NORMALIZE;
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_evaluate: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    auto* st = const_cast<prc_gpu_store*>(store);
    store_for_scene(ctx, st);
    EvalRun er;
    er.want_grad = (flags & PRC_EVAL_WANT_GRAD) != 0;
    er.per_species = (flags & PRC_EVAL_PER_SPECIES) != 0;
    er.legacy = (flags & PRC_EVAL_LEGACY_SCORE) != 0;
    er.deterministic = (flags & PRC_EVAL_DETERMINISTIC) != 0;
    const double scale = (flags & PRC_EVAL_NORMALIZE) && st->n_global ? 1.0 / (double)st->n_global : 1.0;
    er.grad_scale = scale;
    const unsigned long long key = params_key(ctx, params, st, flags);
    const bool reuse = er.want_grad && ctx->last_fwd_store == st && ctx->last_fwd_gen == ctx->fwd_gen &&
                       ctx->last_fwd_key == key;
    if (er.want_grad && opts && opts->pixel_weights) {
        CK(cudaMemcpyAsync(ctx->weights.p, opts->pixel_weights, (size_t)ctx->n_pix * 8,
                           cudaMemcpyHostToDevice, ctx->stream));
        er.weights = ctx->weights.p;
    }
    unsigned long long cl;
    if (reuse) {  // images, event cache, prep fields and Phong values are still current
        cudaStream_t q = ctx->stream;
        for (int i = 0; i < 4; ++i) CK(cudaEventRecord(ctx->ev[i], q));
        EvalArgs ea = eval_args(ctx, st, er, ctx->phong.p);
        run_gradient(ctx, st, ea, er.per_species ? ctx->dsc.n_species : 1, scale);
        cl = ctx->last_fwd_clamps;
    } else {
        Resolved r = resolve_params(ctx, params, st);
        cl = run_eval(ctx, st, r, er, nullptr);
        CK(launch_scale(ctx->images.p, ctx->n_pix, scale, ctx->stream, &ctx->launches));
        ctx->last_fwd_store = st;
        ctx->last_fwd_gen = ctx->fwd_gen;
        ctx->last_fwd_key = key;
    }
    copy_out(ctx, res->images, ctx->images.p, (size_t)ctx->n_pix);
    const DScene& s = ctx->dsc;
    const int n_out = er.per_species ? s.n_species : 1;
    const bool grad_beta_out = er.want_grad && s.has_medium && (s.unknown >= 0 || er.per_species) && ctx->grad_res;
    res->grad_kappa = res->grad_gamma = 0.0;
    if (er.want_grad) {
        if (grad_beta_out) copy_out(ctx, res->grad_beta, ctx->grad_res, (size_t)n_out * ctx->V);
        double gp[2] = {0, 0};
        CK(cudaMemcpyAsync(gp, ctx->g_phong.p, sizeof gp, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaEventRecord(ctx->ev[5], ctx->stream));
        record_timings(ctx);
        res->grad_kappa = gp[0] * scale;
        res->grad_gamma = gp[1] * scale;
    } else {
        CK(cudaEventRecord(ctx->ev[5], ctx->stream));
        record_timings(ctx);
    }
    ctx->last_fwd_clamps = cl;
    res->clamp_events = cl;
    res->mean_correction = 1.0;
    if (flags & PRC_EVAL_SELF_NORMALIZE) {
        // pathstore.cpp:334-359: scale /= mean correction factor over the store; applied to
        // the returned copies (the device images stay those of the cached forward)
        const double mean = mean_correction(ctx, st, er);
        res->mean_correction = mean;
        // a detached shard (world > 1, no communicator) holds a partial sum only: it returns
        // its partial mean (shard sum / global count) and leaves the division to the caller
        const bool detached = ctx->world > 1 && !ctx->comm;
        if (mean > 0.0 && !detached) {
            const double inv = 1.0 / mean;
            if (res->images)
                for (long long i = 0; i < ctx->n_pix; ++i) res->images[i] *= inv;
            if (grad_beta_out && res->grad_beta)
                for (long long i = 0; i < (long long)n_out * ctx->V; ++i) res->grad_beta[i] *= inv;
            res->grad_kappa *= inv;
            res->grad_gamma *= inv;
        }
    }
    ABI_CATCH
}

// Mean correction_factor over the store (all ranks) under the context's current
// evaluation fields (EvalOptions::self_normalize, pathstore.cpp:334-359).
static double mean_correction(prc_gpu_ctx* c, prc_gpu_store* st, const EvalRun& er, double* per_path) {
    cudaStream_t q = c->stream;
    c->selfn.grow(1);
    CK(cudaMemsetAsync(c->selfn.p, 0, sizeof(double), q));
    CK(cudaMemsetAsync(c->err.p, 0, sizeof(int), q));
    if (st->mat) {
        CK(launch_mat_correction(c->dsc, st->mat_view(), st->m_ctx, c->selfn.p, c->err.p, per_path, q,
                                 &c->launches));
    } else {
        // the padded dbeta table is refreshed by mode-0 forwards only (run_forward)
        if (c->mode != 0 && c->dsc.pad_walk)
            CK(launch_pad_tables(c->dsc, c->bt_tot.p, c->dbeta.p, c->bt_pad.p, c->db_pad.p, q, &c->launches));
        const EvalArgs ea = eval_args(c, st, er, c->phong.p);
        CK(launch_correction(c->dsc, st->view(), ea, c->selfn.p, c->err.p, per_path, q, &c->launches));
    }
    c->allreduce(c->selfn.p, 1);
    double sum = 0.0;
    int errf = 0;
    CK(cudaMemcpyAsync(&sum, c->selfn.p, sizeof sum, cudaMemcpyDeviceToHost, q));
    CK(cudaMemcpyAsync(&errf, c->err.p, sizeof errf, cudaMemcpyDeviceToHost, q));
    c->sync();
    if (errf) throw Err(PRC_ERR_NUMERIC, "correction_factor: zero reference extinction at a vertex");
    return st->n_global ? sum / (double)st->n_global : 1.0;
}

PRC_EXPORT int prc_gpu_correction_factors(prc_gpu_ctx* ctx, const prc_gpu_store* store,
                                          const prc_gpu_params* params_t, double* out) {
    if (!ctx || !store || !out) return fail(PRC_ERR_INVALID, "prc_gpu_correction_factors: null argument");
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_correction_factors: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    auto* st = const_cast<prc_gpu_store*>(store);
    store_for_scene(ctx, st);
    EvalRun er;
    const Resolved r = resolve_params(ctx, params_t, st);
    run_eval(ctx, st, r, er, nullptr);  // the evaluation fields under params_t
    DBuf<double> pp;
    pp.alloc(std::max<unsigned long long>(st->n, 1));
    mean_correction(ctx, st, er, pp.p);
    copy_out(ctx, out, pp.p, (size_t)st->n);
    ctx->sync();
    ABI_CATCH
}

// ------------------------------------------------------------------ Algorithm 2 (device)
static void opt_init(prc_gpu_ctx* c, const prc_gpu_params* initial, const double* gt,
                     const prc_gpu_adam_config* adam) {
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    if (s.unknown >= 0) {
        c->opt_mode = 0;
        c->opt_n = c->V;
        c->opt_x.alloc((size_t)c->V);
        if (initial && initial->beta) {
            if ((long long)initial->n_beta != c->V) throw Err(PRC_ERR_CONFIG, "initial beta size != voxel count");
            CK(cudaMemcpyAsync(c->opt_x.p, initial->beta, (size_t)c->V * 8, cudaMemcpyHostToDevice, q));
        } else {
            CK(cudaMemcpyAsync(c->opt_x.p, c->scene_sp.p + (size_t)s.unknown * c->V, (size_t)c->V * 8,
                               cudaMemcpyDeviceToDevice, q));
        }
    } else if (s.target >= 0) {
        c->opt_mode = 1;
        c->opt_n = 2;
        c->opt_x.alloc(2);
        const double kg[2] = {initial ? initial->kappa_s : c->scene_kappa,
                              initial ? initial->gamma : c->scene_gamma};
        CK(cudaMemcpyAsync(c->opt_x.p, kg, sizeof kg, cudaMemcpyHostToDevice, q));
    } else {
        throw Err(PRC_ERR_CONFIG, "scene declares no unknown species or target surface");
    }
    c->opt_m1.alloc((size_t)c->opt_n);
    c->opt_m2.alloc((size_t)c->opt_n);
    CK(cudaMemsetAsync(c->opt_m1.p, 0, c->opt_m1.bytes(), q));
    CK(cudaMemsetAsync(c->opt_m2.p, 0, c->opt_m2.bytes(), q));
    c->opt_gt.alloc((size_t)c->n_pix);
    CK(cudaMemcpyAsync(c->opt_gt.p, gt, (size_t)c->n_pix * 8, cudaMemcpyHostToDevice, q));
    c->adam = adam ? *adam : prc_gpu_adam_config{1e7, 0.9, 0.999, 1e-8, 1, nullptr, 0};
    c->n_step_scale = adam && adam->step_scale ? adam->n_step_scale : 0;
    c->opt_step_scale.alloc((size_t)std::max(1, c->n_step_scale));
    if (c->n_step_scale)
        CK(cudaMemcpyAsync(c->opt_step_scale.p, adam->step_scale, (size_t)c->n_step_scale * 8,
                           cudaMemcpyHostToDevice, q));
    c->opt_t = 0;
    c->sync();
    c->opt_ready = true;
}

// Current sampling species values (device fp64) for a resample under the iterate.
static void bind_trace_species(prc_gpu_ctx* c) {
    const DScene& s = c->dsc;
    CK(launch_set_species(s.n_species, c->V, s.unknown, c->scene_sp.p,
                          c->opt_mode == 0 ? c->opt_x.p : nullptr, c->trace_sp.p, c->stream,
                          &c->launches));
}

// adam_step (inverse.cpp:41-67) on the device-resident unknowns with gradient g (device,
// opt_n values): the same operations in the same order, so the update is the reference's
// bit for bit (bias corrections c1, c2 from std::pow on the host, as there).
static void adam_update(prc_gpu_ctx* c, const double* g) {
    ++c->opt_t;
    const double c1 = 1.0 - std::pow(c->adam.eta1, (double)c->opt_t);
    const double c2 = 1.0 - std::pow(c->adam.eta2, (double)c->opt_t);
    CK(launch_adam(c->opt_x.p, c->opt_m1.p, c->opt_m2.p, g, c->opt_n, c->adam.alpha, c->adam.eta1,
                   c->adam.eta2, c->adam.eps_guard, c1, c2, c->opt_step_scale.p, c->n_step_scale,
                   c->opt_mode == 0 ? (c->adam.project_nonneg ? 0 : 2) : 1, c->stream, &c->launches));
}

static double opt_step(prc_gpu_ctx* c, prc_gpu_store* st) {
    const DScene& s = c->dsc;
    cudaStream_t q = c->stream;
    Resolved r;
    for (int j = 0; j < s.n_species; ++j) r.src[j] = c->scene_sp.p + (size_t)j * c->V;
    const double* phong_dev = nullptr;
    if (c->opt_mode == 0) {
        r.src[s.unknown] = c->opt_x.p;
        r.kappa = c->scene_kappa;
        r.gamma = c->scene_gamma;
    } else {
        phong_dev = c->opt_x.p;
    }
    EvalRun er;
    EvalArgs ea;
    run_forward(c, st, r, er, phong_dev, ea);  // K3 + K4 (+ image allreduce)
    const double scale = 1.0 / (double)st->n_global;
    CK(launch_scale(c->images.p, c->n_pix, scale, q, &c->launches));
    CK(cudaMemsetAsync(c->loss.p, 0, 8, q));
    CK(launch_loss_residual(c->images.p, c->opt_gt.p, c->n_pix, c->weights.p, c->loss.p, q, &c->launches));
    ea.weights = c->weights.p;  // K5 with residual weights (+ gradient allreduce)
    ea.per_species = c->opt_per_species && s.has_medium ? 1 : 0;
    ea.do_beta = s.has_medium && (s.unknown >= 0 || ea.per_species) ? 1 : 0;
    // per-type mode (config (c)): grad_j = g_span + g_vert[j] for every species j; the
    // optimiser updates the unknown species' slice
    run_gradient(c, st, ea, ea.per_species ? s.n_species : 1, scale);
    const double* g;
    if (c->opt_mode == 0) {
        g = c->grad_res + (ea.per_species ? (size_t)s.unknown * c->V : 0);
    } else {
        CK(launch_scale(c->g_phong.p, 2, scale, q, &c->launches));
        g = c->g_phong.p;
    }
    adam_update(c, g);
    double loss = 0.0;
    CK(cudaMemcpyAsync(&loss, c->loss.p, 8, cudaMemcpyDeviceToHost, q));
    CK(cudaEventRecord(c->ev[5], q));
    record_timings(c);
    if (!std::isfinite(loss))
        throw Err(PRC_ERR_NUMERIC, "reconstruct: non-finite loss at iteration " + std::to_string(c->opt_t - 1));
    return loss;
}

PRC_EXPORT int prc_gpu_opt_init(prc_gpu_ctx* ctx, const prc_gpu_params* initial,
                                const double* gt_images, const prc_gpu_adam_config* adam) {
    if (!ctx || !gt_images) return fail(PRC_ERR_INVALID, "prc_gpu_opt_init: null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    opt_init(ctx, initial, gt_images, adam);
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_opt_step(prc_gpu_ctx* ctx, const prc_gpu_store* store, double* loss_out) {
    if (!ctx || !store) return fail(PRC_ERR_INVALID, "prc_gpu_opt_step: null argument");
    if (!ctx->opt_ready) return fail(PRC_ERR_INVALID, "prc_gpu_opt_step: optimizer not initialised");
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_opt_step: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    store_for_scene(ctx, const_cast<prc_gpu_store*>(store));
    const double l = opt_step(ctx, const_cast<prc_gpu_store*>(store));
    if (loss_out) *loss_out = l;
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_opt_adam_step(prc_gpu_ctx* ctx, const double* grad, uint64_t n) {
    if (!ctx || !grad) return fail(PRC_ERR_INVALID, "prc_gpu_opt_adam_step: null argument");
    if (!ctx->opt_ready) return fail(PRC_ERR_INVALID, "prc_gpu_opt_adam_step: optimizer not initialised");
    if ((long long)n != ctx->opt_n) return fail(PRC_ERR_CONFIG, "prc_gpu_opt_adam_step: gradient size != unknowns");
    ABI_TRY
    auto _lk = begin(ctx);
    DBuf<double> g;
    g.alloc((size_t)n);
    CK(cudaMemcpyAsync(g.p, grad, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    adam_update(ctx, g.p);
    ctx->sync();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_opt_params(prc_gpu_ctx* ctx, double* beta_out, double* kappa_s, double* gamma) {
    if (!ctx) return fail(PRC_ERR_INVALID, "prc_gpu_opt_params: null argument");
    if (!ctx->opt_ready) return fail(PRC_ERR_INVALID, "optimizer not initialised");
    ABI_TRY
    auto _lk = begin(ctx);
    if (ctx->opt_mode == 0) {
        copy_out(ctx, beta_out, ctx->opt_x.p, (size_t)ctx->V);
        if (kappa_s) *kappa_s = ctx->scene_kappa;
        if (gamma) *gamma = ctx->scene_gamma;
    } else {
        double kg[2];
        CK(cudaMemcpyAsync(kg, ctx->opt_x.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        if (kappa_s) *kappa_s = kg[0];
        if (gamma) *gamma = kg[1];
    }
    ctx->sync();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_opt_images(prc_gpu_ctx* ctx, double* images_out) {
    if (!ctx || !images_out) return fail(PRC_ERR_INVALID, "prc_gpu_opt_images: null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    copy_out(ctx, images_out, ctx->images.p, (size_t)ctx->n_pix);
    ctx->sync();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_reconstruct(prc_gpu_ctx* ctx, const prc_gpu_params* initial,
                                   const double* gt_images, const prc_gpu_adam_config* adam,
                                   const prc_gpu_reconstruct_opts* o, double* loss_history,
                                   uint64_t* phases_out) {
    if (!ctx || !gt_images || !o) return fail(PRC_ERR_INVALID, "prc_gpu_reconstruct: null argument");
    if (o->n_paths == 0) return fail(PRC_ERR_CONFIG, "reconstruct: n_paths must be >= 1");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    opt_init(ctx, initial, gt_images, adam);
    const int n_r = std::max(1, o->recycle_period);
    std::unique_ptr<prc_gpu_store> store;
    uint64_t phases = 0;
    for (int t = 0; t < o->max_iterations; ++t) {
        if (t % n_r == 0) {  // resample + sort (inverse.cpp:175-204)
            store.reset();
            bind_trace_species(ctx);
            double kg[2] = {ctx->scene_kappa, ctx->scene_gamma};
            if (ctx->opt_mode == 1) {
                CK(cudaMemcpyAsync(kg, ctx->opt_x.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
                ctx->sync();
            }
            prc_gpu_render_opts ro{o->n_paths, o->seed + 0x9E3779B97F4A7C15ull * (phases + 1),
                                   o->max_bounces, -1};
            store = trace_store(ctx, &ro, ctx->trace_sp.p, kg[0], kg[1], nullptr, true);
            sort_store(ctx, store.get());
            store->generation = (uint64_t)t;
            ++phases;
        }
        const double l = opt_step(ctx, store.get());
        if (loss_history) loss_history[t] = l;
    }
    if (phases_out) *phases_out = phases;
    ABI_CATCH
}

// ----------------------------------------------------------- Algorithm-2 driver (§8(f) 1)
// Host utilities in the reference's arithmetic order (inverse.cpp:103-133, io.cpp:32-76,
// 147-155); the carve test runs on the device.

static void downsample(int n_img, const int* rows, const int* cols, const double* in, int ro, int co,
                       double* out) {  // downsample_images, inverse.cpp:116-133
    size_t ii = 0, oo = 0;
    for (int k = 0; k < n_img; ++k) {
        const int r0 = rows[k], c0 = cols[k];
        double* o = out + oo;
        if (r0 == ro && c0 == co) {
            std::memcpy(o, in + ii, (size_t)r0 * c0 * 8);
        } else {
            std::fill(o, o + (size_t)ro * co, 0.0);
            for (int r = 0; r < r0; ++r) {
                const int cr = r * ro / r0;
                for (int c = 0; c < c0; ++c) o[(size_t)cr * co + (size_t)(c * co / c0)] += in[ii + (size_t)r * c0 + c];
            }
        }
        ii += (size_t)r0 * c0;
        oo += (size_t)ro * co;
    }
}

static void metrics_host(const double* e, const double* t, uint64_t n, double* eps, double* delta) {
    double diff = 0.0, nt = 0.0, ne = 0.0;  // inverse.cpp:103-114
    for (uint64_t i = 0; i < n; ++i) {
        diff += std::abs(t[i] - e[i]);
        nt += std::abs(t[i]);
        ne += std::abs(e[i]);
    }
    if (nt == 0.0) throw Err(PRC_ERR_CONFIG, "metrics: zero-norm truth");
    *eps = diff / nt;
    *delta = (nt - ne) / nt;
}

template <class T>
static void put_raw(std::ofstream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

static void save_grid_host(const std::string& path, const int dims[3], const double org[3], const double vs[3],
                           int unit, const double* values) {  // save_grid, io.cpp:59-76
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Err(PRC_ERR_IO, "save_grid: cannot open " + path);
    os.write("VGRD", 4);
    put_raw<uint32_t>(os, 1u);
    for (int a = 0; a < 3; ++a) put_raw<uint32_t>(os, (uint32_t)dims[a]);
    for (int a = 0; a < 3; ++a) put_raw<double>(os, org[a]);
    for (int a = 0; a < 3; ++a) put_raw<double>(os, vs[a]);
    put_raw<uint8_t>(os, (uint8_t)unit);
    const size_t n = (size_t)dims[0] * dims[1] * dims[2];
    for (size_t i = 0; i < n; ++i) put_raw<float>(os, (float)values[i]);
    if (!os) throw Err(PRC_ERR_IO, "save_grid: write failure on " + path);
}

static void save_csv_host(const std::vector<prc_gpu_iteration_log>& rows, const std::string& path) {
    std::ofstream os(path);  // save_csv, io.cpp:147-155
    if (!os) throw Err(PRC_ERR_IO, "save_csv: cannot open " + path);
    os << "iter,time_s,loss,eps,delta,stage\r\n";
    os.precision(17);
    for (const auto& r : rows)
        os << r.iter << "," << r.time_s << "," << r.loss << "," << r.eps << "," << r.delta << "," << r.stage << "\r\n";
}

// Re-finalizes every detector at rows[k] x cols[k] and resizes the pixel buffers.
static void set_resolution(prc_gpu_ctx* c, const std::vector<int>& rows, const std::vector<int>& cols) {
    const long long n_pix = finalize_detectors(c->dsc, c->det_desc.data(), (int)c->det_desc.size(), rows.data(),
                                               cols.data(), c->det_finalized);
    c->n_pix = n_pix;
    c->images.alloc((size_t)n_pix);
    c->weights.alloc((size_t)n_pix);
    c->opt_gt.alloc((size_t)n_pix);
    nvls_setup(c);
    ++c->geo_gen;  // pixel_of changes with the resolution
    ++c->fwd_gen;
}

PRC_EXPORT int prc_gpu_reconstruct_schedule(prc_gpu_ctx* ctx, const prc_gpu_params* initial,
                                            const double* gt_images, const prc_gpu_adam_config* adam,
                                            const prc_gpu_schedule* sch, prc_gpu_iteration_log* history,
                                            uint64_t* phases_out, uint64_t* truncated_out) {
    if (!ctx || !gt_images || !sch) return fail(PRC_ERR_INVALID, "prc_gpu_reconstruct_schedule: null argument");
    if (sch->n_stages < 1 || !sch->stages)
        return fail(PRC_ERR_CONFIG, "reconstruct: schedule needs at least one stage");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    const auto t_start = std::chrono::steady_clock::now();
    const int n_det = ctx->dsc.n_det;
    std::vector<int> base_rows(n_det), base_cols(n_det);
    for (int k = 0; k < n_det; ++k) {
        base_rows[k] = ctx->dsc.det[k].rows;
        base_cols[k] = ctx->dsc.det[k].cols;
    }
    const std::vector<double> gt_full(gt_images, gt_images + ctx->n_pix);
    struct Restore {  // the scene's own resolution and ground truth come back on every exit
        prc_gpu_ctx* c;
        const std::vector<int>& r;
        const std::vector<int>& k;
        const std::vector<double>& gt;
        ~Restore() {
            try {
                set_resolution(c, r, k);
                CK(cudaMemcpyAsync(c->opt_gt.p, gt.data(), gt.size() * 8, cudaMemcpyHostToDevice, c->stream));
                c->sync();
            } catch (...) {
                c->opt_ready = false;
            }
        }
    } restore{ctx, base_rows, base_cols, gt_full};
    opt_init(ctx, initial, gt_full.data(), adam);
    std::vector<double> truth;
    if (sch->truth) {
        if (ctx->opt_mode == 0) {
            if (!sch->truth->beta || (long long)sch->truth->n_beta != ctx->V)
                throw Err(PRC_ERR_CONFIG, "truth beta size != voxel count");
            truth.assign(sch->truth->beta, sch->truth->beta + ctx->V);
        } else {
            truth = {sch->truth->kappa_s, sch->truth->gamma};
        }
    }
    const bool ckpt = sch->checkpoint_dir && sch->checkpoint_dir[0] && sch->checkpoint_every > 0;
    const bool want_x = !truth.empty() || ckpt;
    std::vector<double> x_host;
    std::vector<prc_gpu_iteration_log> rows;
    std::vector<double> loss_hist;
    const int n_r = std::max(1, sch->recycle_period);
    // inverse.cpp:249-258 takes the window as given (0 advances at the first check); a
    // negative window would index past the loss history there, so it is rejected here
    if (sch->saturation_window < 0) throw Err(PRC_ERR_CONFIG, "reconstruct: saturation_window must be >= 0");
    const int w = sch->saturation_window;
    const double rel = sch->saturation_rel_improvement;
    int stage = 0, applied = -1, pending = 0, stage_start = 0;
    uint64_t phases = 0, truncated = 0;
    std::vector<int> cur_rows = base_rows, cur_cols = base_cols;
    std::unique_ptr<prc_gpu_store> store;
    for (int t = 0; t < sch->max_iterations; ++t) {
        if (t % n_r == 0) {  // resample boundary (inverse.cpp:175-205)
            if (pending != applied) {
                stage = pending;
                applied = stage;
                stage_start = t;
                const prc_gpu_stage& st = sch->stages[stage];
                for (int k = 0; k < n_det; ++k) {
                    if (st.rows > 0) cur_rows[k] = st.rows;
                    if (st.cols > 0) cur_cols[k] = st.cols;
                }
                store.reset();
                set_resolution(ctx, cur_rows, cur_cols);
                std::vector<double> g((size_t)ctx->n_pix);
                downsample(n_det, base_rows.data(), base_cols.data(), gt_full.data(), cur_rows[0], cur_cols[0],
                           g.data());
                if ((long long)g.size() != ctx->n_pix)
                    throw Err(PRC_ERR_CONFIG, "reconstruct: stage resolution must be the same for every detector");
                CK(cudaMemcpyAsync(ctx->opt_gt.p, g.data(), g.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            }
            store.reset();
            bind_trace_species(ctx);
            double kg[2] = {ctx->scene_kappa, ctx->scene_gamma};
            if (ctx->opt_mode == 1) {
                CK(cudaMemcpyAsync(kg, ctx->opt_x.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
                ctx->sync();
            }
            const uint64_t n_paths = sch->stages[stage].n_paths;
            if (n_paths == 0) throw Err(PRC_ERR_CONFIG, "reconstruct: stage n_paths must be >= 1");
            prc_gpu_render_opts ro{n_paths, sch->seed + 0x9E3779B97F4A7C15ull * (phases + 1),
                                   sch->max_bounces > 0 ? sch->max_bounces : 500, -1};
            store = trace_store(ctx, &ro, ctx->trace_sp.p, kg[0], kg[1], nullptr, true);
            truncated += global_count(ctx, store->truncated);
            sort_store(ctx, store.get());
            store->generation = (uint64_t)t;
            ++phases;
        }
        if (want_x) {  // the unknowns before this iteration's update (inverse.cpp:215-236)
            x_host.resize((size_t)ctx->opt_n);
            CK(cudaMemcpyAsync(x_host.data(), ctx->opt_x.p, x_host.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
            ctx->sync();
        }
        const double l = opt_step(ctx, store.get());  // loss, gradient, ADAM
        loss_hist.push_back(l);
        prc_gpu_iteration_log row{};
        row.iter = t;
        row.time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
        row.loss = l;
        row.stage = stage;
        if (!truth.empty()) metrics_host(x_host.data(), truth.data(), truth.size(), &row.eps, &row.delta);
        rows.push_back(row);
        if (history) history[t] = row;
        if (sch->on_iteration) sch->on_iteration(&row, sch->user);  // ReconstructOptions::on_iteration
        if (ckpt && ctx->rank == 0 && (t + 1) % sch->checkpoint_every == 0) {  // replicas agree: rank 0 writes
            const std::string dir(sch->checkpoint_dir);
            if (ctx->opt_mode == 0 && ctx->dsc.has_medium)
                save_grid_host(dir + "/checkpoint_" + std::to_string(t) + ".vgrd", ctx->dsc.dims, ctx->dsc.gorg,
                               ctx->dsc.vs, sch->length_unit, x_host.data());
            save_csv_host(rows, dir + "/loss.csv");
        }
        // stage saturation (inverse.cpp:249-258)
        const int since = t - stage_start;
        if (pending == stage && stage + 1 < sch->n_stages && since >= w) {
            const double past = loss_hist[(size_t)(t - w)], now = loss_hist.back();
            if (past > 0.0 && (past - now) / past < rel) pending = stage + 1;
        }
    }
    if (phases_out) *phases_out = phases;
    if (truncated_out) *truncated_out = truncated;
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_space_carve(prc_gpu_ctx* ctx, const double* gt_images, double threshold_fraction,
                                   double fill_extinction, uint8_t* mask_out, double* beta_out) {
    if (!ctx || !gt_images) return fail(PRC_ERR_INVALID, "prc_gpu_space_carve: null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    const DScene& s = ctx->dsc;
    if (s.n_det < 2) throw Err(PRC_ERR_INVALID, "space_carve: needs at least 2 detectors");
    if (!s.has_medium) throw Err(PRC_ERR_INVALID, "space_carve: scene has no medium");
    std::vector<double> thr((size_t)s.n_det, 0.0);
    for (int k = 0; k < s.n_det; ++k) {  // view maxima (inverse.cpp:76-78)
        double mx = 0.0;
        const long long n = (long long)s.det[k].rows * s.det[k].cols;
        for (long long p = 0; p < n; ++p) mx = std::max(mx, gt_images[s.det[k].img_off + p]);
        thr[(size_t)k] = threshold_fraction * mx;
    }
    cudaStream_t q = ctx->stream;
    DBuf<double> dgt, dthr, dbeta;
    DBuf<uint8_t> dmask;
    dgt.alloc((size_t)ctx->n_pix);
    dthr.alloc(thr.size());
    dmask.alloc((size_t)ctx->V);
    dbeta.alloc((size_t)ctx->V);
    CK(cudaMemcpyAsync(dgt.p, gt_images, (size_t)ctx->n_pix * 8, cudaMemcpyHostToDevice, q));
    CK(cudaMemcpyAsync(dthr.p, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, q));
    CK(launch_space_carve(s, dgt.p, dthr.p, fill_extinction, dmask.p, dbeta.p, q, &ctx->launches));
    if (mask_out) CK(cudaMemcpyAsync(mask_out, dmask.p, (size_t)ctx->V, cudaMemcpyDeviceToHost, q));
    if (beta_out) CK(cudaMemcpyAsync(beta_out, dbeta.p, (size_t)ctx->V * 8, cudaMemcpyDeviceToHost, q));
    ctx->sync();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_metrics(const double* estimate, const double* truth, uint64_t n, double* eps,
                               double* delta) {
    if (!estimate || !truth || !eps || !delta) return fail(PRC_ERR_INVALID, "prc_gpu_metrics: null argument");
    try {
        metrics_host(estimate, truth, n, eps, delta);
        return PRC_OK;
    } catch (const Err& e) {
        return fail(e.code, e.what());
    }
}

PRC_EXPORT int prc_gpu_downsample_images(int n_images, const int* rows, const int* cols, const double* images,
                                         int rows_out, int cols_out, double* out) {
    if (!rows || !cols || !images || !out) return fail(PRC_ERR_INVALID, "prc_gpu_downsample_images: null argument");
    if (n_images < 0 || rows_out <= 0 || cols_out <= 0) return fail(PRC_ERR_CONFIG, "downsample: bad sizes");
    for (int k = 0; k < n_images; ++k)
        if (rows[k] <= 0 || cols[k] <= 0) return fail(PRC_ERR_CONFIG, "downsample: bad image size");
    downsample(n_images, rows, cols, images, rows_out, cols_out, out);
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_save_grid(const char* path, const int dims[3], const prc_vec3* origin,
                                 const prc_vec3* voxel_size, int length_unit, const double* values) {
    if (!path || !dims || !origin || !voxel_size || !values) return fail(PRC_ERR_INVALID, "prc_gpu_save_grid: null argument");
    try {
        const double o[3] = {origin->x, origin->y, origin->z}, v[3] = {voxel_size->x, voxel_size->y, voxel_size->z};
        save_grid_host(path, dims, o, v, length_unit, values);
        return PRC_OK;
    } catch (const Err& e) {
        return fail(e.code, e.what());
    }
}

template <class T>
static T get_raw(std::ifstream& is) {
    T v{};
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
}

PRC_EXPORT int prc_gpu_load_grid(const char* path, int dims_out[3], prc_vec3* origin_out, prc_vec3* voxel_size_out,
                                 int* length_unit_out, double* values_out, uint64_t capacity) {
    if (!path) return fail(PRC_ERR_INVALID, "prc_gpu_load_grid: null path");
    std::ifstream is(path, std::ios::binary);  // load_grid, io.cpp:32-57
    if (!is) return fail(PRC_ERR_IO, std::string("load_grid: cannot open ") + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "VGRD", 4) != 0)
        return fail(PRC_ERR_IO, std::string("load_grid: bad magic at offset 0 in ") + path);
    if (get_raw<uint32_t>(is) != 1u) return fail(PRC_ERR_IO, std::string("load_grid: unsupported version in ") + path);
    int dims[3];
    for (int a = 0; a < 3; ++a) {
        const uint32_t d = get_raw<uint32_t>(is);
        if (d == 0 || d > (1u << 20)) return fail(PRC_ERR_IO, std::string("load_grid: bad dims in ") + path);
        dims[a] = (int)d;
    }
    double o[3], v[3];
    for (int a = 0; a < 3; ++a) o[a] = get_raw<double>(is);
    for (int a = 0; a < 3; ++a) v[a] = get_raw<double>(is);
    const uint8_t tag = get_raw<uint8_t>(is);
    if (tag > 1) return fail(PRC_ERR_IO, std::string("load_grid: bad unit tag in ") + path);
    const uint64_t count = (uint64_t)dims[0] * dims[1] * dims[2];
    std::vector<float> raw(count);
    is.read(reinterpret_cast<char*>(raw.data()), (std::streamsize)(count * sizeof(float)));
    if (!is) return fail(PRC_ERR_IO, std::string("load_grid: truncated payload in ") + path);
    if (dims_out)
        for (int a = 0; a < 3; ++a) dims_out[a] = dims[a];
    if (origin_out) *origin_out = prc_vec3{o[0], o[1], o[2]};
    if (voxel_size_out) *voxel_size_out = prc_vec3{v[0], v[1], v[2]};
    if (length_unit_out) *length_unit_out = tag;
    if (values_out) {
        if (capacity < count) return fail(PRC_ERR_INVALID, "load_grid: capacity too small");
        for (uint64_t i = 0; i < count; ++i) values_out[i] = raw[i];
    }
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_last_timings(const prc_gpu_ctx* ctx, double* ms8) {
    if (!ctx || !ms8) return fail(PRC_ERR_INVALID, "null argument");
    for (int i = 0; i < 8; ++i) ms8[i] = ctx->last_ms[i];
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_timer_start(prc_gpu_ctx* ctx) {
    if (!ctx) return fail(PRC_ERR_INVALID, "null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    if (!ctx->timer[0]) {
        CK(cudaEventCreate(&ctx->timer[0]));
        CK(cudaEventCreate(&ctx->timer[1]));
    }
    CK(cudaEventRecord(ctx->timer[0], ctx->stream));
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_timer_stop(prc_gpu_ctx* ctx, double* ms) {
    if (!ctx || !ms || !ctx->timer[0]) return fail(PRC_ERR_INVALID, "timer not started");
    ABI_TRY
    auto _lk = begin(ctx);
    CK(cudaEventRecord(ctx->timer[1], ctx->stream));
    CK(cudaEventSynchronize(ctx->timer[1]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]));
    *ms = f;
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_store_stats(prc_gpu_ctx* ctx, const prc_gpu_store* store, uint64_t* out4) {
    if (!ctx || !store || !out4) return fail(PRC_ERR_INVALID, "null argument");
    if (store->ctx != ctx) return fail(PRC_ERR_INVALID, "prc_gpu_store_stats: the store belongs to another context");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    store_for_scene(ctx, const_cast<prc_gpu_store*>(store));
    DBuf<unsigned long long> d;
    d.alloc(4);
    CK(cudaMemsetAsync(d.p, 0, 32, ctx->stream));
    CK(launch_stats(ctx->dsc, const_cast<prc_gpu_store*>(store)->view(), d.p, ctx->stream,
                    &ctx->launches));
    ctx->allreduce_u64(d.p, 4);
    CK(cudaMemcpyAsync(out4, d.p, 32, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_debug_checks(prc_gpu_ctx* ctx, uint32_t* flags_out, int* checked_build) {
    if (!ctx || !flags_out) return fail(PRC_ERR_INVALID, "prc_gpu_debug_checks: null argument");
#ifdef PRC_CHECKED
    if (checked_build) *checked_build = 1;
#else
    if (checked_build) *checked_build = 0;
#endif
    ABI_TRY
    auto _lk = begin(ctx);
    *flags_out = 0;
    if (ctx->check.p) {
        unsigned f = 0;
        CK(cudaMemcpy(&f, ctx->check.p, sizeof f, cudaMemcpyDeviceToHost));
        CK(cudaMemset(ctx->check.p, 0, sizeof f));
        *flags_out = f;
    }
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_kernel_launches(const prc_gpu_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return fail(PRC_ERR_INVALID, "null argument");
    *out = ctx->launches;
    return PRC_OK;
}

PRC_EXPORT int prc_gpu_debug_philox(prc_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t n,
                                    uint32_t* out) {
    if (!ctx || !out) return fail(PRC_ERR_INVALID, "null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    DBuf<uint32_t> d;
    d.alloc(std::max<uint64_t>(n, 1));
    CK(launch_philox(seed, stream, n, d.p, ctx->stream, &ctx->launches));
    if (n) CK(cudaMemcpyAsync(out, d.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    ABI_CATCH
}

static int debug_walk(prc_gpu_ctx* ctx, uint64_t n, const double* rays, uint32_t* counts_out,
                      uint32_t* voxels_out, double* lengths_out, uint64_t cap, bool pad) {
    if (!ctx || !rays || !counts_out) return fail(PRC_ERR_INVALID, "null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    if (!ctx->dsc.has_medium) throw Err(PRC_ERR_CONFIG, "scene has no medium grid");
    if (pad && !ctx->pad_ok) throw Err(PRC_ERR_CONFIG, "padded walks are not valid for this scene");
    cudaStream_t q = ctx->stream;
    DBuf<double> dr;
    DBuf<uint32_t> dc;
    dr.alloc(std::max<uint64_t>(7 * n, 1));
    dc.alloc(std::max<uint64_t>(n, 1));
    if (n) CK(cudaMemcpyAsync(dr.p, rays, 7 * n * 8, cudaMemcpyHostToDevice, q));
    CK(launch_walk(ctx->dsc, dr.p, (long long)n, dc.p, nullptr, nullptr, nullptr, q, &ctx->launches, pad));
    if (n) CK(cudaMemcpyAsync(counts_out, dc.p, n * 4, cudaMemcpyDeviceToHost, q));
    ctx->sync();
    if (voxels_out && lengths_out) {
        std::vector<unsigned long long> off(n + 1, 0);
        for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + counts_out[i];
        if (off[n] > cap) throw Err(PRC_ERR_INVALID, "debug_walk: capacity too small");
        DBuf<unsigned long long> doff;
        DBuf<uint32_t> dv;
        DBuf<double> dl;
        doff.alloc(std::max<uint64_t>(n, 1));
        dv.alloc(std::max<unsigned long long>(off[n], 1));
        dl.alloc(std::max<unsigned long long>(off[n], 1));
        if (n) CK(cudaMemcpyAsync(doff.p, off.data(), n * 8, cudaMemcpyHostToDevice, q));
        CK(launch_walk(ctx->dsc, dr.p, (long long)n, dc.p, doff.p, dv.p, dl.p, q, &ctx->launches, pad));
        if (off[n]) {
            CK(cudaMemcpyAsync(voxels_out, dv.p, off[n] * 4, cudaMemcpyDeviceToHost, q));
            CK(cudaMemcpyAsync(lengths_out, dl.p, off[n] * 8, cudaMemcpyDeviceToHost, q));
        }
        ctx->sync();
    }
    ABI_CATCH
}

PRC_EXPORT int prc_gpu_debug_walk(prc_gpu_ctx* ctx, uint64_t n, const double* rays, uint32_t* counts_out,
                                  uint32_t* voxels_out, double* lengths_out, uint64_t cap) {
    return debug_walk(ctx, n, rays, counts_out, voxels_out, lengths_out, cap, false);
}

PRC_EXPORT int prc_gpu_debug_walk_padded(prc_gpu_ctx* ctx, uint64_t n, const double* rays, uint32_t* counts_out,
                                         uint32_t* voxels_out, double* lengths_out, uint64_t cap) {
    return debug_walk(ctx, n, rays, counts_out, voxels_out, lengths_out, cap, true);
}

PRC_EXPORT int prc_gpu_debug_pixel_of(prc_gpu_ctx* ctx, int det, uint64_t n, const double* pts,
                                      int32_t* out) {
    if (!ctx || !pts || !out) return fail(PRC_ERR_INVALID, "null argument");
    ABI_TRY
    auto _lk = begin(ctx);
    ctx->check_scene();
    if (det < 0 || det >= ctx->dsc.n_det) throw Err(PRC_ERR_INVALID, "detector index out of range");
    cudaStream_t q = ctx->stream;
    DBuf<double> dp;
    DBuf<int32_t> dout;
    dp.alloc(std::max<uint64_t>(3 * n, 1));
    dout.alloc(std::max<uint64_t>(n, 1));
    if (n) CK(cudaMemcpyAsync(dp.p, pts, 3 * n * 8, cudaMemcpyHostToDevice, q));
    CK(launch_pixel_of(ctx->dsc, det, dp.p, (long long)n, dout.p, q, &ctx->launches));
    if (n) CK(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, q));
    ctx->sync();
    ABI_CATCH
}
