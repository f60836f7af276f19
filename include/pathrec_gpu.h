/*
 * pathrec_gpu.h — C ABI of the B200-native Path Sorting + Path Recycling engine.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2110.00085,
 * reference `pathrec`, /root/reference/proj).  The reference's C++ calls that the
 * recycling loop is made of, and the entry point here that replaces each one:
 *
 *   pathrec::render(scene, {keep_paths})      transport.hpp:174, transport.cpp:405-454
 *        -> prc_gpu_render                      (K1 trace + K4 fresh evaluation)
 *   pathrec::sort_by_size(store)              pathstore.hpp:28, pathstore.cpp:261-267
 *        -> prc_gpu_sort_by_size                (K2 stable counting sort by B)
 *   pathrec::evaluate_store(scene, store, t, opt)   pathstore.hpp:64, pathstore.cpp:315-368
 *        -> prc_gpu_evaluate                    (K3 prep, K4 forward, K5 gradient)
 *   pathrec::recycled_render(...)             pathstore.hpp:68, pathstore.cpp:370-375
 *        -> prc_gpu_evaluate with want_grad = 0
 *   pathrec::grad_forward(...)                gradient.hpp:40, gradient.cpp:111-128
 *        -> prc_gpu_evaluate with want_grad = 1
 *   pathrec::reconstruct / adam_step / loss   inverse.hpp:274-295, inverse.cpp:11-67,154-263
 *        -> prc_gpu_opt_* (device-resident Algorithm 2 iteration) and prc_gpu_reconstruct
 *   pathrec::save_store / load_store (PSTR v1) pathstore.cpp:410-516
 *        -> prc_gpu_store_export_pstr / prc_gpu_store_import_pstr
 *
 * Around the loop (the Algorithm-2 driver):
 *   reconstruct with a stage schedule          inverse.cpp:154-263, inverse.hpp:23-34
 *        -> prc_gpu_reconstruct_schedule
 *   space_carve / metrics / downsample_images inverse.cpp:69-133
 *        -> prc_gpu_space_carve (device), prc_gpu_metrics, prc_gpu_downsample_images
 *   save_grid / load_grid (VGRD v1), save_csv   io.cpp:32-76, 147-155
 *        -> prc_gpu_save_grid / prc_gpu_load_grid, checkpoints of the schedule
 *
 * Conventions follow the reference C ABI (include/pathrec.h:11-23, src/capi.cpp:17-32):
 * opaque handles, int error codes, a thread-local last-error string, no exceptions
 * across the boundary, caller-owned option structs, one *_free per handle.
 * Every entry point is synchronous.  Plain pointers and sizes only; no torch types.
 */
#ifndef PATHREC_GPU_H
#define PATHREC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: same values as the reference enum (pathrec.h:13-19) plus CUDA. */
enum {
    PRC_OK = 0,
    PRC_ERR_CONFIG = 1,  /* bad option values, malformed scene */
    PRC_ERR_IO = 2,      /* missing or unreadable/unwritable files */
    PRC_ERR_NUMERIC = 3, /* non-finite results, aborted optimization */
    PRC_ERR_INVALID = 4, /* null handles, out-of-range indices */
    PRC_ERR_CUDA = 5     /* device / driver / NCCL failure (no CPU fallback exists) */
};

/* ---------------------------------------------------------------------------
 * Scene description (value mirror of pathrec::Scene, scene.hpp:26-107).
 * All arrays are borrowed for the duration of the call that receives them.
 * ------------------------------------------------------------------------- */

typedef struct {
    double x, y, z;
} prc_vec3;

/* PhaseFunction::Kind (phase.hpp:19) */
enum { PRC_PHASE_HG = 0, PRC_PHASE_RAYLEIGH = 1 };
/* Surface::Kind (scene.hpp:79), Brdf::Kind (brdf.hpp:41) */
enum { PRC_SURF_SPHERE = 0, PRC_SURF_FACE = 1 };
enum { PRC_BRDF_DIFFUSE = 0, PRC_BRDF_PHONG = 1 };
/* LightSource::Kind (scene.hpp:57) */
enum { PRC_LIGHT_SUN = 0, PRC_LIGHT_POINT = 1 };

/* ParticleSpecies (scene.hpp:26-32).  All species share one grid geometry. */
typedef struct {
    const double* extinction; /* voxel_count values, x-fastest (grid.hpp:15-24) */
    double albedo;
    int phase_kind;           /* PRC_PHASE_* */
    double g;                 /* HG asymmetry (ignored for Rayleigh) */
    int unknown;              /* tomography target (at most one, scene.cpp:145-147) */
} prc_species_desc;

/* Surface + Sphere + BoxFace + Brdf (scene.hpp:63-86, brdf.hpp:12-63) */
typedef struct {
    int kind;                 /* PRC_SURF_* */
    prc_vec3 center;          /* sphere */
    double radius;
    int axis;                 /* face: plane axis 0..2 */
    double coord;             /* face: plane coordinate */
    double lo[2], hi[2];      /* face: extents on the other two axes, in axis order */
    double normal_sign;       /* face: +1 normal toward +axis */
    int brdf_kind;            /* PRC_BRDF_* */
    double albedo;            /* diffuse albedo */
    double kappa_s, gamma;    /* Phong lobe */
    int target;               /* reflectometry unknown surface (Phong) */
} prc_surface_desc;

/* LightSource (scene.hpp:56-61) */
typedef struct {
    int kind;                 /* PRC_LIGHT_* */
    prc_vec3 position;        /* point light */
    prc_vec3 direction;       /* sun propagation direction */
    double radiance;
} prc_light_desc;

/* Detector (scene.hpp:34-54); the frame is derived as Detector::finalize (scene.cpp:8-14). */
typedef struct {
    prc_vec3 position;
    prc_vec3 direction;
    prc_vec3 up;
    int rows, cols;
    double fov;               /* full horizontal field of view [rad] */
} prc_detector_desc;

typedef struct {
    prc_vec3 bounds_min, bounds_max;   /* Scene::bounds */
    int dims[3];                       /* GridGeometry (ignored when n_species == 0) */
    prc_vec3 grid_origin, voxel_size;
    int n_species;
    const prc_species_desc* species;
    int n_surfaces;
    const prc_surface_desc* surfaces;
    prc_light_desc light;
    int n_detectors;
    const prc_detector_desc* detectors;
    /* Nonzero when Scene::finalize (scene.cpp:8-14, 69-75) already ran on the host: detector
     * and sun directions are unit vectors and are used as given.  Zero (the default): the
     * engine finalizes them itself, exactly once. */
    int finalized;
} prc_scene_desc;

/* ParamSet (transport.hpp:63-67): the unknowns decoupled from the scene.
 * beta: unknown species' extinction per voxel (n_beta == voxel_count) or NULL to
 * use the scene's values.  species_beta (extension for per-type work, config (c)):
 * optional array of n_species pointers overriding every species; NULL entries keep
 * the scene's (or `beta`'s) values. */
typedef struct {
    const double* beta;
    uint64_t n_beta;
    double kappa_s, gamma;
    const double* const* species_beta;
} prc_gpu_params;

/* ---------------------------------------------------------------------------
 * Context: one per process; owns the device(s), streams, the scene copy and the
 * NCCL communicator.  Paths are sharded over ranks by contiguous stream ranges.
 * ------------------------------------------------------------------------- */

typedef struct prc_gpu_ctx prc_gpu_ctx;
typedef struct prc_gpu_store prc_gpu_store;

const char* prc_gpu_version(void);
const char* prc_gpu_last_error(void);

/* Single-GPU context on CUDA device `device`. */
int prc_gpu_ctx_create(int device, prc_gpu_ctx** out);
/* One process per GPU: joins an NCCL communicator of `world` ranks.  nccl_id is the
 * 128-byte ncclUniqueId produced by prc_gpu_nccl_unique_id on rank 0 and broadcast
 * by the caller (e.g. through torch.distributed). */
int prc_gpu_nccl_unique_id(void* out128);
/* nccl_id NULL with world > 1: a detached shard without a communicator.  The context
 * traces / imports rank `rank`'s stream range and every result it returns (images,
 * gradients, clamp and truncation counts) is that shard's partial sum, still normalised by
 * the global path count; the caller reduces them (e.g. over MPI or torch.distributed).
 * With PRC_EVAL_SELF_NORMALIZE a detached shard returns its results undivided and its
 * partial mean_correction (shard sum / global count): the caller sums both and divides. */
int prc_gpu_ctx_create_rank(int device, int rank, int world, const void* nccl_id,
                            prc_gpu_ctx** out);
/* The contiguous stream range [lo, hi) rank `rank` of `world` owns out of n paths
 * (floor(n r / w) .. floor(n (r+1) / w)).  Host-only, no device needed. */
int prc_gpu_shard_range(uint64_t n, int rank, int world, uint64_t* lo, uint64_t* hi);
/* Destroys the context (its stores stay freeable) and returns the device's cached blocks. */
void prc_gpu_ctx_destroy(prc_gpu_ctx* ctx);
int prc_gpu_ctx_rank(const prc_gpu_ctx* ctx, int* rank, int* world);
/* Device memory: freed buffers of >= 1 MB (a freed store's arrays, scratch) are kept by the
 * engine and reused by later allocations of nearly the same size -- the resample of the
 * recycling loop frees one path-store generation and allocates the next -- instead of
 * being returned to the driver.  They are returned when a context on that device is
 * destroyed, when an engine allocation fails, or by this call (every device).  A caller
 * that shares the GPU with another allocator (e.g. torch) can call it after freeing
 * stores. */
int prc_gpu_release_cached_memory(void);
/* Engine knobs (all give the same results up to the order of floating-point sums):
 * - "mode": 0 = event-major wavefront over Morton-ordered interaction vertices
 *   (default), 1 = fused thread-per-path (the paper's mapping);
 * - "packet" 1..4: LE rays per thread walked in lockstep by the gradient kernel (default 3);
 * - "spread": Morton distance between the packets of one warp (default 0: chosen from
 *   the vertex density per gradient copy);
 * - "per_species" 1: the device-resident iteration (prc_gpu_opt_step) computes per-type
 *   gradients of every species (config (c)); the optimiser still updates the unknown one;
 * - "pad" 0: no guard-free walks over the padded voxel layout (default 1);
 * - "grad_copies": copies of the padded gradient the gradient kernel reduces into (0 =
 *   default: 8, up to 32 while they fit in 64 MB, fewer when they would exceed 2 GB;
 *   applied at the next scene upload);
 * - "events" 0: no compact event list for scenes without a medium (default 1: after the
 *   first forward over a store, forwards and gradients run over its events only);
 * - "nvls" 1: images and gradients reduced over ranks by NVLS multicast (2 = the fold
 *   without multicast, one rank; applied at the next scene upload). */
int prc_gpu_ctx_set_option(prc_gpu_ctx* ctx, const char* key, int64_t value);

/* Uploads (and validates, finalizes) the scene; replaces any previous scene and
 * frees every store built against it. */
int prc_gpu_scene_upload(prc_gpu_ctx* ctx, const prc_scene_desc* scene);
int prc_gpu_scene_voxel_count(const prc_gpu_ctx* ctx, uint64_t* out);
/* Total image pixels over detectors (images are concatenated detector-major). */
int prc_gpu_scene_pixel_count(const prc_gpu_ctx* ctx, uint64_t* out);

/* ---------------------------------------------------------------------------
 * Path generation (K1) — pathrec::render (transport.cpp:405-454).
 * ------------------------------------------------------------------------- */

typedef struct {
    uint64_t n_paths;         /* global path count (all ranks) */
    uint64_t seed;
    int max_bounces;          /* <= 0: default 500 */
    int max_scatter_events;   /* < 0: unlimited (RenderOptions, transport.hpp:154-161) */
} prc_gpu_render_opts;

/* Traces n_paths paths under `params` (NULL: scene values; bind_params semantics,
 * inverse.cpp:144-150) and evaluates them at that point (the fresh image, bit-reproducible
 * for fixed seed and n_paths).  images_out: host buffer of pixel_count doubles, normalised
 * by 1/N; NULL skips the fresh evaluation (trace only, as a resample of reconstruct).
 * store_out: non-NULL keeps the path store (keep_paths). */
int prc_gpu_render(prc_gpu_ctx* ctx, const prc_gpu_render_opts* opts, const prc_gpu_params* params,
                   double* images_out, uint64_t* truncated_out, prc_gpu_store** store_out);

/* K2: stable sort by ascending B (pathstore.cpp:261-267); re-lays the device store
 * out bucket-major so a warp of consecutive paths reads coalesced records. */
int prc_gpu_sort_by_size(prc_gpu_ctx* ctx, prc_gpu_store* store);

typedef struct {
    uint64_t n_paths;          /* paths in this rank's shard */
    uint64_t n_paths_global;   /* normalisation count */
    uint64_t stream_base;      /* first global stream id of this shard */
    uint64_t segments;         /* S = sum of B (dead final segments included) */
    uint64_t vertices;         /* sum of (B + 1) */
    uint64_t interaction_vertices; /* sum of (B - 1) */
    uint64_t truncated;
    uint64_t seed, generation;
    int sorted;
    int max_size;              /* max B */
    uint64_t device_bytes;     /* device memory held by the store */
    int materialized;          /* imported with PRC_IMPORT_MATERIALIZE */
} prc_gpu_store_info;

int prc_gpu_store_info_get(const prc_gpu_store* store, prc_gpu_store_info* out);
/* Stream ids in storage order (PathStore::records[i].stream). */
int prc_gpu_store_streams(const prc_gpu_store* store, uint64_t* out);
/* correction_factor (pathstore.cpp:269-294) of every path of this shard under params_t
 * (NULL: the scene's values) against the store's reference parameters, in storage order
 * (prc_gpu_store_streams gives each position's stream id); out has prc_gpu_store_info.n
 * entries.  The mean of these over the store is EvalOptions::self_normalize's divisor. */
int prc_gpu_correction_factors(prc_gpu_ctx* ctx, const prc_gpu_store* store, const prc_gpu_params* params_t,
                               double* out);
/* Path sizes B in storage order. */
int prc_gpu_store_sizes(const prc_gpu_store* store, uint32_t* out);
/* PSTR v1 interchange (pathstore.cpp:410-516).  Export materialises every span and
 * event on the device.  Import accepts reference-written files. */
int prc_gpu_store_export_pstr(prc_gpu_ctx* ctx, const prc_gpu_store* store, const char* path);
int prc_gpu_store_import_pstr(prc_gpu_ctx* ctx, const char* path, prc_gpu_store** out);
/* load_store with options.  PRC_IMPORT_MATERIALIZE keeps the file's own segment spans,
 * events and LE spans on the device and evaluates them as eval_record reads them
 * (pathstore.cpp:115-238): the reference's voxel ids and span lengths, fp64 throughout.
 * Without it (prc_gpu_store_import_pstr) spans are recomputed by the DDA along chord
 * directions (voxel ids identical, lengths within rounding) and the store runs on the
 * recycling kernels.  A materialized store exports its records verbatim (sorted:
 * in storage order), byte-identical to the reference's save_store of the same store. */
enum { PRC_IMPORT_MATERIALIZE = 1 };
int prc_gpu_store_import_pstr_ex(prc_gpu_ctx* ctx, const char* path, int flags, prc_gpu_store** out);
int prc_gpu_store_set_generation(prc_gpu_store* store, uint64_t generation);
/* A store belongs to the context that made it: passing it with another context returns
 * PRC_ERR_INVALID.  prc_gpu_store_free is valid before or after that context is destroyed
 * (a store outliving its context can only be freed). */
void prc_gpu_store_free(prc_gpu_store* store);

/* ---------------------------------------------------------------------------
 * Recycled evaluation (K3/K4/K5) — pathrec::evaluate_store (pathstore.cpp:315-368).
 * ------------------------------------------------------------------------- */

enum {
    PRC_EVAL_NORMALIZE = 1,     /* divide by the global record count (default on) */
    PRC_EVAL_WANT_GRAD = 2,
    PRC_EVAL_LEGACY_SCORE = 4,  /* pathstore.cpp:98-101 */
    PRC_EVAL_SELF_NORMALIZE = 8,/* divide by the mean correction factor (pathstore.cpp:334-359) */
    PRC_EVAL_PER_SPECIES = 16,  /* per-type gradients: grad_out holds n_species x V */
    PRC_EVAL_DETERMINISTIC = 32 /* bit-reproducible images (exact fixed-point pixel sums,
                                   two forward passes); prc_gpu_render always does this */
};

typedef struct {
    int flags;                    /* PRC_EVAL_* */
    const double* pixel_weights;  /* host, pixel_count doubles (residuals) or NULL = 1 */
} prc_gpu_eval_opts;

typedef struct {
    double* images;      /* host, pixel_count doubles, or NULL */
    double* grad_beta;   /* host, V doubles (or n_species*V with PER_SPECIES), or NULL */
    double grad_kappa, grad_gamma;
    uint64_t clamp_events;
    double mean_correction;
} prc_gpu_eval_result;

int prc_gpu_evaluate(prc_gpu_ctx* ctx, const prc_gpu_store* store, const prc_gpu_params* params,
                     const prc_gpu_eval_opts* opts, prc_gpu_eval_result* result);

/* ---------------------------------------------------------------------------
 * Device-resident Algorithm 2 (inverse.cpp:154-263): the recycled iteration
 * K3 -> K4 -> allreduce(images) -> loss/residual -> K5 -> allreduce(grad) -> K6 ADAM,
 * with parameters, moments and the ground truth resident in HBM.
 * ------------------------------------------------------------------------- */

typedef struct {
    double alpha, eta1, eta2, eps_guard;  /* AdamConfig (inverse.hpp:11-21) */
    int project_nonneg;
    const double* step_scale;             /* n_step_scale multipliers or NULL */
    int n_step_scale;
} prc_gpu_adam_config;

/* gt_images: host, pixel_count doubles.  initial: starting unknowns. */
int prc_gpu_opt_init(prc_gpu_ctx* ctx, const prc_gpu_params* initial, const double* gt_images,
                     const prc_gpu_adam_config* adam);
/* One recycled iteration over `store`; loss_out receives 0.5*||F - gt||^2. */
int prc_gpu_opt_step(prc_gpu_ctx* ctx, const prc_gpu_store* store, double* loss_out);
/* adam_step (inverse.cpp:41-67) with a caller-given gradient over the flattened unknowns
 * (tomography: V values; reflectometry: dkappa_s, dgamma): one K6 update of the device-
 * resident state, bit-identical to the reference's.  n must equal the unknown count. */
int prc_gpu_opt_adam_step(prc_gpu_ctx* ctx, const double* grad, uint64_t n);
/* Copies the current unknowns out (beta: V doubles or NULL). */
int prc_gpu_opt_params(prc_gpu_ctx* ctx, double* beta_out, double* kappa_s, double* gamma);
/* Current device forward images (pixel_count doubles) of the last step. */
int prc_gpu_opt_images(prc_gpu_ctx* ctx, double* images_out);

typedef struct {
    uint64_t seed;
    uint64_t n_paths;
    int max_bounces;
    int recycle_period;       /* N_r (Schedule::recycle_period) */
    int max_iterations;
} prc_gpu_reconstruct_opts;

/* Algorithm 2 with a single stage: resample + sort every N_r iterations (seed
 * schedule of inverse.cpp:193), otherwise recycle.  loss_history: max_iterations
 * doubles or NULL.  sampling_phases_out may be NULL. */
int prc_gpu_reconstruct(prc_gpu_ctx* ctx, const prc_gpu_params* initial, const double* gt_images,
                        const prc_gpu_adam_config* adam, const prc_gpu_reconstruct_opts* opts,
                        double* loss_history, uint64_t* sampling_phases_out);

/* ---------------------------------------------------------------------------
 * The Algorithm-2 driver around the loop (inverse.cpp:69-263, io.cpp:32-76, 147-155).
 * ------------------------------------------------------------------------- */

typedef struct {              /* Stage (inverse.hpp:23-26) */
    int rows, cols;           /* detector resolution; <= 0 keeps the current value */
    uint64_t n_paths;
} prc_gpu_stage;

struct prc_gpu_iteration_log_s; /* prc_gpu_iteration_log, below */

typedef struct {              /* Schedule (inverse.hpp:28-35) + ReconstructOptions (:66-76) */
    uint64_t seed;
    int max_bounces;          /* trace budget (RenderOptions::max_bounces, default 500) */
    int recycle_period;       /* N_r */
    int max_iterations;
    const prc_gpu_stage* stages;
    int n_stages;             /* >= 1 */
    int saturation_window;    /* default 20 */
    double saturation_rel_improvement;  /* default 0.01 */
    int checkpoint_every;     /* 0 disables checkpoints */
    const char* checkpoint_dir;         /* NULL or "" disables checkpoints; rank 0 writes */
    int length_unit;          /* VGRD unit tag of the checkpoints (LengthUnit) */
    const prc_gpu_params* truth;        /* optional ground-truth unknowns for eps/delta */
    /* ReconstructOptions::on_iteration (inverse.hpp:75): called once per iteration after
     * logging, before the checkpoint and the update; may be NULL. */
    void (*on_iteration)(const struct prc_gpu_iteration_log_s* row, void* user);
    void* user;
} prc_gpu_schedule;

typedef struct prc_gpu_iteration_log_s { /* IterationLog (inverse.hpp:46-53) */
    int iter;
    double time_s, loss, eps, delta;
    int stage;
} prc_gpu_iteration_log;

/* reconstruct() with a stage schedule (inverse.cpp:154-263): at every resample
 * boundary (t % N_r == 0) a pending stage change is applied first -- every detector
 * takes the stage's rows/cols and the ground truth is block-sum downsampled to it --
 * then paths are traced under the iterate with the stage's n_paths (seed schedule of
 * inverse.cpp:193) and sorted.  Each iteration logs (loss, eps/delta against `truth`),
 * optionally checkpoints the pre-update unknowns (VGRD) and the history (CSV) to
 * checkpoint_dir, then takes the residual-weighted gradient and the ADAM step.  A stage
 * saturates when the relative loss improvement over saturation_window iterations falls
 * below saturation_rel_improvement.  gt_images are at the uploaded detector resolution.
 * The scene's detector resolution is restored on return.  history: max_iterations rows
 * or NULL; the counters may be NULL. */
int prc_gpu_reconstruct_schedule(prc_gpu_ctx* ctx, const prc_gpu_params* initial, const double* gt_images,
                                 const prc_gpu_adam_config* adam, const prc_gpu_schedule* schedule,
                                 prc_gpu_iteration_log* history, uint64_t* sampling_phases_out,
                                 uint64_t* truncated_paths_out);

/* space_carve (inverse.cpp:69-101) on the device: a voxel is occupied when its centre
 * projects into every detector at a pixel above threshold_fraction of that view's
 * maximum in gt_images (host, uploaded resolution).  mask_out: voxel_count bytes;
 * beta_out: voxel_count doubles (fill_extinction where occupied, else 0); either may
 * be NULL.  PRC_ERR_INVALID with fewer than 2 detectors or without a medium. */
int prc_gpu_space_carve(prc_gpu_ctx* ctx, const double* gt_images, double threshold_fraction,
                        double fill_extinction, uint8_t* mask_out, double* beta_out);

/* metrics (inverse.cpp:103-114): eps = sum|t - e| / sum|t|, delta = (sum|t| - sum|e|) / sum|t|.
 * Host arithmetic in the reference's order. */
int prc_gpu_metrics(const double* estimate, const double* truth, uint64_t n, double* eps, double* delta);

/* downsample_images (inverse.cpp:116-133): block sums of n_images images, image i of
 * rows[i] x cols[i] (row-major, concatenated), to rows_out x cols_out each (copied when
 * equal).  out: n_images * rows_out * cols_out doubles. */
int prc_gpu_downsample_images(int n_images, const int* rows, const int* cols, const double* images,
                              int rows_out, int cols_out, double* out);

/* VGRD v1 (io.cpp:32-76): "VGRD", u32 1, u32 dims[3], f64 origin[3], f64 voxel_size[3],
 * u8 unit, f32 values[prod dims].  save_grid writes values as f32; load_grid fills
 * dims/origin/voxel_size/unit (any may be NULL) and, when values_out is non-NULL,
 * capacity >= prod dims values (f64). */
int prc_gpu_save_grid(const char* path, const int dims[3], const prc_vec3* origin, const prc_vec3* voxel_size,
                      int length_unit, const double* values);
int prc_gpu_load_grid(const char* path, int dims_out[3], prc_vec3* origin_out, prc_vec3* voxel_size_out,
                      int* length_unit_out, double* values_out, uint64_t capacity);

/* ---------------------------------------------------------------------------
 * Timing and device-side diagnostics (used by tests and bench; not on the API path).
 * ------------------------------------------------------------------------- */

/* Milliseconds of the most recent evaluate / opt_step kernels, measured with CUDA
 * events on the launching stream: [0] prep, [1] forward (K4), [2] image allreduce +
 * loss, [3] gradient (K5), [4] grad allreduce + ADAM, [5] total, [6] the per-path part of
 * K4 (k_prefix), [7] the per-path part of K5 (k_path_gradient). */
int prc_gpu_last_timings(const prc_gpu_ctx* ctx, double* ms8);
/* CUDA events recorded on the context's stream: start / stop -> elapsed ms. */
int prc_gpu_timer_start(prc_gpu_ctx* ctx);
int prc_gpu_timer_stop(prc_gpu_ctx* ctx, double* ms);
/* Device counting pass over a store (no gathers): out[0] events, out[1] live path-span
 * incidences (segments 1..B-1), out[2] LE span incidences, out[3] all path spans. */
int prc_gpu_store_stats(prc_gpu_ctx* ctx, const prc_gpu_store* store, uint64_t* out4);
/* Range-check word of a checked build (libpathrec_gpu_checked.so, built with
 * -DPRC_CHECKED): bit k set when an access of class k left its table (0 padded gathers,
 * 1 padded reductions, 2 pixel indices, 3 voxel indices, 4 event-cache slots).  Reads and
 * clears it; *checked_build tells whether this library checks at all (0: flags stay 0). */
int prc_gpu_debug_checks(prc_gpu_ctx* ctx, uint32_t* flags_out, int* checked_build);
/* Number of kernels this library launched since ctx creation. */
int prc_gpu_kernel_launches(const prc_gpu_ctx* ctx, uint64_t* out);

/* Philox4x32-10 words from the device generator (rng.hpp:11-61): n words of stream. */
int prc_gpu_debug_philox(prc_gpu_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t n,
                         uint32_t* out);
/* Device fp64 DDA (traverse.hpp:45-116) over n rays against the uploaded grid.
 * rays: n x 7 doubles (origin xyz, direction xyz, max_distance).
 * counts_out[n]; when voxels_out/lengths_out are non-NULL they receive the spans of
 * all rays concatenated (capacity `cap`). */
int prc_gpu_debug_walk(prc_gpu_ctx* ctx, uint64_t n, const double* rays, uint32_t* counts_out,
                       uint32_t* voxels_out, double* lengths_out, uint64_t cap);
/* The guard-free walk the wavefront kernels use on the padded voxel layout (one border
 * voxel per face; voxels_out are padded indices (ix+1) + (nx+2)((iy+1) + (ny+2)(iz+1))).
 * Its spans are the reference walk's spans plus at most three trailing spans in border
 * voxels of total length ~1e-13 |t|.  PRC_ERR_CONFIG when the scene fails the padded
 * walk's preconditions. */
int prc_gpu_debug_walk_padded(prc_gpu_ctx* ctx, uint64_t n, const double* rays, uint32_t* counts_out,
                              uint32_t* voxels_out, double* lengths_out, uint64_t cap);
/* Device Detector::pixel_of (scene.cpp:16-28) for n points against detector det. */
int prc_gpu_debug_pixel_of(prc_gpu_ctx* ctx, int det, uint64_t n, const double* points,
                           int32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PATHREC_GPU_H */
