/*
 * pathrec.h -- the reference's coarse C API (reference include/pathrec.h, src/capi.cpp),
 * served by the B200 engine.
 *
 * A C caller of the reference library switches by compiling against this directory and
 * linking paper_2110_00085_b200/libpathrec_gpu.so instead of libpathrec.so.  Every entry
 * point keeps the reference's name, argument meaning, option defaults and error codes
 * (the enum lives in pathrec_gpu.h, same values plus PRC_ERR_CUDA).  Underneath, the
 * scene is uploaded to the process's default device context (CUDA device $LOCAL_RANK,
 * else 0) and the work runs through the fine-grained engine API of pathrec_gpu.h:
 *
 *   prc_scene_load       load_scene (io.cpp:190-278): JSON scene, VGRD species grids
 *   prc_render           render (transport.cpp:405-454)   -> prc_gpu_render
 *   prc_reconstruct      reconstruct (inverse.cpp:154-263) -> prc_gpu_space_carve +
 *                        prc_gpu_reconstruct_schedule, ground truth from gt_dir PFMs
 *   prc_result_* / prc_grid_*   PFM / PGM / VGRD / CSV writers (io.cpp:32-155)
 *
 * Two calls differ from the reference by design: `workers` is ignored (the work runs on
 * the GPU), and prc_selftest checks the device path (Philox known answer, DDA known
 * answer, phase-function normalisation) instead of the reference's Monte-Carlo oracles,
 * which are out of scope.
 */
#ifndef PATHREC_H
#define PATHREC_H

#include <stddef.h>
#include <stdint.h>

#include "pathrec_gpu.h" /* PRC_OK / PRC_ERR_* (pathrec.h:13-19 values) */

#ifdef __cplusplus
extern "C" {
#endif

typedef struct prc_scene prc_scene;   /* a loaded scene (host) */
typedef struct prc_result prc_result; /* images, or the result of an optimisation */
typedef struct prc_grid prc_grid;     /* a VGRD voxel grid */

const char* prc_version(void);
const char* prc_last_error(void); /* thread-local, as capi.cpp:17-22 */

/* Scene (capi.cpp:58-96). */
int prc_scene_load(const char* path, prc_scene** out);
void prc_scene_free(prc_scene* scene);
int prc_scene_validate(const prc_scene* scene, char* buf, size_t buflen, int* n_violations);
int prc_scene_detector_count(const prc_scene* scene, int* out);
/* Engine extension: the loaded scene as the flat descriptor prc_gpu_scene_upload takes;
 * borrowed, valid until prc_scene_free. */
int prc_scene_describe(const prc_scene* scene, const prc_scene_desc** out, int* length_unit);

/* Forward render (capi.cpp:98-122).  store_dump_path: PSTR v1 of the traced paths. */
typedef struct {
    uint64_t n_paths;
    uint64_t seed;
    int workers;                 /* ignored */
    int max_bounces;             /* <= 0: 500 */
    const char* store_dump_path; /* may be NULL */
} prc_render_opts;

int prc_render(const prc_scene* scene, const prc_render_opts* opts, prc_result** out);

/* Inverse problem (capi.cpp:124-204): tomography when the scene flags an unknown species
 * (space-carved start), reflectometry when it flags a target surface. */
typedef struct {
    uint64_t seed;
    uint64_t n_paths;           /* first stage; each further stage doubles it (<= 0: 1e5) */
    int workers;                /* ignored */
    int max_bounces;            /* <= 0: 500 */
    int recycle_period;         /* <= 0: 30 */
    int max_iterations;
    int n_stages;               /* <= 0: 1 */
    double alpha;               /* <= 0: 1e7 */
    double carve_threshold;     /* <= 0: 0.02 of each view's maximum */
    double carve_fill;
    double init_kappa, init_gamma;
    double gamma_step_scale;    /* <= 0: 1 */
    const char* gt_dir;         /* gt_000.pfm, gt_001.pfm, ... one per detector (required) */
    const char* out_dir;        /* loss.csv and a VGRD checkpoint every 25 iterations; may be NULL */
    const char* truth_grid;     /* VGRD truth for eps / delta; may be NULL */
    double truth_kappa, truth_gamma; /* reflectometry truth, used when either is > 0 */
} prc_reconstruct_opts;

int prc_reconstruct(const prc_scene* scene, const prc_reconstruct_opts* opts, prc_result** out);

/* Results (capi.cpp:206-296). */
int prc_result_image(const prc_result* result, int detector, const double** data, int* rows, int* cols);
int prc_result_save_pfm(const prc_result* result, int detector, const char* path);
int prc_result_save_pgm(const prc_result* result, int detector, const char* path);
int prc_result_params(const prc_result* result, double* kappa_s, double* gamma);
int prc_result_grid_save(const prc_result* result, const char* path);
int prc_result_final_loss(const prc_result* result, double* loss);
int prc_result_save_csv(const prc_result* result, const char* path);
void prc_result_free(prc_result* result);

/* VGRD grids (capi.cpp:298-334). */
int prc_grid_load(const char* path, prc_grid** out);
int prc_grid_save(const prc_grid* grid, const char* path);
int prc_grid_metrics(const prc_grid* estimate, const prc_grid* truth, double* eps, double* delta);
void prc_grid_free(prc_grid* grid);

int prc_selftest(void);

#ifdef __cplusplus
}
#endif

#endif /* PATHREC_H */
