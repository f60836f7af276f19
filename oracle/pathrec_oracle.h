/*
 * pathrec_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the reference
 * path (arXiv 2110.00085 reference `pathrec`).  Used exclusively by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline leg as the checker; the
 * product (paper_2110_00085_b200/) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement bit-for-bit against the
 * reference library compiled in place (oracle/_ref) and against the committed golden
 * vectors (tests/golden/, written by tests/golden/make_golden.py from the reference).
 */
#ifndef PATHREC_ORACLE_H
#define PATHREC_ORACLE_H

#include <stdint.h>

#include "pathrec_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_store orc_store;

const char* orc_last_error(void);

/* Philox4x32-10 words (rng.hpp:11-61). */
int orc_philox(uint64_t seed, uint64_t stream, uint64_t n, uint32_t* out);
/* walk_voxels (traverse.hpp:45-116) over n rays (n x 7 doubles). */
int orc_walk(const prc_scene_desc* d, uint64_t n, const double* rays, uint32_t* counts,
             uint32_t* vox, double* len, uint64_t cap);
/* Detector::pixel_of (scene.cpp:16-28). */
int orc_pixel_of(const prc_scene_desc* d, int det, uint64_t n, const double* pts, int32_t* out);

/* render (transport.cpp:405-454); keep != 0 returns the store. */
int orc_render(const prc_scene_desc* d, const prc_gpu_params* params, uint64_t n, uint64_t seed,
               int max_bounces, int max_events, int keep, double* images_out,
               uint64_t* trunc_out, orc_store** store_out);
/* sort_by_size (pathstore.cpp:261-267). */
int orc_sort_by_size(orc_store* s);
/* evaluate_store (pathstore.cpp:315-368); params NULL = store reference parameters. */
int orc_evaluate(const prc_scene_desc* d, const orc_store* s, const prc_gpu_params* params,
                 int flags, const double* weights, double* images, double* grad, double* gk,
                 double* gg, uint64_t* clamps, double* mean_corr);
int orc_save_pstr(const orc_store* s, const char* path);
int orc_load_pstr(const char* path, orc_store** out);
uint64_t orc_store_count(const orc_store* s);
/* Deep copy of records [lo, hi) (multi-rank decomposition tests). */
orc_store* orc_store_slice(const orc_store* s, uint64_t lo, uint64_t hi);
int orc_store_streams(const orc_store* s, uint64_t* out);
int orc_store_sizes(const orc_store* s, uint32_t* out);
/* Per-store statistics: [0] S, [1] vertices, [2] events, [3] LE spans,
 * [4] live path spans (segments 1..B-1), [5] all path spans, [6] truncated. */
int orc_store_stats(const orc_store* s, double* out7);
void orc_store_free(orc_store* s);

#ifdef __cplusplus
}
#endif

#endif
