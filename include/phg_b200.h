/*
 * phg_b200.h -- C ABI of the B200-native PHG (Parallel Hair Growing) tracer.
 *
 * Drop-in for the reference's grow-step boundary
 *   strandkit.phg.trace_batch(vol, seed_pos, seed_dir, params,
 *                             at_cap=None, live_counts=None, near_occ=None)
 *   (/root/reference/pkg/src/strandkit/phg.py:67-163)
 * and its sampler
 *   strandkit.volume.sample_orientation_batch(vol, pts, prev_dirs)
 *   (/root/reference/pkg/src/strandkit/volume.py:183-224).
 * The reference has no FFI of its own (pure Python); the binding a maintainer
 * adds is a ctypes stub that replaces the module attribute
 * strandkit.phg.trace_batch, which every caller resolves at call time
 * (phg.py:233,240,283,288).
 *
 * Conventions: plain pointers and sizes only.  Every array pointer may be a
 * HOST pointer (pageable or pinned) or a DEVICE pointer of the field's GPU;
 * the library detects which and stages host data itself.  `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  Functions never
 * throw; they return a phg_status and phg_last_error() describes the failure
 * (thread-local).  Arithmetic is IEEE binary64 in the reference's own
 * evaluation order, so results are bit-identical to the reference.
 */
#ifndef PHG_B200_H
#define PHG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PHG_ABI_VERSION 2 /* 2: phg_params_v1.max_turn_cos, phg_trace_rows */

typedef enum {
    PHG_OK = 0,
    PHG_ERR_INVALID = 1,  /* bad argument / shape     -> strandkit DataError / ConfigError */
    PHG_ERR_CUDA = 2,     /* CUDA runtime failure     -> strandkit PipelineError */
    PHG_ERR_OOM = 3,      /* device allocation failed -> strandkit PipelineError */
    PHG_ERR_CAPACITY = 4, /* caller output buffer too small (required size reported) */
    PHG_ERR_STATE = 5     /* call order violated (e.g. gather before trace) */
} phg_status;

/* Packed, device-resident orientation/occupancy field (OOVolume, volume.py:21-56). */
typedef struct phg_field phg_field;
/* Per-caller context: scratch memory and the result of the last trace. */
typedef struct phg_ctx phg_ctx;

/* Trace parameters: the trace-relevant subset of PhgParams (phg.py:24-43). */
typedef struct {
    double step_mm;       /* PhgParams.step_mm */
    double min_support;   /* PhgParams.min_support */
    double steer;         /* PhgParams.steer (used only when a near-occupancy map is set) */
    int32_t max_vertices; /* PhgParams.max_vertices (>= 1) */
    int32_t probe_steps;  /* PhgParams.probe_steps */
    int32_t coast_steps;  /* PhgParams.coast_steps */
    uint32_t flags;       /* PHG_FLAG_* */
    double max_turn_cos;  /* with PHG_FLAG_TURN_STOP: cos of the largest turn a step may make */
} phg_params_v1;

#define PHG_FLAG_STRICT 0x1u   /* PhgParams.strict: lockstep per-step commits to live_counts */
#define PHG_FLAG_NO_ORDER 0x2u /* disable the locality (Morton) seed ordering; output order is
                                  seed order either way */
#define PHG_FLAG_TURN_STOP 0x4u /* opt-in angle stop, NOT in the reference (whose stop tests are
                                   phg.py:119-142): a step whose direction d' has
                                   dot(d, d') < max_turn_cos against the previous step direction d
                                   ends the strand before appending, like the bounds test */

/* ---- field (replaces the OOVolume arrays read by volume.py:205-212) ---------- */

/* ori: (nx,ny,nz,3) float32 C-order; occ: (nx,ny,nz) bool/uint8.  Copied and packed
 * to float4 (ori.xyz, occ) on the current device. nx*ny*nz must be < 2^32. */
phg_status phg_field_create(phg_field** out, const float* ori, const uint8_t* occ, int64_t nx,
                            int64_t ny, int64_t nz, const double origin[3], double voxel_size,
                            void* stream);
/* at_cap: (nx,ny,nz) bool plane (phg.py:236) or NULL to clear.  Stored as a 1-bit plane. */
phg_status phg_field_set_cap(phg_field* f, const uint8_t* at_cap, void* stream);
/* near_occ: (nx,ny,nz,3) int64 nearest-occupied map (phg.py:57-64) or NULL to clear. */
phg_status phg_field_set_near(phg_field* f, const int64_t* near_occ, void* stream);
phg_status phg_field_destroy(phg_field* f);
/* dims / device of a field (for callers' validation) */
phg_status phg_field_info(const phg_field* f, int64_t dims[3], int* device);

/* ---- field replication across GPUs (multi-GPU setup) -------------------------
 * The packed field is one device buffer plus two scalars, so ranks can replicate it with one
 * broadcast over NVLink instead of each rank uploading and packing the host arrays.
 * phg_field_packed: the padded packed voxel buffer (device pointer, bytes) and its flags.
 * phg_field_create_packed: a field of the given geometry whose packed buffer the caller then
 *   fills (e.g. the NCCL broadcast of another rank's phg_field_packed buffer), followed by
 *   phg_field_packed_done (derived structures: the block sign bounds in the voxels' low .w
 *   bits, recomputed from the buffer, and the optional bricked copy).  The buffer format is
 *   this library build's own; it is meant for replication between ranks running the same
 *   build. */
phg_status phg_field_packed(const phg_field* f, void** vox, int64_t* bytes, int32_t* zeroed,
                            float* maxabs);
phg_status phg_field_create_packed(phg_field** out, int64_t nx, int64_t ny, int64_t nz,
                                   const double origin[3], double voxel_size, int32_t zeroed,
                                   float maxabs, void* stream);
phg_status phg_field_packed_done(phg_field* f, void* stream);

/* ---- context ---------------------------------------------------------------- */
phg_status phg_ctx_create(phg_ctx** out);
phg_status phg_ctx_destroy(phg_ctx* c);

/* ---- trace (replaces trace_batch, phg.py:67-163) ----------------------------
 * Phase 1: trace n seeds.  seed_pos/seed_dir: (n,3) float64.  live_counts:
 * (nx,ny,nz) uint16, read and updated in place in strict mode (phg.py:150-154),
 * ignored otherwise (may be NULL; strict mode then starts from zeros).
 * Writes offsets (n+1) int64 (CSR row starts of the kept vertices, phg.py:159-162)
 * and entered (n) uint8, and returns the total kept vertex count in *n_verts_out.
 * Blocks until *n_verts_out is known (offsets/entered copies are complete on return). */
phg_status phg_trace(phg_ctx* c, const phg_field* f, const phg_params_v1* p,
                     const double* seed_pos, const double* seed_dir, int64_t n,
                     uint16_t* live_counts, int64_t* offsets, uint8_t* entered,
                     int64_t* n_verts_out, void* stream);
/* Phase 2: write the kept vertices of the last phg_trace on this context as a
 * (n_verts,3) float64 CSR payload.  verts_cap is in vertices. Blocks when verts is host memory. */
phg_status phg_gather(phg_ctx* c, double* verts, int64_t verts_cap, void* stream);

/* Device-resident strand rows: the reference's own trace buffer `buf` (N, max_vertices, 3)
 * (phg.py:85) with its per-seed `keep` (phg.py:159-161), i.e. strand i's vertices are
 *   rows[row(i) * row_stride .. + 3 * lengths[i]]   (f64 x,y,z; row(i) = rowmap ? rowmap[i] : i)
 * which is exactly buf[i, :keep] -- the array trace_batch returns for seed i, without the
 * per-strand copy into a list (phg.py:162) or our CSR gather.  Every pointer is device memory
 * owned by the context and valid until the next trace on it. */
typedef struct {
    const double* rows;        /* strand rows, row_stride doubles apart */
    const int32_t* rowmap;     /* (n) row of seed i, or NULL: row i */
    const int64_t* lengths;    /* (n) kept vertex count of seed i (len(vertices_i)) */
    const uint8_t* entered;    /* (n) entered flag of seed i */
    int64_t row_stride;        /* doubles per row: max_vertices rounded up to 4, times 3 */
    int64_t n;                 /* seeds */
    const uint64_t* counters;  /* device: [0] accepted steps (vertices appended before the
                                  trailing-coast trim), [1] sum of lengths (kept vertices) */
} phg_rows_v1;

/* Trace n seeds into device-resident strand rows (relaxed mode, phg_field's cap plane as in
 * phg_trace).  Asynchronous: enqueues the locality sort and the trace kernel on `stream` and
 * returns without waiting; `out` is filled at once, its contents are ready when the stream
 * reaches them.  Seeds may be host or device memory (host seeds are staged synchronously).
 * The sum of lengths minus n is the reference's step count sum(len(vertices) - 1). */
phg_status phg_trace_rows(phg_ctx* c, const phg_field* f, const phg_params_v1* p,
                          const double* seed_pos, const double* seed_dir, int64_t n,
                          phg_rows_v1* out, void* stream);

/* End-to-end variant of phg_trace + phg_gather for HOST seeds and HOST outputs: seeds are
 * traced in chunks of `chunk` (<= 0: n/8, at least 131072) and the D2H copy of chunk k's
 * vertices (on an internal copy stream) overlaps the device work of chunk k+1.  offsets
 * (n+1) i64, entered (n) u8, verts (verts_cap,3) f64: pinned host memory gives the overlap.
 * Relaxed mode only (strict mode couples all seeds per step).  If the vertices exceed
 * verts_cap, returns PHG_ERR_CAPACITY with the required count in *n_verts_out (offsets and
 * entered are still written). */
phg_status phg_trace_to_host(phg_ctx* c, const phg_field* f, const phg_params_v1* p,
                             const double* seed_pos, const double* seed_dir, int64_t n,
                             int64_t chunk, int64_t* offsets, uint8_t* entered, double* verts,
                             int64_t verts_cap, int64_t* n_verts_out, void* stream);

/* ---- rank-order concatenation on one GPU over peer memory (multi-GPU) -------
 * The CSR gather of the last phg_trace, fused with the concatenation on the root GPU: the
 * gather kernel writes this rank's strands straight into the root's global CSR (peer memory
 * over NVLink, opened with phg_ipc_open) at the rank's global bases, so the "gather to root"
 * collective costs no separate copy.
 * phg_gather_to: verts/offsets/entered are the GLOBAL buffers ((M,3) f64, (N+1) i64, (N) u8,
 *   device or peer memory); vert_base / strand_base this rank's place in them (exclusive
 *   sums of the ranks before it).  Enqueued on `stream`.
 * phg_ipc_alloc / phg_ipc_free: a device buffer whose CUDA IPC handle (64 bytes) other
 *   processes open with phg_ipc_open (a device pointer to the same memory; phg_ipc_close). */
phg_status phg_gather_to(phg_ctx* c, double* verts, int64_t* offsets, uint8_t* entered,
                         int64_t vert_base, int64_t strand_base, void* stream);
phg_status phg_ipc_alloc(int64_t bytes, void** dev_ptr, uint8_t handle[64]);
phg_status phg_ipc_free(void* dev_ptr);
phg_status phg_ipc_open(const uint8_t handle[64], void** dev_ptr);
phg_status phg_ipc_close(void* dev_ptr);

/* Checked build only (libphg_b200_checked.so, compiled with PHG_CHECKED; the stand-in for
 * compute-sanitizer): waits for the device, then reports device-side index-check violations
 * of the hot kernels (with the first failing check's site id) and the number of live library
 * buffers whose canary guards (4 KiB before and after every allocation) were overwritten.
 * A release build returns PHG_ERR_STATE. */
phg_status phg_debug_checks(int64_t* dcheck_violations, int64_t* first_site,
                            int64_t* guard_violations);
/* 1 in the checked build, else 0 */
int phg_is_checked_build(void);

/* Accepted integration steps of the last phg_trace, phg_trace_rows (waits for its stream) or
 * phg_trace_to_host call on the context:
 * one total over all strands (sum of vertices appended, before the trailing-coast trim). */
phg_status phg_last_steps(phg_ctx* c, int64_t* total_steps);

/* ---- device batch driver (replaces init_guide_strands, phg.py:210-260, with
 * _trace_field_seeds, phg.py:263-303) ---------------------------------------------------- */
typedef struct {
    int32_t batch_size;    /* PhgParams.batch_size: seeds per deferred-commit batch */
    int32_t occupancy_cap; /* PhgParams.occupancy_cap: at_cap = counts >= cap (phg.py:236) */
    int32_t field_seeds;   /* PhgParams.field_seeds: 0 disables the field pass */
    int32_t reserved;
} phg_grow_params_v1;

/* Scalp seeds/normals (n,3) f64 (scalp.seeds / scalp.seed_normals); counts: (nx,ny,nz)
 * uint16 vol.counts, read and updated in place exactly as the reference updates it.  The
 * segments stay on the context: *n_segments strands, *n_verts vertices.  report =
 * {n_never_entered, n_scalp_segments, n_field_seeds_traced, n_field_segments}.
 * The field's cap plane is consumed (cleared on return). */
phg_status phg_grow_init(phg_ctx* c, phg_field* f, const phg_params_v1* p,
                         const phg_grow_params_v1* g, const double* seeds, const double* normals,
                         int64_t n, uint16_t* counts, int64_t* n_segments, int64_t* n_verts,
                         int64_t report[4], void* stream);
/* The same driver as batch-level steps, for callers that interleave their own work between
 * deferred-commit batches (the multi-GPU driver exchanges commits between ranks):
 *   phg_grow_begin         load vol.counts, reset the session
 *   phg_grow_scalp_batch   one batch of scalp seeds (phg.py:229-251) -> out = {segments
 *                          added, commit ids exported}; export_commits=0 commits directly
 *   phg_grow_field_begin   select the field seeds from the current counts (phg.py:266-275)
 *   phg_grow_field_batch   field seeds [first, first+nb): +d / -d traces, join, keep, commit
 *   phg_grow_commits       copy the last batch's exported commit ids (one per segment and
 *                          distinct voxel; u32 linear voxel index)
 *   phg_grow_apply         counts[id] += 1 for each id (the union of all ranks' exports)
 *   phg_grow_end           write vol.counts back, finish the segment set (-> phg_grow_fetch,
 *                          phg_link with offsets == NULL) */
phg_status phg_grow_begin(phg_ctx* c, phg_field* f, const phg_params_v1* p,
                          const phg_grow_params_v1* g, const uint16_t* counts, void* stream);
phg_status phg_grow_scalp_batch(phg_ctx* c, const double* seeds, const double* normals,
                                int64_t nb, int32_t export_commits, int64_t out[2], void* stream);
phg_status phg_grow_field_begin(phg_ctx* c, int64_t* n_field_seeds, void* stream);
phg_status phg_grow_field_batch(phg_ctx* c, int64_t first, int64_t nb, int32_t export_commits,
                                int64_t out[2], void* stream);
phg_status phg_grow_commits(phg_ctx* c, uint32_t* ids, void* stream);
phg_status phg_grow_apply(phg_ctx* c, const uint32_t* ids, int64_t n, void* stream);
phg_status phg_grow_end(phg_ctx* c, uint16_t* counts, int64_t* n_segments, int64_t* n_verts,
                        int64_t report[4], void* stream);

/* Segments of the last phg_grow_init in order (scalp segments in seed order, then field
 * segments): offsets (n_segments+1) i64, verts (n_verts,3) f64, rooted (n_segments) u8
 * (1 = Strand(rooted=True, source="traced"), 0 = Strand(rooted=False, source="field")).
 * Any pointer may be NULL (skipped); host or device memory. */
phg_status phg_grow_fetch(phg_ctx* c, int64_t* offsets, double* verts, uint8_t* rooted,
                          void* stream);

/* ---- linking + attachment (replaces compute_links / connect_segments, phg.py:337-413,
 * attach_to_scalp, phg.py:419-439, and the tangents of grow, phg.py:467-468) ------------- */
typedef struct {
    double link_dist_mm;     /* PhgParams.link_dist_mm */
    double link_cos_gate;    /* np.cos(np.deg2rad(link_angle_deg)) computed by the caller */
    double smooth_strength;  /* PhgParams.smooth_strength */
    double step_mm;          /* PhgParams.step_mm (resampling step) */
    double attach_radius_mm; /* PhgParams.attach_radius_mm */
    int32_t tangent_window;  /* PhgParams.tangent_window */
    int32_t smooth;          /* PhgParams.smooth */
    int32_t smooth_iters;    /* PhgParams.smooth_iters */
    int32_t attach;          /* 1: attach_to_scalp with the given scalp vertices; 0: skip */
} phg_link_params_v1;

/* Segments as CSR (offsets (n+1) i64, verts f64, rooted u8, source u8 with 0 traced, 1 field,
 * 2 linked, 3 attached) -- or offsets == NULL to take the last phg_grow_init result of the
 * context.  scalp: (n_scalp,3) f64 scalp.vertices (attach only).  Results stay on the context;
 * counts_out = {n_strands, n_verts, n_links, n_unrooted}. */
phg_status phg_link(phg_ctx* c, const int64_t* offsets, const double* verts,
                    const uint8_t* rooted, const uint8_t* source, int64_t n,
                    const double* scalp, int64_t n_scalp, const phg_link_params_v1* lp,
                    int64_t counts_out[4], void* stream);
/* Strands of the last phg_link: offsets (n_strands+1), verts / tangents (n_verts,3) f64,
 * rooted / source (n_strands) u8, links (n_links,2) i64 in acceptance order.  NULL skips. */
phg_status phg_link_fetch(phg_ctx* c, int64_t* offsets, double* verts, double* tangents,
                          uint8_t* rooted, uint8_t* source, int64_t* links, void* stream);

/* ---- wire formats ------------------------------------------------------------------
 * STND image (write_strands, strands.py:63-69) of a CSR strand set: u32 magic 0x444E5453,
 * u32 count, per strand u32 n + n*3 float32 (vertices rounded to nearest).  `out` must hold
 * 8 + 4*n_strands + 12*offsets[n_strands] bytes; host or device pointers. */
phg_status phg_stnd_encode(const int64_t* offsets, const double* verts, int64_t n_strands,
                           uint8_t* out, void* stream);
/* Field straight from an OOVL payload (read_volume, volume.py:248-266): bits =
 * np.packbits(occ) ((nx*ny*nz+7)/8 bytes, MSB first), ori_occupied = (n_occ,3) float32 of the
 * occupied voxels in C order.  PHG_ERR_INVALID if n_occ != number of set bits (truncated). */
phg_status phg_field_from_oovl(phg_field** out, const uint8_t* bits, const float* ori_occupied,
                               int64_t n_occ, int64_t nx, int64_t ny, int64_t nz,
                               const double origin[3], double voxel_size, void* stream);

/* ---- sampler (replaces sample_orientation_batch, volume.py:183-224) --------- */
phg_status phg_sample(const phg_field* f, const double* pts, const double* prev, int64_t n,
                      double* dirs, uint8_t* has, double* support, void* stream);

/* ---- diagnostics -------------------------------------------------------------- */
const char* phg_last_error(void);
int phg_abi_version(void);
/* device time (ms) of the last trace kernel launch on this context (CUDA events on `stream`) */
phg_status phg_last_kernel_ms(phg_ctx* c, float* trace_ms, float* total_ms);
/* name of the trace-kernel variant the last trace used (env PHG_VARIANT=<index> selects one;
 * all variants are bit-identical) and the number of compiled variants */
const char* phg_last_variant(phg_ctx* c);
/* sampler form the last trace used, chosen per field (all bit-identical): "exact" (a field
 * with non-finite ori, steering, strict mode), "fast" (all ori finite: zeroed padded field),
 * "fast-pow2" (and a power-of-two voxel size) */
const char* phg_last_sampler(phg_ctx* c);
/* device self-test of the arithmetic building blocks: runs n randomized and edge-case
 * operand pairs through the kernel's shared-reciprocal division and the compiler's own
 * IEEE division and reports how many results differ bitwise (must be 0) */
phg_status phg_selftest(int64_t n, uint64_t seed, int64_t* mismatches, void* stream);
int phg_num_variants(void);

#ifdef __cplusplus
}
#endif
#endif /* PHG_B200_H */
