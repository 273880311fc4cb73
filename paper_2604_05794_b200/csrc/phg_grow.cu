// phg_grow.cu -- device batch driver: strandkit.phg.init_guide_strands on the GPU.
//
// Reference: /root/reference/pkg/src/strandkit/phg.py
//   init_guide_strands   :210-260  scalp seeds in deferred-commit batches; per batch the frozen
//                                  at_cap = counts >= occupancy_cap (:236), trace, keep segments
//                                  with entered && len >= 2 (:242-246), commit each segment's
//                                  unique in-bounds voxels to counts (:247-251)
//   _trace_field_seeds   :263-303  occupied voxels with counts == 0 (:266) strided to field_seeds
//                                  (:269-271), centres + unit ori (:272-275), per batch trace +d
//                                  and -d (:291-292), join reverse(bwd) + fwd[1:] (:294), keep
//                                  len >= 4 and (ef or eb) (:295), commit (:298-302)
//   strict mode                    per-step commits inside the trace, no segment commits
// Kernels here: cap_from_counts (at_cap bit plane), segment_select, commit_kernel (per-segment
// set of voxels via a warp-private shared-memory hash set, then one atomicAdd per distinct
// voxel), gather_scalp / gather_joined (compaction into the output CSR), field-seed
// selection (CUB DeviceSelect + numpy-exact linspace striding).

#include <thrust/iterator/counting_iterator.h>

#include "phg_core.cuh"

using namespace phg;

namespace phg {
namespace {

constexpr int kCommitWarps = 4;  // warps per CTA of the commit kernel

// at_cap = counts >= cap with vol.counts' uint16 semantics, packed 32 voxels per word
__global__ void cap_from_counts_kernel(const uint32_t* __restrict__ counts, long long nvox,
                                       uint32_t cap, uint32_t* __restrict__ bits) {
    const long long nwords = (nvox + 31) / 32;
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long w = warp; w < nwords; w += nwarps) {
        const long long i = w * 32 + lane;
        const bool b = i < nvox && (counts[i] & 0xffffu) >= cap;
        const unsigned m = __ballot_sync(kFull, b);
        if (lane == 0) bits[w] = m;
    }
}

// scalp segments: valid = entered && len >= 2 (phg.py:243); lens zeroed for invalid ones
__global__ void segment_select_kernel(const long long* __restrict__ keep,
                                      const uint8_t* __restrict__ entered, long long n,
                                      long long* __restrict__ lens, long long* __restrict__ segf,
                                      uint8_t* __restrict__ valid,
                                      unsigned long long* __restrict__ never_entered) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool v = entered[i] && keep[i] >= 2;
    lens[i] = v ? keep[i] : 0;
    segf[i] = v ? 1 : 0;
    valid[i] = v ? 1 : 0;
    if (!entered[i]) atomicAdd(never_entered, 1ull);
}

// field segments: joined length (phg.py:294) and validity (phg.py:295)
__global__ void join_select_kernel(const long long* __restrict__ keep_f,
                                   const uint8_t* __restrict__ ent_f,
                                   const long long* __restrict__ keep_b,
                                   const uint8_t* __restrict__ ent_b, long long n,
                                   long long* __restrict__ lens, long long* __restrict__ segf,
                                   uint8_t* __restrict__ valid) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long lf = keep_f[i], lb = keep_b[i];
    const long long L = lb > 1 ? lb + lf - 1 : lf;
    const bool v = L >= 4 && (ent_f[i] || ent_b[i]);
    lens[i] = v ? L : 0;
    segf[i] = v ? 1 : 0;
    valid[i] = v ? 1 : 0;
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t lin, int bits) {
    return (lin * 2654435761u) >> (32 - bits);
}

// Insert lin into the warp's set; true if it was not present.  Entries are (epoch << 32 | lin);
// entries of older epochs count as empty, so the table is never cleared between segments.
__device__ __forceinline__ bool set_insert(unsigned long long* T, int bits, uint32_t epoch,
                                           uint32_t lin) {
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t h = hash_slot(lin, bits);
    const unsigned long long mine = ((unsigned long long)epoch << 32) | lin;
    while (true) {
        const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(T + h);
        if ((uint32_t)(cur >> 32) == epoch) {
            if ((uint32_t)cur == lin) return false;
            h = (h + 1) & mask;
            continue;
        }
        const unsigned long long old = atomicCAS(T + h, cur, mine);
        if (old == cur) return true;
        // another lane claimed this slot first: re-examine it
    }
}

// counts[lin] += 1, keeping the at_cap plane (counts >= cap, phg.py:236) current
// incrementally: without uint16 wrap-around counts only grow, so a voxel turns "at cap" exactly
// when its count reaches cap; a wrap raises `wrapped`, which forces a full rebuild
__device__ __forceinline__ void bump_count(uint32_t* __restrict__ counts,
                                           uint32_t* __restrict__ cap_bits, uint32_t cap,
                                           unsigned int* __restrict__ wrapped, uint32_t lin) {
    const uint32_t now = (atomicAdd(counts + lin, 1u) + 1u) & 0xffffu;
    if (now == cap) atomicOr(cap_bits + (lin >> 5), 1u << (lin & 31));
    if (now == 0u) atomicOr(wrapped, 1u);
}

// Where a segment's distinct voxels go: straight into counts (one rank), or appended to an
// export list that every rank applies after an all-gather (multi-rank driver).
struct CommitSink {
    uint32_t* counts;
    uint32_t* cap_bits;
    uint32_t cap;
    unsigned int* wrapped;
    uint32_t* export_ids;                 // nullptr: commit directly
    unsigned long long* export_cursor;
};

// Add the vertices of one slab row to the warp's set; commit newly seen in-bounds voxels.
__device__ __forceinline__ void commit_row(const FieldView& F, const double* __restrict__ row,
                                           long long L, unsigned long long* T, int bits,
                                           uint32_t epoch, const CommitSink& K, int lane) {
    // the next pass's vertex is loaded before this pass's hash insert and atomics, so the load
    // latency overlaps them
    double nx_ = 0.0, ny_ = 0.0, nz_ = 0.0;
    if (lane < L) {
        nx_ = row[3 * lane + 0];
        ny_ = row[3 * lane + 1];
        nz_ = row[3 * lane + 2];
    }
    for (long long k = lane; k < L; k += 32) {
        const double px = nx_, py = ny_, pz = nz_;
        if (k + 32 < L) {
            nx_ = row[3 * (k + 32) + 0];
            ny_ = row[3 * (k + 32) + 1];
            nz_ = row[3 * (k + 32) + 2];
        }
        // vol.voxel_of (volume.py:42-45) and in_bounds (:47-49)
        const int vx = floor_idx(grid_coord(F, px - F.ox));
        const int vy = floor_idx(grid_coord(F, py - F.oy));
        const int vz = floor_idx(grid_coord(F, pz - F.oz));
        if ((unsigned)vx < (unsigned)F.nx && (unsigned)vy < (unsigned)F.ny &&
            (unsigned)vz < (unsigned)F.nz) {
            const uint32_t lin = ((uint32_t)vx * F.ny + vy) * F.nz + vz;
            if (set_insert(T, bits, epoch, lin)) {
                if (K.export_ids)
                    K.export_ids[atomicAdd(K.export_cursor, 1ull)] = lin;
                else
                    bump_count(K.counts, K.cap_bits, K.cap, K.wrapped, lin);
            }
        }
    }
}

// apply exported commits (all ranks' lists): counts[id] += 1 for each id
__global__ void apply_commits_kernel(const uint32_t* __restrict__ ids, long long n,
                                     uint32_t* __restrict__ counts, uint32_t* __restrict__ cap_bits,
                                     uint32_t cap, unsigned int* __restrict__ wrapped) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        bump_count(counts, cap_bits, cap, wrapped, ids[i]);
}

// undo exported commits (rollback of an optimistic window): counts[id] -= 1
__global__ void uncommit_kernel(const uint32_t* __restrict__ ids, long long n,
                                uint32_t* __restrict__ counts) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        atomicSub(counts + ids[i], 1u);
}

// sum of the appended vertex counts of a traced window (bounds its kept vertices)
__global__ void sum_nverts_kernel(const int32_t* __restrict__ nv, long long n,
                                  unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc += (unsigned long long)nv[i];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// device output totals of asynchronous posts: dtot = {segments, vertices}
__global__ void set_totals_kernel(long long* dtot, long long segs, long long verts) {
    dtot[0] = segs;
    dtot[1] = verts;
}
__global__ void advance_totals_kernel(long long* dtot, const long long* __restrict__ sidx_end,
                                      const long long* __restrict__ voff_end) {
    dtot[0] += *sidx_end;
    dtot[1] += *voff_end;
}

// vol.counts[unique voxels of each valid segment] += 1 (phg.py:248-251, :299-302).  One warp per
// segment; for joined field segments the set spans both traces (voxels(bwd) U voxels(fwd)).
// GLOBAL_TABLE: the per-warp table lives in global memory (very long segments).
template <bool GLOBAL_TABLE>
__global__ void commit_kernel(FieldView F, Rows slab_a, const long long* __restrict__ keep_a,
                              Rows slab_b, const long long* __restrict__ keep_b,
                              const uint8_t* __restrict__ valid, long long n,
                              CommitSink K, int bits, unsigned long long* __restrict__ gtables) {
    extern __shared__ unsigned long long smem_tables[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const long long gwarp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long* T = GLOBAL_TABLE ? gtables + ((size_t)gwarp << bits)
                                         : smem_tables + ((size_t)wib << bits);
    for (long long j = lane; j < (1ll << bits); j += 32) T[j] = 0ull;  // epoch 0 = empty
    __syncwarp();
    uint32_t epoch = 0;
    for (long long i = gwarp; i < n; i += nwarps) {
        if (!valid[i]) continue;
        ++epoch;
        commit_row(F, slab_a.row(i), keep_a[i], T, bits, epoch, K, lane);
        if (slab_b.base) commit_row(F, slab_b.row(i), keep_b[i], T, bits, epoch, K,
                               lane);
        __syncwarp();
    }
}

// scalp segments -> output CSR (rows of valid strands, in seed order)
__global__ void gather_scalp_kernel(Rows slab,
                                    const long long* __restrict__ keep,
                                    const uint8_t* __restrict__ valid,
                                    const long long* __restrict__ voff,
                                    const long long* __restrict__ sidx, long long n,
                                    long long vbase, long long sbase, long long* __restrict__ out_off,
                                    double* __restrict__ out_v, uint8_t* __restrict__ rooted,
                                    const long long* __restrict__ dtot) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    if (dtot) {  // asynchronous posts: output bases kept on the device
        sbase = dtot[0];
        vbase = dtot[1];
    }
    for (long long i = warp; i < n; i += nwarps) {
        if (!valid[i]) continue;
        const long long o = vbase + voff[i];
        if (lane == 0) {
            out_off[sbase + sidx[i]] = o;
            rooted[sbase + sidx[i]] = 1;
        }
        copy_strand(slab.row(i), out_v + o * 3, keep[i] * 3, lane);
    }
}

// field segments: v = concat(bwd[::-1], fwd[1:]) if len(bwd) > 1 else fwd (phg.py:294)
__global__ void gather_joined_kernel(Rows slab_f, Rows slab_b,
                                     const long long* __restrict__ keep_f,
                                     const long long* __restrict__ keep_b,
                                     const uint8_t* __restrict__ valid,
                                     const long long* __restrict__ voff,
                                     const long long* __restrict__ sidx, long long n,
                                     long long vbase, long long sbase,
                                     long long* __restrict__ out_off, double* __restrict__ out_v,
                                     uint8_t* __restrict__ rooted,
                                     const long long* __restrict__ dtot) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    if (dtot) {
        sbase = dtot[0];
        vbase = dtot[1];
    }
    for (long long i = warp; i < n; i += nwarps) {
        if (!valid[i]) continue;
        const long long o = vbase + voff[i];
        if (lane == 0) {
            out_off[sbase + sidx[i]] = o;
            rooted[sbase + sidx[i]] = 0;
        }
        const double* f = slab_f.row(i);
        const double* b = slab_b.row(i);
        const long long lf = keep_f[i], lb = keep_b[i];
        double* dst = out_v + o * 3;
        if (lb > 1) {
            for (long long j = lane; j < lb * 3; j += 32) {  // reversed vertex order
                const long long k = j / 3, c = j - 3 * k;
                dst[j] = b[3 * (lb - 1 - k) + c];
            }
            dst += lb * 3;
            for (long long j = lane; j < (lf - 1) * 3; j += 32) dst[j] = f[3 + j];
        } else {
            copy_strand(f, dst, lf * 3, lane);
        }
    }
}

// unvisited = argwhere(occ & (counts == 0)) (phg.py:266): flag per voxel
__global__ void unvisited_flag_kernel(FieldView F, const uint32_t* __restrict__ counts,
                                      long long nvox, uint8_t* __restrict__ flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x)
        flag[i] = (occ_live(F.vox[vox_index_lin(F, (uint32_t)i)].w) && (counts[i] & 0xffffu) == 0u)
                      ? 1
                      : 0;
}

// unvisited[np.linspace(0, U - 1, m).astype(np.int64)] (phg.py:269-271), numpy-exact:
// y_k = k * ((U-1)/(m-1)) + 0.0 truncated toward zero, last element = U - 1
__global__ void stride_pick_kernel(const uint32_t* __restrict__ unvisited, long long U, long long m,
                                   uint32_t* __restrict__ picked) {
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= m) return;
    long long idx;
    if (m == 1) {
        idx = 0;
    } else if (k == m - 1) {
        idx = U - 1;
    } else {
        const double step = (double)(U - 1) / (double)(m - 1);
        idx = (long long)((double)k * step + 0.0);
    }
    picked[k] = unvisited[idx];
}

// centres + unit ori of the picked voxels, dropping |ori| <= 1e-9 (phg.py:272-275)
__global__ void field_seed_kernel(FieldView F, const uint32_t* __restrict__ lin, long long m,
                                  double* __restrict__ pos, double* __restrict__ dir,
                                  uint8_t* __restrict__ keepf) {
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const uint32_t l = lin[k];
    const uint32_t z = l % (uint32_t)F.nz, y = (l / (uint32_t)F.nz) % (uint32_t)F.ny,
                   x = l / ((uint32_t)F.nz * (uint32_t)F.ny);
    // vol.centers: origin + (idx + 0.5) * voxel_size
    pos[3 * k + 0] = F.ox + ((double)x + 0.5) * F.vs;
    pos[3 * k + 1] = F.oy + ((double)y + 0.5) * F.vs;
    pos[3 * k + 2] = F.oz + ((double)z + 0.5) * F.vs;
    const float4 v = F.vox[vox_index(F, (int)x, (int)y, (int)z)];
    double ox = (double)v.x, oy = (double)v.y, oz = (double)v.z;
    const double n = nrm3(ox, oy, oz);
    keepf[k] = (n > 1e-9) ? 1 : 0;
    scale_unit(ox, oy, oz, n);  // geom.normalize
    dir[3 * k + 0] = ox;
    dir[3 * k + 1] = oy;
    dir[3 * k + 2] = oz;
}

__global__ void row_gather_kernel(const double* __restrict__ src_pos,
                                  const double* __restrict__ src_dir,
                                  const uint32_t* __restrict__ rows, long long n,
                                  double* __restrict__ pos, double* __restrict__ dir) {
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t r = rows[k];
    for (int c = 0; c < 3; ++c) {
        pos[3 * k + c] = src_pos[3 * (size_t)r + c];
        dir[3 * k + c] = src_dir[3 * (size_t)r + c];
    }
}

__global__ void negate_kernel(const double* __restrict__ a, double* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = -1.0 * a[i];  // sign * db with sign = -1.0 (phg.py:288,292)
}

__global__ void u16_to_u32(const uint16_t* __restrict__ a, uint32_t* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}

__global__ void u32_to_u16(const uint32_t* __restrict__ a, uint16_t* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = (uint16_t)(a[i] & 0xffffu);
}

void swap_buf(DevBuf& a, DevBuf& b) { a.swap(b); }

// ---- speculative deferred-commit batches ------------------------------------------------------
// Every batch of a phase is traced in ONE launch against the cap plane P0 at the start of the
// phase; batch b must see the plane P_b after batches < b committed (phg.py:236).  Counts only
// grow (a uint16 wrap ends the speculation), so P0 is a subset of P_b, and a cap probe
// differs between the two planes only where P_b holds a voxel P0 did not -- there the strand
// dies instead of continuing (phg.py:140-142).  Up to its first such probe the strand is the
// same under both planes, so its exact trace under P_b is the speculative one truncated there.
//
// A probe is a step that appends vertex t while entered (some step <= t was supported,
// phg.py:127) into a voxel other than that of vertex t-1 (t = 1: always; phg.py:139, the
// trace kernel's new_vox).  Truncating at t keeps vertices [0, t) and, the strand being
// entered, keep = max(last supported step <= t, 1) of them (phg.py:124, :158).  The trace kernel
// records which appended steps were supported (TraceRecord); vertex cells are recomputed from
// the slab with the kernel's own arithmetic.  One warp per strand, 32 vertices per pass.
__global__ void spec_truncate_kernel(FieldView F, Rows slab,
                                     const uint32_t* __restrict__ bits, int words,
                                     const int32_t* __restrict__ nverts, long long n,
                                     long long* __restrict__ keep) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < n; i += nwarps) {
        const int m = nverts[i];
        const double* row = slab.row(i);
        const uint32_t* b = bits + (size_t)i * words;
        // bit t (1 <= t < m) of the words: step t was supported; the first one enters
        int first_sup = INT_MAX;
        for (int w = 0; 32 * w < m && first_sup == INT_MAX; ++w) {
            uint32_t x = b[w];
            if (w == 0) x &= ~1u;
            const int valid = m - 32 * w;
            if (valid < 32) x &= (1u << valid) - 1u;
            if (x) first_sup = 32 * w + __ffs(x) - 1;
        }
        if (first_sup == INT_MAX) continue;  // never entered: no cap probes at all
        int cut = -1;
        uint32_t carry = 0xffffffffu;  // cell of the last vertex of the previous pass
        for (int base = 0; base < m && cut < 0; base += 32) {
            const int t = base + lane;
            const bool step = t >= 1 && t < m;
            uint32_t lin = 0xffffffffu;
            if (step) {
                const int vx = floor_sat(grid_coord(F, row[3 * t + 0] - F.ox));
                const int vy = floor_sat(grid_coord(F, row[3 * t + 1] - F.oy));
                const int vz = floor_sat(grid_coord(F, row[3 * t + 2] - F.oz));
                lin = ((uint32_t)vx * F.ny + vy) * F.nz + vz;
            }
            uint32_t prev = __shfl_up_sync(kFull, lin, 1);
            if (lane == 0) prev = carry;
            const bool probe = step && t >= first_sup && (t == 1 || lin != prev) &&
                               ((__ldg(F.cap + (lin >> 5)) >> (lin & 31)) & 1u);
            const unsigned hit = __ballot_sync(kFull, probe);
            if (hit) cut = base + __ffs(hit) - 1;
            carry = __shfl_sync(kFull, lin, 31);
        }
        if (cut < 0 || lane != 0) continue;
        int last = 1;  // strand_init's last_sup
        for (int w = cut >> 5; w >= 0; --w) {
            uint32_t x = b[w];
            if (w == 0) x &= ~1u;
            if (w == (cut >> 5) && (cut & 31) != 31) x &= (2u << (cut & 31)) - 1u;
            if (x) {
                last = 32 * w + 31 - __clz(x);
                break;
            }
        }
        keep[i] = last > 1 ? last : 1;
    }
}

// grow `b` to hold `need` bytes keeping its first `used` bytes
phg_status grow_keep(DevBuf& b, size_t used, size_t need, cudaStream_t st) {
    if (need <= b.cap) return PHG_OK;
    DevBuf nb;
    PHG_TRY(nb.ensure(std::max(need, b.cap * 2)));
    if (used) PHG_CUDA(cudaMemcpyAsync(nb.p, b.p, used, cudaMemcpyDeviceToDevice, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    swap_buf(b, nb);
    return PHG_OK;
}

// ---- the batch-driver session ---------------------------------------------------------------
// State of one init_guide_strands run, kept on the context between the batch-level entry points
// (phg_grow_begin .. phg_grow_end); phg_grow_init composes them for the single-GPU case.
struct GrowSession {
    phg_field* f = nullptr;
    phg_params_v1 p{};
    phg_grow_params_v1 g{};
    bool strict = false;
    uint32_t* counts = nullptr;  // device uint32 plane (vol.counts), c->counts32
    long long segs = 0, verts = 0, scalp_segs = 0, n_field = 0;
    DevBuf misc;                 // [0] never-entered scalp seeds, [1] (u32) count wrapped
    bool cap_valid = false;      // f->cap == (counts >= cap) for the current counts
    DevBuf export_ids;           // commits of the last batch (multi-rank mode)
    long long n_export = 0;
    long long nf_seeds = 0;      // field seeds selected by phg_grow_field_begin
    DevBuf dtot;                 // [0] segments, [1] vertices, [2] never-entered snapshot
};

struct GrowCtx {  // per-call view
    phg_ctx* c;
    GrowSession* s;
    cudaStream_t st;
};

phg_status set_cap_plane(GrowCtx& G) {
    GrowSession& S = *G.s;
    if (S.strict) {
        S.f->has_cap = false;
        return PHG_OK;
    }
    S.f->has_cap = true;
    if (S.cap_valid) return PHG_OK;  // maintained incrementally by the commits
    const long long V = S.f->nvox();
    PHG_TRY(S.f->cap.ensure((size_t)((V + 31) / 32) * 4));
    cap_from_counts_kernel<<<grid_for((V + 31) / 32 * 32, 256, num_sms() * 16), 256, 0, G.st>>>(
        S.counts, V, (uint32_t)S.g.occupancy_cap, S.f->cap.as<uint32_t>());
    PHG_CUDA(cudaGetLastError());
    S.cap_valid = true;
    return PHG_OK;
}

CommitSink direct_sink(GrowSession& S) {
    return CommitSink{S.counts, S.f->cap.as<uint32_t>(), (uint32_t)S.g.occupancy_cap,
                      (unsigned int*)(S.misc.as<unsigned long long>() + 1), nullptr, nullptr};
}

// rows of the last trace_core launch on the context
Rows slab_rows(const GrowCtx& G) {
    return Rows{G.c->slab.as<double>(), G.c->rows_by_queue ? G.c->rowmap.as<int32_t>() : nullptr,
                row_stride_doubles(G.s->p.max_vertices)};
}

phg_status launch_commit(GrowCtx& G, Rows slab_a, const long long* keep_a, Rows slab_b,
                         const long long* keep_b, const uint8_t* valid,
                         long long n, CommitSink K) {
    GrowSession& S = *G.s;
    const FieldView F = S.f->view();
    const long long max_entries = (long long)S.p.max_vertices * (slab_b.base ? 2 : 1);
    int bits = 6;
    while ((1ll << bits) < 2 * max_entries) ++bits;
    const size_t table_bytes = (size_t)8 << bits;
    // as many warps as the per-warp tables let an SM hold (up to 32): each warp walks a few
    // segments with a dependent load -> hash -> atomic chain, so warps in flight set the pace
    const bool smem_tables = table_bytes * kCommitWarps <= 200 * 1024;
    const int per_sm =
        smem_tables ? (int)std::max<size_t>(kCommitWarps, std::min<size_t>(32, (200 * 1024) / table_bytes))
                    : 16;
    const int warps_total = num_sms() * per_sm;
    const int blocks = std::max(1, std::min(warps_total / kCommitWarps,
                                            (int)((n + kCommitWarps - 1) / kCommitWarps)));
    if (smem_tables) {
        const size_t smem = table_bytes * kCommitWarps;
        PHG_CUDA(cudaFuncSetAttribute(commit_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        commit_kernel<false><<<blocks, 32 * kCommitWarps, smem, G.st>>>(
            F, slab_a, keep_a, slab_b, keep_b, valid, n, K, bits, nullptr);
    } else {
        PHG_TRY(G.c->g_hash.ensure(table_bytes * (size_t)blocks * kCommitWarps));
        commit_kernel<true><<<blocks, 32 * kCommitWarps, 0, G.st>>>(
            F, slab_a, keep_a, slab_b, keep_b, valid, n, K, bits,
            G.c->g_hash.as<unsigned long long>());
    }
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// commit a batch: directly, or (export) into S.export_ids for an all-gather by the caller
phg_status commit_batch(GrowCtx& G, Rows slab_a, const long long* keep_a, Rows slab_b,
                        const long long* keep_b, const uint8_t* valid,
                        long long n, long long max_ids, bool export_commits) {
    GrowSession& S = *G.s;
    S.n_export = 0;
    if (S.strict) return PHG_OK;  // strict mode commits inside the trace
    if (!export_commits) return launch_commit(G, slab_a, keep_a, slab_b, keep_b, valid, n,
                                              direct_sink(S));
    PHG_TRY(S.export_ids.ensure((size_t)std::max<long long>(max_ids, 1) * 4));
    unsigned long long* cursor = S.misc.as<unsigned long long>() + 2;
    PHG_CUDA(cudaMemsetAsync(cursor, 0, 8, G.st));
    CommitSink K = direct_sink(S);
    K.export_ids = S.export_ids.as<uint32_t>();
    K.export_cursor = cursor;
    PHG_TRY(launch_commit(G, slab_a, keep_a, slab_b, keep_b, valid, n, K));
    PHG_CUDA(cudaMemcpyAsync(G.c->host_total + 3, cursor, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    S.n_export = G.c->host_total[3];
    return PHG_OK;
}

// scans of lens / segment flags -> per-strand output offsets; returns batch totals (syncs)
phg_status batch_offsets(GrowCtx& G, long long n, long long* lens, long long* segf,
                         long long* voff, long long* sidx, long long* nv, long long* ns) {
    GrowSession& S = *G.s;
    PHG_TRY(scan_lengths(G.c, lens, n, voff, G.st));
    PHG_TRY(scan_lengths(G.c, segf, n, sidx, G.st));
    PHG_CUDA(cudaMemcpyAsync(G.c->host_total, voff + n, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaMemcpyAsync(G.c->host_total + 1, sidx + n, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaMemcpyAsync(G.c->host_total + 2, S.misc.as<unsigned long long>() + 1, 8,
                             cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    *nv = G.c->host_total[0];
    *ns = G.c->host_total[1];
    if (G.c->host_total[2]) {  // a count wrapped past 65535: rebuild the cap plane exactly
        S.cap_valid = false;
        PHG_CUDA(cudaMemsetAsync(S.misc.as<unsigned long long>() + 1, 0, 8, G.st));
    }
    return PHG_OK;
}

phg_status ensure_output(GrowCtx& G, long long add_segs, long long add_verts) {
    GrowSession& S = *G.s;
    PHG_TRY(grow_keep(G.c->g_out_off, (size_t)S.segs * 8, (size_t)(S.segs + add_segs + 1) * 8,
                      G.st));
    PHG_TRY(grow_keep(G.c->g_out_rooted, (size_t)S.segs, (size_t)(S.segs + add_segs + 1), G.st));
    PHG_TRY(grow_keep(G.c->g_out_verts, (size_t)S.verts * 24,
                      (size_t)(S.verts + add_verts + 1) * 24, G.st));
    return PHG_OK;
}

// per-batch scratch: lens, segment flags, their scans, validity
struct BatchScratch {
    long long *lens, *segf, *voff, *sidx;
    uint8_t* valid;
};

phg_status batch_scratch(GrowCtx& G, long long n, BatchScratch& B) {
    PHG_TRY(G.c->g_misc.ensure((size_t)(n + 1) * 8 * 4 + (size_t)n + 64));
    char* base = (char*)G.c->g_misc.p;
    B.lens = (long long*)base;
    B.segf = B.lens + (n + 1);
    B.voff = B.segf + (n + 1);
    B.sidx = B.voff + (n + 1);
    B.valid = (uint8_t*)(B.sidx + (n + 1));
    return PHG_OK;
}

// segments, commits and output of one traced batch of scalp seeds (phg.py:242-251)
phg_status scalp_post(GrowCtx& G, Rows slab, const long long* keep, const uint8_t* ent,
                      long long nb, bool export_commits, long long* segs_added) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    BatchScratch B;
    PHG_TRY(batch_scratch(G, nb, B));
    segment_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(
        keep, ent, nb, B.lens, B.segf, B.valid, S.misc.as<unsigned long long>());
    PHG_CUDA(cudaGetLastError());
    // direct commits go before the synchronising offsets step, which also picks up a uint16
    // wrap flag they may raise; exported commits need the batch size to size their list
    if (!export_commits)
        PHG_TRY(commit_batch(G, slab, keep, Rows{}, nullptr, B.valid, nb, 0, false));
    long long nv = 0, ns = 0;
    PHG_TRY(batch_offsets(G, nb, B.lens, B.segf, B.voff, B.sidx, &nv, &ns));
    if (export_commits)
        PHG_TRY(commit_batch(G, slab, keep, Rows{}, nullptr, B.valid, nb, nv, true));
    PHG_TRY(ensure_output(G, ns, nv));
    gather_scalp_kernel<<<grid_for(nb * 32, 256, num_sms() * kCopyCtasPerSm), 256, 0, G.st>>>(
        slab, keep, B.valid, B.voff, B.sidx, nb, S.verts,
        S.segs, c->g_out_off.as<long long>(), c->g_out_verts.as<double>(),
        c->g_out_rooted.as<uint8_t>(), nullptr);
    PHG_CUDA(cudaGetLastError());
    S.segs += ns;
    S.verts += nv;
    S.scalp_segs = S.segs;
    *segs_added = ns;
    return PHG_OK;
}

// one deferred-commit batch of scalp seeds (phg.py:229-251)
phg_status scalp_batch(GrowCtx& G, const double* d_pos, const double* d_dir, long long nb,
                       bool export_commits, long long* segs_added) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    *segs_added = 0;
    S.n_export = 0;
    if (nb == 0) return PHG_OK;
    PHG_TRY(set_cap_plane(G));
    PHG_TRY(trace_core(c, S.f, &S.p, d_pos, d_dir, nb, S.strict ? S.counts : nullptr, G.st,
                       nullptr, true));
    return scalp_post(G, slab_rows(G), c->keep.as<long long>(), c->entered.as<uint8_t>(),
                      nb, export_commits, segs_added);
}

// field seeds (phg.py:266-275): unvisited occupied voxels, strided, centres + unit ori
phg_status field_begin(GrowCtx& G) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    S.nf_seeds = 0;
    S.n_field = 0;
    const long long V = S.f->nvox();
    const FieldView F = S.f->view();
    long long* d_count = (long long*)c->counters.p + 4;
    thrust::counting_iterator<uint32_t> iota(0);
    PHG_TRY(c->g_flags.ensure((size_t)V));
    PHG_TRY(c->g_sel.ensure((size_t)V * 4));
    uint8_t* flags = c->g_flags.as<uint8_t>();
    uint32_t* unvisited = c->g_sel.as<uint32_t>();
    unvisited_flag_kernel<<<grid_for(V, 256, num_sms() * 16), 256, 0, G.st>>>(F, S.counts, V,
                                                                              flags);
    PHG_CUDA(cudaGetLastError());
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, iota, flags, unvisited, d_count, V, G.st);
    PHG_TRY(c->cub_tmp.ensure(tmp));
    PHG_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, flags, unvisited, d_count, V,
                                        G.st));
    PHG_CUDA(cudaMemcpyAsync(c->host_total, d_count, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    const long long U = c->host_total[0];
    if (U == 0 || S.g.field_seeds <= 0) return PHG_OK;
    long long m = U;
    const uint32_t* picked = unvisited;
    if (U > S.g.field_seeds) {
        m = S.g.field_seeds;
        PHG_TRY(c->g_pick.ensure((size_t)m * 4));
        stride_pick_kernel<<<grid_for(m, 256), 256, 0, G.st>>>(unvisited, U, m,
                                                                c->g_pick.as<uint32_t>());
        PHG_CUDA(cudaGetLastError());
        picked = c->g_pick.as<uint32_t>();
    }
    PHG_TRY(c->g_raw.ensure((size_t)m * 48 + (size_t)m));
    double* raw_pos = c->g_raw.as<double>();
    double* raw_dir = raw_pos + 3 * m;
    uint8_t* keepf = (uint8_t*)(raw_dir + 3 * m);
    field_seed_kernel<<<grid_for(m, 256), 256, 0, G.st>>>(F, picked, m, raw_pos, raw_dir, keepf);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(c->g_rows.ensure((size_t)m * 4));
    uint32_t* rows = c->g_rows.as<uint32_t>();
    tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, iota, keepf, rows, d_count, m, G.st);
    PHG_TRY(c->cub_tmp.ensure(tmp));
    PHG_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, keepf, rows, d_count, m, G.st));
    PHG_CUDA(cudaMemcpyAsync(c->host_total, d_count, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    const long long nf = c->host_total[0];
    S.nf_seeds = nf;
    S.n_field = nf;
    if (nf == 0) return PHG_OK;
    PHG_TRY(c->g_fpos.ensure((size_t)nf * 24));
    PHG_TRY(c->g_fdir.ensure((size_t)nf * 24));
    row_gather_kernel<<<grid_for(nf, 256), 256, 0, G.st>>>(raw_pos, raw_dir, rows, nf,
                                                           c->g_fpos.as<double>(),
                                                           c->g_fdir.as<double>());
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// joins, commits and output of one traced batch of field seeds (phg.py:294-302); rows of the
// forward traces in slab_f/keep_f/ent_f, of the backward ones in slab_b/keep_b/ent_b
phg_status field_post(GrowCtx& G, Rows slab_f, const long long* keep_f,
                      const uint8_t* ent_f, Rows slab_b, const long long* keep_b,
                      const uint8_t* ent_b, long long nb, bool export_commits,
                      long long* segs_added) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    BatchScratch B;
    PHG_TRY(batch_scratch(G, nb, B));
    join_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(keep_f, ent_f, keep_b, ent_b, nb,
                                                            B.lens, B.segf, B.valid);
    PHG_CUDA(cudaGetLastError());
    if (!export_commits)
        PHG_TRY(commit_batch(G, slab_f, keep_f, slab_b, keep_b, B.valid, nb, 0, false));
    long long nv = 0, ns = 0;
    PHG_TRY(batch_offsets(G, nb, B.lens, B.segf, B.voff, B.sidx, &nv, &ns));
    // a joined segment's voxels are those of its two traces: at most L + 1 distinct ids
    if (export_commits)
        PHG_TRY(commit_batch(G, slab_f, keep_f, slab_b, keep_b, B.valid, nb, nv + ns, true));
    PHG_TRY(ensure_output(G, ns, nv));
    gather_joined_kernel<<<grid_for(nb * 32, 256, num_sms() * kCopyCtasPerSm), 256, 0, G.st>>>(
        slab_f, slab_b, keep_f, keep_b, B.valid, B.voff, B.sidx, nb, S.verts, S.segs,
        c->g_out_off.as<long long>(), c->g_out_verts.as<double>(), c->g_out_rooted.as<uint8_t>(),
        nullptr);
    PHG_CUDA(cudaGetLastError());
    S.segs += ns;
    S.verts += nv;
    *segs_added = ns;
    return PHG_OK;
}

// one batch of field seeds [first, first + nb): trace +d and -d against the same frozen plane,
// join, keep, commit (phg.py:277-302)
phg_status field_batch(GrowCtx& G, long long first, long long nb, bool export_commits,
                       long long* segs_added) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    *segs_added = 0;
    S.n_export = 0;
    if (nb == 0) return PHG_OK;
    const double* pos = c->g_fpos.as<double>() + 3 * first;
    const double* dir = c->g_fdir.as<double>() + 3 * first;
    PHG_TRY(set_cap_plane(G));
    Rows slab_f, slab_b;
    const long long *keep_f, *keep_b;
    const uint8_t *ent_f, *ent_b;
    if (!S.strict) {
        // relaxed mode: +d and -d see the same frozen plane (no commits in between), so both
        // directions run as ONE launch of 2*nb seeds: rows [0, nb) forward, [nb, 2nb) backward
        PHG_TRY(c->g_neg_dir.ensure((size_t)nb * 24 * 4));
        double* pos2 = c->g_neg_dir.as<double>();
        double* dir2 = pos2 + 6 * nb;
        PHG_CUDA(cudaMemcpyAsync(pos2, pos, (size_t)nb * 24, cudaMemcpyDeviceToDevice, G.st));
        PHG_CUDA(cudaMemcpyAsync(pos2 + 3 * nb, pos, (size_t)nb * 24, cudaMemcpyDeviceToDevice,
                                 G.st));
        PHG_CUDA(cudaMemcpyAsync(dir2, dir, (size_t)nb * 24, cudaMemcpyDeviceToDevice, G.st));
        negate_kernel<<<grid_for(nb * 3, 256, num_sms() * 16), 256, 0, G.st>>>(dir, dir2 + 3 * nb,
                                                                                nb * 3);
        PHG_CUDA(cudaGetLastError());
        PHG_TRY(trace_core(c, S.f, &S.p, pos2, dir2, 2 * nb, nullptr, G.st, nullptr, true));
        slab_f = slab_rows(G);
        slab_b = slab_f.sub(nb);
        keep_f = c->keep.as<long long>();
        keep_b = keep_f + nb;
        ent_f = c->entered.as<uint8_t>();
        ent_b = ent_f + nb;
    } else {
        // strict: the -d trace sees the counts the +d trace committed (phg.py:283, :291-292)
        PHG_TRY(trace_core(c, S.f, &S.p, pos, dir, nb, S.counts, G.st));
        swap_buf(c->slab, c->g_slab2);  // keep the forward trace aside
        swap_buf(c->keep, c->g_keep2);
        swap_buf(c->entered, c->g_ent2);
        PHG_TRY(c->g_neg_dir.ensure((size_t)nb * 24));
        double* ndir = c->g_neg_dir.as<double>();
        negate_kernel<<<grid_for(nb * 3, 256, num_sms() * 16), 256, 0, G.st>>>(dir, ndir, nb * 3);
        PHG_CUDA(cudaGetLastError());
        PHG_TRY(trace_core(c, S.f, &S.p, pos, ndir, nb, S.counts, G.st));
        // (strict traces keep seed rows: no locality order)
        const size_t rs = row_stride_doubles(S.p.max_vertices);
        slab_f = Rows{c->g_slab2.as<double>(), nullptr, rs};
        keep_f = c->g_keep2.as<long long>();
        ent_f = c->g_ent2.as<uint8_t>();
        slab_b = Rows{c->slab.as<double>(), nullptr, rs};
        keep_b = c->keep.as<long long>();
        ent_b = c->entered.as<uint8_t>();
    }
    return field_post(G, slab_f, keep_f, ent_f, slab_b, keep_b, ent_b, nb, export_commits,
                      segs_added);
}

// ---- speculative phases of phg_grow_init (see spec_truncate_kernel) ---------------------------
phg_status rec_buffers(GrowCtx& G, long long n, TraceRecord& R) {
    const int words = (G.s->p.max_vertices + 31) / 32;
    PHG_TRY(G.c->g_rec_bits.ensure((size_t)n * words * 4));
    PHG_TRY(G.c->g_rec_nv.ensure((size_t)n * 4));
    R = TraceRecord{G.c->g_rec_bits.as<uint32_t>(), G.c->g_rec_nv.as<int32_t>(), words};
    return PHG_OK;
}

// exact trace of rows [first, first + nb) under the current plane: truncate in place (keep)
phg_status spec_truncate(GrowCtx& G, const TraceRecord& R, long long first, long long nb) {
    GrowSession& S = *G.s;
    spec_truncate_kernel<<<grid_for(nb * 32, 256, num_sms() * 16), 256, 0, G.st>>>(
        S.f->view(), slab_rows(G).sub(first),
        R.bits + (size_t)first * R.words, R.words, R.nverts + first, nb,
        G.c->keep.as<long long>() + first);
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// PHG_DRIVER_SPEC=0 turns the speculation off (per-batch traces, for comparison)
bool spec_enabled() {
    const char* e = getenv("PHG_DRIVER_SPEC");
    return !(e && e[0] == '0');
}

// every scalp batch (phg.py:229-251): one trace against the plane at the start, then per
// batch in order: truncate to the current plane, select, commit, emit.  After a uint16 wrap
// the plane is no longer a superset of the start plane: the remaining batches trace afresh.
// Seeds per speculative launch: whole batches, about four times the trace kernel's resident
// lanes (16 batches of the reference's 16384 on a B200).  One launch for the whole phase
// traces every strand to full length against an empty plane; windows re-freeze the plane, so
// later launches stop at the caps earlier batches filled (measured on 1M C3 seeds: 30.8 ms
// for one launch, 22.1 ms for 16-batch windows, 29.7 ms for 4).  PHG_SPEC_WINDOW=<batches>
// overrides.
long long spec_window(long long bs) {
    const char* e = getenv("PHG_SPEC_WINDOW");
    long long w = (e && *e) ? atoll(e) : 0;
    if (w <= 0) w = std::max(1ll, (4ll * num_sms() * 4 * kTPB + bs / 2) / bs);
    return w * bs;
}

// ---- optimistic windows: batch posts without host synchronisation -------------------------
// Inside a speculative window the batches are posted back to back: segments, commits, offsets
// and gathers all run on the stream, with the output bases kept on the device (S.dtot) and the
// outputs preallocated for the whole window.  The host looks once per window.  A uint16 count
// wrap (rare) makes the incremental cap plane unusable for the batches after it: the window is
// then rolled back exactly (its commits undone, outputs and counters restored) and redone one
// traced batch at a time, as the synchronous driver does after a wrap.

// Post one scalp batch without synchronising (valid, commit, offsets, gather, totals).
phg_status scalp_post_async(GrowCtx& G, Rows slab, const long long* keep, const uint8_t* ent,
                            long long nb) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    BatchScratch B;
    PHG_TRY(batch_scratch(G, nb, B));
    segment_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(
        keep, ent, nb, B.lens, B.segf, B.valid, S.misc.as<unsigned long long>());
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(commit_batch(G, slab, keep, Rows{}, nullptr, B.valid, nb, 0, false));
    PHG_TRY(scan_lengths(c, B.lens, nb, B.voff, G.st));
    PHG_TRY(scan_lengths(c, B.segf, nb, B.sidx, G.st));
    long long* dtot = S.dtot.as<long long>();
    gather_scalp_kernel<<<grid_for(nb * 32, 256, num_sms() * kCopyCtasPerSm), 256, 0, G.st>>>(
        slab, keep, B.valid, B.voff, B.sidx, nb, 0, 0, c->g_out_off.as<long long>(),
        c->g_out_verts.as<double>(), c->g_out_rooted.as<uint8_t>(), dtot);
    advance_totals_kernel<<<1, 1, 0, G.st>>>(dtot, B.sidx + nb, B.voff + nb);
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// Post one field batch (joins) without synchronising.
phg_status field_post_async(GrowCtx& G, Rows slab_f, const long long* keep_f, const uint8_t* ent_f,
                            Rows slab_b, const long long* keep_b, const uint8_t* ent_b,
                            long long nb) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    BatchScratch B;
    PHG_TRY(batch_scratch(G, nb, B));
    join_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(keep_f, ent_f, keep_b, ent_b, nb,
                                                            B.lens, B.segf, B.valid);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(commit_batch(G, slab_f, keep_f, slab_b, keep_b, B.valid, nb, 0, false));
    PHG_TRY(scan_lengths(c, B.lens, nb, B.voff, G.st));
    PHG_TRY(scan_lengths(c, B.segf, nb, B.sidx, G.st));
    long long* dtot = S.dtot.as<long long>();
    gather_joined_kernel<<<grid_for(nb * 32, 256, num_sms() * kCopyCtasPerSm), 256, 0, G.st>>>(
        slab_f, slab_b, keep_f, keep_b, B.valid, B.voff, B.sidx, nb, 0, 0,
        c->g_out_off.as<long long>(), c->g_out_verts.as<double>(), c->g_out_rooted.as<uint8_t>(),
        dtot);
    advance_totals_kernel<<<1, 1, 0, G.st>>>(dtot, B.sidx + nb, B.voff + nb);
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// Window start (after its trace): outputs sized by the trace's appended vertex counts (a kept
// segment never has more), device totals = host totals, never-entered counter snapshot.
phg_status window_begin(GrowCtx& G, long long add_segs, const TraceRecord& R, long long n) {
    GrowSession& S = *G.s;
    unsigned long long* sum = S.dtot.as<unsigned long long>() + 4;
    PHG_CUDA(cudaMemsetAsync(sum, 0, 8, G.st));
    sum_nverts_kernel<<<grid_for(n, 256, num_sms() * 8), 256, 0, G.st>>>(R.nverts, n, sum);
    PHG_CUDA(cudaGetLastError());
    PHG_CUDA(cudaMemcpyAsync(G.c->host_total, sum, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    PHG_TRY(ensure_output(G, add_segs, G.c->host_total[0]));
    set_totals_kernel<<<1, 1, 0, G.st>>>(S.dtot.as<long long>(), S.segs, S.verts);
    PHG_CUDA(cudaGetLastError());
    PHG_CUDA(cudaMemcpyAsync(S.dtot.as<long long>() + 2, S.misc.p, 8, cudaMemcpyDeviceToDevice,
                             G.st));
    return PHG_OK;
}

// Window end (synchronises): adopt the device totals, or report a count wrap.
phg_status window_end(GrowCtx& G, bool* wrapped) {
    GrowSession& S = *G.s;
    long long* h = G.c->host_total;
    PHG_CUDA(cudaMemcpyAsync(h, S.dtot.p, 16, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaMemcpyAsync(h + 2, S.misc.as<unsigned long long>() + 1, 8,
                             cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    *wrapped = h[2] != 0;
    if (!*wrapped) {
        S.segs = h[0];
        S.verts = h[1];
    }
    return PHG_OK;
}

// Undo one posted batch's commits exactly: its segments' distinct voxels, exported and
// decremented.  valid is recomputed from the (truncated) keep arrays the post used.
phg_status uncommit_batch(GrowCtx& G, Rows slab_a, const long long* keep_a, const uint8_t* ent_a,
                          Rows slab_b, const long long* keep_b, const uint8_t* ent_b,
                          long long nb) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    BatchScratch B;
    PHG_TRY(batch_scratch(G, nb, B));
    if (slab_b.base)
        join_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(keep_a, ent_a, keep_b, ent_b, nb,
                                                                B.lens, B.segf, B.valid);
    else  // the never-entered count is restored from its window snapshot: count into a dummy
        segment_select_kernel<<<grid_for(nb, 256), 256, 0, G.st>>>(
            keep_a, ent_a, nb, B.lens, B.segf, B.valid, S.dtot.as<unsigned long long>() + 3);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(scan_lengths(c, B.lens, nb, B.voff, G.st));
    PHG_CUDA(cudaMemcpyAsync(c->host_total, B.voff + nb, 8, cudaMemcpyDeviceToHost, G.st));
    PHG_CUDA(cudaStreamSynchronize(G.st));
    const long long nv = c->host_total[0];
    const long long max_ids = nv + (slab_b.base ? nb : 0);
    PHG_TRY(commit_batch(G, slab_a, keep_a, slab_b, keep_b, B.valid, nb, max_ids, true));
    if (S.n_export)
        uncommit_kernel<<<grid_for(S.n_export, 256, num_sms() * 16), 256, 0, G.st>>>(
            S.export_ids.as<uint32_t>(), S.n_export, S.counts);
    PHG_CUDA(cudaGetLastError());
    S.n_export = 0;
    return PHG_OK;
}

// After a wrap inside a window: counters back to the window start, cap plane to be rebuilt.
phg_status window_restore(GrowCtx& G) {
    GrowSession& S = *G.s;
    PHG_CUDA(cudaMemcpyAsync(S.misc.p, S.dtot.as<long long>() + 2, 8, cudaMemcpyDeviceToDevice,
                             G.st));
    PHG_CUDA(cudaMemsetAsync(S.misc.as<unsigned long long>() + 1, 0, 8, G.st));
    S.cap_valid = false;
    return PHG_OK;
}

phg_status scalp_phase_spec(GrowCtx& G, const double* pos, const double* dir, long long n) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    const long long bs = S.g.batch_size;
    const long long win = spec_window(bs);
    long long added = 0;
    for (long long w0 = 0; w0 < n; w0 += win) {
        const long long nw = std::min(win, n - w0);
        PHG_TRY(set_cap_plane(G));
        TraceRecord R;
        PHG_TRY(rec_buffers(G, nw, R));
        PHG_TRY(trace_core(c, S.f, &S.p, pos + 3 * w0, dir + 3 * w0, nw, nullptr, G.st, &R,
                           true));
        PHG_TRY(window_begin(G, nw, R, nw));
        const Rows rows = slab_rows(G);
        const long long* keep = c->keep.as<long long>();
        const uint8_t* ent = c->entered.as<uint8_t>();
        for (long long b0 = 0; b0 < nw; b0 += bs) {
            const long long nb = std::min(bs, nw - b0);
            if (b0 > 0) PHG_TRY(spec_truncate(G, R, b0, nb));  // the window's first batch saw
                                                                // the plane it was traced with
            PHG_TRY(scalp_post_async(G, rows.sub(b0), keep + b0, ent + b0, nb));
        }
        bool wrapped = false;
        PHG_TRY(window_end(G, &wrapped));
        if (!wrapped) {
            S.scalp_segs = S.segs;
            continue;
        }
        // a count wrapped: undo the window, then trace every remaining batch afresh
        for (long long b0 = 0; b0 < nw; b0 += bs) {
            const long long nb = std::min(bs, nw - b0);
            PHG_TRY(uncommit_batch(G, rows.sub(b0), keep + b0, ent + b0, Rows{}, nullptr, nullptr,
                                   nb));
        }
        PHG_TRY(window_restore(G));
        for (long long r0 = w0; r0 < n; r0 += bs)
            PHG_TRY(scalp_batch(G, pos + 3 * r0, dir + 3 * r0, std::min(bs, n - r0), false,
                                &added));
        return PHG_OK;
    }
    return PHG_OK;
}

// every field batch (phg.py:277-302) the same way: one launch of all +d rows [0, nf) and -d
// rows [nf, 2nf) against the plane after the scalp phase, posted as one optimistic window
phg_status field_phase_spec(GrowCtx& G) {
    GrowSession& S = *G.s;
    phg_ctx* c = G.c;
    const long long nf = S.nf_seeds, bs = S.g.batch_size;
    if (nf == 0) return PHG_OK;
    PHG_TRY(set_cap_plane(G));
    const double* pos = c->g_fpos.as<double>();
    const double* dir = c->g_fdir.as<double>();
    PHG_TRY(c->g_neg_dir.ensure((size_t)nf * 24 * 4));
    double* pos2 = c->g_neg_dir.as<double>();
    double* dir2 = pos2 + 6 * nf;
    PHG_CUDA(cudaMemcpyAsync(pos2, pos, (size_t)nf * 24, cudaMemcpyDeviceToDevice, G.st));
    PHG_CUDA(cudaMemcpyAsync(pos2 + 3 * nf, pos, (size_t)nf * 24, cudaMemcpyDeviceToDevice, G.st));
    PHG_CUDA(cudaMemcpyAsync(dir2, dir, (size_t)nf * 24, cudaMemcpyDeviceToDevice, G.st));
    negate_kernel<<<grid_for(nf * 3, 256, num_sms() * 16), 256, 0, G.st>>>(dir, dir2 + 3 * nf,
                                                                            nf * 3);
    PHG_CUDA(cudaGetLastError());
    TraceRecord R;
    PHG_TRY(rec_buffers(G, 2 * nf, R));
    PHG_TRY(trace_core(c, S.f, &S.p, pos2, dir2, 2 * nf, nullptr, G.st, &R, true));
    PHG_TRY(window_begin(G, nf, R, 2 * nf));
    long long added = 0;
    const Rows slab = slab_rows(G);
    const long long* keep = c->keep.as<long long>();
    const uint8_t* ent = c->entered.as<uint8_t>();
    for (long long b0 = 0; b0 < nf; b0 += bs) {
        const long long nb = std::min(bs, nf - b0);
        if (b0 > 0) {
            PHG_TRY(spec_truncate(G, R, b0, nb));
            PHG_TRY(spec_truncate(G, R, nf + b0, nb));
        }
        PHG_TRY(field_post_async(G, slab.sub(b0), keep + b0, ent + b0, slab.sub(nf + b0),
                                 keep + nf + b0, ent + nf + b0, nb));
    }
    bool wrapped = false;
    PHG_TRY(window_end(G, &wrapped));
    if (!wrapped) return PHG_OK;
    for (long long b0 = 0; b0 < nf; b0 += bs) {
        const long long nb = std::min(bs, nf - b0);
        PHG_TRY(uncommit_batch(G, slab.sub(b0), keep + b0, ent + b0, slab.sub(nf + b0),
                               keep + nf + b0, ent + nf + b0, nb));
    }
    PHG_TRY(window_restore(G));
    for (long long r0 = 0; r0 < nf; r0 += bs)
        PHG_TRY(field_batch(G, r0, std::min(bs, nf - r0), false, &added));
    return PHG_OK;
}

GrowSession* session(phg_ctx* c) { return static_cast<GrowSession*>(c->grow_session); }

}  // namespace

void grow_session_free(void* s) { delete static_cast<GrowSession*>(s); }

}  // namespace phg

extern "C" {

phg_status phg_grow_begin(phg_ctx* c, phg_field* f, const phg_params_v1* p,
                          const phg_grow_params_v1* g, const uint16_t* counts, void* stream) {
    if (!c || !f || !p || !g || !counts) return fail(PHG_ERR_INVALID, "phg_grow_begin: null argument");
    if (g->batch_size < 1 || g->occupancy_cap < 1)
        return fail(PHG_ERR_INVALID, "phg_grow_begin: invalid batch_size / occupancy_cap");
    if (p->max_vertices < 1)
        return fail(PHG_ERR_INVALID, "phg_grow_begin: max_vertices must be >= 1");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != f->device)
        return fail(PHG_ERR_INVALID, "phg_grow_begin: field lives on device %d", f->device);
    cudaStream_t st = as_stream(stream);
    c->grow_ready = false;
    if (!c->grow_session) c->grow_session = new GrowSession();
    GrowSession& S = *session(c);
    S.f = f;
    S.p = *p;
    S.g = *g;
    S.strict = (p->flags & PHG_FLAG_STRICT) != 0;
    S.segs = S.verts = S.scalp_segs = S.n_field = S.n_export = S.nf_seeds = 0;
    S.cap_valid = false;
    const long long V = f->nvox();
    PHG_TRY(c->counts32.ensure((size_t)V * 4));
    S.counts = c->counts32.as<uint32_t>();
    const void* d_counts = nullptr;
    PHG_TRY(to_device(counts, (size_t)V * 2, c->live_stage, &d_counts, st));
    u16_to_u32<<<grid_for(V, 256, num_sms() * 16), 256, 0, st>>>((const uint16_t*)d_counts,
                                                                S.counts, V);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(c->counters.ensure(64));
    PHG_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, st));
    PHG_TRY(S.misc.ensure(64));
    PHG_CUDA(cudaMemsetAsync(S.misc.p, 0, 64, st));
    PHG_TRY(S.dtot.ensure(64));
    PHG_CUDA(cudaMemsetAsync(S.dtot.p, 0, 64, st));
    PHG_CUDA(cudaStreamSynchronize(st));  // host counts may be released after return
    return PHG_OK;
}

phg_status phg_grow_scalp_batch(phg_ctx* c, const double* seeds, const double* normals,
                                int64_t nb, int32_t export_commits, int64_t out[2], void* stream) {
    PHG_RANGE("phg/grow_scalp_batch");
    if (!c || !out || nb < 0 || (nb > 0 && (!seeds || !normals)))
        return fail(PHG_ERR_INVALID, "phg_grow_scalp_batch: bad argument");
    if (!session(c)) return fail(PHG_ERR_STATE, "phg_grow_scalp_batch: no phg_grow_begin");
    cudaStream_t st = as_stream(stream);
    GrowCtx G{c, session(c), st};
    const void *d_pos = nullptr, *d_dir = nullptr;
    PHG_TRY(to_device(seeds, (size_t)nb * 24, c->g_seeds_pos, &d_pos, st));
    PHG_TRY(to_device(normals, (size_t)nb * 24, c->g_seeds_dir, &d_dir, st));
    long long added = 0;
    PHG_TRY(scalp_batch(G, (const double*)d_pos, (const double*)d_dir, nb, export_commits != 0,
                        &added));
    out[0] = added;
    out[1] = G.s->n_export;
    return PHG_OK;
}

phg_status phg_grow_field_begin(phg_ctx* c, int64_t* n_field_seeds, void* stream) {
    if (!c || !n_field_seeds) return fail(PHG_ERR_INVALID, "phg_grow_field_begin: null argument");
    if (!session(c)) return fail(PHG_ERR_STATE, "phg_grow_field_begin: no phg_grow_begin");
    GrowCtx G{c, session(c), as_stream(stream)};
    PHG_TRY(field_begin(G));
    *n_field_seeds = G.s->nf_seeds;
    return PHG_OK;
}

phg_status phg_grow_field_batch(phg_ctx* c, int64_t first, int64_t nb, int32_t export_commits,
                                int64_t out[2], void* stream) {
    PHG_RANGE("phg/grow_field_batch");
    if (!c || !out || first < 0 || nb < 0)
        return fail(PHG_ERR_INVALID, "phg_grow_field_batch: bad argument");
    if (!session(c)) return fail(PHG_ERR_STATE, "phg_grow_field_batch: no phg_grow_begin");
    GrowCtx G{c, session(c), as_stream(stream)};
    if (first + nb > G.s->nf_seeds)
        return fail(PHG_ERR_INVALID, "phg_grow_field_batch: [%lld, %lld) beyond %lld field seeds",
                    (long long)first, (long long)(first + nb), G.s->nf_seeds);
    long long added = 0;
    PHG_TRY(field_batch(G, first, nb, export_commits != 0, &added));
    out[0] = added;
    out[1] = G.s->n_export;
    return PHG_OK;
}

phg_status phg_grow_commits(phg_ctx* c, uint32_t* ids, void* stream) {
    if (!c || !session(c)) return fail(PHG_ERR_STATE, "phg_grow_commits: no session");
    GrowSession& S = *session(c);
    if (S.n_export && !ids) return fail(PHG_ERR_INVALID, "phg_grow_commits: null ids");
    cudaStream_t st = as_stream(stream);
    if (S.n_export)
        PHG_CUDA(cudaMemcpyAsync(ids, S.export_ids.p, (size_t)S.n_export * 4, cudaMemcpyDefault, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

phg_status phg_grow_apply(phg_ctx* c, const uint32_t* ids, int64_t n, void* stream) {
    PHG_RANGE("phg/grow_apply");
    if (!c || !session(c)) return fail(PHG_ERR_STATE, "phg_grow_apply: no session");
    if (n < 0 || (n > 0 && !ids)) return fail(PHG_ERR_INVALID, "phg_grow_apply: bad ids");
    GrowSession& S = *session(c);
    if (S.strict || n == 0) return PHG_OK;
    cudaStream_t st = as_stream(stream);
    DevBuf stage;
    const void* d_ids = nullptr;
    PHG_TRY(to_device(ids, (size_t)n * 4, stage, &d_ids, st));
    GrowCtx G{c, &S, st};
    PHG_TRY(set_cap_plane(G));  // the plane must exist before incremental updates
    const CommitSink K = direct_sink(S);
    apply_commits_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(
        (const uint32_t*)d_ids, n, K.counts, K.cap_bits, K.cap, K.wrapped);
    PHG_CUDA(cudaGetLastError());
    // a wrapped count invalidates the incremental plane
    PHG_CUDA(cudaMemcpyAsync(c->host_total + 2, S.misc.as<unsigned long long>() + 1, 8,
                             cudaMemcpyDeviceToHost, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    if (c->host_total[2]) {
        S.cap_valid = false;
        PHG_CUDA(cudaMemsetAsync(S.misc.as<unsigned long long>() + 1, 0, 8, st));
    }
    return PHG_OK;
}

phg_status phg_grow_end(phg_ctx* c, uint16_t* counts, int64_t* n_segments, int64_t* n_verts,
                        int64_t report[4], void* stream) {
    if (!c || !session(c)) return fail(PHG_ERR_STATE, "phg_grow_end: no session");
    if (!counts || !n_segments || !n_verts || !report)
        return fail(PHG_ERR_INVALID, "phg_grow_end: null argument");
    GrowSession& S = *session(c);
    cudaStream_t st = as_stream(stream);
    GrowCtx G{c, &S, st};
    S.f->has_cap = false;  // the driver overwrote the field's cap plane; leave none behind
    const long long V = S.f->nvox();
    const bool counts_dev = is_device_ptr(counts);
    PHG_TRY(c->live_stage.ensure((size_t)V * 2));
    uint16_t* dst16 = counts_dev ? counts : c->live_stage.as<uint16_t>();
    u32_to_u16<<<grid_for(V, 256, num_sms() * 16), 256, 0, st>>>(S.counts, dst16, V);
    PHG_CUDA(cudaGetLastError());
    if (!counts_dev) PHG_TRY(copy_d2h(counts, dst16, (size_t)V * 2, st));
    unsigned long long never = 0;
    PHG_CUDA(cudaMemcpyAsync(&never, S.misc.p, 8, cudaMemcpyDeviceToHost, st));
    PHG_TRY(ensure_output(G, 0, 0));
    PHG_CUDA(cudaMemcpyAsync(c->g_out_off.as<long long>() + S.segs, &S.verts, 8,
                             cudaMemcpyHostToDevice, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    report[0] = (int64_t)never;
    report[1] = S.scalp_segs;
    report[2] = S.n_field;
    report[3] = S.segs - S.scalp_segs;
    *n_segments = S.segs;
    *n_verts = S.verts;
    c->grow_segs = S.segs;
    c->grow_verts = S.verts;
    c->grow_ready = true;
    return PHG_OK;
}

phg_status phg_grow_init(phg_ctx* c, phg_field* f, const phg_params_v1* p,
                         const phg_grow_params_v1* g, const double* seeds, const double* normals,
                         int64_t n, uint16_t* counts, int64_t* n_segments, int64_t* n_verts,
                         int64_t report[4], void* stream) {
    PHG_RANGE("phg/grow_init");
    if (!c || !f || !p || !g || !counts || !n_segments || !n_verts || !report)
        return fail(PHG_ERR_INVALID, "phg_grow_init: null argument");
    if (n < 0) return fail(PHG_ERR_INVALID, "phg_grow_init: negative seed count");
    if (n > 0 && (!seeds || !normals)) return fail(PHG_ERR_INVALID, "phg_grow_init: null seeds");
    cudaStream_t st = as_stream(stream);
    PHG_TRY(phg_grow_begin(c, f, p, g, counts, stream));
    GrowCtx G{c, session(c), st};
    const void *d_pos = nullptr, *d_dir = nullptr;
    if (n > 0) {
        PHG_TRY(to_device(seeds, (size_t)n * 24, c->g_seeds_pos, &d_pos, st));
        PHG_TRY(to_device(normals, (size_t)n * 24, c->g_seeds_dir, &d_dir, st));
    }
    PHG_CUDA(cudaEventRecord(c->ev[0], st));  // device window: uploads done .. downloads begin
    phg_status s = PHG_OK;
    const long long bs = g->batch_size;
    long long added = 0;
    const bool spec = !G.s->strict && spec_enabled();
    if (spec && n > 0) {
        s = scalp_phase_spec(G, (const double*)d_pos, (const double*)d_dir, n);
    } else {
        for (long long b0 = 0; s == PHG_OK && b0 < n; b0 += bs)
            s = scalp_batch(G, (const double*)d_pos + 3 * b0, (const double*)d_dir + 3 * b0,
                            std::min(bs, n - b0), false, &added);
    }
    if (s == PHG_OK && n > 0 && g->field_seeds > 0) {
        s = field_begin(G);
        if (s == PHG_OK && spec) {
            s = field_phase_spec(G);
        } else {
            for (long long b0 = 0; s == PHG_OK && b0 < G.s->nf_seeds; b0 += bs)
                s = field_batch(G, b0, std::min(bs, G.s->nf_seeds - b0), false, &added);
        }
    }
    if (s != PHG_OK) {
        f->has_cap = false;
        return s;
    }
    PHG_CUDA(cudaEventRecord(c->ev[2], st));
    PHG_TRY(phg_grow_end(c, counts, n_segments, n_verts, report, stream));
    cudaEventElapsedTime(&c->last_total_ms, c->ev[0], c->ev[2]);
    return PHG_OK;
}

phg_status phg_grow_fetch(phg_ctx* c, int64_t* offsets, double* verts, uint8_t* rooted,
                          void* stream) {
    if (!c) return fail(PHG_ERR_INVALID, "phg_grow_fetch: null context");
    if (!c->grow_ready) return fail(PHG_ERR_STATE, "phg_grow_fetch: no completed phg_grow_init");
    cudaStream_t st = as_stream(stream);
    if (offsets)
        PHG_CUDA(cudaMemcpyAsync(offsets, c->g_out_off.p, (size_t)(c->grow_segs + 1) * 8,
                                 cudaMemcpyDefault, st));
    if (verts && c->grow_verts) {
        PHG_CUDA(cudaStreamSynchronize(st));
        PHG_TRY(copy_d2h(verts, c->g_out_verts.p, (size_t)c->grow_verts * 24, st));
    }
    if (rooted && c->grow_segs)
        PHG_CUDA(cudaMemcpyAsync(rooted, c->g_out_rooted.p, (size_t)c->grow_segs,
                                 cudaMemcpyDefault, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

}  // extern "C"
