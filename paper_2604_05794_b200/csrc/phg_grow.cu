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

// Add the vertices of one slab row to the warp's set, counting newly seen in-bounds voxels.
__device__ __forceinline__ void commit_row(const FieldView& F, const double* __restrict__ row,
                                           long long L, unsigned long long* T, int bits,
                                           uint32_t epoch, uint32_t* __restrict__ counts,
                                           uint32_t* __restrict__ cap_bits, uint32_t cap,
                                           unsigned int* __restrict__ wrapped, int lane) {
    for (long long k = lane; k < L; k += 32) {
        // vol.voxel_of (volume.py:42-45) and in_bounds (:47-49)
        const int vx = floor_idx(grid_coord(F, row[3 * k + 0] - F.ox));
        const int vy = floor_idx(grid_coord(F, row[3 * k + 1] - F.oy));
        const int vz = floor_idx(grid_coord(F, row[3 * k + 2] - F.oz));
        if ((unsigned)vx < (unsigned)F.nx && (unsigned)vy < (unsigned)F.ny &&
            (unsigned)vz < (unsigned)F.nz) {
            const uint32_t lin = ((uint32_t)vx * F.ny + vy) * F.nz + vz;
            if (set_insert(T, bits, epoch, lin)) {
                // keep the at_cap plane (counts >= cap, phg.py:236) current incrementally:
                // without uint16 wrap-around counts only grow, so a voxel turns "at cap"
                // exactly when its count reaches cap; a wrap forces a full rebuild
                const uint32_t now = (atomicAdd(counts + lin, 1u) + 1u) & 0xffffu;
                if (now == cap) atomicOr(cap_bits + (lin >> 5), 1u << (lin & 31));
                if (now == 0u) atomicOr(wrapped, 1u);
            }
        }
    }
}

// vol.counts[unique voxels of each valid segment] += 1 (phg.py:248-251, :299-302).  One warp per
// segment; for joined field segments the set spans both traces (voxels(bwd) U voxels(fwd)).
// GLOBAL_TABLE: the per-warp table lives in global memory (very long segments).
template <bool GLOBAL_TABLE>
__global__ void commit_kernel(FieldView F, const double* __restrict__ slab_a,
                              const long long* __restrict__ keep_a,
                              const double* __restrict__ slab_b,
                              const long long* __restrict__ keep_b,
                              const uint8_t* __restrict__ valid, long long n, size_t row_stride,
                              uint32_t* __restrict__ counts, uint32_t* __restrict__ cap_bits,
                              uint32_t cap, unsigned int* __restrict__ wrapped, int bits,
                              unsigned long long* __restrict__ gtables) {
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
        commit_row(F, slab_a + (size_t)i * row_stride, keep_a[i], T, bits, epoch, counts,
                   cap_bits, cap, wrapped, lane);
        if (slab_b) commit_row(F, slab_b + (size_t)i * row_stride, keep_b[i], T, bits, epoch,
                               counts, cap_bits, cap, wrapped, lane);
        __syncwarp();
    }
}

// scalp segments -> output CSR (rows of valid strands, in seed order)
__global__ void gather_scalp_kernel(const double* __restrict__ slab, size_t row_stride,
                                    const long long* __restrict__ keep,
                                    const uint8_t* __restrict__ valid,
                                    const long long* __restrict__ voff,
                                    const long long* __restrict__ sidx, long long n,
                                    long long vbase, long long sbase, long long* __restrict__ out_off,
                                    double* __restrict__ out_v, uint8_t* __restrict__ rooted) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < n; i += nwarps) {
        if (!valid[i]) continue;
        const long long o = vbase + voff[i];
        if (lane == 0) {
            out_off[sbase + sidx[i]] = o;
            rooted[sbase + sidx[i]] = 1;
        }
        const double* src = slab + (size_t)i * row_stride;
        double* dst = out_v + o * 3;
        const long long len = keep[i] * 3;
        for (long long j = lane; j < len; j += 32) dst[j] = src[j];
    }
}

// field segments: v = concat(bwd[::-1], fwd[1:]) if len(bwd) > 1 else fwd (phg.py:294)
__global__ void gather_joined_kernel(const double* __restrict__ slab_f,
                                     const double* __restrict__ slab_b, size_t row_stride,
                                     const long long* __restrict__ keep_f,
                                     const long long* __restrict__ keep_b,
                                     const uint8_t* __restrict__ valid,
                                     const long long* __restrict__ voff,
                                     const long long* __restrict__ sidx, long long n,
                                     long long vbase, long long sbase,
                                     long long* __restrict__ out_off, double* __restrict__ out_v,
                                     uint8_t* __restrict__ rooted) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < n; i += nwarps) {
        if (!valid[i]) continue;
        const long long o = vbase + voff[i];
        if (lane == 0) {
            out_off[sbase + sidx[i]] = o;
            rooted[sbase + sidx[i]] = 0;
        }
        const double* f = slab_f + (size_t)i * row_stride;
        const double* b = slab_b + (size_t)i * row_stride;
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
            for (long long j = lane; j < lf * 3; j += 32) dst[j] = f[j];
        }
    }
}

// unvisited = argwhere(occ & (counts == 0)) (phg.py:266): flag per voxel
__global__ void unvisited_flag_kernel(const float4* __restrict__ vox,
                                      const uint32_t* __restrict__ counts, long long nvox,
                                      uint8_t* __restrict__ flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x)
        flag[i] = (vox[i].w != 0.0f && (counts[i] & 0xffffu) == 0u) ? 1 : 0;
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
    const float4 v = F.vox[l];
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

void swap_buf(DevBuf& a, DevBuf& b) {
    std::swap(a.p, b.p);
    std::swap(a.cap, b.cap);
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

struct GrowState {
    phg_ctx* c;
    phg_field* f;
    const phg_params_v1* p;
    const phg_grow_params_v1* g;
    cudaStream_t st;
    bool strict;
    uint32_t* counts;    // device uint32 plane (vol.counts)
    long long segs = 0;  // output segments so far
    long long verts = 0; // output vertices so far
    unsigned long long* misc = nullptr;  // [0] never_entered, [1] (u32) count wrapped
    bool cap_valid = false;              // f->cap == (counts >= cap) for the current counts
};

phg_status set_cap_plane(GrowState& S) {
    if (S.strict) {
        S.f->has_cap = false;
        return PHG_OK;
    }
    S.f->has_cap = true;
    if (S.cap_valid) return PHG_OK;  // maintained incrementally by the commit kernel
    const long long V = S.f->nvox();
    PHG_TRY(S.f->cap.ensure((size_t)((V + 31) / 32) * 4));
    cap_from_counts_kernel<<<grid_for((V + 31) / 32 * 32, 256, num_sms() * 16), 256, 0, S.st>>>(
        S.counts, V, (uint32_t)S.g->occupancy_cap, S.f->cap.as<uint32_t>());
    PHG_CUDA(cudaGetLastError());
    S.cap_valid = true;
    return PHG_OK;
}

phg_status launch_commit(GrowState& S, const double* slab_a, const long long* keep_a,
                         const double* slab_b, const long long* keep_b, const uint8_t* valid,
                         long long n) {
    const FieldView F = S.f->view();
    const size_t rs = row_stride_doubles(S.p->max_vertices);
    const long long max_entries = (long long)S.p->max_vertices * (slab_b ? 2 : 1);
    int bits = 6;
    while ((1ll << bits) < 2 * max_entries) ++bits;
    const size_t table_bytes = (size_t)8 << bits;
    const int warps_total = num_sms() * 16;
    if (table_bytes * kCommitWarps <= 200 * 1024) {
        const size_t smem = table_bytes * kCommitWarps;
        PHG_CUDA(cudaFuncSetAttribute(commit_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int blocks = std::max(1, std::min(warps_total / kCommitWarps,
                                                (int)((n + kCommitWarps - 1) / kCommitWarps)));
        commit_kernel<false><<<blocks, 32 * kCommitWarps, smem, S.st>>>(
            F, slab_a, keep_a, slab_b, keep_b, valid, n, rs, S.counts, S.f->cap.as<uint32_t>(),
            (uint32_t)S.g->occupancy_cap, (unsigned int*)(S.misc + 1), bits, nullptr);
    } else {
        const int blocks = std::max(1, std::min(warps_total / kCommitWarps,
                                                (int)((n + kCommitWarps - 1) / kCommitWarps)));
        PHG_TRY(S.c->g_hash.ensure(table_bytes * (size_t)blocks * kCommitWarps));
        commit_kernel<true><<<blocks, 32 * kCommitWarps, 0, S.st>>>(
            F, slab_a, keep_a, slab_b, keep_b, valid, n, rs, S.counts, S.f->cap.as<uint32_t>(),
            (uint32_t)S.g->occupancy_cap, (unsigned int*)(S.misc + 1), bits,
            S.c->g_hash.as<unsigned long long>());
    }
    PHG_CUDA(cudaGetLastError());
    return PHG_OK;
}

// scans of lens / segment flags -> per-strand output offsets; returns batch totals (syncs)
phg_status batch_offsets(GrowState& S, long long n, long long* lens, long long* segf,
                         long long* voff, long long* sidx, long long* nv, long long* ns) {
    PHG_TRY(scan_lengths(S.c, lens, n, voff, S.st));
    PHG_TRY(scan_lengths(S.c, segf, n, sidx, S.st));
    PHG_CUDA(cudaMemcpyAsync(S.c->host_total, voff + n, 8, cudaMemcpyDeviceToHost, S.st));
    PHG_CUDA(cudaMemcpyAsync(S.c->host_total + 1, sidx + n, 8, cudaMemcpyDeviceToHost, S.st));
    PHG_CUDA(cudaMemcpyAsync(S.c->host_total + 2, S.misc + 1, 8, cudaMemcpyDeviceToHost, S.st));
    PHG_CUDA(cudaStreamSynchronize(S.st));
    *nv = S.c->host_total[0];
    *ns = S.c->host_total[1];
    if (S.c->host_total[2]) {  // a count wrapped past 65535: rebuild the cap plane exactly
        S.cap_valid = false;
        PHG_CUDA(cudaMemsetAsync(S.misc + 1, 0, 8, S.st));
    }
    return PHG_OK;
}

phg_status ensure_output(GrowState& S, long long add_segs, long long add_verts) {
    PHG_TRY(grow_keep(S.c->g_out_off, (size_t)S.segs * 8, (size_t)(S.segs + add_segs + 1) * 8,
                      S.st));
    PHG_TRY(grow_keep(S.c->g_out_rooted, (size_t)S.segs, (size_t)(S.segs + add_segs + 1), S.st));
    PHG_TRY(grow_keep(S.c->g_out_verts, (size_t)S.verts * 24,
                      (size_t)(S.verts + add_verts + 1) * 24, S.st));
    return PHG_OK;
}

// per-batch scratch: lens, segment flags, their scans, validity
struct BatchScratch {
    long long *lens, *segf, *voff, *sidx;
    uint8_t* valid;
};

phg_status batch_scratch(GrowState& S, long long n, BatchScratch& B) {
    PHG_TRY(S.c->g_misc.ensure((size_t)(n + 1) * 8 * 4 + (size_t)n + 64));
    char* base = (char*)S.c->g_misc.p;
    B.lens = (long long*)base;
    B.segf = B.lens + (n + 1);
    B.voff = B.segf + (n + 1);
    B.sidx = B.voff + (n + 1);
    B.valid = (uint8_t*)(B.sidx + (n + 1));
    return PHG_OK;
}

phg_status scalp_pass(GrowState& S, const double* d_pos, const double* d_dir, long long n) {
    const long long bs = S.g->batch_size;
    for (long long b0 = 0; b0 < n; b0 += bs) {
        const long long nb = std::min(bs, n - b0);
        PHG_TRY(set_cap_plane(S));
        PHG_TRY(trace_core(S.c, S.f, S.p, d_pos + 3 * b0, d_dir + 3 * b0, nb,
                           S.strict ? S.counts : nullptr, S.st));
        BatchScratch B;
        PHG_TRY(batch_scratch(S, nb, B));
        const long long* keep = S.c->keep.as<long long>();
        segment_select_kernel<<<grid_for(nb, 256), 256, 0, S.st>>>(
            keep, S.c->entered.as<uint8_t>(), nb, B.lens, B.segf, B.valid, S.misc);
        PHG_CUDA(cudaGetLastError());
        if (!S.strict)
            PHG_TRY(launch_commit(S, S.c->slab.as<double>(), keep, nullptr, nullptr, B.valid, nb));
        long long nv = 0, ns = 0;
        PHG_TRY(batch_offsets(S, nb, B.lens, B.segf, B.voff, B.sidx, &nv, &ns));
        PHG_TRY(ensure_output(S, ns, nv));
        gather_scalp_kernel<<<grid_for(nb * 32, 256, num_sms() * 16), 256, 0, S.st>>>(
            S.c->slab.as<double>(), row_stride_doubles(S.p->max_vertices), keep, B.valid, B.voff,
            B.sidx, nb, S.verts, S.segs, S.c->g_out_off.as<long long>(),
            S.c->g_out_verts.as<double>(), S.c->g_out_rooted.as<uint8_t>());
        PHG_CUDA(cudaGetLastError());
        S.segs += ns;
        S.verts += nv;
    }
    return PHG_OK;
}

phg_status field_pass(GrowState& S, long long* n_field_seeds) {
    *n_field_seeds = 0;
    phg_ctx* c = S.c;
    const long long V = S.f->nvox();
    const FieldView F = S.f->view();
    long long* d_count = (long long*)c->counters.p + 4;
    thrust::counting_iterator<uint32_t> iota(0);
    // 1. unvisited occupied voxels, ascending linear index == np.argwhere's C order
    PHG_TRY(c->g_flags.ensure((size_t)V));
    PHG_TRY(c->g_sel.ensure((size_t)V * 4));
    uint8_t* flags = c->g_flags.as<uint8_t>();
    uint32_t* unvisited = c->g_sel.as<uint32_t>();
    unvisited_flag_kernel<<<grid_for(V, 256, num_sms() * 16), 256, 0, S.st>>>(F.vox, S.counts, V,
                                                                              flags);
    PHG_CUDA(cudaGetLastError());
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, iota, flags, unvisited, d_count, V, S.st);
    PHG_TRY(c->cub_tmp.ensure(tmp));
    PHG_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, flags, unvisited, d_count, V,
                                        S.st));
    PHG_CUDA(cudaMemcpyAsync(c->host_total, d_count, 8, cudaMemcpyDeviceToHost, S.st));
    PHG_CUDA(cudaStreamSynchronize(S.st));
    const long long U = c->host_total[0];
    if (U == 0) return PHG_OK;
    // 2. stride down to field_seeds voxels
    long long m = U;
    const uint32_t* picked = unvisited;
    if (U > S.g->field_seeds) {
        m = S.g->field_seeds;
        PHG_TRY(c->g_pick.ensure((size_t)m * 4));
        stride_pick_kernel<<<grid_for(m, 256), 256, 0, S.st>>>(unvisited, U, m,
                                                                c->g_pick.as<uint32_t>());
        PHG_CUDA(cudaGetLastError());
        picked = c->g_pick.as<uint32_t>();
    }
    // 3. centres + unit orientation, then drop rows with |ori| <= 1e-9
    PHG_TRY(c->g_raw.ensure((size_t)m * 48 + (size_t)m));
    double* raw_pos = c->g_raw.as<double>();
    double* raw_dir = raw_pos + 3 * m;
    uint8_t* keepf = (uint8_t*)(raw_dir + 3 * m);
    field_seed_kernel<<<grid_for(m, 256), 256, 0, S.st>>>(F, picked, m, raw_pos, raw_dir, keepf);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(c->g_rows.ensure((size_t)m * 4));
    uint32_t* rows = c->g_rows.as<uint32_t>();
    tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, iota, keepf, rows, d_count, m, S.st);
    PHG_TRY(c->cub_tmp.ensure(tmp));
    PHG_CUDA(cub::DeviceSelect::Flagged(c->cub_tmp.p, tmp, iota, keepf, rows, d_count, m, S.st));
    PHG_CUDA(cudaMemcpyAsync(c->host_total, d_count, 8, cudaMemcpyDeviceToHost, S.st));
    PHG_CUDA(cudaStreamSynchronize(S.st));
    const long long nf = c->host_total[0];
    *n_field_seeds = nf;
    if (nf == 0) return PHG_OK;
    PHG_TRY(c->g_fpos.ensure((size_t)nf * 24));
    PHG_TRY(c->g_fdir.ensure((size_t)nf * 24));
    double* pos = c->g_fpos.as<double>();
    double* dir = c->g_fdir.as<double>();
    row_gather_kernel<<<grid_for(nf, 256), 256, 0, S.st>>>(raw_pos, raw_dir, rows, nf, pos, dir);
    PHG_CUDA(cudaGetLastError());
    // 4. batches: trace +d and -d against the same frozen plane, join, keep, commit
    const long long bs = S.g->batch_size;
    const size_t rs = row_stride_doubles(S.p->max_vertices);
    for (long long b0 = 0; b0 < nf; b0 += bs) {
        const long long nb = std::min(bs, nf - b0);
        PHG_TRY(set_cap_plane(S));
        PHG_TRY(trace_core(S.c, S.f, S.p, pos + 3 * b0, dir + 3 * b0, nb,
                           S.strict ? S.counts : nullptr, S.st));
        // keep the forward trace aside
        swap_buf(S.c->slab, S.c->g_slab2);
        swap_buf(S.c->keep, S.c->g_keep2);
        swap_buf(S.c->entered, S.c->g_ent2);
        PHG_TRY(S.c->g_neg_dir.ensure((size_t)nb * 24));
        double* ndir = S.c->g_neg_dir.as<double>();
        negate_kernel<<<grid_for(nb * 3, 256, num_sms() * 16), 256, 0, S.st>>>(dir + 3 * b0, ndir,
                                                                                nb * 3);
        PHG_CUDA(cudaGetLastError());
        if (!S.strict) PHG_TRY(set_cap_plane(S));  // identical plane: no commits in between
        PHG_TRY(trace_core(S.c, S.f, S.p, pos + 3 * b0, ndir, nb, S.strict ? S.counts : nullptr,
                           S.st));
        const double* slab_f = S.c->g_slab2.as<double>();
        const long long* keep_f = S.c->g_keep2.as<long long>();
        const uint8_t* ent_f = S.c->g_ent2.as<uint8_t>();
        const double* slab_b = S.c->slab.as<double>();
        const long long* keep_b = S.c->keep.as<long long>();
        const uint8_t* ent_b = S.c->entered.as<uint8_t>();
        BatchScratch B;
        PHG_TRY(batch_scratch(S, nb, B));
        join_select_kernel<<<grid_for(nb, 256), 256, 0, S.st>>>(keep_f, ent_f, keep_b, ent_b, nb,
                                                                B.lens, B.segf, B.valid);
        PHG_CUDA(cudaGetLastError());
        if (!S.strict) PHG_TRY(launch_commit(S, slab_f, keep_f, slab_b, keep_b, B.valid, nb));
        long long nv = 0, ns = 0;
        PHG_TRY(batch_offsets(S, nb, B.lens, B.segf, B.voff, B.sidx, &nv, &ns));
        PHG_TRY(ensure_output(S, ns, nv));
        gather_joined_kernel<<<grid_for(nb * 32, 256, num_sms() * 16), 256, 0, S.st>>>(
            slab_f, slab_b, rs, keep_f, keep_b, B.valid, B.voff, B.sidx, nb, S.verts, S.segs,
            S.c->g_out_off.as<long long>(), S.c->g_out_verts.as<double>(),
            S.c->g_out_rooted.as<uint8_t>());
        PHG_CUDA(cudaGetLastError());
        S.segs += ns;
        S.verts += nv;
    }
    return PHG_OK;
}

}  // namespace
}  // namespace phg

extern "C" {

phg_status phg_grow_init(phg_ctx* c, phg_field* f, const phg_params_v1* p,
                         const phg_grow_params_v1* g, const double* seeds, const double* normals,
                         int64_t n, uint16_t* counts, int64_t* n_segments, int64_t* n_verts,
                         int64_t report[4], void* stream) {
    if (!c || !f || !p || !g || !counts || !n_segments || !n_verts || !report)
        return fail(PHG_ERR_INVALID, "phg_grow_init: null argument");
    if (n < 0) return fail(PHG_ERR_INVALID, "phg_grow_init: negative seed count");
    if (n > 0 && (!seeds || !normals))
        return fail(PHG_ERR_INVALID, "phg_grow_init: null seeds");
    if (g->batch_size < 1 || g->occupancy_cap < 1)
        return fail(PHG_ERR_INVALID, "phg_grow_init: invalid batch_size / occupancy_cap");
    if (p->max_vertices < 1)
        return fail(PHG_ERR_INVALID, "phg_grow_init: max_vertices must be >= 1");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != f->device)
        return fail(PHG_ERR_INVALID, "phg_grow_init: field lives on device %d", f->device);
    cudaStream_t st = as_stream(stream);
    c->grow_ready = false;
    GrowState S{c, f, p, g, st, (p->flags & PHG_FLAG_STRICT) != 0, nullptr};
    const long long V = f->nvox();
    PHG_TRY(c->counts32.ensure((size_t)V * 4));
    S.counts = c->counts32.as<uint32_t>();
    const bool counts_dev = is_device_ptr(counts);
    const void* d_counts = nullptr;
    PHG_TRY(to_device(counts, (size_t)V * 2, c->live_stage, &d_counts, st));
    u16_to_u32<<<grid_for(V, 256, num_sms() * 16), 256, 0, st>>>((const uint16_t*)d_counts,
                                                                S.counts, V);
    PHG_CUDA(cudaGetLastError());
    PHG_TRY(c->counters.ensure(64));
    PHG_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, st));
    DevBuf misc_buf;  // [0] = never-entered scalp seeds
    PHG_TRY(misc_buf.ensure(64));
    PHG_CUDA(cudaMemsetAsync(misc_buf.p, 0, 64, st));
    unsigned long long* misc = misc_buf.as<unsigned long long>();
    S.misc = misc;
    const void *d_pos = nullptr, *d_dir = nullptr;
    if (n > 0) {
        PHG_TRY(to_device(seeds, (size_t)n * 24, c->g_seeds_pos, &d_pos, st));
        PHG_TRY(to_device(normals, (size_t)n * 24, c->g_seeds_dir, &d_dir, st));
    }
    PHG_CUDA(cudaEventRecord(c->ev[0], st));  // device window: uploads done .. downloads begin
    phg_status s = PHG_OK;
    if (n > 0) s = scalp_pass(S, (const double*)d_pos, (const double*)d_dir, n);
    long long scalp_segs = S.segs;
    long long n_field = 0;
    if (s == PHG_OK && n > 0 && g->field_seeds > 0) s = field_pass(S, &n_field);
    f->has_cap = false;  // the driver overwrote the field's cap plane; leave none behind
    if (s != PHG_OK) return s;
    PHG_CUDA(cudaEventRecord(c->ev[2], st));
    // counts back to vol.counts (uint16 wrap like np ndarray +=)
    uint16_t* dst16 = counts_dev ? counts : c->live_stage.as<uint16_t>();
    u32_to_u16<<<grid_for(V, 256, num_sms() * 16), 256, 0, st>>>(S.counts, dst16, V);
    PHG_CUDA(cudaGetLastError());
    if (!counts_dev)
        PHG_CUDA(cudaMemcpyAsync(counts, dst16, (size_t)V * 2, cudaMemcpyDeviceToHost, st));
    unsigned long long never = 0;
    PHG_CUDA(cudaMemcpyAsync(&never, misc, 8, cudaMemcpyDeviceToHost, st));
    PHG_TRY(ensure_output(S, 0, 0));
    PHG_CUDA(cudaMemcpyAsync(c->g_out_off.as<long long>() + S.segs, &S.verts, 8,
                             cudaMemcpyHostToDevice, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    cudaEventElapsedTime(&c->last_total_ms, c->ev[0], c->ev[2]);
    report[0] = (int64_t)never;
    report[1] = scalp_segs;
    report[2] = n_field;
    report[3] = S.segs - scalp_segs;
    *n_segments = S.segs;
    *n_verts = S.verts;
    c->grow_segs = S.segs;
    c->grow_verts = S.verts;
    c->grow_ready = true;
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
    if (verts && c->grow_verts)
        PHG_CUDA(cudaMemcpyAsync(verts, c->g_out_verts.p, (size_t)c->grow_verts * 24,
                                 cudaMemcpyDefault, st));
    if (rooted && c->grow_segs)
        PHG_CUDA(cudaMemcpyAsync(rooted, c->g_out_rooted.p, (size_t)c->grow_segs,
                                 cudaMemcpyDefault, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

}  // extern "C"
