// phg_io.cu -- reference wire formats straight to / from device memory.
//
//   phg_stnd_encode      STND image of a CSR strand set (strands.py:63-69 write_strands):
//                        u32 magic 0x444E5453, u32 count, per strand u32 n + n*3 float32
//   phg_field_from_oovl  OOVL payload -> packed float4 field (volume.py:248-266 read_volume):
//                        np.packbits(occ) bits (MSB first) + float32 ori of occupied voxels
//                        in C order, scattered by the rank of each set bit

#include "phg_core.cuh"

using namespace phg;

namespace phg {
namespace {

constexpr uint32_t kStrandMagic = 0x444E5453u;  // "STND" (strands.py:16)

// byte offset of strand i's header: 8 + 4*i + 12*offsets[i]
__global__ void stnd_encode_kernel(const long long* __restrict__ off, const double* __restrict__ v,
                                   long long n, uint8_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    if (warp == 0 && lane == 0) {
        reinterpret_cast<uint32_t*>(out)[0] = kStrandMagic;
        reinterpret_cast<uint32_t*>(out)[1] = (uint32_t)n;
    }
    for (long long i = warp; i < n; i += nwarps) {
        const long long o = off[i], len = off[i + 1] - o;
        uint8_t* base = out + 8 + 4 * i + 12 * o;
        if (lane == 0) *reinterpret_cast<uint32_t*>(base) = (uint32_t)len;
        float* dst = reinterpret_cast<float*>(base + 4);
        const double* src = v + 3 * o;
        for (long long j = lane; j < 3 * len; j += 32) dst[j] = __double2float_rn(src[j]);
    }
}

__global__ void byte_popc_kernel(const uint8_t* __restrict__ bits, long long nbytes,
                                 uint32_t* __restrict__ pc) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nbytes;
         i += (long long)gridDim.x * blockDim.x)
        pc[i] = __popc((uint32_t)bits[i]);
}

// voxel i is bit (7 - i%8) of byte i/8 (np.packbits, bitorder="big"); its ori is row
// rank(i) = (set bits before byte i/8) + (set bits above it within the byte)
// Unoccupied voxels keep the zeros of the freshly cleared padded field (read_volume fills
// their ori with 0, so the packing is the zeroed one whenever the payload is finite).
__global__ void oovl_scatter_kernel(FieldView F, const uint8_t* __restrict__ bits,
                                    const unsigned long long* __restrict__ byte_rank,
                                    const float* __restrict__ ori, long long nvox,
                                    float4* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvox;
         i += (long long)gridDim.x * blockDim.x) {
        const uint32_t b = bits[i >> 3];
        const int k = (int)(i & 7);
        if ((b >> (7 - k)) & 1u) {
            const unsigned long long r = byte_rank[i >> 3] + __popc(b >> (8 - k));
            out[vox_index_lin(F, (uint32_t)i)] =
                make_float4(ori[3 * r], ori[3 * r + 1], ori[3 * r + 2], occ_flag(true));
        }
    }
}

}  // namespace
}  // namespace phg

extern "C" {

phg_status phg_stnd_encode(const int64_t* offsets, const double* verts, int64_t n_strands,
                           uint8_t* out, void* stream) {
    PHG_RANGE("phg/stnd_encode");
    if (!offsets || !out || n_strands < 0) return fail(PHG_ERR_INVALID, "phg_stnd_encode: bad args");
    cudaStream_t st = as_stream(stream);
    DevBuf s_off, s_v, s_out;
    const void* d_off = nullptr;
    PHG_TRY(to_device(offsets, (size_t)(n_strands + 1) * 8, s_off, &d_off, st));
    long long total = 0;
    PHG_CUDA(cudaMemcpyAsync(&total, (const long long*)d_off + n_strands, 8, cudaMemcpyDefault, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    if (total > 0 && !verts) return fail(PHG_ERR_INVALID, "phg_stnd_encode: null verts");
    const void* d_v = nullptr;
    PHG_TRY(to_device(verts, (size_t)total * 24, s_v, &d_v, st));
    const size_t bytes = 8 + 4 * (size_t)n_strands + 12 * (size_t)total;
    const bool out_dev = is_device_ptr(out);
    uint8_t* d_out = out;
    if (!out_dev) {
        PHG_TRY(s_out.ensure(bytes));
        d_out = s_out.as<uint8_t>();
    }
    stnd_encode_kernel<<<grid_for(std::max<long long>(n_strands, 1) * 32, 256, num_sms() * 16), 256,
                         0, st>>>((const long long*)d_off, (const double*)d_v, n_strands, d_out);
    PHG_CUDA(cudaGetLastError());
    if (!out_dev) PHG_TRY(copy_d2h(out, d_out, bytes, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

phg_status phg_field_from_oovl(phg_field** out, const uint8_t* bits, const float* ori_occupied,
                               int64_t n_occ, int64_t nx, int64_t ny, int64_t nz,
                               const double origin[3], double voxel_size, void* stream) {
    PHG_RANGE("phg/field_from_oovl");
    if (!out || !bits || !origin || n_occ < 0)
        return fail(PHG_ERR_INVALID, "phg_field_from_oovl: null argument");
    *out = nullptr;
    if (!field_dims_ok(nx, ny, nz)) return fail(PHG_ERR_INVALID, "phg_field_from_oovl: bad dims");
    if (!(voxel_size > 0) || !std::isfinite(voxel_size))
        return fail(PHG_ERR_INVALID, "phg_field_from_oovl: voxel_size must be positive");
    cudaStream_t st = as_stream(stream);
    const long long V = nx * ny * nz, nbytes = (V + 7) / 8;
    DevBuf s_bits, s_ori, pc, rank;
    const void *d_bits = nullptr, *d_ori = nullptr;
    PHG_TRY(to_device(bits, (size_t)nbytes, s_bits, &d_bits, st));
    PHG_TRY(to_device(ori_occupied, (size_t)n_occ * 12, s_ori, &d_ori, st));
    PHG_TRY(pc.ensure((size_t)nbytes * 4));
    PHG_TRY(rank.ensure((size_t)(nbytes + 1) * 8));
    byte_popc_kernel<<<grid_for(nbytes, 256, num_sms() * 16), 256, 0, st>>>(
        (const uint8_t*)d_bits, nbytes, pc.as<uint32_t>());
    PHG_CUDA(cudaGetLastError());
    // exclusive scan of per-byte popcounts (64-bit ranks)
    unsigned long long* r = rank.as<unsigned long long>();
    PHG_CUDA(cudaMemsetAsync(r, 0, 8, st));
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, pc.as<uint32_t>(), r + 1, nbytes, st);
    DevBuf cub_tmp;
    PHG_TRY(cub_tmp.ensure(tmp));
    PHG_CUDA(cub::DeviceScan::InclusiveSum(cub_tmp.p, tmp, pc.as<uint32_t>(), r + 1, nbytes, st));
    unsigned long long total = 0;
    PHG_CUDA(cudaMemcpyAsync(&total, r + nbytes, 8, cudaMemcpyDeviceToHost, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    // bits past nvox in the last byte are padding (np.unpackbits(...)[:nvox] ignores them)
    unsigned long long pad = 0;
    if (V % 8) {
        uint8_t last = 0;
        PHG_CUDA(cudaMemcpy(&last, (const uint8_t*)d_bits + nbytes - 1, 1, cudaMemcpyDefault));
        pad = __builtin_popcount((unsigned)(last & ((1u << (8 - V % 8)) - 1u)));
    }
    if ((long long)(total - pad) != n_occ)
        return fail(PHG_ERR_INVALID,
                    "phg_field_from_oovl: truncated orientation payload (%llu occupied, %lld rows)",
                    total - pad, (long long)n_occ);
    phg_field* f = new phg_field();
    cudaGetDevice(&f->device);
    f->nx = nx;
    f->ny = ny;
    f->nz = nz;
    for (int k = 0; k < 3; ++k) f->origin[k] = origin[k];
    f->vs = voxel_size;
    phg_status s = field_alloc_padded(f, st);
    if (s == PHG_OK) s = field_check_finite(f, (const float*)d_ori, 3 * n_occ, st);
    if (s != PHG_OK) {
        delete f;
        return s;
    }
    oovl_scatter_kernel<<<grid_for(V, 256, num_sms() * 16), 256, 0, st>>>(
        f->view(), (const uint8_t*)d_bits, r, (const float*)d_ori, V, f->vox.as<float4>());
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        delete f;
        return fail(PHG_ERR_CUDA, "oovl_scatter_kernel: %s", cudaGetErrorString(e));
    }
    s = field_finish(f, st);
    if (s != PHG_OK) {
        delete f;
        return s;
    }
    *out = f;
    return PHG_OK;
}

}  // extern "C"
