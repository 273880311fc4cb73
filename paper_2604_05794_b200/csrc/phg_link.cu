// phg_link.cu -- segment linking, chain assembly and scalp attachment (the rest of phg.grow).
//
// Reference: /root/reference/pkg/src/strandkit/phg.py
//   _end_tangent/_start_tangent  :309-316  windowed end/start tangents
//   compute_links                :337-377  end_i -> start_j pairs with d < link_dist and
//                                          dot(et_i, st_j) > cos(angle), greedy in (d, i, j) order,
//                                          each end/start used once, union-find rejects cycles
//   _smooth / connect_segments   :380-413  chains concatenated, Laplacian-smoothed when merged,
//                                          resampled uniformly (geom.py:82-95 with np.interp)
//   attach_to_scalp              :419-439  nearest scalp vertex to either end (lowest id on ties,
//                                          spatial.py:54-65), prepended, strand reversed if the
//                                          tail is closer
//   grow                         :467-468  polyline_tangents (geom.py:98-103)
// Device: endpoint/tangent kernel, uniform-grid radius search (CUB-sorted cell keys), candidate
// pairs sorted by (d, i, j) with two stable radix sorts, chain assembly + smoothing + arc length
// + numpy-exact interp resampling, brute-force exact nearest scalp vertex, tangents.
// Host (native C++): the greedy union-find acceptance over the sorted pairs (inherently
// sequential, O(pairs)) and the chain walk.

#include <vector>

#include "phg_core.cuh"

using namespace phg;

namespace phg {
namespace {

// ---- endpoints and windowed tangents ------------------------------------------------------
__device__ __forceinline__ void unit_v(double& x, double& y, double& z) { unit3(x, y, z); }

__global__ void endpoints_kernel(const long long* __restrict__ off, const double* __restrict__ v,
                                 long long n, int window, double* __restrict__ start,
                                 double* __restrict__ end, double* __restrict__ st,
                                 double* __restrict__ et) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long o = off[i], len = off[i + 1] - o;
    const double* p = v + 3 * o;
    const long long k = min((long long)window, len - 1);
    const double* last = p + 3 * (len - 1);
    for (int c = 0; c < 3; ++c) {
        start[3 * i + c] = p[c];
        end[3 * i + c] = last[c];
    }
    // _start_tangent: normalize(v[k] - v[0]); _end_tangent: normalize(v[-1] - v[-1-k])
    double sx = p[3 * k] - p[0], sy = p[3 * k + 1] - p[1], sz = p[3 * k + 2] - p[2];
    unit_v(sx, sy, sz);
    const double* b = last - 3 * k;
    double ex = last[0] - b[0], ey = last[1] - b[1], ez = last[2] - b[2];
    unit_v(ex, ey, ez);
    st[3 * i] = sx;
    st[3 * i + 1] = sy;
    st[3 * i + 2] = sz;
    et[3 * i] = ex;
    et[3 * i + 1] = ey;
    et[3 * i + 2] = ez;
}

struct Grid {
    double ox, oy, oz, h;  // cell = floor((p - o) / h)
    int nx, ny, nz;
};

__device__ __forceinline__ int cell_of(double p, double o, double h, int n) {
    const double g = floor((p - o) / h);
    return g < 0 ? 0 : (g > n - 1 ? n - 1 : (int)g);
}

__device__ __forceinline__ unsigned long long cell_key(int x, int y, int z) {
    return ((unsigned long long)x << 42) | ((unsigned long long)y << 21) | (unsigned long long)z;
}

__global__ void start_keys_kernel(const double* __restrict__ start, long long n, Grid G,
                                  unsigned long long* __restrict__ keys, int* __restrict__ ids) {
    long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (j >= n) return;
    keys[j] = cell_key(cell_of(start[3 * j], G.ox, G.h, G.nx), cell_of(start[3 * j + 1], G.oy, G.h, G.ny),
                       cell_of(start[3 * j + 2], G.oz, G.h, G.nz));
    ids[j] = (int)j;
}

__device__ __forceinline__ long long lower_bound_key(const unsigned long long* a, long long n,
                                                     unsigned long long k) {
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// For end i: every start j in the 27 neighbouring cells with d < r (d as numpy computes
// np.linalg.norm(points[idx] - q): sqrt((dx*dx + dy*dy) + dz*dz)), j != i and
// dot(et_i, st_j) > gate.  WRITE=false counts, WRITE=true emits at out_off[i].
template <bool WRITE>
__global__ void pairs_kernel(const double* __restrict__ start, const double* __restrict__ end,
                             const double* __restrict__ st, const double* __restrict__ et,
                             long long n, Grid G, const unsigned long long* __restrict__ skeys,
                             const int* __restrict__ sids, double r, double gate,
                             long long* __restrict__ count, const long long* __restrict__ out_off,
                             double* __restrict__ pd, unsigned long long* __restrict__ pij) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double qx = end[3 * i], qy = end[3 * i + 1], qz = end[3 * i + 2];
    const double tx = et[3 * i], ty = et[3 * i + 1], tz = et[3 * i + 2];
    const int cx = cell_of(qx, G.ox, G.h, G.nx), cy = cell_of(qy, G.oy, G.h, G.ny),
              cz = cell_of(qz, G.oz, G.h, G.nz);
    long long c = 0;
    long long w = WRITE ? out_off[i] : 0;
    for (int dx = -1; dx <= 1; ++dx) {
        const int x = cx + dx;
        if (x < 0 || x >= G.nx) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= G.ny) continue;
            for (int dz = -1; dz <= 1; ++dz) {
                const int z = cz + dz;
                if (z < 0 || z >= G.nz) continue;
                const unsigned long long k = cell_key(x, y, z);
                for (long long s = lower_bound_key(skeys, n, k); s < n && skeys[s] == k; ++s) {
                    const int j = sids[s];
                    if (j == i) continue;
                    const double ax = start[3 * j] - qx, ay = start[3 * j + 1] - qy,
                                 az = start[3 * j + 2] - qz;
                    const double d = sqrt((ax * ax + ay * ay) + az * az);
                    if (!(d < r)) continue;
                    const double dot = (tx * st[3 * j] + ty * st[3 * j + 1]) + tz * st[3 * j + 2];
                    if (!(dot > gate)) continue;
                    if (WRITE) {
                        pd[w] = d;
                        pij[w] = ((unsigned long long)i << 32) | (unsigned int)j;
                        ++w;
                    } else {
                        ++c;
                    }
                }
            }
        }
    }
    if (!WRITE) count[i] = c;
}

__global__ void dbits_kernel(const double* __restrict__ d, const long long* __restrict__ perm,
                             long long n, unsigned long long* __restrict__ out) {
    long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k < n) out[k] = (unsigned long long)__double_as_longlong(d[perm ? perm[k] : k]);
}

// ---- chain assembly -----------------------------------------------------------------------
// chain c: member segments members[moff[c] .. moff[c+1]); concatenated into buf at coff[c];
// smoothing (phg._smooth) when merged; arc lengths s (polyline_lengths) and totals.
__global__ void chain_concat_kernel(const long long* __restrict__ seg_off,
                                    const double* __restrict__ v, const int* __restrict__ members,
                                    const long long* __restrict__ moff,
                                    const long long* __restrict__ coff, long long nchains,
                                    double* __restrict__ buf) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = warp; c < nchains; c += nw) {
        long long o = coff[c];
        for (long long m = moff[c]; m < moff[c + 1]; ++m) {
            const int sgi = members[m];
            const long long a = seg_off[sgi], len = seg_off[sgi + 1] - a;
            for (long long j = lane; j < 3 * len; j += 32) buf[3 * o + j] = v[3 * a + j];
            o += len;
        }
    }
}

// one Jacobi smoothing iteration v[1:-1] += s * (0.5 * (v[:-2] + v[2:]) - v[1:-1]) (phg.py:385)
__global__ void smooth_iter_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                   const long long* __restrict__ coff,
                                   const uint8_t* __restrict__ do_smooth, long long nchains,
                                   double strength) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = warp; c < nchains; c += nw) {
        const long long o = coff[c], len = coff[c + 1] - o;
        const bool sm = do_smooth[c] && len >= 3;
        for (long long j = lane; j < 3 * len; j += 32) {
            const long long k = j / 3;
            double val = src[3 * o + j];
            if (sm && k > 0 && k < len - 1) {
                const double avg = 0.5 * (src[3 * o + j - 3] + src[3 * o + j + 3]);
                val = val + strength * (avg - val);
            }
            dst[3 * o + j] = val;
        }
    }
}

// polyline_lengths (geom.py:76-79): s_0 = 0, s_k = s_{k-1} + |v_k - v_{k-1}| (sequential cumsum)
__global__ void arclen_kernel(const double* __restrict__ buf, const long long* __restrict__ coff,
                              long long nchains, double* __restrict__ s, double step,
                              long long* __restrict__ nout) {
    long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= nchains) return;
    const long long o = coff[c], len = coff[c + 1] - o;
    double acc = 0.0;
    s[o] = 0.0;
    for (long long k = 1; k < len; ++k) {
        const double* a = buf + 3 * (o + k - 1);
        const double dx = a[3] - a[0], dy = a[4] - a[1], dz = a[5] - a[2];
        acc = acc + sqrt((dx * dx + dy * dy) + dz * dz);
        s[o + k] = acc;
    }
    // resample_polyline_uniform: n = max(1, int(round(total / step))) -> n + 1 points;
    // fewer than 2 input vertices: copied as is (and later dropped, len < 2)
    if (len < 2) {
        nout[c] = len;
    } else {
        const long long m = (long long)rint(acc / step);  // Python round(): half to even
        nout[c] = (m < 1 ? 1 : m) + 1;
    }
}

// np.interp(x, xp, fp) for sorted xp, numpy 2.x arr_interp semantics (left = fp[0], right = fp[-1])
__device__ __forceinline__ double np_interp(double x, const double* xp, const double* fp3,
                                            int comp, long long n) {
    if (x != x) return x;
    if (x > xp[n - 1]) return fp3[3 * (n - 1) + comp];
    if (x < xp[0]) return fp3[comp];
    long long lo = 0, hi = n;  // j = (first index with xp[j] > x) - 1
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (x >= xp[mid]) lo = mid + 1; else hi = mid;
    }
    const long long j = lo - 1;
    if (j == n - 1) return fp3[3 * j + comp];
    if (xp[j] == x) return fp3[3 * j + comp];
    const double y0 = fp3[3 * j + comp], y1 = fp3[3 * (j + 1) + comp];
    const double slope = (y1 - y0) / (xp[j + 1] - xp[j]);
    double r = slope * (x - xp[j]) + y0;
    if (r != r) {
        r = slope * (x - xp[j + 1]) + y1;
        if (r != r && y0 == y1) r = y0;
    }
    return r;
}

// resample_polyline_uniform (geom.py:82-95): grid = np.linspace(0, total, n + 1)
__global__ void resample_kernel(const double* __restrict__ buf, const double* __restrict__ s,
                                const long long* __restrict__ coff,
                                const long long* __restrict__ roff, long long nchains,
                                double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = warp; c < nchains; c += nw) {
        const long long o = coff[c], len = coff[c + 1] - o;
        const long long ro = roff[c], cnt = roff[c + 1] - ro;
        if (len < 2) {  // geom: `if len(verts) < 2: return verts.copy()`
            for (long long j = lane; j < 3 * len; j += 32) out[3 * ro + j] = buf[3 * o + j];
            continue;
        }
        const double total = s[o + len - 1];
        const long long div = cnt - 1;
        const double step = total / (double)div;
        for (long long k = lane; k < cnt; k += 32) {
            double g;
            if (k == cnt - 1) g = total;                          // y[-1] = stop
            else if (step == 0.0) g = ((double)k / (double)div) * total;  // any_step_zero
            else g = (double)k * step + 0.0;
            for (int comp = 0; comp < 3; ++comp)
                out[3 * (ro + k) + comp] = np_interp(g, s + o, buf + 3 * o, comp, len);
        }
    }
}

// ---- attachment -------------------------------------------------------------------------
// SpatialIndex.nearest (spatial.py:54-65): minimal |p - q| (numpy row norm), lowest id on ties
__device__ __forceinline__ void nearest_scalp(const double* __restrict__ sv, long long ns,
                                              double qx, double qy, double qz, int lane,
                                              double& best_d, long long& best_i) {
    double bd = __longlong_as_double(0x7ff0000000000000ll);
    long long bi = -1;
    for (long long k = lane; k < ns; k += 32) {
        const double dx = sv[3 * k] - qx, dy = sv[3 * k + 1] - qy, dz = sv[3 * k + 2] - qz;
        const double d = sqrt((dx * dx + dy * dy) + dz * dz);
        if (d < bd || (d == bd && k < bi)) {
            bd = d;
            bi = k;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(kFull, bd, o);
        const long long oi = __shfl_xor_sync(kFull, bi, o);
        if (od < bd || (od == bd && oi >= 0 && (bi < 0 || oi < bi))) {
            bd = od;
            bi = oi;
        }
    }
    best_d = bd;
    best_i = bi;
}

// attach decision per strand: mode 0 keep, 1 prepend head's scalp vertex, 2 prepend tail's and
// reverse (phg.py:425-438); unrooted strands beyond the radius stay as they are
__global__ void attach_kernel(const double* __restrict__ v, const long long* __restrict__ roff,
                              const uint8_t* __restrict__ rooted, long long nstr,
                              const double* __restrict__ sv, long long ns, double radius,
                              uint8_t* __restrict__ mode, long long* __restrict__ sid,
                              long long* __restrict__ newlen,
                              unsigned long long* __restrict__ n_unrooted) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = warp; c < nstr; c += nw) {
        const long long o = roff[c], len = roff[c + 1] - o;
        if (rooted[c] || ns == 0) {
            if (lane == 0) {
                mode[c] = 0;
                newlen[c] = len;
                if (!rooted[c]) atomicAdd(n_unrooted, 1ull);
            }
            continue;
        }
        double hd, td;
        long long hid, tid;
        nearest_scalp(sv, ns, v[3 * o], v[3 * o + 1], v[3 * o + 2], lane, hd, hid);
        const double* t = v + 3 * (o + len - 1);
        nearest_scalp(sv, ns, t[0], t[1], t[2], lane, td, tid);
        if (lane == 0) {
            const double mn = hd < td ? hd : td;  // Python min(hd, td)
            if (mn >= radius) {
                mode[c] = 0;
                newlen[c] = len;
                atomicAdd(n_unrooted, 1ull);
            } else if (td < hd) {
                mode[c] = 2;
                sid[c] = tid;
                newlen[c] = len + 1;
            } else {
                mode[c] = 1;
                sid[c] = hid;
                newlen[c] = len + 1;
            }
        }
    }
}

// final strands + polyline_tangents (geom.py:98-103): unit forward differences, last repeated
__global__ void finalize_kernel(const double* __restrict__ v, const long long* __restrict__ roff,
                                const uint8_t* __restrict__ mode, const long long* __restrict__ sid,
                                const double* __restrict__ sv, const long long* __restrict__ foff,
                                long long nstr, double* __restrict__ out,
                                double* __restrict__ tan) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long c = warp; c < nstr; c += nw) {
        const long long o = roff[c], len = roff[c + 1] - o;
        const long long fo = foff[c], flen = foff[c + 1] - fo;
        const int md = mode[c];
        for (long long j = lane; j < 3 * flen; j += 32) {
            const long long k = j / 3, comp = j - 3 * k;
            double val;
            if (md == 0) val = v[3 * (o + k) + comp];
            else if (k == 0) val = sv[3 * sid[c] + comp];
            else if (md == 1) val = v[3 * (o + k - 1) + comp];
            else val = v[3 * (o + len - k) + comp];  // reversed strand after the scalp vertex
            out[3 * fo + j] = val;
        }
        __syncwarp();
        for (long long k = lane; k < flen; k += 32) {
            const long long a = (k < flen - 1) ? k : flen - 2;
            if (a < 0) {  // single-vertex strand: np.diff is empty; tangents undefined
                tan[3 * (fo + k)] = tan[3 * (fo + k) + 1] = tan[3 * (fo + k) + 2] = 0.0;
                continue;
            }
            const double* p = out + 3 * (fo + a);
            double dx = p[3] - p[0], dy = p[4] - p[1], dz = p[5] - p[2];
            unit3(dx, dy, dz);
            tan[3 * (fo + k)] = dx;
            tan[3 * (fo + k) + 1] = dy;
            tan[3 * (fo + k) + 2] = dz;
        }
    }
}

template <class T>
phg_status d2h(std::vector<T>& h, const void* d, size_t n, cudaStream_t st) {
    h.resize(n);
    if (n) PHG_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

template <class T>
phg_status h2d(DevBuf& b, const std::vector<T>& h, cudaStream_t st) {
    PHG_TRY(b.ensure(std::max<size_t>(h.size() * sizeof(T), 8)));
    if (!h.empty())
        PHG_CUDA(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return PHG_OK;
}

}  // namespace
}  // namespace phg

extern "C" {

phg_status phg_link(phg_ctx* c, const int64_t* offsets, const double* verts,
                    const uint8_t* rooted, const uint8_t* source, int64_t n,
                    const double* scalp, int64_t n_scalp, const phg_link_params_v1* lp,
                    int64_t counts_out[4], void* stream) {
    PHG_RANGE("phg/link");
    if (!c || !lp || !counts_out || n < 0 || n_scalp < 0)
        return fail(PHG_ERR_INVALID, "phg_link: bad argument");
    if (!(lp->link_dist_mm > 0)) return fail(PHG_ERR_INVALID, "phg_link: link_dist_mm must be > 0");
    if (!(lp->step_mm > 0)) return fail(PHG_ERR_INVALID, "phg_link: step_mm must be > 0");
    cudaStream_t st = as_stream(stream);
    c->link_ready = false;
    // ---- inputs: explicit CSR, or the last phg_grow_init result when offsets == NULL
    const long long* d_off;
    const double* d_v;
    const uint8_t *d_root, *d_src;
    if (offsets) {
        if (n > 0 && (!verts || !rooted || !source))
            return fail(PHG_ERR_INVALID, "phg_link: null segment arrays");
        const void* p = nullptr;
        PHG_TRY(to_device(offsets, (size_t)(n + 1) * 8, c->l_in_off, &p, st));
        d_off = (const long long*)p;
        long long total = 0;
        PHG_CUDA(cudaMemcpyAsync(&total, d_off + n, 8, cudaMemcpyDefault, st));
        PHG_CUDA(cudaStreamSynchronize(st));
        PHG_TRY(to_device(verts, (size_t)total * 24, c->l_in_v, &p, st));
        d_v = (const double*)p;
        PHG_TRY(to_device(rooted, (size_t)n, c->l_in_r, &p, st));
        d_root = (const uint8_t*)p;
        PHG_TRY(to_device(source, (size_t)n, c->l_in_s, &p, st));
        d_src = (const uint8_t*)p;
    } else {
        if (!c->grow_ready) return fail(PHG_ERR_STATE, "phg_link: no phg_grow_init result");
        n = c->grow_segs;
        d_off = c->g_out_off.as<long long>();
        d_v = c->g_out_verts.as<double>();
        d_root = c->g_out_rooted.as<uint8_t>();
        d_src = nullptr;  // traced if rooted else field
    }
    if (n >= (1ll << 31)) return fail(PHG_ERR_INVALID, "phg_link: more than 2^31 segments");
    std::vector<long long> h_off;
    PHG_TRY(d2h(h_off, d_off, (size_t)n + 1, st));
    std::vector<uint8_t> h_root, h_src;
    PHG_TRY(d2h(h_root, d_root, (size_t)n, st));
    if (d_src) {
        PHG_TRY(d2h(h_src, d_src, (size_t)n, st));
    } else {
        h_src.resize(n);
        for (long long i = 0; i < n; ++i) h_src[i] = h_root[i] ? 0 : 1;
    }
    // ---- 1. endpoints and tangents
    PHG_TRY(c->l_end.ensure((size_t)std::max<long long>(n, 1) * 96));
    double* start = c->l_end.as<double>();
    double* end = start + 3 * n;
    double* stg = end + 3 * n;
    double* etg = stg + 3 * n;
    std::vector<std::pair<long long, long long>> sorted_pairs;
    long long P = 0;
    if (n > 0) {
        endpoints_kernel<<<grid_for(n, 128), 128, 0, st>>>(d_off, d_v, n, lp->tangent_window, start,
                                                           end, stg, etg);
        PHG_CUDA(cudaGetLastError());
        // ---- 2. uniform grid over the starts (cell >= link_dist; 21 bits per axis)
        std::vector<double> h_start;
        PHG_TRY(d2h(h_start, start, (size_t)n * 3, st));
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (long long j = 0; j < n; ++j)
            for (int k = 0; k < 3; ++k) {
                const double x = h_start[3 * j + k];
                if (x == x) {
                    lo[k] = std::min(lo[k], x);
                    hi[k] = std::max(hi[k], x);
                }
            }
        Grid G;
        double h = lp->link_dist_mm;
        for (int k = 0; k < 3; ++k) {
            if (lo[k] > hi[k]) lo[k] = hi[k] = 0.0;
            h = std::max(h, (hi[k] - lo[k]) / 1.0e6);
        }
        G.ox = lo[0];
        G.oy = lo[1];
        G.oz = lo[2];
        G.h = h;
        G.nx = (int)((hi[0] - lo[0]) / h) + 1;
        G.ny = (int)((hi[1] - lo[1]) / h) + 1;
        G.nz = (int)((hi[2] - lo[2]) / h) + 1;
        PHG_TRY(c->l_keys.ensure((size_t)n * 8 * 2));
        PHG_TRY(c->l_ids.ensure((size_t)n * 4 * 2));
        unsigned long long* k0 = c->l_keys.as<unsigned long long>();
        unsigned long long* k1 = k0 + n;
        int* i0 = c->l_ids.as<int>();
        int* i1 = i0 + n;
        start_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(start, n, G, k0, i0);
        PHG_CUDA(cudaGetLastError());
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, i0, i1, (int)n, 0, 63, st);
        PHG_TRY(c->cub_tmp.ensure(tmp));
        PHG_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, k0, k1, i0, i1, (int)n, 0, 63,
                                                 st));
        // ---- 3. candidate pairs: count, scan, write
        PHG_TRY(c->l_cnt.ensure((size_t)(n + 1) * 16));
        long long* cnt = c->l_cnt.as<long long>();
        long long* poff = cnt + (n + 1);
        pairs_kernel<false><<<grid_for(n, 128), 128, 0, st>>>(start, end, stg, etg, n, G, k1, i1,
                                                              lp->link_dist_mm, lp->link_cos_gate,
                                                              cnt, nullptr, nullptr, nullptr);
        PHG_CUDA(cudaGetLastError());
        PHG_TRY(scan_lengths(c, cnt, n, poff, st));
        PHG_CUDA(cudaMemcpyAsync(&P, poff + n, 8, cudaMemcpyDeviceToHost, st));
        PHG_CUDA(cudaStreamSynchronize(st));
        if (P >= (1ll << 31))
            return fail(PHG_ERR_INVALID, "phg_link: %lld candidate pairs exceed 2^31", P);
        if (P > 0) {
            PHG_TRY(c->l_pd.ensure((size_t)P * 8));
            PHG_TRY(c->l_pij.ensure((size_t)P * 8 * 4));
            double* pd = c->l_pd.as<double>();
            unsigned long long* ij0 = c->l_pij.as<unsigned long long>();
            unsigned long long* ij1 = ij0 + P;
            unsigned long long* db0 = ij1 + P;
            unsigned long long* db1 = db0 + P;
            pairs_kernel<true><<<grid_for(n, 128), 128, 0, st>>>(start, end, stg, etg, n, G, k1,
                                                                 i1, lp->link_dist_mm,
                                                                 lp->link_cos_gate, nullptr, poff,
                                                                 pd, ij0);
            PHG_CUDA(cudaGetLastError());
            // (d, i, j) order: sort by (i<<32|j) carrying d, then stable sort by d's bits
            PHG_TRY(c->l_pd2.ensure((size_t)P * 8));
            double* pd2 = c->l_pd2.as<double>();
            tmp = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp, ij0, ij1, pd, pd2, (int)P, 0, 64, st);
            PHG_TRY(c->cub_tmp.ensure(tmp));
            PHG_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, ij0, ij1, pd, pd2, (int)P,
                                                     0, 64, st));
            dbits_kernel<<<grid_for(P, 256), 256, 0, st>>>(pd2, nullptr, P, db0);
            PHG_CUDA(cudaGetLastError());
            tmp = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp, db0, db1, ij1, ij0, (int)P, 0, 64, st);
            PHG_TRY(c->cub_tmp.ensure(tmp));
            PHG_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tmp, db0, db1, ij1, ij0, (int)P,
                                                     0, 64, st));
            std::vector<unsigned long long> h_ij;
            PHG_TRY(d2h(h_ij, ij0, (size_t)P, st));
            sorted_pairs.resize(P);
            for (long long k = 0; k < P; ++k)
                sorted_pairs[k] = {(long long)(h_ij[k] >> 32), (long long)(h_ij[k] & 0xffffffffull)};
        }
    }
    // ---- 4. greedy acceptance with union-find (phg.py:365-377), native host code
    std::vector<long long> parent(n), nxt(n, -1);
    std::vector<char> end_used(n, 0), start_used(n, 0), has_prev(n, 0);
    for (long long i = 0; i < n; ++i) parent[i] = i;
    auto find = [&](long long a) {
        while (parent[a] != a) {
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        return a;
    };
    std::vector<long long> links;
    for (const auto& pr : sorted_pairs) {
        const long long i = pr.first, j = pr.second;
        if (end_used[i] || start_used[j]) continue;
        const long long ri = find(i), rj = find(j);
        if (ri == rj) continue;
        parent[rj] = ri;
        end_used[i] = start_used[j] = 1;
        links.push_back(i);
        links.push_back(j);
        nxt[i] = j;
        has_prev[j] = 1;
    }
    // ---- 5. chains (connect_segments, phg.py:395-412)
    std::vector<int> members;
    std::vector<long long> moff(1, 0), coff(1, 0);
    std::vector<uint8_t> ch_smooth, ch_root, ch_src;
    for (long long i = 0; i < n; ++i) {
        if (has_prev[i]) continue;
        long long L = 0, j = i;
        int cnt_m = 0;
        while (true) {
            members.push_back((int)j);
            L += h_off[j + 1] - h_off[j];
            ++cnt_m;
            if (nxt[j] < 0) break;
            j = nxt[j];
        }
        const bool merged = cnt_m > 1;
        moff.push_back((long long)members.size());
        coff.push_back(coff.back() + L);
        ch_smooth.push_back(merged && lp->smooth ? 1 : 0);
        ch_root.push_back(h_root[i]);
        ch_src.push_back(merged ? 2 : h_src[i]);
    }
    const long long nch = (long long)ch_root.size();
    const long long ML = coff.back();
    std::vector<long long> h_roff, h_foff;
    long long nstr = 0, nverts = 0;
    unsigned long long n_unrooted = 0;
    if (nch > 0) {
        DevBuf& d_members = c->l_members;
        PHG_TRY(h2d(d_members, members, st));
        PHG_TRY(h2d(c->l_moff, moff, st));
        PHG_TRY(h2d(c->l_coff, coff, st));
        PHG_TRY(h2d(c->l_smooth, ch_smooth, st));
        PHG_TRY(c->l_buf.ensure((size_t)std::max<long long>(ML, 1) * 24 * 2));
        double* b0 = c->l_buf.as<double>();
        double* b1 = b0 + 3 * ML;
        const long long* d_coff = c->l_coff.as<long long>();
        chain_concat_kernel<<<grid_for(nch * 32, 256, num_sms() * 16), 256, 0, st>>>(
            d_off, d_v, d_members.as<int>(), c->l_moff.as<long long>(), d_coff, nch, b0);
        PHG_CUDA(cudaGetLastError());
        double* cur = b0;
        double* oth = b1;
        for (int it = 0; it < lp->smooth_iters && lp->smooth; ++it) {
            smooth_iter_kernel<<<grid_for(nch * 32, 256, num_sms() * 16), 256, 0, st>>>(
                cur, oth, d_coff, c->l_smooth.as<uint8_t>(), nch, lp->smooth_strength);
            PHG_CUDA(cudaGetLastError());
            std::swap(cur, oth);
        }
        PHG_TRY(c->l_arc.ensure((size_t)std::max<long long>(ML, 1) * 8 + (size_t)(nch + 1) * 16));
        double* s = c->l_arc.as<double>();
        long long* nout = (long long*)(s + ML);
        arclen_kernel<<<grid_for(nch, 128), 128, 0, st>>>(cur, d_coff, nch, s, lp->step_mm, nout);
        PHG_CUDA(cudaGetLastError());
        std::vector<long long> h_nout;
        PHG_TRY(d2h(h_nout, nout, (size_t)nch, st));
        // resampled chains; strands with < 2 vertices are dropped (phg.py:410-411)
        std::vector<long long> rof(1, 0);
        for (long long k = 0; k < nch; ++k) rof.push_back(rof.back() + h_nout[k]);
        PHG_TRY(h2d(c->l_roff, rof, st));
        PHG_TRY(c->l_res.ensure((size_t)std::max<long long>(rof.back(), 1) * 24));
        resample_kernel<<<grid_for(nch * 32, 256, num_sms() * 16), 256, 0, st>>>(
            cur, s, d_coff, c->l_roff.as<long long>(), nch, c->l_res.as<double>());
        PHG_CUDA(cudaGetLastError());
        // keep strands with >= 2 vertices (compaction of the chain list, order preserved)
        std::vector<long long> keep_idx;
        for (long long k = 0; k < nch; ++k)
            if (h_nout[k] >= 2) keep_idx.push_back(k);
        nstr = (long long)keep_idx.size();
        std::vector<long long> koff(1, 0);
        std::vector<uint8_t> k_root, k_src;
        for (long long k : keep_idx) {
            koff.push_back(koff.back() + h_nout[k]);
            k_root.push_back(ch_root[k]);
            k_src.push_back(ch_src[k]);
        }
        if ((long long)keep_idx.size() != nch) {  // rare: copy kept rows contiguously
            std::vector<double> h_res;
            PHG_TRY(d2h(h_res, c->l_res.p, (size_t)rof.back() * 3, st));
            std::vector<double> packed;
            for (long long k : keep_idx)
                packed.insert(packed.end(), h_res.begin() + 3 * rof[k], h_res.begin() + 3 * rof[k + 1]);
            PHG_TRY(h2d(c->l_res, packed, st));
        }
        h_roff = koff;
        // ---- 6. attachment decisions and final assembly with tangents
        PHG_TRY(h2d(c->l_roff, koff, st));
        PHG_TRY(h2d(c->l_kroot, k_root, st));
        const void* d_scalp = nullptr;
        if (lp->attach && n_scalp > 0)
            PHG_TRY(to_device(scalp, (size_t)n_scalp * 24, c->l_scalp, &d_scalp, st));
        PHG_TRY(c->l_att.ensure((size_t)std::max<long long>(nstr, 1) * 17 + 64));
        long long* sid = c->l_att.as<long long>();
        long long* newlen = sid + nstr;
        uint8_t* mode = (uint8_t*)(newlen + nstr);
        DevBuf cnt_buf;
        PHG_TRY(cnt_buf.ensure(8));
        PHG_CUDA(cudaMemsetAsync(cnt_buf.p, 0, 8, st));
        attach_kernel<<<grid_for(std::max<long long>(nstr, 1) * 32, 256, num_sms() * 16), 256, 0,
                        st>>>(c->l_res.as<double>(), c->l_roff.as<long long>(),
                              c->l_kroot.as<uint8_t>(), nstr, (const double*)d_scalp,
                              (lp->attach ? n_scalp : 0), lp->attach_radius_mm, mode, sid, newlen,
                              cnt_buf.as<unsigned long long>());
        PHG_CUDA(cudaGetLastError());
        std::vector<long long> h_newlen;
        PHG_TRY(d2h(h_newlen, newlen, (size_t)nstr, st));
        std::vector<uint8_t> h_mode;
        PHG_TRY(d2h(h_mode, mode, (size_t)nstr, st));
        PHG_CUDA(cudaMemcpyAsync(&n_unrooted, cnt_buf.p, 8, cudaMemcpyDeviceToHost, st));
        h_foff.assign(1, 0);
        for (long long k = 0; k < nstr; ++k) h_foff.push_back(h_foff.back() + h_newlen[k]);
        nverts = h_foff.back();
        PHG_TRY(h2d(c->l_foff, h_foff, st));
        PHG_TRY(c->l_out_v.ensure((size_t)std::max<long long>(nverts, 1) * 24));
        PHG_TRY(c->l_out_t.ensure((size_t)std::max<long long>(nverts, 1) * 24));
        finalize_kernel<<<grid_for(std::max<long long>(nstr, 1) * 32, 256, num_sms() * 16), 256, 0,
                          st>>>(c->l_res.as<double>(), c->l_roff.as<long long>(), mode, sid,
                                (const double*)d_scalp, c->l_foff.as<long long>(), nstr,
                                c->l_out_v.as<double>(), c->l_out_t.as<double>());
        PHG_CUDA(cudaGetLastError());
        PHG_CUDA(cudaStreamSynchronize(st));
        c->l_rooted.resize(nstr);
        c->l_source.resize(nstr);
        for (long long k = 0; k < nstr; ++k) {
            c->l_rooted[k] = h_mode[k] ? 1 : k_root[k];
            c->l_source[k] = h_mode[k] ? 3 : k_src[k];
        }
    }
    c->l_offsets = h_foff.empty() ? std::vector<long long>(1, 0) : h_foff;
    c->l_links = links;
    c->l_nstr = nstr;
    c->l_nverts = nverts;
    c->link_ready = true;
    counts_out[0] = nstr;
    counts_out[1] = nverts;
    counts_out[2] = (int64_t)(links.size() / 2);
    counts_out[3] = (int64_t)n_unrooted;
    return PHG_OK;
}

phg_status phg_link_fetch(phg_ctx* c, int64_t* offsets, double* verts, double* tangents,
                          uint8_t* rooted, uint8_t* source, int64_t* links, void* stream) {
    if (!c) return fail(PHG_ERR_INVALID, "phg_link_fetch: null context");
    if (!c->link_ready) return fail(PHG_ERR_STATE, "phg_link_fetch: no completed phg_link");
    cudaStream_t st = as_stream(stream);
    const long long ns = c->l_nstr, nv = c->l_nverts;
    if (offsets)
        PHG_CUDA(cudaMemcpyAsync(offsets, c->l_offsets.data(), (size_t)(ns + 1) * 8,
                                 cudaMemcpyDefault, st));
    if (verts && nv)
        PHG_CUDA(cudaMemcpyAsync(verts, c->l_out_v.p, (size_t)nv * 24, cudaMemcpyDefault, st));
    if (tangents && nv)
        PHG_CUDA(cudaMemcpyAsync(tangents, c->l_out_t.p, (size_t)nv * 24, cudaMemcpyDefault, st));
    if (rooted && ns)
        PHG_CUDA(cudaMemcpyAsync(rooted, c->l_rooted.data(), (size_t)ns, cudaMemcpyDefault, st));
    if (source && ns)
        PHG_CUDA(cudaMemcpyAsync(source, c->l_source.data(), (size_t)ns, cudaMemcpyDefault, st));
    if (links && !c->l_links.empty())
        PHG_CUDA(cudaMemcpyAsync(links, c->l_links.data(), c->l_links.size() * 8, cudaMemcpyDefault,
                                 st));
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

}  // extern "C"
