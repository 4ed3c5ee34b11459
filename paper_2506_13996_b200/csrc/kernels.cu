// HBM-bound kernels of the layer step: RMSNorm fwd/bwd, Ulysses pack/unpack (K1/K2), label /
// position-id pre-passes (K10), row-wise cross-entropy, deterministic reductions, SGD update.
// All use 128-bit vectorised, coalesced accesses and 64-bit indexing (N*h reaches 2^32 at 1M tokens).
#include <algorithm>

#include "common.h"
#include "launch.h"
#include "prof.h"
#include "sm100.cuh"

namespace spt {

static inline int grid_for(int64_t work, int threads, int per_sm = 8) {
    int64_t g = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * per_sm));
}

// ------------------------------------------------------------------ block reduce helpers
template <int MAXW>
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = 0.f;
    for (int i = 0; i < nw; ++i) t += red[i];  // fixed order -> deterministic
    return t;
}

// ------------------------------------------------------------------ RMSNorm
// One thread owns 8 consecutive columns (one uint4); blockDim = max(32, h/8).
// The next row's 16-byte loads are issued (kept packed, 4 registers each) before the current row's block
// reduction, so two rows per CTA are in flight; the arithmetic is unchanged (bitwise equal to one row at a time).
__device__ __forceinline__ void unpack8(const uint4 w, float* v) {
    float2 a = unpack_bf16x2(w.x), b = unpack_bf16x2(w.y), c = unpack_bf16x2(w.z), d = unpack_bf16x2(w.w);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y; v[6] = d.x; v[7] = d.y;
}
__device__ __forceinline__ uint4 ld16(const bf16* p) { return *reinterpret_cast<const uint4*>(p); }

// REGS: register cap (32 for h <= 5120, no spills: four 512-thread / three 640-thread CTAs per SM, 107 vs 124 us at
// 48 registers for the L1 shape, tools/rms_bench.py; 64 for up to 1024 threads)
template <int REGS>
__global__ void __maxnreg__(REGS) rmsnorm_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g, bf16* __restrict__ y,
                                   float* __restrict__ rstd, int64_t n, int h, float eps) {
    __shared__ float red[32];
    const int c = threadIdx.x * 8;
    const bool act = c < h;
    float gv[8];
    if (act) load8(g + c, gv);
    uint4 xq = make_uint4(0, 0, 0, 0);
    if (act && blockIdx.x < n) xq = ld16(x + (int64_t)blockIdx.x * h + c);
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t rn = r + gridDim.x;
        uint4 xqn = make_uint4(0, 0, 0, 0);
        if (act && rn < n) xqn = ld16(x + rn * h + c);
        float xv[8];
        unpack8(xq, xv);
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) ss += xv[i] * xv[i];
        const float tot = block_sum<32>(ss, red);
        const float rs = rsqrtf(tot / (float)h + eps);
        if (act) {
            float o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = xv[i] * rs * gv[i];
            store8(y + r * h + c, o);
        }
        if (threadIdx.x == 0) rstd[r] = rs;
        xq = xqn;
    }
}

__global__ void __launch_bounds__(1024, 1) rmsnorm_bwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                   const float* __restrict__ rstd, const bf16* __restrict__ dy,
                                   const bf16* __restrict__ dres, bf16* __restrict__ dx, float* __restrict__ part,
                                   int64_t n, int h, int64_t rows_per_cta) {
    __shared__ float red[32];
    const int c = threadIdx.x * 8;
    const bool act = c < h;
    // inactive lanes (h/8 not a multiple of 32) must contribute exact zeros to the row dot
    float gv[8] = {0, 0, 0, 0, 0, 0, 0, 0}, dga[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (act) load8(g + c, gv);
    const int64_t r0 = blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    const uint4 z = make_uint4(0, 0, 0, 0);
    uint4 xq = z, dq = z, rq = z;
    float rs = 0.f;
    if (r0 < r1) {
        if (act) {
            xq = ld16(x + r0 * h + c);
            dq = ld16(dy + r0 * h + c);
            if (dres) rq = ld16(dres + r0 * h + c);
        }
        rs = rstd[r0];
    }
    for (int64_t r = r0; r < r1; ++r) {
        uint4 xqn = z, dqn = z, rqn = z;  // next row, in flight during this row's reduction
        float rsn = 0.f;
        if (r + 1 < r1) {
            if (act) {
                xqn = ld16(x + (r + 1) * h + c);
                dqn = ld16(dy + (r + 1) * h + c);
                if (dres) rqn = ld16(dres + (r + 1) * h + c);
            }
            rsn = rstd[r + 1];
        }
        float xv[8], dv[8];
        unpack8(xq, xv);
        unpack8(dq, dv);
        float dot = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) dot += dv[i] * gv[i] * xv[i] * rs;
        const float tot = block_sum<32>(dot, red) / (float)h;
        if (act) {
            float o[8], rr[8];
            unpack8(rq, rr);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float xh = xv[i] * rs;
                o[i] = rs * (dv[i] * gv[i] - xh * tot) + rr[i];
                dga[i] += dv[i] * xh;
            }
            store8(dx + r * h + c, o);
        }
        xq = xqn;
        dq = dqn;
        rq = rqn;
        rs = rsn;
    }
    if (act) {
        float4* p = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * h + c);
        p[0] = make_float4(dga[0], dga[1], dga[2], dga[3]);
        p[1] = make_float4(dga[4], dga[5], dga[6], dga[7]);
    }
}

__global__ void colsum_accum_kernel(const float* __restrict__ part, int nparts, int h, float* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= h) return;
    float s = 0.f;
    for (int i = 0; i < nparts; ++i) s += part[(int64_t)i * h + c];
    out[c] += s;
}

static int rms_threads(int64_t h) {
    SPT_CHECK(h % 8 == 0 && h / 8 <= 1024, SPT_ERR_SHAPE, "rmsnorm: hidden must be a multiple of 8 and <= 8192");
    return std::max<int>(32, (int)((h / 8 + 31) / 32 * 32));
}

void rmsnorm_fwd(const void* x, const void* gamma, void* y, float* rstd, int64_t n, int64_t h, float eps,
                 cudaStream_t st) {
    if (n == 0) return;
    const int th = rms_threads(h);
    if (th <= 640)
        rmsnorm_fwd_kernel<32><<<grid_for(n, 1, 4), th, 0, st>>>((const bf16*)x, (const bf16*)gamma, (bf16*)y, rstd,
                                                                 n, (int)h, eps);
    else
        rmsnorm_fwd_kernel<64><<<grid_for(n, 1, 4), th, 0, st>>>((const bf16*)x, (const bf16*)gamma, (bf16*)y, rstd,
                                                                  n, (int)h, eps);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

static int rms_bwd_ctas(int64_t n) { return (int)std::min<int64_t>(n, (int64_t)num_sms() * 4); }

size_t rmsnorm_bwd_workspace(int64_t n, int64_t h) { return (size_t)std::max(1, rms_bwd_ctas(n)) * h * 4; }

void rmsnorm_bwd(const void* x, const void* gamma, const float* rstd, const void* dy, const void* dres, void* dx,
                 float* dgamma_accum, void* ws, int64_t n, int64_t h, cudaStream_t st) {
    if (n == 0) return;
    const int th = rms_threads(h);
    const int ctas = rms_bwd_ctas(n);
    const int64_t per = (n + ctas - 1) / ctas;
    const int used = (int)((n + per - 1) / per);
    rmsnorm_bwd_kernel<<<used, th, 0, st>>>((const bf16*)x, (const bf16*)gamma, rstd, (const bf16*)dy,
                                            (const bf16*)dres, (bf16*)dx, (float*)ws, n, (int)h, per);
    count_launch();
    SPT_CUDA(cudaGetLastError());
    colsum_accum_kernel<<<(int)((h + 255) / 256), 256, 0, st>>>((const float*)ws, used, (int)h, dgamma_accum);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ Ulysses reshard K1 / K2
// K1: send[j][t][a][:] = src[t][head_map[j*heads_out + a]][:]   (payload layout :351)
__global__ void reshard_pack_kernel(const uint4* __restrict__ src, int64_t s_loc, int heads_in, int vpd, int P,
                                    int heads_out, const int32_t* __restrict__ head_map, const RowTab dst) {
    const int64_t total = (int64_t)P * s_loc * heads_out * vpd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int v = (int)(i % vpd);
        int64_t q = i / vpd;
        const int a = (int)(q % heads_out);
        q /= heads_out;
        const int64_t t = q % s_loc;
        const int j = (int)(q / s_loc);
        const int hsrc = __ldg(head_map + j * heads_out + a);
        static_cast<uint4*>(dst.p[j])[((dst.row_off + t) * heads_out + a) * vpd + v] =
            __ldg(src + (t * heads_in + hsrc) * vpd + v);
    }
}

// K2: dst[t][h][:] = sum_e recv[i_e][t][a_e][:] over the listed sources, rank order
__global__ void reshard_unpack_kernel(const RowTab recv, int64_t s_loc, int heads_in, int vpd,
                                      int heads_out, const int32_t* __restrict__ gather, int max_src,
                                      uint4* __restrict__ dst) {
    const int64_t total = s_loc * heads_out * vpd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int v = (int)(i % vpd);
        int64_t q = i / vpd;
        const int h = (int)(q % heads_out);
        const int64_t t = q / heads_out;
        const int32_t* gl = gather + h * max_src;
        const int g0 = __ldg(gl);
        auto src_of = [&](int gidx) {
            const int rank = gidx / heads_in, slot = gidx % heads_in;
            return static_cast<const uint4*>(recv.p[rank]) + ((recv.row_off + t) * heads_in + slot) * vpd + v;
        };
        int nsrc = 1;
        while (nsrc < max_src && __ldg(gl + nsrc) >= 0) ++nsrc;
        if (nsrc == 1) {
            dst[i] = *src_of(g0);  // plain permutation: bit-exact (plain loads: the source may be a peer's buffer)
        } else {
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int e = 0; e < nsrc; ++e) {
                uint4 w = *src_of(__ldg(gl + e));
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    float2 f = unpack_bf16x2(ws[k]);
                    acc[2 * k] += f.x;
                    acc[2 * k + 1] += f.y;
                }
            }
            uint4 o;
            o.x = pack_bf16x2(acc[0], acc[1]);
            o.y = pack_bf16x2(acc[2], acc[3]);
            o.z = pack_bf16x2(acc[4], acc[5]);
            o.w = pack_bf16x2(acc[6], acc[7]);
            dst[i] = o;
        }
    }
}

// Row-parallel variants for head_dim in {32, 64, 128} (VPD = head_dim / 8 uint4 per head): one warp per
// destination row ((rank, token) for K1, token for K2), index maps staged in shared memory, one integer
// division per row instead of several per 16-byte element, and loads batched ahead of the stores so each
// lane keeps several 16-byte requests in flight (the generic kernels above were issue-bound at ~60% of
// the HBM copy bandwidth).
// RoPE rotation of 8 consecutive pairs (j = 8 gi .. 8 gi + 7 of the first half against the second half) at
// position p, Llama / HF rotate_half convention with HF's fp32 angles; explicit roundings so the standalone
// kernel and the pack/unpack-fused kernels produce identical bits.
// The (cos, sin) of one (position, j): HF's fp32 angle p * theta^(-2j/d).  Used by rope_table_kernel and by
// the kernels when no table is given, so both paths give identical bits.
__device__ __forceinline__ void rope_cos_sin(float p, int j, int d, float theta, float& cs, float& sn) {
    const float inv_freq = 1.f / powf(theta, (float)(2 * j) / (float)d);
    sincosf(p * inv_freq, &sn, &cs);
}

// tab: NULL (angles computed here: accurate sincosf of arguments up to ~1e6 rad takes the slow range
// reduction, which made the kernels ALU-bound) or the (cos, sin) row of this position, entries 8 gi .. 8 gi + 7.
__device__ __forceinline__ void rope_rotate8(const float* a, const float* b, float p, int gi, int d, float theta,
                                             float sgn, float* o1, float* o2, const float2* tab = nullptr) {
    float2 cst[8];
    if (tab) {
        const float4* t4 = reinterpret_cast<const float4*>(tab + gi * 8);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float4 v = __ldg(t4 + k);
            cst[2 * k] = make_float2(v.x, v.y);
            cst[2 * k + 1] = make_float2(v.z, v.w);
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float sn, cs;
        if (tab) {
            cs = cst[k].x;
            sn = cst[k].y;
        } else {
            rope_cos_sin(p, gi * 8 + k, d, theta, cs, sn);
        }
        sn *= sgn;
        o1[k] = __fsub_rn(__fmul_rn(a[k], cs), __fmul_rn(b[k], sn));
        o2[k] = __fadd_rn(__fmul_rn(b[k], cs), __fmul_rn(a[k], sn));
    }
}

// The (cos, sin) row of position pi in a table of npos rows, or NULL (in-kernel angles) without a table or when
// pi is outside it: a packed chunk whose position_ids run past the table must not read out of bounds (the
// error flag turns the step into a ValidationError when the host reads it).
__device__ __forceinline__ const float2* rope_row(const float2* tab, int64_t pi, int64_t npos, int row,
                                                  int32_t* err) {
    if (!tab) return nullptr;
    if (pi < 0 || pi >= npos) {
        if (err) *err = 4;
        return nullptr;
    }
    return tab + pi * row;
}

__device__ __forceinline__ void u4_to_f8(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 v = unpack_bf16x2(w[k]);
        f[2 * k] = v.x;
        f[2 * k + 1] = v.y;
    }
}

__device__ __forceinline__ uint4 f8_to_u4(const float* f) {
    return make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                      pack_bf16x2(f[6], f[7]));
}

// K1 pack with RoPE fused: the q and k heads (source head < n_rot) are rotated on the
// way from the token rows to the per-peer send buffer, replacing the separate in-place rope pass.  A lane
// handles one (head, chunk pair): chunk c of the first half of the head row and chunk c of the second half.
template <int VPD>
__global__ void __launch_bounds__(256) reshard_pack_rope_kernel(const uint4* __restrict__ src, int64_t s_loc,
                                                                int heads_in, int P, int heads_out,
                                                                const int32_t* __restrict__ head_map,
                                                                const RowTab dst, int n_rot,
                                                                const int64_t* __restrict__ pos, int64_t pos_offset,
                                                                float theta, const float2* __restrict__ tab,
                                                                int64_t npos, int32_t* err) {
    extern __shared__ int32_t smap[];  // [P][heads_out]
    for (int i = threadIdx.x; i < P * heads_out; i += blockDim.x) smap[i] = head_map[i];
    __syncthreads();
    constexpr int HP = VPD / 2;  // chunk pairs per head
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)P * s_loc;
    const int row_pairs = heads_out * HP;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < nrows; r += nw) {
        const int j = (int)(r / s_loc);
        const int64_t t = r - (int64_t)j * s_loc;
        const int64_t pi = pos ? pos[t] : pos_offset + t;
        const float p = (float)pi;
        const float2* trow = rope_row(tab, pi, npos, VPD * 4, err);
        const uint4* srow = src + t * heads_in * VPD;
        uint4* drow = static_cast<uint4*>(dst.p[j]) + (dst.row_off + t) * heads_out * VPD;
        const int32_t* m = smap + j * heads_out;
        for (int e = lane; e < row_pairs; e += 32) {
            const int hs = e / HP, c = e - hs * HP;
            const int sh = m[hs];
            uint4 a = __ldg(srow + sh * VPD + c), b = __ldg(srow + sh * VPD + c + HP);
            if (sh < n_rot) {
                float fa[8], fb[8], o1[8], o2[8];
                u4_to_f8(a, fa);
                u4_to_f8(b, fb);
                rope_rotate8(fa, fb, p, c, VPD * 8, theta, 1.f, o1, o2, trow);
                a = f8_to_u4(o1);
                b = f8_to_u4(o2);
            }
            drow[hs * VPD + c] = a;
            drow[hs * VPD + c + HP] = b;
        }
    }
}

// K2 unpack of d(q, k, v) with the inverse RoPE fused: replicas summed in fp32 (rank order) and rounded to
// bf16 exactly as the plain unpack writes them, then the q / k heads (< n_rot) rotated back.
template <int VPD>
__global__ void __launch_bounds__(256) reshard_unpack_rope_kernel(const RowTab recv, int64_t s_loc,
                                                                  int heads_in, int heads_out,
                                                                  const int32_t* __restrict__ gather, int max_src,
                                                                  uint4* __restrict__ dst, int n_rot,
                                                                  const int64_t* __restrict__ pos, int64_t pos_offset,
                                                                  float theta, const float2* __restrict__ tab,
                                                                  int64_t npos, int32_t* err) {
    extern __shared__ int32_t sg[];  // [heads_out][max_src]
    for (int i = threadIdx.x; i < heads_out * max_src; i += blockDim.x) sg[i] = gather[i];
    __syncthreads();
    constexpr int HP = VPD / 2;
    const int lane = threadIdx.x & 31;
    const int row_pairs = heads_out * HP;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < s_loc; t += nw) {
        const int64_t roff = (recv.row_off + t) * heads_in * VPD;
        uint4* drow = dst + t * heads_out * VPD;
        const int64_t pi = pos ? pos[t] : pos_offset + t;
        const float p = (float)pi;
        const float2* crow = rope_row(tab, pi, npos, VPD * 4, err);
        for (int e = lane; e < row_pairs; e += 32) {
            const int h = e / HP, c = e - h * HP;
            const int32_t* gl = sg + h * max_src;
            auto at = [&](int g, int v) {
                return static_cast<const uint4*>(recv.p[g / heads_in]) + roff + (g % heads_in) * VPD + v;
            };
            uint4 a = *at(gl[0], c), b = *at(gl[0], c + HP);
            if (max_src > 1 && gl[1] >= 0) {  // replica sum in fp32, rank order (as reshard_unpack_rows_kernel)
                float fa[8], fb[8];
                u4_to_f8(a, fa);
                u4_to_f8(b, fb);
                for (int sidx = 1; sidx < max_src && gl[sidx] >= 0; ++sidx) {
                    float ga[8], gb[8];
                    u4_to_f8(*at(gl[sidx], c), ga);
                    u4_to_f8(*at(gl[sidx], c + HP), gb);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        fa[k] += ga[k];
                        fb[k] += gb[k];
                    }
                }
                a = f8_to_u4(fa);
                b = f8_to_u4(fb);
            }
            if (h < n_rot) {
                float fa[8], fb[8], o1[8], o2[8];
                u4_to_f8(a, fa);
                u4_to_f8(b, fb);
                rope_rotate8(fa, fb, p, c, VPD * 8, theta, -1.f, o1, o2, crow);
                a = f8_to_u4(o1);
                b = f8_to_u4(o2);
            }
            drow[h * VPD + c] = a;
            drow[h * VPD + c + HP] = b;
        }
    }
}

template <int VPD>
__global__ void __launch_bounds__(256) reshard_pack_rows_kernel(const uint4* __restrict__ src, int64_t s_loc,
                                                                int heads_in, int P, int heads_out,
                                                                const int32_t* __restrict__ head_map,
                                                                const RowTab dst) {
    extern __shared__ int32_t smap[];  // [P][heads_out]
    for (int i = threadIdx.x; i < P * heads_out; i += blockDim.x) smap[i] = head_map[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)P * s_loc;
    const int row_elems = heads_out * VPD;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < nrows; r += nw) {
        const int j = (int)(r / s_loc);
        const int64_t t = r - (int64_t)j * s_loc;
        const uint4* srow = src + t * heads_in * VPD;
        uint4* drow = static_cast<uint4*>(dst.p[j]) + (dst.row_off + t) * row_elems;
        const int32_t* m = smap + j * heads_out;
        for (int e0 = 0; e0 < row_elems; e0 += 32 * 4) {
            uint4 buf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < row_elems) buf[u] = __ldg(srow + m[e / VPD] * VPD + (e % VPD));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < row_elems) drow[e] = buf[u];
            }
        }
    }
}

template <int VPD>
__global__ void __launch_bounds__(256) reshard_unpack_rows_kernel(const RowTab recv, int64_t s_loc,
                                                                  int heads_in, int heads_out,
                                                                  const int32_t* __restrict__ gather, int max_src,
                                                                  uint4* __restrict__ dst) {
    extern __shared__ int32_t sg[];  // [heads_out][max_src] (rank*heads_in + slot, -1 = unused)
    for (int i = threadIdx.x; i < heads_out * max_src; i += blockDim.x) sg[i] = gather[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int row_elems = heads_out * VPD;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = w0; t < s_loc; t += nw) {
        const int64_t roff = (recv.row_off + t) * heads_in * VPD;
        uint4* drow = dst + t * row_elems;
        for (int e0 = 0; e0 < row_elems; e0 += 32 * 4) {
            uint4 buf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e >= row_elems) continue;
                const int h = e / VPD, v = e % VPD;
                const int32_t* gl = sg + h * max_src;
                auto at = [&](int g) {
                    return static_cast<const uint4*>(recv.p[g / heads_in]) + roff + (g % heads_in) * VPD + v;
                };
                buf[u] = *at(gl[0]);
                if (max_src > 1 && gl[1] >= 0) {  // replicate_kv backward: fp32 sum in rank order
                    float acc[8];
                    {
                        const uint32_t ws[4] = {buf[u].x, buf[u].y, buf[u].z, buf[u].w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float2 f = unpack_bf16x2(ws[k]);
                            acc[2 * k] = f.x;
                            acc[2 * k + 1] = f.y;
                        }
                    }
                    for (int s = 1; s < max_src && gl[s] >= 0; ++s) {
                        const uint4 w = *at(gl[s]);
                        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float2 f = unpack_bf16x2(ws[k]);
                            acc[2 * k] += f.x;
                            acc[2 * k + 1] += f.y;
                        }
                    }
                    buf[u].x = pack_bf16x2(acc[0], acc[1]);
                    buf[u].y = pack_bf16x2(acc[2], acc[3]);
                    buf[u].z = pack_bf16x2(acc[4], acc[5]);
                    buf[u].w = pack_bf16x2(acc[6], acc[7]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < row_elems) drow[e] = buf[u];
            }
        }
    }
}

static int reshard_rows_grid(int64_t rows) {
    const int64_t blocks = (rows + 7) / 8;  // 8 warps (rows) per block per pass
    return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)num_sms() * 8));
}

RowTab contiguous_rows(const void* base, int P, int64_t s_loc, int64_t row_bytes) {
    SPT_CHECK(P >= 1 && P <= kMaxSP, SPT_ERR_CONFIG, "SP degree must be in [1, " + std::to_string(kMaxSP) + "]");
    RowTab t{};
    for (int j = 0; j < P; ++j) t.p[j] = (char*)base + (size_t)j * s_loc * row_bytes;
    t.row_off = 0;
    return t;
}

void reshard_pack(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                  const int32_t* head_map, const RowTab& dst, cudaStream_t st) {
    SPT_CHECK(head_dim % 8 == 0, SPT_ERR_SHAPE, "head_dim must be a multiple of 8");
    SPT_CHECK(P >= 1 && P <= kMaxSP, SPT_ERR_CONFIG, "SP degree out of range");
    const int vpd = head_dim / 8;
    const int64_t total = (int64_t)P * s_loc * heads_out * vpd;
    if (total == 0) return;
    const size_t smem = (size_t)P * heads_out * 4;
    if ((vpd == 4 || vpd == 8 || vpd == 16) && smem <= 48 * 1024) {
        const int g = reshard_rows_grid((int64_t)P * s_loc);
        auto k = vpd == 16 ? reshard_pack_rows_kernel<16> : vpd == 8 ? reshard_pack_rows_kernel<8> : reshard_pack_rows_kernel<4>;
        k<<<g, 256, smem, st>>>((const uint4*)src, s_loc, heads_in, P, heads_out, head_map, dst);
    } else {
        reshard_pack_kernel<<<grid_for(total, 256), 256, 0, st>>>((const uint4*)src, s_loc, heads_in, vpd, P, heads_out,
                                                                   head_map, dst);
    }
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void reshard_pack(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                  const int32_t* head_map, void* dst, cudaStream_t st) {
    reshard_pack(src, s_loc, heads_in, head_dim, P, heads_out, head_map,
                 contiguous_rows(dst, P, s_loc, (int64_t)heads_out * head_dim * 2), st);
}

void reshard_unpack(const RowTab& recv, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                    const int32_t* gather, int max_src, void* dst, cudaStream_t st) {
    SPT_CHECK(head_dim % 8 == 0, SPT_ERR_SHAPE, "head_dim must be a multiple of 8");
    (void)P;
    const int vpd = head_dim / 8;
    const int64_t total = s_loc * heads_out * vpd;
    if (total == 0) return;
    const size_t smem = (size_t)heads_out * max_src * 4;
    if ((vpd == 4 || vpd == 8 || vpd == 16) && smem <= 48 * 1024) {
        const int g = reshard_rows_grid(s_loc);
        auto k = vpd == 16 ? reshard_unpack_rows_kernel<16>
                           : vpd == 8 ? reshard_unpack_rows_kernel<8> : reshard_unpack_rows_kernel<4>;
        k<<<g, 256, smem, st>>>(recv, s_loc, heads_in, heads_out, gather, max_src, (uint4*)dst);
    } else {
        reshard_unpack_kernel<<<grid_for(total, 256), 256, 0, st>>>(recv, s_loc, heads_in, vpd, heads_out, gather,
                                                                     max_src, (uint4*)dst);
    }
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void reshard_unpack(const void* recv, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                    const int32_t* gather, int max_src, void* dst, cudaStream_t st) {
    reshard_unpack(contiguous_rows(recv, P, s_loc, (int64_t)heads_in * head_dim * 2), s_loc, heads_in, head_dim, P,
                   heads_out, gather, max_src, dst, st);
}

bool reshard_pack_rope(const void* src, int64_t s_loc, int heads_in, int head_dim, int P, int heads_out,
                       const int32_t* head_map, const RowTab& dst, int n_rot, const int64_t* pos, int64_t pos_offset,
                       float theta, cudaStream_t st, const void* tab, int64_t npos, int32_t* err) {
    const int vpd = head_dim / 8;
    const size_t smem = (size_t)P * heads_out * 4;
    if (head_dim % 16 != 0 || !(vpd == 4 || vpd == 8 || vpd == 16) || smem > 48 * 1024) return false;
    if ((int64_t)P * s_loc * heads_out == 0) return true;
    const int g = reshard_rows_grid((int64_t)P * s_loc);
    auto k = vpd == 16 ? reshard_pack_rope_kernel<16> : vpd == 8 ? reshard_pack_rope_kernel<8> : reshard_pack_rope_kernel<4>;
    k<<<g, 256, smem, st>>>((const uint4*)src, s_loc, heads_in, P, heads_out, head_map, dst, n_rot, pos, pos_offset,
                            theta, (const float2*)tab, npos, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
    return true;
}

bool reshard_unpack_rope(const RowTab& recv, int64_t s_loc, int heads_in, int head_dim, int heads_out,
                         const int32_t* gather, int max_src, void* dst, int n_rot, const int64_t* pos,
                         int64_t pos_offset, float theta, cudaStream_t st, const void* tab, int64_t npos,
                         int32_t* err) {
    const int vpd = head_dim / 8;
    const size_t smem = (size_t)heads_out * max_src * 4;
    if (head_dim % 16 != 0 || !(vpd == 4 || vpd == 8 || vpd == 16) || smem > 48 * 1024) return false;
    if (s_loc * heads_out == 0) return true;
    const int g = reshard_rows_grid(s_loc);
    auto k = vpd == 16 ? reshard_unpack_rope_kernel<16>
                       : vpd == 8 ? reshard_unpack_rope_kernel<8> : reshard_unpack_rope_kernel<4>;
    k<<<g, 256, smem, st>>>(recv, s_loc, heads_in, heads_out, gather, max_src, (uint4*)dst, n_rot, pos, pos_offset,
                            theta, (const float2*)tab, npos, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
    return true;
}

// ------------------------------------------------------------------ RoPE
// In-place rotary embedding of the first n_rot heads of each token row of x [n][heads][d] (bf16), Llama / HF
// rotate_half convention: (x1, x2) -> (x1 cos - x2 sin, x2 cos + x1 sin) with angle = pos * theta^(-2j/d)
// computed in fp32 exactly as HF does; inverse = the transpose rotation (backward).  pos: DEVICE int64 [n]
// or NULL (then pos = pos_offset + t).  One thread per (token, head, 8 consecutive j): 16-byte loads/stores.
__global__ void rope_kernel(bf16* __restrict__ x, int64_t n, int heads, int n_rot, int d,
                            const int64_t* __restrict__ pos, int64_t pos_offset, float theta, int inverse,
                            const float2* __restrict__ tab, int64_t npos, int32_t* err) {
    const int half = d / 2, g8 = half / 8;  // 8-wide groups per half
    const int64_t total = n * n_rot * g8;
    const float sgn = inverse ? -1.f : 1.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int gi = (int)(i % g8);
        const int64_t q = i / g8;
        const int hh = (int)(q % n_rot);
        const int64_t t = q / n_rot;
        const int64_t pi = pos ? pos[t] : pos_offset + t;
        const float p = (float)pi;
        bf16* row = x + (t * heads + hh) * d;
        float a[8], b[8];
        load8(row + gi * 8, a);
        load8(row + half + gi * 8, b);
        float o1[8], o2[8];
        rope_rotate8(a, b, p, gi, d, theta, sgn, o1, o2, rope_row(tab, pi, npos, half, err));
        store8(row + gi * 8, o1);
        store8(row + half + gi * 8, o2);
    }
}

// Angle table for positions [0, npos): tab[p][j] = (cos, sin) of HF's fp32 angle, bit-identical to the in-kernel
// computation (rope_cos_sin).  npos * d/2 * 8 bytes (16.8 MB for 32K positions at d=128).
__global__ void rope_table_kernel(float2* __restrict__ tab, int64_t npos, int d, float theta) {
    const int half = d / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npos * half; i += (int64_t)gridDim.x * blockDim.x) {
        float cs, sn;
        rope_cos_sin((float)(i / half), (int)(i % half), d, theta, cs, sn);
        tab[i] = make_float2(cs, sn);
    }
}

void rope_table(void* tab, int64_t npos, int d, float theta, cudaStream_t st) {
    SPT_CHECK(d % 16 == 0 && theta > 0.f, SPT_ERR_CONFIG, "rope table: head_dim % 16 and theta > 0");
    if (npos == 0) return;
    rope_table_kernel<<<grid_for(npos * (d / 2), 256), 256, 0, st>>>((float2*)tab, npos, d, theta);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void rope_apply(void* x, int64_t n, int heads, int n_rot, int d, const int64_t* pos, int64_t pos_offset, float theta,
                bool inverse, cudaStream_t st, const void* tab, int64_t npos, int32_t* err) {
    SPT_CHECK(d % 16 == 0, SPT_ERR_SHAPE, "rope: head_dim must be a multiple of 16");
    SPT_CHECK(theta > 0.f, SPT_ERR_CONFIG, "rope: theta must be > 0");
    const int64_t total = n * n_rot * (d / 16);
    if (total == 0) return;
    rope_kernel<<<grid_for(total, 256), 256, 0, st>>>((bf16*)x, n, heads, n_rot, d, pos, pos_offset, theta,
                                                      inverse ? 1 : 0, (const float2*)tab, npos, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ K10 label / position pre-passes
__global__ void label_stats_kernel(const int64_t* __restrict__ labels, int64_t n, int64_t V, int64_t* count,
                                   int32_t* err) {
    __shared__ long long red[32];
    long long c = 0;
    int bad = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t l = labels[i];
        if (l == -100) continue;
        if (l < 0 || l >= V) bad = 1;
        else ++c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    if (bad && (threadIdx.x & 31) == 0) *err = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        *count += t;
    }
}

void label_stats(const int64_t* labels, int64_t n, int64_t vocab, int64_t* count_accum, int32_t* err,
                 cudaStream_t st) {
    if (n == 0) return;
    label_stats_kernel<<<1, 1024, 0, st>>>(labels, n, vocab, count_accum, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

__global__ void segment_starts_kernel(const int64_t* __restrict__ pos, int64_t n, int32_t* __restrict__ starts,
                                      int32_t* err) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = pos[t];
        const bool ok = (t == 0) ? (p == 0) : (p == 0 || p == pos[t - 1] + 1);
        if (!ok) *err = 2;
        starts[t] = (int32_t)(t - p);
    }
}

void segment_starts(const int64_t* pos, int64_t n, int32_t* starts, int32_t* err, cudaStream_t st) {
    if (n == 0) return;
    segment_starts_kernel<<<grid_for(n, 256), 256, 0, st>>>(pos, n, starts, err);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ cross-entropy rows
// One CTA per row: one pass online (max, sumexp), block combine, then dlogits = (p - onehot) * scale.
__global__ void __launch_bounds__(512) ce_rows_kernel(const float* __restrict__ logits, const int64_t* __restrict__ labels,
                                                      int64_t V, const float* __restrict__ scale_dev,
                                                      float* __restrict__ loss_rows, bf16* __restrict__ dlogits,
                                                      int32_t* err) {
    __shared__ float sm_m[32], sm_s[32];
    __shared__ float sh_lse;
    const int64_t r = blockIdx.x;
    const float* row = logits + r * V;
    const int64_t label = labels[r];
    const bool valid = label != -100 && label >= 0 && label < V;
    if (label != -100 && !valid && threadIdx.x == 0) *err = 1;
    bf16* drow = dlogits + r * V;
    const int64_t nv = V / 8;  // V % 8 == 0 enforced by host
    if (!valid) {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) reinterpret_cast<uint4*>(drow)[i] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) loss_rows[r] = 0.f;
        return;
    }
    float m = -INFINITY, s = 0.f;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const float4 a = reinterpret_cast<const float4*>(row)[2 * i];
        const float4 b = reinterpret_cast<const float4*>(row)[2 * i + 1];
        const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        float mx = v[0];
#pragma unroll
        for (int k = 1; k < 8; ++k) mx = fmaxf(mx, v[k]);
        const float nm = fmaxf(m, mx);
        float acc = s * __expf(m - nm);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += __expf(v[k] - nm);
        s = acc;
        m = nm;
    }
    // warp combine
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
        const float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sm_m[w] = m;
        sm_s[w] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            const float nm = fmaxf(M, sm_m[i]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - nm)) + (sm_m[i] == -INFINITY ? 0.f : sm_s[i] * __expf(sm_m[i] - nm));
            M = nm;
        }
        const float lse = M + __logf(S);
        sh_lse = lse;
        loss_rows[r] = lse - row[label];
    }
    __syncthreads();
    const float lse = sh_lse;
    const float scale = *scale_dev;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const float4 a = reinterpret_cast<const float4*>(row)[2 * i];
        const float4 b = reinterpret_cast<const float4*>(row)[2 * i + 1];
        float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = __expf(v[k] - lse);
            if (8 * i + k == label) v[k] -= 1.f;
            v[k] *= scale;
        }
        store8(drow + 8 * i, v);
    }
}

// Variant fed by the logits GEMM's epilogue statistics: per (row, 256-column tile) (max, sum exp(x - max)).
// The row's log-sum-exp is combined from ntile pairs, so the fp32 logits are read exactly once.
__global__ void __launch_bounds__(512) ce_rows_stats_kernel(const float* __restrict__ logits,
                                                            const float2* __restrict__ stats, int ntile,
                                                            const int64_t* __restrict__ labels, int64_t V,
                                                            const float* __restrict__ scale_dev,
                                                            float* __restrict__ loss_rows, bf16* __restrict__ dlogits,
                                                            int32_t* err) {
    __shared__ float sm_m[32], sm_s[32];
    __shared__ float sh_lse;
    const int64_t r = blockIdx.x;
    const float* row = logits + r * V;
    const int64_t label = labels[r];
    const bool valid = label != -100 && label >= 0 && label < V;
    if (label != -100 && !valid && threadIdx.x == 0) *err = 1;
    bf16* drow = dlogits + r * V;
    const int64_t nv = V / 8;
    if (!valid) {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) reinterpret_cast<uint4*>(drow)[i] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) loss_rows[r] = 0.f;
        return;
    }
    float m = -INFINITY, s = 0.f;
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) {
        const float2 p = stats[r * ntile + i];
        const float nm = fmaxf(m, p.x);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (p.x == -INFINITY ? 0.f : p.y * __expf(p.x - nm));
        m = nm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
        const float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sm_m[w] = m;
        sm_s[w] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            const float nm = fmaxf(M, sm_m[i]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - nm)) + (sm_m[i] == -INFINITY ? 0.f : sm_s[i] * __expf(sm_m[i] - nm));
            M = nm;
        }
        const float lse = M + __logf(S);
        sh_lse = lse;
        loss_rows[r] = lse - row[label];
    }
    __syncthreads();
    const float lse = sh_lse;
    const float scale = *scale_dev;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(row) + 2 * i);
        const float4 b = __ldcs(reinterpret_cast<const float4*>(row) + 2 * i + 1);
        float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = __expf(v[k] - lse);
            if (8 * i + k == label) v[k] -= 1.f;
            v[k] *= scale;
        }
        store8(drow + 8 * i, v);
    }
}

// Variant fed by the EPI_EXP_STATS logits epilogue (the fp32 logits never reach memory): e = exp(x - m_t) in
// bf16 per (row, 256-column tile t), stats (m_t, sum e), the fp32 label logit.  lse = combine(stats), then
// p = e * exp(m_t - lse): one multiply by a per-tile factor instead of an exponential per element, and the
// dlogits overwrite e in place.  Traffic per row: 2V read + 2V write (the fp32 form moves 4V + 2V plus the
// epilogue's 4V write).
constexpr int CE_MAX_TILES = 1024;  // V <= 262144
__global__ void __launch_bounds__(512) ce_rows_exp_kernel(bf16* __restrict__ e_dlogits, const float2* __restrict__ stats,
                                                          int ntile, const int64_t* __restrict__ labels,
                                                          const float* __restrict__ label_logit, int64_t V,
                                                          const float* __restrict__ scale_dev,
                                                          float* __restrict__ loss_rows, int32_t* err) {
    __shared__ float sm_m[32], sm_s[32];
    __shared__ float fac[CE_MAX_TILES];
    __shared__ float sh_lse;
    const int64_t r = blockIdx.x;
    const int64_t label = labels[r];
    const bool valid = label != -100 && label >= 0 && label < V;
    if (label != -100 && !valid && threadIdx.x == 0) *err = 1;
    uint4* drow = reinterpret_cast<uint4*>(e_dlogits + r * V);
    const int64_t nv = V / 8;
    if (!valid) {
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) drow[i] = make_uint4(0, 0, 0, 0);
        if (threadIdx.x == 0) loss_rows[r] = 0.f;
        return;
    }
    float m = -INFINITY, s = 0.f;
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) {
        const float2 p = stats[r * ntile + i];
        const float nm = fmaxf(m, p.x);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (p.x == -INFINITY ? 0.f : p.y * __expf(p.x - nm));
        m = nm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
        const float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sm_m[w] = m;
        sm_s[w] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY, S = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            const float nm = fmaxf(M, sm_m[i]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - nm)) + (sm_m[i] == -INFINITY ? 0.f : sm_s[i] * __expf(sm_m[i] - nm));
            M = nm;
        }
        const float lse = M + __logf(S);
        sh_lse = lse;
        loss_rows[r] = lse - label_logit[r];
    }
    __syncthreads();
    const float lse = sh_lse;
    const float scale = *scale_dev;
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) fac[i] = __expf(stats[r * ntile + i].x - lse) * scale;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const uint4 u = __ldcs(drow + i);
        const float f = fac[i >> 5];  // 32 uint4 = 256 columns per stats tile
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
        float v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = __uint_as_float(w4[k] << 16) * f;
            v[2 * k + 1] = __uint_as_float(w4[k] & 0xffff0000u) * f;
        }
        const int64_t j = label - 8 * i;
        if (j >= 0 && j < 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k == j) v[k] -= scale;
        }
        store8(e_dlogits + r * V + 8 * i, v);
    }
}

void ce_rows_exp(void* e_dlogits, const float* stats, int ntile, const int64_t* labels, const float* label_logit,
                 int64_t rows, int64_t V, const float* scale_dev, float* loss_rows, int32_t* err, cudaStream_t st) {
    SPT_CHECK(V % 8 == 0, SPT_ERR_SHAPE, "vocab must be a multiple of 8");
    SPT_CHECK(ntile <= CE_MAX_TILES, SPT_ERR_SHAPE, "vocab too large for the fused CE pass (max 262144)");
    if (rows == 0) return;
    prof_run(P_CE, 0, 4.0 * rows * V, st, [&] {
        ce_rows_exp_kernel<<<(unsigned)rows, 512, 0, st>>>((bf16*)e_dlogits, (const float2*)stats, ntile, labels,
                                                           label_logit, V, scale_dev, loss_rows, err);
        count_launch("ce_rows_exp");
    });
    SPT_CUDA(cudaGetLastError());
}

void ce_rows_stats(const float* logits, const float* stats, int ntile, const int64_t* labels, int64_t rows, int64_t V,
                   const float* scale_dev, float* loss_rows, void* dlogits, int32_t* err, cudaStream_t st) {
    SPT_CHECK(V % 8 == 0, SPT_ERR_SHAPE, "vocab must be a multiple of 8");
    if (rows == 0) return;
    prof_run(P_CE, 0, 4.0 * rows * V + 2.0 * rows * V, st, [&] {
        ce_rows_stats_kernel<<<(unsigned)rows, 512, 0, st>>>(logits, (const float2*)stats, ntile, labels, V, scale_dev,
                                                             loss_rows, (bf16*)dlogits, err);
        count_launch("ce_rows_stats");
    });
    SPT_CUDA(cudaGetLastError());
}

void ce_rows(const float* logits, const int64_t* labels, int64_t rows, int64_t V, const float* scale_dev,
             float* loss_rows, void* dlogits, int32_t* err, cudaStream_t st) {
    SPT_CHECK(V % 8 == 0, SPT_ERR_SHAPE, "vocab must be a multiple of 8");
    if (rows == 0) return;
    prof_run(P_CE, 0, 6.0 * rows * V, st, [&] {
        ce_rows_kernel<<<(unsigned)rows, 512, 0, st>>>(logits, labels, V, scale_dev, loss_rows, (bf16*)dlogits, err);
        count_launch("ce_rows");
    });
    SPT_CUDA(cudaGetLastError());
}

__global__ void sum_rows_kernel(const float* __restrict__ v, int64_t n, double* accum) {
    __shared__ double red[32];
    double s = 0.0;
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t a = threadIdx.x * per, b = min(n, a + per);
    for (int64_t i = a; i < b; ++i) s += (double)v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        *accum += t;
    }
}

void sum_rows(const float* v, int64_t n, double* accum, cudaStream_t st) {
    if (n == 0) return;
    sum_rows_kernel<<<1, 1024, 0, st>>>(v, n, accum);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

__global__ void finalize_scale_kernel(const int64_t* count, float* scale) {
    const int64_t c = *count;
    *scale = c > 0 ? (float)(1.0 / (double)c) : 0.f;
}
__global__ void finalize_loss_kernel(const double* sum, const int64_t* count, float* loss) {
    const int64_t c = *count;
    *loss = c > 0 ? (float)(*sum / (double)c) : 0.f;
}
__global__ void window_accumulate_kernel(const double* loss_sum, const int64_t* count, double* win_sum,
                                         int64_t* win_count, int first) {
    *win_sum = (first ? 0.0 : *win_sum) + *loss_sum;
    *win_count = (first ? 0 : *win_count) + *count;
}
void window_accumulate(const double* loss_sum, const int64_t* count, double* win_sum, int64_t* win_count, bool first,
                       cudaStream_t st) {
    window_accumulate_kernel<<<1, 1, 0, st>>>(loss_sum, count, win_sum, win_count, first ? 1 : 0);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}
__global__ void window_finalize_kernel(const double* win_sum, const int64_t* win_count, double* loss_sum,
                                       int64_t* count, float* loss) {
    *loss_sum = *win_sum;
    *count = *win_count;
    *loss = *win_count > 0 ? (float)(*win_sum / (double)*win_count) : 0.f;
}
void window_finalize(const double* win_sum, const int64_t* win_count, double* loss_sum, int64_t* count, float* loss,
                     cudaStream_t st) {
    window_finalize_kernel<<<1, 1, 0, st>>>(win_sum, win_count, loss_sum, count, loss);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}
__global__ void scale_by_inverse_count_kernel(float* g, int64_t n, const int64_t* count) {
    const int64_t c = *count;
    const float s = c > 0 ? (float)(1.0 / (double)c) : 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g[i] *= s;
}
void scale_by_inverse_count(float* g, int64_t n, const int64_t* count, cudaStream_t st) {
    scale_by_inverse_count_kernel<<<148 * 8, 256, 0, st>>>(g, n, count);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}
void finalize_scale(const int64_t* count, float* scale, cudaStream_t st) {
    finalize_scale_kernel<<<1, 1, 0, st>>>(count, scale);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}
void finalize_loss(const double* loss_sum, const int64_t* count, float* loss_out, cudaStream_t st) {
    finalize_loss_kernel<<<1, 1, 0, st>>>(loss_sum, count, loss_out);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ SGD + weight layout helpers
__global__ void sgd_kernel(bf16* __restrict__ w, const float* __restrict__ g, int64_t n, float lr) {
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i < n; i += (int64_t)gridDim.x * blockDim.x * 8) {
        float wv[8];
        load8(w + i, wv);
        const float4 a = *reinterpret_cast<const float4*>(g + i), b = *reinterpret_cast<const float4*>(g + i + 4);
        const float gv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) wv[k] -= lr * gv[k];
        store8(w + i, wv);
    }
}
void sgd_update(void* w, const float* g, int64_t n, float lr, cudaStream_t st) {
    SPT_CHECK(n % 8 == 0, SPT_ERR_SHAPE, "sgd: size must be a multiple of 8");
    if (n == 0) return;
    sgd_kernel<<<grid_for(n / 8, 256), 256, 0, st>>>((bf16*)w, g, n, lr);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

__global__ void interleave_gu_kernel(const uint4* __restrict__ wg, const uint4* __restrict__ wu, uint4* __restrict__ out,
                                     int64_t inter, int64_t vrow) {
    const int64_t total = 2 * inter * vrow;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / vrow, v = i % vrow;
        const int64_t blk = r / 64, w = r % 64;
        if (w < 32) {
            if (wg) out[i] = wg[(blk * 32 + w) * vrow + v];
        } else if (wu) {
            out[i] = wu[(blk * 32 + w - 32) * vrow + v];
        }
    }
}
void interleave_gu(const void* wg, const void* wu, void* wgu, int64_t inter, int64_t h, cudaStream_t st) {
    SPT_CHECK(inter % 32 == 0 && h % 8 == 0, SPT_ERR_SHAPE, "intermediate must be a multiple of 32");
    interleave_gu_kernel<<<grid_for(2 * inter * h / 8, 256), 256, 0, st>>>((const uint4*)wg, (const uint4*)wu,
                                                                           (uint4*)wgu, inter, h / 8);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}
__global__ void deinterleave_gu_kernel(const float4* __restrict__ gu, float4* __restrict__ g, float4* __restrict__ u,
                                       int64_t inter, int64_t vrow) {
    const int64_t total = 2 * inter * vrow;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / vrow, v = i % vrow;
        const int64_t blk = r / 64, w = r % 64;
        if (w < 32) g[(blk * 32 + w) * vrow + v] = gu[i];
        else u[(blk * 32 + w - 32) * vrow + v] = gu[i];
    }
}
void deinterleave_gu_f32(const float* gu, float* g, float* u, int64_t inter, int64_t h, cudaStream_t st) {
    deinterleave_gu_kernel<<<grid_for(2 * inter * h / 4, 256), 256, 0, st>>>((const float4*)gu, (float4*)g, (float4*)u,
                                                                             inter, h / 4);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

}  // namespace spt

namespace spt {

// ------------------------------------------------------------------ checkpoint replay verification
// (autograd.hpp:26-30: the replay of a checkpointed region must be bit-identical to its recorded forward)
// Order-independent 64-bit fingerprint of a bf16 buffer: sum mod 2^64 of a mixed (index, bits) word per
// element, so the atomics' arrival order cannot change it; any bit flip changes it.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fingerprint_kernel(const uint16_t* __restrict__ x, int64_t n, uint64_t* out) {
    uint64_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += mix64(((uint64_t)i << 16) | x[i]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)out, (unsigned long long)acc);
}

__global__ void fingerprint_compare_kernel(const uint64_t* want, const uint64_t* got, int32_t* err, int32_t tag) {
    if (*want != *got && *err == 0) *err = tag;
}

__global__ void flip_bit_kernel(uint16_t* x) { x[0] ^= 1; }

void fingerprint_bf16(const void* x, int64_t n, uint64_t* out, cudaStream_t st) {
    fingerprint_kernel<<<grid_for(n, 256), 256, 0, st>>>((const uint16_t*)x, n, out);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void fingerprint_compare(const uint64_t* want, const uint64_t* got, int32_t* err, int32_t tag, cudaStream_t st) {
    fingerprint_compare_kernel<<<1, 1, 0, st>>>(want, got, err, tag);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

void flip_lowest_bit(void* x, cudaStream_t st) {
    flip_bit_kernel<<<1, 1, 0, st>>>((uint16_t*)x);
    count_launch();
    SPT_CUDA(cudaGetLastError());
}

}  // namespace spt
