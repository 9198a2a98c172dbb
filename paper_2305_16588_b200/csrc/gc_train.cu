// Trainer helper kernels: the GraphSAGE mean aggregation straight from the gathered
// feature rows. For the first layer the children of a tree level are rows of the
// batch's feature matrix X[U, D] named by their relabelled ids, so
//   agg[i] = mean_{k in [off[i], off[i+1])} X[idx[k]]
// is computed without materialising X[idx] (at C2 that is 768K x 100 fp32 per batch).
// Warp per segment, lanes over the feature dimension (float4 when D % 4 == 0); the
// sum runs in child order, as torch.segment_reduce's does, in fp32.
#include <cuda_bf16.h>

#include "gc_common.cuh"

namespace gc {

template <bool VEC4>
__global__ void __launch_bounds__(256) k_segment_mean_gather(const float* __restrict__ x, int dim,
                                                             const int64_t* __restrict__ idx,
                                                             const int64_t* __restrict__ off, int64_t segs,
                                                             float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < segs; i += warps) {
        const int64_t a = off[i], b = off[i + 1];
        const float inv = b > a ? 1.0f / (float)(b - a) : 0.0f;
        if (VEC4) {
            const int d4 = dim / 4;
            for (int c = lane; c < d4; c += 32) {
                float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int64_t k = a; k < b; ++k) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(x + idx[k] * dim) + c);
                    s.x += v.x;
                    s.y += v.y;
                    s.z += v.z;
                    s.w += v.w;
                }
                reinterpret_cast<float4*>(out + i * dim)[c] = make_float4(s.x * inv, s.y * inv, s.z * inv, s.w * inv);
            }
        } else {
            for (int c = lane; c < dim; c += 32) {
                float s = 0.f;
                for (int64_t k = a; k < b; ++k) s += __ldg(x + idx[k] * dim + c);
                out[i * dim + c] = s * inv;
            }
        }
    }
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_segment_mean_gather(const float* d_x, int dim, const int64_t* d_idx, const int64_t* d_offsets, int64_t segs,
                           float* d_out, void* stream) {
    GC_REQUIRE(dim >= 1 && segs >= 0, GC_ERR_VALUE, "gc_segment_mean_gather: bad sizes");
    if (segs == 0) return GC_OK;
    int64_t g = (segs + 7) / 8;
    if (g > (int64_t)sm_count() * 64) g = (int64_t)sm_count() * 64;
    const bool vec4 = dim % 4 == 0 && (uintptr_t)d_x % 16 == 0 && (uintptr_t)d_out % 16 == 0;
    if (vec4)
        k_segment_mean_gather<true><<<(unsigned)g, 256, 0, as_stream(stream)>>>(d_x, dim, d_idx, d_offsets, segs, d_out);
    else
        k_segment_mean_gather<false><<<(unsigned)g, 256, 0, as_stream(stream)>>>(d_x, dim, d_idx, d_offsets, segs,
                                                                                 d_out);
    GC_CHECK_LAUNCH("gc_segment_mean_gather");
    return GC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------
// Tree trainer kernels: GraphSAGE / GCN over the sampled position trees with a
// hand-written forward and backward (train.TreeTrainer). Positions of all levels are
// stacked (level 0 = seeds first); every position has at most one parent, so the
// backward of the neighbour aggregation is a gather from the parent row — no atomics.
// Batches are staged into padded, fixed-shape buffers so one CUDA graph per step
// replays for every batch; the batch index is read from device memory.
namespace gc {

__global__ void k_tree_stage(gc_tree_src_t s, const int32_t* __restrict__ d_batch, int64_t total,
                             int32_t* __restrict__ loc, int32_t* __restrict__ cbeg, int32_t* __restrict__ cdeg,
                             int32_t* __restrict__ level_counts, int64_t* __restrict__ labels) {
    const int b = *d_batch;
    const int L = s.hops;
    if (blockIdx.x == 0 && threadIdx.x <= (unsigned)L)
        level_counts[threadIdx.x] = s.counts[(int64_t)threadIdx.x * s.counts_stride + b];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        int64_t base = 0;
        while (k < L && p >= base + s.caps[k]) base += s.caps[k++];
        const int64_t i = p - base;
        const int64_t cnt = s.counts[(int64_t)k * s.counts_stride + b];
        const bool real = i < cnt;
        const int64_t li = (int64_t)b * s.local_stride[k] + i;
        loc[p] = !real ? 0
                 : s.local_bits == 16 ? (int32_t)reinterpret_cast<const uint16_t*>(s.local[k])[li]
                                      : s.local[k][li];
        if (k == 0 && labels) labels[i] = real ? s.labels[(uint32_t)s.seeds[(int64_t)b * s.seeds_stride + i]] : -100;
        if (k < L) {
            const int64_t nbase = base + s.caps[k];
            const int32_t* off = s.offsets[k] + (int64_t)b * s.offsets_stride[k];
            int32_t o0 = 0, d = 0;
            if (real) {
                o0 = off[i];
                d = off[i + 1] - o0;
            }
            cbeg[p] = (int32_t)(nbase + o0);
            cdeg[p] = d;
        }
    }
}

// 16-byte vectors of T: 4 fp32 or 8 bf16 elements, widened to fp32 in registers
template <typename T>
struct Vec {
    static constexpr int N = 16 / sizeof(T);
};
__device__ __forceinline__ void vload(const float* p, float (&v)[4]) {
    const float4 r = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
}
__device__ __forceinline__ void vload(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
// raw 16-byte loads kept packed in registers until used (4 registers per vector)
__device__ __forceinline__ uint4 rload(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void unpack(uint4 r, float (&v)[4]) {
    v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y); v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
}
__device__ __forceinline__ void unpack(uint4 r, float (&v)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
// store N elements (any N multiple of 2) as fp32 or bf16
template <int N>
__device__ __forceinline__ void vstore(float* p, const float (&v)[N], float s) {
#pragma unroll
    for (int i = 0; i < N; i += 4)
        *reinterpret_cast<float4*>(p + i) = make_float4(v[i] * s, v[i + 1] * s, v[i + 2] * s, v[i + 3] * s);
}
template <int N>
__device__ __forceinline__ void vstore(__nv_bfloat16* p, const float (&v)[N], float s) {
    uint32_t w[N / 2];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i] * s, v[2 * i + 1] * s);
        w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    if constexpr (N == 8) {
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
        *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
    }
}

// forward aggregation, warp per output position, lanes over 16-byte column groups:
//   SAGE: out[p] = [ f(in[row(p)]), mean_{c in children(p)} f(in[row(c)]) ]   (2*dim columns)
//   GCN:  out[p] = ( f(in[row(p)]) + sum_c f(in[row(c)]) ) / (deg(p) + 1)      (dim columns)
// f = ReLU when the input rows are a layer's pre-activations (RELU), else identity.
// row(q) = batch_row0 + (rowmap ? rowmap[q] : q). Children are consecutive positions;
// 4 child rows are loaded before any is summed (summed in child order, in fp32).
template <typename TI, typename TO, int MODE, bool RELU>
__global__ void __launch_bounds__(256, 4) k_tree_aggregate(const TI* __restrict__ in, int64_t in_stride, int dim,
                                                        const int32_t* __restrict__ rowmap,
                                                        const int32_t* __restrict__ cbeg,
                                                        const int32_t* __restrict__ cdeg, int64_t p_out,
                                                        TO* __restrict__ out, int64_t out_stride,
                                                        const int32_t* __restrict__ d_batch, int64_t batch_rows) {
    constexpr int N = Vec<TI>::N;
    const int lane = threadIdx.x & 31;
    const int64_t row0 = d_batch ? (int64_t)(*d_batch) * batch_rows : 0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); p < p_out; p += warps) {
        const int32_t c0 = cbeg[p], d = cdeg[p];
        const TI* self = in + (row0 + (rowmap ? __ldg(rowmap + p) : p)) * in_stride;
        for (int c = lane * N; c < dim; c += 32 * N) {
            float acc[N], v[N];
#pragma unroll
            for (int i = 0; i < N; ++i) acc[i] = 0.f;
            const uint4 sr = rload(self + c);
            int32_t j = 0;
            for (; j + 4 <= d; j += 4) {
                uint4 w[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t q = c0 + j + u;
                    w[u] = rload(in + (row0 + (rowmap ? __ldg(rowmap + q) : q)) * in_stride + c);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    unpack(w[u], v);
#pragma unroll
                    for (int i = 0; i < N; ++i) acc[i] += RELU ? fmaxf(v[i], 0.f) : v[i];
                }
            }
            for (; j < d; ++j) {
                const int64_t q = c0 + j;
                unpack(rload(in + (row0 + (rowmap ? __ldg(rowmap + q) : q)) * in_stride + c), v);
#pragma unroll
                for (int i = 0; i < N; ++i) acc[i] += RELU ? fmaxf(v[i], 0.f) : v[i];
            }
            unpack(sr, v);
            if (RELU) {
#pragma unroll
                for (int i = 0; i < N; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            TO* o = out + p * out_stride;
            if (MODE == 0) {
                vstore<N>(o + c, v, 1.0f);
                vstore<N>(o + dim + c, acc, d ? 1.0f / (float)d : 0.0f);
            } else {
#pragma unroll
                for (int i = 0; i < N; ++i) acc[i] += v[i];
                vstore<N>(o + c, acc, 1.0f / (float)(d + 1));
            }
        }
    }
}

// backward of the aggregation, fused with the ReLU mask of the input pre-activations z.
// Row q of g (q < p_in) receives cs(q) * dA[q, self cols] when q < p_out and
// cc(p) * dA[p, child cols] when q is a child of p:
//   SAGE: self cols [0, dim), child cols [dim, 2 dim), cs = 1, cc = 1/deg(p)
//   GCN:  both [0, dim), cs = 1/(deg(q)+1), cc = 1/(deg(p)+1)
// and g[q] = [z[q] > 0] * that. Work is parent-centric — a warp takes a parent p, loads
// dA[p, child cols] once and walks its consecutive children, 4 rows in flight — plus
// warps for the level-0 rows (no parent) and for 32-row chunks of every level, which
// zero the padded rows (no parent, no gradient) past the batch's count.
struct TreeBwd {
    const void* dA;
    int64_t dA_stride;
    int dim;
    const int32_t* cbeg;
    const int32_t* cdeg;
    int64_t p_out, p_in;
    const void* h;
    int64_t h_stride;
    void* g;
    int64_t g_stride;
    int nlev;  // levels spanned by rows [0, p_in)
    int64_t base[GC_TREE_MAX_LEVELS + 1];
    int64_t chunk0[GC_TREE_MAX_LEVELS + 1];  // first zeroing task of level k (k >= 1)
    const int32_t* level_counts;
};

template <typename T, int MODE>
__device__ __forceinline__ void bwd_row(const TreeBwd& a, int64_t q, float cs, const uint4& pr, float cc, int c,
                                        uint4 self_raw, uint4 z_raw) {
    constexpr int N = Vec<T>::N;
    float v[N], fa[N], fz[N];
    if (cc != 0.f) {
        unpack(pr, fa);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = fa[i] * cc;
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = 0.f;
    }
    if (cs != 0.f) {
        unpack(self_raw, fa);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] += fa[i] * cs;
    }
    if (a.h) {
        unpack(z_raw, fz);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = fz[i] > 0.f ? v[i] : 0.f;
    }
    vstore<N>(static_cast<T*>(a.g) + q * a.g_stride + c, v, 1.0f);
}

template <typename T, int MODE>
__global__ void __launch_bounds__(256, 4) k_tree_aggregate_bwd(TreeBwd a, int64_t tasks) {
    constexpr int N = Vec<T>::N;
    const int lane = threadIdx.x & 31;
    const T* dA = static_cast<const T*>(a.dA);
    const T* h = static_cast<const T*>(a.h);
    const int child_col = MODE == 0 ? a.dim : 0;
    const int64_t B0 = a.base[1] < a.p_in ? a.base[1] : a.p_in;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); t < tasks; t += warps) {
        if (t < B0) {  // level-0 row: self part only
            const int64_t q = t;
            const float cs = MODE == 0 ? 1.0f : 1.0f / (float)(a.cdeg[q] + 1);
            for (int c = lane * N; c < a.dim; c += 32 * N)
                bwd_row<T, MODE>(a, q, q < a.p_out ? cs : 0.f, zero, 0.f, c,
                                 q < a.p_out ? rload(dA + q * a.dA_stride + c) : zero,
                                 h ? rload(h + q * a.h_stride + c) : zero);
            continue;
        }
        if (t < B0 + a.p_out) {  // parent p: its consecutive children
            const int64_t p = t - B0;
            const int32_t c0 = a.cbeg[p], d = a.cdeg[p];
            if (d == 0) continue;
            const float cc = MODE == 0 ? 1.0f / (float)d : 1.0f / (float)(d + 1);
            for (int c = lane * N; c < a.dim; c += 32 * N) {
                const uint4 pr = rload(dA + p * a.dA_stride + child_col + c);
                constexpr int RU = sizeof(T) == 2 ? 2 : 4;  // rows in flight (bf16: 64 registers)
                int32_t j = 0;
                for (; j < d; j += RU) {
                    uint4 sr[RU], zr[RU];
                    float cs[RU];
#pragma unroll
                    for (int u = 0; u < RU; ++u) {
                        const int64_t q = c0 + j + u;
                        sr[u] = zr[u] = zero;
                        cs[u] = 0.f;
                        if (j + u < d) {
                            if (q < a.p_out) {
                                cs[u] = MODE == 0 ? 1.0f : 1.0f / (float)(a.cdeg[q] + 1);
                                sr[u] = rload(dA + q * a.dA_stride + c);
                            }
                            if (h) zr[u] = rload(h + q * a.h_stride + c);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < RU; ++u)
                        if (j + u < d) bwd_row<T, MODE>(a, c0 + j + u, cs[u], pr, cc, c, sr[u], zr[u]);
                }
            }
            continue;
        }
        // zeroing task: 32 rows of level k past the batch's count (padding: no parent)
        const int64_t z = t - B0 - a.p_out;
        int k = 1;
        while (k + 1 < a.nlev && z >= a.chunk0[k + 1]) ++k;
        const int64_t r0 = a.base[k] + (z - a.chunk0[k]) * 32;
        const int64_t first_pad = a.base[k] + a.level_counts[k];
        const int64_t r1 = min(r0 + 32, min(a.base[k + 1], a.p_in));
        for (int64_t q = max(r0, first_pad); q < r1; ++q)
            for (int c = lane * N; c < a.dim; c += 32 * N)
                *reinterpret_cast<uint4*>(static_cast<T*>(a.g) + q * a.g_stride + c) = zero;
    }
}

static inline unsigned warp_grid(int64_t rows) {
    int64_t g = (rows + 7) / 8;
    const int64_t cap = (int64_t)sm_count() * 64;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}


// ---- classifier head: logits, cross entropy and its backward in three launches
// (replaces ~20 small torch kernels per step). T is the activation type: inputs are
// rounded to it exactly as the torch path casts them (bf16 operands, fp32 sums).
template <typename T>
__device__ __forceinline__ float act_round(float x) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(__float2bfloat16(x));
    return x;
}
__device__ __forceinline__ float act_load(const float* p) { return *p; }
__device__ __forceinline__ float act_load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <typename T>
__device__ __forceinline__ T act_cast(float x);
template <>
__device__ __forceinline__ float act_cast<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 act_cast<__nv_bfloat16>(float x) { return __float2bfloat16(x); }


// One CTA of kHeadWarps warps per seed row r: top = relu(z[r]); logits = top . W_act^T
// + b (warps split the classes, lanes the hidden units: coalesced rows of W, fixed-order
// warp sums); log-softmax; rowloss[r] = -logp[y] / nvalid; dlog[r] = (softmax -
// onehot(y)) / nvalid (0 for padding, label < 0); g[r] = (dlog_act . W_act) * (z[r] > 0)
// with threads over the hidden units. A row is little work, so several warps share it:
// the kernel is latency-bound and needs the parallelism.
constexpr int kHeadWarps = 8;

template <typename T>
__global__ void __launch_bounds__(32 * kHeadWarps) k_tree_head_rows(
    const T* __restrict__ z, int64_t z_stride, int hid, int64_t rows, const float* __restrict__ W,
    const float* __restrict__ bias, int C, const int64_t* __restrict__ labels, const int32_t* __restrict__ nvalid,
    float* __restrict__ dlog, float* __restrict__ rowloss, T* __restrict__ g, int64_t g_stride) {
    extern __shared__ float sh[];
    float* top = sh;       // [hid]
    float* dl = sh + hid;  // [C]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = blockIdx.x;
    const T* zr = z + r * z_stride;
    for (int h = threadIdx.x; h < hid; h += blockDim.x) {
        const float v = act_load(zr + h);
        top[h] = v > 0.f ? v : 0.f;
    }
    __syncthreads();
    for (int c = warp; c < C; c += kHeadWarps) {
        const float* w = W + (int64_t)c * hid;
        float part = 0.f;
        for (int h = lane; h < hid; h += 32) part = fmaf(top[h], act_round<T>(__ldg(w + h)), part);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        if (lane == 0) dl[c] = part + bias[c];
    }
    __syncthreads();
    if (warp == 0) {
        const float nv = (float)max(*nvalid, 1);
        const int64_t y = labels[r];
        float mx = -INFINITY;
        for (int c = lane; c < C; c += 32) mx = fmaxf(mx, dl[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        float se = 0.f;
        for (int c = lane; c < C; c += 32) se += __expf(dl[c] - mx);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
        const float lse = mx + __logf(se);
        const bool valid = y >= 0;
        if (lane == 0) rowloss[r] = 0.f;
        __syncwarp();
        for (int c = lane; c < C; c += 32) {
            const float lp = dl[c] - lse;
            if (valid && c == y) rowloss[r] = -lp / nv;
            const float d = valid ? (__expf(lp) - (c == y ? 1.f : 0.f)) / nv : 0.f;
            dl[c] = d;
            dlog[r * C + c] = d;
        }
    }
    __syncthreads();
    T* gr = g + r * g_stride;
    for (int h = threadIdx.x; h < hid; h += blockDim.x) {
        float acc = 0.f;
        for (int c = 0; c < C; ++c) acc = fmaf(act_round<T>(dl[c]), act_round<T>(__ldg(W + (int64_t)c * hid + h)), acc);
        gr[h] = act_cast<T>(top[h] > 0.f ? acc : 0.f);
    }
}

constexpr int kHeadChunkRows = 32;

// dW partials: part[chunk][c][h] = sum over the chunk's rows of dlog_act[r,c] * top[r,h],
// and part[chunk][c][hid] = the chunk's sum of dlog[r,c] (the bias gradient)
template <typename T>
__global__ void k_tree_head_dw(const T* __restrict__ z, int64_t z_stride, int hid, int64_t rows, int C,
                               const float* __restrict__ dlog, float* __restrict__ part) {
    const int c = blockIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * kHeadChunkRows;
    const int64_t r1 = min(rows, r0 + kHeadChunkRows);
    float* out = part + ((int64_t)blockIdx.y * C + c) * (hid + 1);
    for (int h = threadIdx.x; h < hid; h += blockDim.x) {
        float acc = 0.f;
        for (int64_t r = r0; r < r1; ++r) {
            const float t = act_load(z + r * z_stride + h);
            acc = fmaf(act_round<T>(dlog[r * C + c]), t > 0.f ? t : 0.f, acc);
        }
        out[h] = acc;
    }
    if (threadIdx.x < 32) {  // the chunk's bias-gradient share, lanes over rows, fixed order
        float acc = 0.f;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += 32) acc += dlog[r * C + c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (threadIdx.x == 0) out[hid] = acc;
    }
}

// dW and db: sums of the chunk partials in chunk order; loss: one CTA reduces rowloss
__global__ void k_tree_head_final(const float* __restrict__ part, int chunks, int C, int hid, int64_t rows,
                                  const float* __restrict__ rowloss, float* __restrict__ dW, float* __restrict__ db,
                                  float* __restrict__ loss) {
    const int64_t n = (int64_t)C * (hid + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int k = 0; k < chunks; ++k) acc += part[k * n + i];
        const int64_t c = i / (hid + 1), h = i - c * (hid + 1);
        if (h < hid)
            dW[c * hid + h] = acc;
        else
            db[c] = acc;
    }
    if (blockIdx.x == 0) {
        __shared__ float s_w[32];
        float acc = 0.f;
        for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) acc += rowloss[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_w[w];
            *loss = t;
        }
    }
}

}  // namespace gc

extern "C" {

int gc_tree_stage(const gc_tree_src_t* src, const int32_t* d_batch, int32_t* d_loc, int32_t* d_cbeg, int32_t* d_cdeg,
                  int32_t* d_level_counts, int64_t* d_labels, void* stream) {
    GC_REQUIRE(src && d_batch && d_loc && d_level_counts, GC_ERR_VALUE, "gc_tree_stage: null pointer");
    GC_REQUIRE(src->hops >= 0 && src->hops < GC_TREE_MAX_LEVELS, GC_ERR_VALUE, "gc_tree_stage: bad hop count");
    GC_REQUIRE(src->hops == 0 || (d_cbeg && d_cdeg), GC_ERR_VALUE, "gc_tree_stage: null child arrays");
    int64_t total = 0;
    for (int k = 0; k <= src->hops; ++k) total += src->caps[k];
    if (total == 0) return GC_OK;
    int64_t g = (total + 255) / 256;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_tree_stage<<<(unsigned)g, 256, 0, as_stream(stream)>>>(*src, d_batch, total, d_loc, d_cbeg, d_cdeg,
                                                            d_level_counts, d_labels);
    GC_CHECK_LAUNCH("gc_tree_stage");
    return GC_OK;
}

int gc_tree_aggregate(const void* d_in, int in_dtype, int64_t in_stride, int dim, const int32_t* d_rowmap,
                      const int32_t* d_cbeg, const int32_t* d_cdeg, int64_t p_out, int mode, void* d_out, int out_dtype,
                      int64_t out_stride, const int32_t* d_batch, int64_t batch_rows, void* stream) {
    GC_REQUIRE(mode >= 0 && mode <= 3, GC_ERR_VALUE,
               "gc_tree_aggregate: mode is 0 (SAGE) or 1 (GCN), +2 for ReLU on the input rows");
    GC_REQUIRE((in_dtype == 0 || in_dtype == 1) && (out_dtype == 0 || out_dtype == 1), GC_ERR_VALUE,
               "gc_tree_aggregate: dtype is 0 (fp32) or 1 (bf16)");
    const int vec = in_dtype == 0 ? 4 : 8;
    GC_REQUIRE(dim >= vec && dim % vec == 0 && in_stride % vec == 0 && out_stride % vec == 0, GC_ERR_VALUE,
               "gc_tree_aggregate: dim and strides must be multiples of 16 bytes of the input type");
    GC_REQUIRE(in_dtype == out_dtype || in_dtype == 0, GC_ERR_VALUE, "gc_tree_aggregate: bf16 -> fp32 unsupported");
    if (p_out <= 0) return GC_OK;
    const unsigned g = warp_grid(p_out);
    cudaStream_t s = as_stream(stream);
    const int m = mode & 1;
    const bool relu = (mode & 2) != 0;
#define GC_AGG(TI, TO, M, R)                                                                                        \
    k_tree_aggregate<TI, TO, M, R><<<g, 256, 0, s>>>(static_cast<const TI*>(d_in), in_stride, dim, d_rowmap,       \
                                                     d_cbeg, d_cdeg, p_out, static_cast<TO*>(d_out), out_stride,    \
                                                     d_batch, batch_rows)
#define GC_AGG2(TI, TO)                                  \
    if (m == 0) {                                        \
        if (relu) GC_AGG(TI, TO, 0, true); else GC_AGG(TI, TO, 0, false); \
    } else {                                             \
        if (relu) GC_AGG(TI, TO, 1, true); else GC_AGG(TI, TO, 1, false); \
    }
    using bf = __nv_bfloat16;
    if (in_dtype == 0 && out_dtype == 0) { GC_AGG2(float, float) }
    else if (in_dtype == 0) { GC_AGG2(float, bf) }
    else { GC_AGG2(bf, bf) }
#undef GC_AGG2
#undef GC_AGG
    GC_CHECK_LAUNCH("gc_tree_aggregate");
    return GC_OK;
}

int gc_tree_aggregate_backward(const void* d_dA, int dtype, int64_t dA_stride, int dim, int mode,
                               const int32_t* d_cbeg, const int32_t* d_cdeg, int64_t p_out, int64_t p_in,
                               const void* d_h, int64_t h_stride, void* d_g, int64_t g_stride, int nlevels,
                               const int64_t* level_caps, const int32_t* d_level_counts, void* stream) {
    GC_REQUIRE(mode == 0 || mode == 1, GC_ERR_VALUE, "gc_tree_aggregate_backward: mode is 0 (SAGE) or 1 (GCN)");
    GC_REQUIRE(dtype == 0 || dtype == 1, GC_ERR_VALUE, "gc_tree_aggregate_backward: dtype is 0 (fp32) or 1 (bf16)");
    const int vec = dtype == 0 ? 4 : 8;
    GC_REQUIRE(dim >= vec && dim % vec == 0 && dA_stride % vec == 0 && g_stride % vec == 0 && h_stride % vec == 0,
               GC_ERR_VALUE, "gc_tree_aggregate_backward: dim and strides must be multiples of 16 bytes");
    GC_REQUIRE(nlevels >= 1 && nlevels <= GC_TREE_MAX_LEVELS && level_caps && d_level_counts, GC_ERR_VALUE,
               "gc_tree_aggregate_backward: bad level description");
    GC_REQUIRE(p_out <= p_in, GC_ERR_VALUE, "gc_tree_aggregate_backward: p_out > p_in");
    if (p_in <= 0) return GC_OK;
    TreeBwd a{};
    a.dA = d_dA;
    a.dA_stride = dA_stride;
    a.dim = dim;
    a.cbeg = d_cbeg;
    a.cdeg = d_cdeg;
    a.p_out = p_out;
    a.p_in = p_in;
    a.h = d_h;
    a.h_stride = h_stride;
    a.g = d_g;
    a.g_stride = g_stride;
    a.nlev = nlevels;
    a.level_counts = d_level_counts;
    a.base[0] = 0;
    for (int k = 0; k < nlevels; ++k) a.base[k + 1] = a.base[k] + level_caps[k];
    GC_REQUIRE(a.base[nlevels] == p_in, GC_ERR_VALUE, "gc_tree_aggregate_backward: level caps must sum to p_in");
    int64_t chunks = 0;
    for (int k = 1; k < nlevels; ++k) {
        a.chunk0[k] = chunks;
        chunks += (level_caps[k] + 31) / 32;
    }
    a.chunk0[nlevels] = chunks;
    const int64_t tasks = (p_in < level_caps[0] ? p_in : level_caps[0]) + p_out + chunks;
    const unsigned g = warp_grid(tasks);
    cudaStream_t s = as_stream(stream);
    if (dtype == 0) {
        if (mode == 0) k_tree_aggregate_bwd<float, 0><<<g, 256, 0, s>>>(a, tasks);
        else k_tree_aggregate_bwd<float, 1><<<g, 256, 0, s>>>(a, tasks);
    } else {
        if (mode == 0) k_tree_aggregate_bwd<__nv_bfloat16, 0><<<g, 256, 0, s>>>(a, tasks);
        else k_tree_aggregate_bwd<__nv_bfloat16, 1><<<g, 256, 0, s>>>(a, tasks);
    }
    GC_CHECK_LAUNCH("gc_tree_aggregate_backward");
    return GC_OK;
}

size_t gc_tree_head_work_floats(int64_t rows, int classes, int hid) {
    const int64_t chunks = (rows + kHeadChunkRows - 1) / kHeadChunkRows;
    return (size_t)(rows * classes + rows + chunks * classes * ((int64_t)hid + 1));
}

int gc_tree_head(const void* d_z, int dtype, int64_t z_stride, int hid, int64_t rows, const float* d_W,
                 const float* d_b, int classes, const int64_t* d_labels, const int32_t* d_nvalid, float* d_loss,
                 float* d_dW, float* d_db, void* d_g, int64_t g_stride, float* d_work, size_t work_floats,
                 void* stream) {
    GC_REQUIRE(dtype == 0 || dtype == 1, GC_ERR_VALUE, "gc_tree_head: dtype is 0 (fp32) or 1 (bf16)");
    GC_REQUIRE(hid >= 1 && classes >= 1 && rows >= 1, GC_ERR_VALUE, "gc_tree_head: empty shape");
    GC_REQUIRE(d_work && work_floats >= gc_tree_head_work_floats(rows, classes, hid), GC_ERR_VALUE,
               "gc_tree_head: work buffer too small");
    const size_t smem = (size_t)(hid + classes) * sizeof(float);
    GC_REQUIRE(smem <= 48 * 1024, GC_ERR_VALUE, "gc_tree_head: hidden + classes too wide");
    cudaStream_t s = as_stream(stream);
    float* dlog = d_work;
    float* rowloss = dlog + rows * classes;
    float* part = rowloss + rows;
    const int chunks = (int)((rows + kHeadChunkRows - 1) / kHeadChunkRows);
    const unsigned g1 = (unsigned)rows;
    const dim3 g2(classes, chunks);
    const int t2 = hid < 256 ? (hid + 31) / 32 * 32 : 256;
    if (dtype == 0) {
        k_tree_head_rows<float><<<g1, 32 * kHeadWarps, smem, s>>>(
            static_cast<const float*>(d_z), z_stride, hid, rows, d_W, d_b, classes, d_labels, d_nvalid, dlog, rowloss,
            static_cast<float*>(d_g), g_stride);
        k_tree_head_dw<float><<<g2, t2, 0, s>>>(static_cast<const float*>(d_z), z_stride, hid, rows, classes, dlog,
                                                 part);
    } else {
        using bf = __nv_bfloat16;
        k_tree_head_rows<bf><<<g1, 32 * kHeadWarps, smem, s>>>(
            static_cast<const bf*>(d_z), z_stride, hid, rows, d_W, d_b, classes, d_labels, d_nvalid, dlog, rowloss,
            static_cast<bf*>(d_g), g_stride);
        k_tree_head_dw<bf><<<g2, t2, 0, s>>>(static_cast<const bf*>(d_z), z_stride, hid, rows, classes, dlog, part);
    }
    const int64_t n = (int64_t)classes * (hid + 1);
    unsigned g3 = (unsigned)((n + 255) / 256);
    if (g3 < 1) g3 = 1;
    k_tree_head_final<<<g3, 256, 0, s>>>(part, chunks, classes, hid, rows, rowloss, d_dW, d_db, d_loss);
    GC_CHECK_LAUNCH("gc_tree_head");
    return GC_OK;
}

}  // extern "C"
