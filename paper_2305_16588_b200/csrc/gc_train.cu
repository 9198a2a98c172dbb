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
                             int32_t* __restrict__ parent, int64_t* __restrict__ labels) {
    const int b = *d_batch;
    const int L = s.hops;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        int64_t base = 0;
        while (k < L && p >= base + s.caps[k]) base += s.caps[k++];
        const int64_t i = p - base;
        const int64_t cnt = s.counts[(int64_t)k * s.counts_stride + b];
        const bool real = i < cnt;
        loc[p] = real ? s.local[k][(int64_t)b * s.local_stride[k] + i] : 0;
        if (k == 0) {
            parent[p] = -1;
            if (labels) labels[i] = real ? s.labels[(uint32_t)s.seeds[(int64_t)b * s.seeds_stride + i]] : -100;
        } else if (!real) {
            parent[p] = -1;
        }
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
            for (int32_t j = 0; j < d; ++j) parent[nbase + o0 + j] = (int32_t)p;
        }
    }
}

template <typename T>
struct V4;
template <>
struct V4<float> {
    __device__ static float4 load(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ static void store(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
};
template <>
struct V4<__nv_bfloat16> {
    __device__ static float4 load(const __nv_bfloat16* p) {
        const uint2 raw = __ldg(reinterpret_cast<const uint2*>(p));
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
        return make_float4(a.x, a.y, b.x, b.y);
    }
    __device__ static void store(__nv_bfloat16* p, float4 v) {
        const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
        const __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
        uint2 raw;
        raw.x = *reinterpret_cast<const uint32_t*>(&a);
        raw.y = *reinterpret_cast<const uint32_t*>(&b);
        *reinterpret_cast<uint2*>(p) = raw;
    }
};

__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 f4mul(float4 a, float s) { return make_float4(a.x * s, a.y * s, a.z * s, a.w * s); }

// forward aggregation, warp per output position, lanes over 4-element column groups:
//   SAGE: out[p] = [ in[row(p)], mean_{c in children(p)} in[row(c)] ]      (2*dim columns)
//   GCN:  out[p] = ( in[row(p)] + sum_c in[row(c)] ) / (deg(p) + 1)        (dim columns)
// row(q) = batch_row0 + (rowmap ? rowmap[q] : q); children summed in order, in fp32.
template <typename TI, typename TO, int MODE>
__global__ void __launch_bounds__(256) k_tree_aggregate(const TI* __restrict__ in, int64_t in_stride, int dim,
                                                        const int32_t* __restrict__ rowmap,
                                                        const int32_t* __restrict__ cbeg,
                                                        const int32_t* __restrict__ cdeg, int64_t p_out,
                                                        TO* __restrict__ out, int64_t out_stride,
                                                        const int32_t* __restrict__ d_batch, int64_t batch_rows) {
    const int lane = threadIdx.x & 31;
    const int64_t row0 = d_batch ? (int64_t)(*d_batch) * batch_rows : 0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); p < p_out; p += warps) {
        const int32_t c0 = cbeg[p], d = cdeg[p];
        const TI* self = in + (row0 + (rowmap ? rowmap[p] : p)) * in_stride;
        for (int c = lane * 4; c < dim; c += 128) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int32_t j = 0; j < d; ++j) {
                const int64_t q = c0 + j;
                acc = f4add(acc, V4<TI>::load(in + (row0 + (rowmap ? rowmap[q] : q)) * in_stride + c));
            }
            const float4 sv = V4<TI>::load(self + c);
            TO* o = out + p * out_stride;
            if (MODE == 0) {
                V4<TO>::store(o + c, sv);
                V4<TO>::store(o + dim + c, f4mul(acc, d ? 1.0f / (float)d : 0.0f));
            } else {
                V4<TO>::store(o + c, f4mul(f4add(sv, acc), 1.0f / (float)(d + 1)));
            }
        }
    }
}

// backward of the aggregation, fused with the ReLU mask of the input activations:
//   g[q] = [h[q] > 0] * ( cs(q) * dA[q, self cols]  (q < p_out)
//                       + cc(parent) * dA[parent(q), child cols]  (q has a parent) )
// SAGE: self cols [0, dim), child cols [dim, 2 dim), cs = 1, cc = 1/deg(parent)
// GCN:  both [0, dim), cs = 1/(deg(q)+1), cc = 1/(deg(parent)+1)
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_tree_aggregate_bwd(const T* __restrict__ dA, int64_t dA_stride, int dim,
                                                            const int32_t* __restrict__ parent,
                                                            const int32_t* __restrict__ cdeg, int64_t p_out,
                                                            int64_t p_in, const T* __restrict__ h, int64_t h_stride,
                                                            T* __restrict__ g, int64_t g_stride) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t q = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); q < p_in; q += warps) {
        const int32_t par = parent[q];
        float cs = 0.f, cc = 0.f;
        if (q < p_out) cs = MODE == 0 ? 1.0f : 1.0f / (float)(cdeg[q] + 1);
        if (par >= 0) cc = MODE == 0 ? 1.0f / (float)cdeg[par] : 1.0f / (float)(cdeg[par] + 1);
        const int child_col = MODE == 0 ? dim : 0;
        for (int c = lane * 4; c < dim; c += 128) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (cs != 0.f) v = f4mul(V4<T>::load(dA + q * dA_stride + c), cs);
            if (cc != 0.f) v = f4add(v, f4mul(V4<T>::load(dA + (int64_t)par * dA_stride + child_col + c), cc));
            if (h) {
                const float4 a = V4<T>::load(h + q * h_stride + c);
                v.x = a.x > 0.f ? v.x : 0.f;
                v.y = a.y > 0.f ? v.y : 0.f;
                v.z = a.z > 0.f ? v.z : 0.f;
                v.w = a.w > 0.f ? v.w : 0.f;
            }
            V4<T>::store(g + q * g_stride + c, v);
        }
    }
}

static inline unsigned warp_grid(int64_t rows) {
    int64_t g = (rows + 7) / 8;
    const int64_t cap = (int64_t)sm_count() * 64;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace gc

extern "C" {

int gc_tree_stage(const gc_tree_src_t* src, const int32_t* d_batch, int32_t* d_loc, int32_t* d_cbeg, int32_t* d_cdeg,
                  int32_t* d_parent, int64_t* d_labels, void* stream) {
    GC_REQUIRE(src && d_batch && d_loc && d_parent, GC_ERR_VALUE, "gc_tree_stage: null pointer");
    GC_REQUIRE(src->hops >= 0 && src->hops < GC_TREE_MAX_LEVELS, GC_ERR_VALUE, "gc_tree_stage: bad hop count");
    GC_REQUIRE(src->hops == 0 || (d_cbeg && d_cdeg), GC_ERR_VALUE, "gc_tree_stage: null child arrays");
    int64_t total = 0;
    for (int k = 0; k <= src->hops; ++k) total += src->caps[k];
    if (total == 0) return GC_OK;
    int64_t g = (total + 255) / 256;
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_tree_stage<<<(unsigned)g, 256, 0, as_stream(stream)>>>(*src, d_batch, total, d_loc, d_cbeg, d_cdeg, d_parent,
                                                            d_labels);
    GC_CHECK_LAUNCH("gc_tree_stage");
    return GC_OK;
}

int gc_tree_aggregate(const void* d_in, int in_dtype, int64_t in_stride, int dim, const int32_t* d_rowmap,
                      const int32_t* d_cbeg, const int32_t* d_cdeg, int64_t p_out, int mode, void* d_out, int out_dtype,
                      int64_t out_stride, const int32_t* d_batch, int64_t batch_rows, void* stream) {
    GC_REQUIRE(dim >= 4 && dim % 4 == 0, GC_ERR_VALUE, "gc_tree_aggregate: dim must be a multiple of 4");
    GC_REQUIRE(in_stride % 4 == 0 && out_stride % 4 == 0, GC_ERR_VALUE, "gc_tree_aggregate: strides must be multiples of 4");
    GC_REQUIRE(mode == 0 || mode == 1, GC_ERR_VALUE, "gc_tree_aggregate: mode is 0 (SAGE) or 1 (GCN)");
    GC_REQUIRE((in_dtype == 0 || in_dtype == 1) && (out_dtype == 0 || out_dtype == 1), GC_ERR_VALUE,
               "gc_tree_aggregate: dtype is 0 (fp32) or 1 (bf16)");
    if (p_out <= 0) return GC_OK;
    const unsigned g = warp_grid(p_out);
    cudaStream_t s = as_stream(stream);
#define GC_AGG(TI, TO, M)                                                                                           \
    k_tree_aggregate<TI, TO, M><<<g, 256, 0, s>>>(static_cast<const TI*>(d_in), in_stride, dim, d_rowmap, d_cbeg, \
                                                  d_cdeg, p_out, static_cast<TO*>(d_out), out_stride, d_batch,     \
                                                  batch_rows)
    using bf = __nv_bfloat16;
    if (in_dtype == 0 && out_dtype == 0) { if (mode == 0) GC_AGG(float, float, 0); else GC_AGG(float, float, 1); }
    else if (in_dtype == 0) { if (mode == 0) GC_AGG(float, bf, 0); else GC_AGG(float, bf, 1); }
    else if (out_dtype == 1) { if (mode == 0) GC_AGG(bf, bf, 0); else GC_AGG(bf, bf, 1); }
    else { if (mode == 0) GC_AGG(bf, float, 0); else GC_AGG(bf, float, 1); }
#undef GC_AGG
    GC_CHECK_LAUNCH("gc_tree_aggregate");
    return GC_OK;
}

int gc_tree_aggregate_backward(const void* d_dA, int dtype, int64_t dA_stride, int dim, int mode,
                               const int32_t* d_parent, const int32_t* d_cdeg, int64_t p_out, int64_t p_in,
                               const void* d_h, int64_t h_stride, void* d_g, int64_t g_stride, void* stream) {
    GC_REQUIRE(dim >= 4 && dim % 4 == 0, GC_ERR_VALUE, "gc_tree_aggregate_backward: dim must be a multiple of 4");
    GC_REQUIRE(mode == 0 || mode == 1, GC_ERR_VALUE, "gc_tree_aggregate_backward: mode is 0 (SAGE) or 1 (GCN)");
    GC_REQUIRE(dtype == 0 || dtype == 1, GC_ERR_VALUE, "gc_tree_aggregate_backward: dtype is 0 (fp32) or 1 (bf16)");
    GC_REQUIRE(p_out <= p_in, GC_ERR_VALUE, "gc_tree_aggregate_backward: p_out > p_in");
    if (p_in <= 0) return GC_OK;
    const unsigned g = warp_grid(p_in);
    cudaStream_t s = as_stream(stream);
#define GC_BWD(T, M)                                                                                                \
    k_tree_aggregate_bwd<T, M><<<g, 256, 0, s>>>(static_cast<const T*>(d_dA), dA_stride, dim, d_parent, d_cdeg, \
                                                 p_out, p_in, static_cast<const T*>(d_h), h_stride,              \
                                                 static_cast<T*>(d_g), g_stride)
    if (dtype == 0) { if (mode == 0) GC_BWD(float, 0); else GC_BWD(float, 1); }
    else { if (mode == 0) GC_BWD(__nv_bfloat16, 0); else GC_BWD(__nv_bfloat16, 1); }
#undef GC_BWD
    GC_CHECK_LAUNCH("gc_tree_aggregate_backward");
    return GC_OK;
}

}  // extern "C"
