// Trainer helper kernels: the GraphSAGE mean aggregation straight from the gathered
// feature rows. For the first layer the children of a tree level are rows of the
// batch's feature matrix X[U, D] named by their relabelled ids, so
//   agg[i] = mean_{k in [off[i], off[i+1])} X[idx[k]]
// is computed without materialising X[idx] (at C2 that is 768K x 100 fp32 per batch).
// Warp per segment, lanes over the feature dimension (float4 when D % 4 == 0); the
// sum runs in child order, as torch.segment_reduce's does, in fp32.
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
