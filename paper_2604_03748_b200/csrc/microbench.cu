// microbench.cu — the sampler's own ceiling (SURVEY §8(d) "Denominators": L1/TEX measured per
// layout by a microbenchmark that runs the kernel's exact sample code over warp-coherent
// positions inside an L1-resident 16^3 volume).  Every thread runs light_sum (sampler.cuh, the
// march's light loop: FMUL + 3 FFMA positions, occupancy test, one gather, trilinear) over a
// 16-sample line that stays inside a fully occupied volume, repeated; a warp's 32 rays sit on
// the march's 8 x 4 footprint at a 0.25-voxel pixel pitch.  The result is the peak rate at
// which this sampler can deliver occupied samples when nothing else limits it.
#include "sampler.cuh"

namespace nsl {
namespace {

constexpr int kMbThreads = 128, kMbLine = 16;

template <int LAYOUT>
__global__ void __launch_bounds__(kMbThreads) l1_gather_kernel(Vol v, int reps, float* __restrict__ sink) {
    const int lane = threadIdx.x & 31, warp = (int)((blockIdx.x * kMbThreads + threadIdx.x) >> 5);
    // ray base inside [2, 6)^3 (the 16-sample line of length 16 * 0.55 = 8.8 stays below 15)
    float ux = 2.0f + 0.25f * (float)(lane % 8) + 0.125f * (float)(warp % 16);
    float uy = 2.0f + 0.25f * (float)(lane / 8) + 0.125f * (float)((warp / 16) % 16);
    const float uz = 2.0f + 0.0625f * (float)((warp / 256) % 32);
    const float lx = 0.6f, ly = 0.48f, lz = 0.64f, hl = 0.55f;    // |L| = 1
    uint32_t g = 0;
    float acc = 0.0f;
    for (int r = 0; r < reps; ++r) {
        acc += light_sum<LAYOUT, false>(v, ux, uy, uz, lx, ly, lz, hl, kMbLine, g);
        ux += 1.0f / 1024.0f;          // loop-carried, so the line is not hoisted out
        uy += 1.0f / 2048.0f;
    }
    sink[blockIdx.x * kMbThreads + threadIdx.x] = acc;
}

// Hardware L1/TEX gather ceiling (no sampler arithmetic): every lane issues 16 x reps
// ld.global.nc.v8.f32 -- one 32-B element each, the OCT gather's width -- at element offsets
// lane_off[k][lane] from buf + shift_r (shift_r = r * stride mod span), summing the eight
// floats.  Per load: one IMAD.WIDE, the LDG.256 and seven FADDs (all eight floats used).  With stride 0 every load of
// the launch hits the same few L1-resident lines: the L1 data path's own rate for the lane
// pattern in lane_off.
constexpr int kPkThreads = 256, kPkPat = 16;

__global__ void __launch_bounds__(kPkThreads) l1_peak_kernel(const float* __restrict__ buf,
                                                             const int* __restrict__ lane_off, long long stride,
                                                             long long span, int reps, float* __restrict__ sink) {
    const int lane = threadIdx.x & 31;
    int off[kPkPat];
#pragma unroll
    for (int k = 0; k < kPkPat; ++k) off[k] = __ldg(lane_off + k * 32 + lane);
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    long long shift = 0;
    for (int r = 0; r < reps; ++r) {
        const float* base = buf + 8 * shift;
#pragma unroll
        for (int k0 = 0; k0 < kPkPat; k0 += 4) {       // 4 independent loads in flight per thread
            float v[4][8];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=f"(v[q][0]), "=f"(v[q][1]), "=f"(v[q][2]), "=f"(v[q][3]), "=f"(v[q][4]),
                               "=f"(v[q][5]), "=f"(v[q][6]), "=f"(v[q][7])
                             : "l"(base + 8 * off[k0 + q]));
            // all eight floats are consumed (else ptxas narrows the 256-bit load's register write)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                acc[q] += ((v[q][0] + v[q][1]) + (v[q][2] + v[q][3])) + ((v[q][4] + v[q][5]) + (v[q][6] + v[q][7]));
        }
        shift += stride;
        if (shift >= span) shift -= span;
    }
    sink[(size_t)blockIdx.x * kPkThreads + threadIdx.x] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// Hardware trilinear filtering of a float 3-D texture at index-space positions (the
// paper's "3D texture", filtered by the texture unit): one thread per position.
__global__ void tex_filter_kernel(cudaTextureObject_t t, const float* __restrict__ pos, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // padded index u = texel coordinate + 1/2 (texel c of the padded array holds padded voxel c,
    // sampled at its centre c + 1/2 in unnormalised texture coordinates)
    out[i] = tex3D<float>(t, pos[3 * i] + 0.5f, pos[3 * i + 1] + 0.5f, pos[3 * i + 2] + 0.5f);
}

}  // namespace

cudaError_t launch_tex_filter(cudaTextureObject_t t, const float* pos, int n, float* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    tex_filter_kernel<<<(n + 255) / 256, 256, 0, s>>>(t, pos, n, out);
    return cudaGetLastError();
}

int l1_peak_threads() { return kPkThreads; }
int l1_peak_patterns() { return kPkPat; }
int l1_peak_max_blocks_per_sm() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_peak_kernel, kPkThreads, 0);
    return n;
}
cudaError_t launch_l1_peak(const float* buf, const int* lane_off, long long stride, long long span, int blocks,
                           int reps, float* sink, cudaStream_t s) {
    l1_peak_kernel<<<blocks, kPkThreads, 0, s>>>(buf, lane_off, stride, span, reps, sink);
    return cudaGetLastError();
}

int l1_gather_threads() { return kMbThreads; }
int l1_gather_line() { return kMbLine; }

cudaError_t launch_l1_gather(const FrameParams& p, int blocks, int reps, float* sink, cudaStream_t s) {
    Vol v;
    v.data = p.data;
    v.occ = p.occ;
    v.sy = p.sy;
    v.sz = p.sz;
    v.shift = p.occ_shift;
    v.nbx = p.occ_nbx;
    v.nby = p.occ_nby;
    v.sx1 = p.supp[0];
    v.sy1 = p.supp[1];
    v.sz1 = p.supp[2];
    v.mask_words = p.slab_off;
    switch (p.layout) {
        case kLinearF32: l1_gather_kernel<kLinearF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kQuadF32: l1_gather_kernel<kQuadF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kCornerF16: l1_gather_kernel<kCornerF16><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kOctF32: l1_gather_kernel<kOctF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kBrickOctF32: l1_gather_kernel<kBrickOctF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kTex3dF32: l1_gather_kernel<kTex3dF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        case kMortonOctF32: l1_gather_kernel<kMortonOctF32><<<blocks, kMbThreads, 0, s>>>(v, reps, sink); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int l1_gather_max_blocks_per_sm(int layout) {
    int n = 0;
    switch (layout) {
        case kLinearF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kLinearF32>, kMbThreads, 0); break;
        case kQuadF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kQuadF32>, kMbThreads, 0); break;
        case kCornerF16: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kCornerF16>, kMbThreads, 0); break;
        case kOctF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kOctF32>, kMbThreads, 0); break;
        case kBrickOctF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kBrickOctF32>, kMbThreads, 0); break;
        case kTex3dF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kTex3dF32>, kMbThreads, 0); break;
        case kMortonOctF32: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, l1_gather_kernel<kMortonOctF32>, kMbThreads, 0); break;
    }
    return n;
}

}  // namespace nsl
