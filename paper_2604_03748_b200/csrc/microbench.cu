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

}  // namespace

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
    }
    return n;
}

}  // namespace nsl
