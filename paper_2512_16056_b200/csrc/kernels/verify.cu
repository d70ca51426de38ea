// verify.cu — C4: the seeded offset-unique pattern on the device (SURVEY §8(c) "Input
// generator"), so multi-GiB copies are checked without a device->host round trip.
//
// Word w of the stream for `seed` = splitmix64((seed << 40) ^ w), little endian. This is an
// independent device implementation of the counter-based generator; the host side
// (mma_inputs) has its own. Stream byte o lives in word o / 8 at byte o % 8.
#include <cuda_runtime.h>
#include <stdint.h>

namespace mma {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint8_t stream_byte(uint64_t seed, uint64_t o)
{
    return (uint8_t)(splitmix64((seed << 40) ^ (o >> 3)) >> (8 * (o & 7)));
}

// Each thread owns whole stream words; the first and last partial words go byte by byte.
__global__ void fill_kernel(uint8_t* p, uint64_t bytes, uint64_t seed, uint64_t offset)
{
    const uint64_t head = ((8 - (offset & 7)) & 7) < bytes ? ((8 - (offset & 7)) & 7) : bytes;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    if (tid < head) p[tid] = stream_byte(seed, offset + tid);
    const uint64_t nwords = (bytes - head) >> 3;
    const uint64_t w0 = (offset + head) >> 3;
    uint8_t* q = p + head;
    const bool aligned = (reinterpret_cast<uintptr_t>(q) & 7) == 0;
    for (uint64_t w = tid; w < nwords; w += nthr) {
        const uint64_t val = splitmix64((seed << 40) ^ (w0 + w));
        if (aligned) reinterpret_cast<uint64_t*>(q)[w] = val;
        else for (int b = 0; b < 8; b++) q[8 * w + b] = (uint8_t)(val >> (8 * b));
    }
    const uint64_t done = head + (nwords << 3);
    if (tid < bytes - done) p[done + tid] = stream_byte(seed, offset + done + tid);
}

__device__ __forceinline__ unsigned diff_bytes(uint64_t a, uint64_t b)
{
    uint64_t x = a ^ b;
    unsigned n = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) n += ((x >> (8 * k)) & 0xff) != 0;
    return n;
}

__device__ uint64_t count_mismatch(const uint8_t* p, uint64_t bytes, uint64_t seed,
                                   uint64_t offset, uint64_t tid, uint64_t nthr)
{
    uint64_t bad = 0;
    const uint64_t head = ((8 - (offset & 7)) & 7) < bytes ? ((8 - (offset & 7)) & 7) : bytes;
    if (tid < head) bad += p[tid] != stream_byte(seed, offset + tid);
    const uint64_t nwords = (bytes - head) >> 3;
    const uint64_t w0 = (offset + head) >> 3;
    const uint8_t* q = p + head;
    const bool aligned = (reinterpret_cast<uintptr_t>(q) & 7) == 0;
    for (uint64_t w = tid; w < nwords; w += nthr) {
        const uint64_t val = splitmix64((seed << 40) ^ (w0 + w));
        uint64_t got;
        if (aligned) got = __ldcg(reinterpret_cast<const unsigned long long*>(q) + w);
        else {
            got = 0;
            for (int b = 0; b < 8; b++) got |= (uint64_t)q[8 * w + b] << (8 * b);
        }
        bad += diff_bytes(got, val);
    }
    const uint64_t done = head + (nwords << 3);
    if (tid < bytes - done) bad += p[done + tid] != stream_byte(seed, offset + done + tid);
    return bad;
}

__global__ void verify_kernel(const uint8_t* p, uint64_t bytes, uint64_t seed, uint64_t offset,
                              unsigned long long* mismatches)
{
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t bad = count_mismatch(p, bytes, seed, offset, tid, nthr);
    if (bad) atomicAdd(mismatches, (unsigned long long)bad);
}

// one CTA per segment (grid-stride over segments)
__global__ void verify_segments_kernel(const uint64_t* dst, const uint64_t* off, const uint64_t* len,
                                       uint64_t nsegs, uint64_t seed, unsigned long long* mismatches)
{
    uint64_t bad = 0;
    for (uint64_t k = blockIdx.x; k < nsegs; k += gridDim.x)
        bad += count_mismatch(reinterpret_cast<const uint8_t*>(dst[k]), len[k], seed, off[k],
                              threadIdx.x, blockDim.x);
    if (bad) atomicAdd(mismatches, (unsigned long long)bad);
}

static unsigned grid_for(uint64_t bytes)
{
    uint64_t g = (bytes / 8 + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}

cudaError_t launch_fill(void* p, uint64_t bytes, uint64_t seed, uint64_t offset, cudaStream_t s)
{
    if (!bytes) return cudaSuccess;
    fill_kernel<<<grid_for(bytes), 256, 0, s>>>((uint8_t*)p, bytes, seed, offset);
    return cudaGetLastError();
}

cudaError_t launch_verify(const void* p, uint64_t bytes, uint64_t seed, uint64_t offset,
                          uint64_t* mismatches, cudaStream_t s)
{
    if (!bytes) return cudaSuccess;
    verify_kernel<<<grid_for(bytes), 256, 0, s>>>((const uint8_t*)p, bytes, seed, offset,
                                                   (unsigned long long*)mismatches);
    return cudaGetLastError();
}

cudaError_t launch_verify_segments(const uint64_t* dst, const uint64_t* off, const uint64_t* len,
                                   uint64_t nsegs, uint64_t seed, uint64_t* mismatches, cudaStream_t s)
{
    if (!nsegs) return cudaSuccess;
    unsigned g = nsegs < 148 * 8 ? (unsigned)nsegs : 148 * 8;
    verify_segments_kernel<<<g, 256, 0, s>>>(dst, off, len, nsegs, seed, (unsigned long long*)mismatches);
    return cudaGetLastError();
}

}  // namespace mma
