// engine.h — internal interfaces between the C ABI (api.cpp), the data plane
// (plane.cpp, api.cpp, tune.cpp), the host allocator (hostmem.cpp) and the sm_100a kernels (kernels/*.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kargs.h"

#define MMA_ERR_RELAY_TIMEOUT 2001   // sticky: a relay kernel's bounded spin expired
#define MMA_ERR_NO_MEMOPS 2002       // stream memory operations unavailable

namespace mma {

// kernels/relay.cu: H2D pull on the target (pull = true) or D2H pack on the relay
// bulk: the cp.async.bulk (TMA) form of the copy (contiguous 16-byte-aligned units)
cudaError_t launch_relay(const RelayLaunchArg& a, bool pull, unsigned grid, cudaStream_t s, bool bulk = false);
// kernels/zerocopy.cu
cudaError_t launch_zc(const ZcLaunchArg& a, unsigned grid, cudaStream_t s, bool bulk = false);
cudaError_t launch_zc_dyn(const DynLaunchArg& a, unsigned grid, cudaStream_t s);
// kernels/verify.cu
cudaError_t launch_fill(void* p, uint64_t bytes, uint64_t seed, uint64_t offset, cudaStream_t s);
cudaError_t launch_verify(const void* p, uint64_t bytes, uint64_t seed, uint64_t offset,
                          uint64_t* mismatches, cudaStream_t s);
cudaError_t launch_verify_segments(const uint64_t* dst, const uint64_t* off, const uint64_t* len,
                                   uint64_t nsegs, uint64_t seed, uint64_t* mismatches,
                                   cudaStream_t s);

// hostmem.cpp
int host_alloc(void** ptr, size_t bytes, int numa_mode, int node0);
int host_free(void* ptr);
int host_alloc_size(const void* ptr, size_t* bytes);   // cudaErrorInvalidValue: not a host_alloc base
int host_alloc_ranges(void** ptr, size_t bytes, const uint64_t* range_end, const int* node, int nranges);
int host_page_node(const void* p);
// NUMA node of each host address (2 MiB regions cached; MMA_FAKE_HOST_NODES=K (tests): node =
// (address >> 21) mod K); -1 = unknown
void host_nodes(const void* const* p, size_t n, int* nodes);
int host_numa_count();
// NUMA node of a GPU's PCI device from sysfs (-1 = unknown)
int gpu_numa_node(int dev);
// plane.cpp: the CUDA device behind engine GPU index g (identity unless MMA_VGPUS)
int phys_dev(int g);

}  // namespace mma
