// Exportable device memory (cuMemCreate) and NVLink SHARP multicast objects
// for the symmetric pool, through CUDA driver entry points resolved at run
// time (cudaGetDriverEntryPoint): the library keeps no link-time dependency
// on libcuda, so it still loads on a machine without a GPU driver.
#pragma once

#include <cuda.h>
#include <stddef.h>
#include <stdint.h>

namespace fsdp {
namespace vmm {

// handle types (values of the C ABI's FSDP_HANDLE_*)
constexpr int kFabric = 1;
constexpr int kPosixFd = 2;

struct Mapping {
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr va = 0;
  size_t bytes = 0;
  bool owns_handle = false;
};

// 1 if the driver exposes VMM + multicast on `device`, else 0.
int multicast_supported(int device);
// Allocation granularity that also satisfies the multicast granularity for a
// group of `ndev` devices (so a pool can be bound whole to a multicast object).
int granularity(int device, int htype, int ndev, size_t* out);
// cuMemCreate(bytes) on `device`, exportable as `htype`, mapped read/write.
int create(int device, size_t bytes, int htype, Mapping* out);
// 64-byte shareable handle: fabric handle bytes, or the fd in the first int.
int export_handle(CUmemGenericAllocationHandle h, int htype, void* out64);
// Import a peer's allocation and map it read/write for `device`.
int import_map(int device, const void* handle64, int htype, size_t bytes, Mapping* out);
void unmap(Mapping* m);

// Multicast object over `ndev` devices of `bytes` (granularity-rounded).
int mc_create(int ndev, size_t bytes, int htype, CUmemGenericAllocationHandle* out);
int mc_import(const void* handle64, int htype, CUmemGenericAllocationHandle* out);
int mc_add_device(CUmemGenericAllocationHandle mc, int device);
// Bind `mem` (whole) at multicast offset 0 and map the multicast VA.
int mc_bind_map(CUmemGenericAllocationHandle mc, int device, const Mapping& mem, Mapping* mc_map);
void mc_unbind(CUmemGenericAllocationHandle mc, int device, Mapping* mc_map);
void release_handle(CUmemGenericAllocationHandle h);

}  // namespace vmm
}  // namespace fsdp
