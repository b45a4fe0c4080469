// Exportable pool memory + NVLink SHARP (NVLS) multicast objects via the CUDA
// driver's virtual-memory API, resolved through cudaGetDriverEntryPoint.
//
// Used by fsdp_comm_create_vmm / fsdp_nvls_* (comm.cu): the symmetric pool is
// one cuMemCreate allocation per rank, mapped by peers from an exported
// handle (instead of cudaMalloc + cudaIpc), and bound whole to a multicast
// object of the rank's shard group, so one multimem.st from any member lands
// in every member's pool at the same offset.
#include "vmm.h"

#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace fsdp {
namespace vmm {
namespace {

struct Driver {
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*,
                                           CUmemAllocationHandleType) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                               size_t, unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                      CUmulticastGranularity_flags) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  bool ok = false;
  std::string why;
};

template <typename F>
bool resolve(const char* name, F& fn, std::string& why) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult st;
  cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, CUDART_VERSION, cudaEnableDefault, &st);
  if (e != cudaSuccess || st != cudaDriverEntryPointSuccess || !p) {
    why = std::string("driver entry point ") + name + " unavailable";
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

Driver& drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    std::string& w = d.why;
    d.ok = resolve("cuDeviceGet", d.DeviceGet, w) &&
           resolve("cuDeviceGetAttribute", d.DeviceGetAttribute, w) &&
           resolve("cuMemGetAllocationGranularity", d.MemGetAllocationGranularity, w) &&
           resolve("cuMemCreate", d.MemCreate, w) && resolve("cuMemRelease", d.MemRelease, w) &&
           resolve("cuMemAddressReserve", d.MemAddressReserve, w) &&
           resolve("cuMemAddressFree", d.MemAddressFree, w) && resolve("cuMemMap", d.MemMap, w) &&
           resolve("cuMemUnmap", d.MemUnmap, w) && resolve("cuMemSetAccess", d.MemSetAccess, w) &&
           resolve("cuMemExportToShareableHandle", d.MemExportToShareableHandle, w) &&
           resolve("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle, w) &&
           resolve("cuMulticastCreate", d.MulticastCreate, w) &&
           resolve("cuMulticastAddDevice", d.MulticastAddDevice, w) &&
           resolve("cuMulticastBindMem", d.MulticastBindMem, w) &&
           resolve("cuMulticastUnbind", d.MulticastUnbind, w) &&
           resolve("cuMulticastGetGranularity", d.MulticastGetGranularity, w) &&
           resolve("cuGetErrorString", d.GetErrorString, w);
  });
  return d;
}

int cu_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return fail(FSDP_E_IPC, std::string(what) + ": CUresult " + std::to_string((int)r) +
                              (s ? std::string(" (") + s + ")" : std::string()));
}

#define CU_TRY(expr, what)                        \
  do {                                            \
    CUresult _r = (expr);                         \
    if (_r != CUDA_SUCCESS) return cu_fail(_r, what); \
  } while (0)

CUmemAllocationHandleType cu_htype(int htype) {
  return htype == kFabric ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
}

CUmemAllocationProp alloc_prop(int device, int htype) {
  CUmemAllocationProp p;
  std::memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = cu_htype(htype);
  return p;
}

int need_driver() {
  if (!drv().ok) return fail(FSDP_E_UNSUPPORTED, drv().why);
  return 0;
}

int map_rw(int device, CUmemGenericAllocationHandle h, size_t bytes, CUdeviceptr* va) {
  Driver& d = drv();
  CU_TRY(d.MemAddressReserve(va, bytes, 0, 0, 0), "cuMemAddressReserve");
  CUresult r = d.MemMap(*va, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) { d.MemAddressFree(*va, bytes); *va = 0; return cu_fail(r, "cuMemMap"); }
  CUmemAccessDesc a;
  std::memset(&a, 0, sizeof(a));
  a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  a.location.id = device;
  a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = d.MemSetAccess(*va, bytes, &a, 1);
  if (r != CUDA_SUCCESS) {
    d.MemUnmap(*va, bytes);
    d.MemAddressFree(*va, bytes);
    *va = 0;
    return cu_fail(r, "cuMemSetAccess");
  }
  return 0;
}

}  // namespace

int multicast_supported(int device) {
  if (!drv().ok) { set_error(drv().why); return 0; }
  CUdevice dev;
  if (drv().DeviceGet(&dev, device) != CUDA_SUCCESS) return 0;
  int mc = 0, vm = 0;
  drv().DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  drv().DeviceGetAttribute(&vm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
  if (!(mc && vm)) set_error("device reports no multicast / VMM support");
  return (mc && vm) ? 1 : 0;
}

int granularity(int device, int htype, int ndev, size_t* out) {
  if (int rc = need_driver()) return rc;
  Driver& d = drv();
  CUmemAllocationProp p = alloc_prop(device, htype);
  size_t g = 0;
  CU_TRY(d.MemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
         "cuMemGetAllocationGranularity");
  if (ndev > 0) {
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.numDevices = (unsigned)ndev;
    mp.size = g;
    mp.handleTypes = cu_htype(htype);
    size_t mg = 0;
    CU_TRY(d.MulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM),
           "cuMulticastGetGranularity");
    if (mg > g) g = (mg % g == 0) ? mg : mg * g;   // both are powers of two in practice
  }
  *out = g;
  return 0;
}

int create(int device, size_t bytes, int htype, Mapping* out) {
  if (int rc = need_driver()) return rc;
  Driver& d = drv();
  CUmemAllocationProp p = alloc_prop(device, htype);
  CUmemGenericAllocationHandle h = 0;
  CU_TRY(d.MemCreate(&h, bytes, &p, 0), "cuMemCreate(pool)");
  CUdeviceptr va = 0;
  if (int rc = map_rw(device, h, bytes, &va)) { d.MemRelease(h); return rc; }
  out->handle = h;
  out->va = va;
  out->bytes = bytes;
  out->owns_handle = true;
  return 0;
}

int export_handle(CUmemGenericAllocationHandle h, int htype, void* out64) {
  if (int rc = need_driver()) return rc;
  std::memset(out64, 0, 64);
  if (htype == kFabric) {
    CUmemFabricHandle fh;
    CU_TRY(drv().MemExportToShareableHandle(&fh, h, CU_MEM_HANDLE_TYPE_FABRIC, 0),
           "cuMemExportToShareableHandle(fabric)");
    static_assert(sizeof(fh) <= 64, "fabric handle size");
    std::memcpy(out64, &fh, sizeof(fh));
  } else {
    int fd = -1;
    CU_TRY(drv().MemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
           "cuMemExportToShareableHandle(fd)");
    std::memcpy(out64, &fd, sizeof(fd));
  }
  return 0;
}

static int import_handle(const void* handle64, int htype, CUmemGenericAllocationHandle* h) {
  if (htype == kFabric) {
    CUmemFabricHandle fh;
    std::memcpy(&fh, handle64, sizeof(fh));
    CU_TRY(drv().MemImportFromShareableHandle(h, &fh, CU_MEM_HANDLE_TYPE_FABRIC),
           "cuMemImportFromShareableHandle(fabric)");
  } else {
    int fd = -1;
    std::memcpy(&fd, handle64, sizeof(fd));
    CU_TRY(drv().MemImportFromShareableHandle(h, (void*)(uintptr_t)fd,
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
           "cuMemImportFromShareableHandle(fd)");
  }
  return 0;
}

int import_map(int device, const void* handle64, int htype, size_t bytes, Mapping* out) {
  if (int rc = need_driver()) return rc;
  CUmemGenericAllocationHandle h = 0;
  if (int rc = import_handle(handle64, htype, &h)) return rc;
  CUdeviceptr va = 0;
  if (int rc = map_rw(device, h, bytes, &va)) { drv().MemRelease(h); return rc; }
  out->handle = h;
  out->va = va;
  out->bytes = bytes;
  out->owns_handle = true;
  return 0;
}

void unmap(Mapping* m) {
  if (!drv().ok || !m) return;
  if (m->va) {
    drv().MemUnmap(m->va, m->bytes);
    drv().MemAddressFree(m->va, m->bytes);
  }
  if (m->owns_handle && m->handle) drv().MemRelease(m->handle);
  *m = Mapping();
}

int mc_create(int ndev, size_t bytes, int htype, CUmemGenericAllocationHandle* out) {
  if (int rc = need_driver()) return rc;
  CUmulticastObjectProp mp;
  std::memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)ndev;
  mp.size = bytes;
  mp.handleTypes = cu_htype(htype);
  CU_TRY(drv().MulticastCreate(out, &mp), "cuMulticastCreate");
  return 0;
}

int mc_import(const void* handle64, int htype, CUmemGenericAllocationHandle* out) {
  if (int rc = need_driver()) return rc;
  return import_handle(handle64, htype, out);
}

int mc_add_device(CUmemGenericAllocationHandle mc, int device) {
  if (int rc = need_driver()) return rc;
  CUdevice dev;
  CU_TRY(drv().DeviceGet(&dev, device), "cuDeviceGet");
  CU_TRY(drv().MulticastAddDevice(mc, dev), "cuMulticastAddDevice");
  return 0;
}

int mc_bind_map(CUmemGenericAllocationHandle mc, int device, const Mapping& mem, Mapping* mc_map) {
  if (int rc = need_driver()) return rc;
  CU_TRY(drv().MulticastBindMem(mc, 0, mem.handle, 0, mem.bytes, 0), "cuMulticastBindMem");
  CUdeviceptr va = 0;
  if (int rc = map_rw(device, mc, mem.bytes, &va)) {
    CUdevice dev;
    drv().DeviceGet(&dev, device);
    drv().MulticastUnbind(mc, dev, 0, mem.bytes);
    return rc;
  }
  mc_map->handle = mc;
  mc_map->va = va;
  mc_map->bytes = mem.bytes;
  mc_map->owns_handle = false;
  return 0;
}

void mc_unbind(CUmemGenericAllocationHandle mc, int device, Mapping* mc_map) {
  if (!drv().ok || !mc_map || !mc_map->va) return;
  drv().MemUnmap(mc_map->va, mc_map->bytes);
  drv().MemAddressFree(mc_map->va, mc_map->bytes);
  CUdevice dev;
  if (drv().DeviceGet(&dev, device) == CUDA_SUCCESS) drv().MulticastUnbind(mc, dev, 0, mc_map->bytes);
  *mc_map = Mapping();
}

void release_handle(CUmemGenericAllocationHandle h) {
  if (drv().ok && h) drv().MemRelease(h);
}

}  // namespace vmm
}  // namespace fsdp
