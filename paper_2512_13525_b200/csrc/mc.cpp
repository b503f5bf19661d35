// mc.cpp — NVLS multicast transport of the box exchange (host side).
//
// One multicast object spans every rank of the box.  Each rank binds its own
// physical backing to it and maps it twice: the multicast mapping (mc_va),
// where a store is replicated by the NVSwitch into every rank's backing and a
// multimem.ld_reduce returns the sum over every rank's backing, and a unicast
// mapping of its own backing (uc_va) for plain loads/stores.  Dispatch thus
// leaves an attention GPU once (not once per MoE GPU), and the combine's
// reduction over MoE GPUs happens in the switch.
//
// Creation order (CUDA multicast rules): rank 0 creates the object and exports
// a POSIX file descriptor; the others import it (the descriptor travels over a
// Unix socket, dist.py); every rank adds its device; only then does every rank
// bind and map its backing.  Driver entry points are resolved through the
// runtime (no libcuda link dependency).
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>

#include "internal.h"

namespace janus {
namespace {

struct Drv {
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceGetAttribute = nullptr;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemGetAllocationGranularity) memGranularity = nullptr;
  decltype(&cuMemAddressReserve) addressReserve = nullptr;
  decltype(&cuMemAddressFree) addressFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  bool ok = false;
};

template <class F>
bool resolve(F &f, const char *name) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  f = reinterpret_cast<F>(p);
  return true;
}

const Drv &drv() {
  static Drv d = [] {
    Drv x;
    x.ok = resolve(x.deviceGet, "cuDeviceGet") &&
           resolve(x.deviceGetAttribute, "cuDeviceGetAttribute") &&
           resolve(x.mcCreate, "cuMulticastCreate") &&
           resolve(x.mcAddDevice, "cuMulticastAddDevice") &&
           resolve(x.mcBindMem, "cuMulticastBindMem") &&
           resolve(x.mcUnbind, "cuMulticastUnbind") &&
           resolve(x.mcGranularity, "cuMulticastGetGranularity") &&
           resolve(x.memCreate, "cuMemCreate") && resolve(x.memRelease, "cuMemRelease") &&
           resolve(x.memGranularity, "cuMemGetAllocationGranularity") &&
           resolve(x.addressReserve, "cuMemAddressReserve") &&
           resolve(x.addressFree, "cuMemAddressFree") && resolve(x.memMap, "cuMemMap") &&
           resolve(x.memUnmap, "cuMemUnmap") && resolve(x.memSetAccess, "cuMemSetAccess") &&
           resolve(x.exportHandle, "cuMemExportToShareableHandle") &&
           resolve(x.importHandle, "cuMemImportFromShareableHandle");
    return x;
  }();
  return d;
}

std::string cu_err(const char *what, CUresult r) {
  return std::string("xfer multicast: ") + what + " failed (CUresult " + std::to_string((int)r) +
         ")";
}

#define CU_TRY(call, what)                      \
  do {                                          \
    CUresult r_ = (call);                       \
    if (r_ != CUDA_SUCCESS) return cu_err(what, r_); \
  } while (0)

size_t up(size_t v, size_t a) { return (v + a - 1) / a * a; }

CUmemAllocationProp backing_prop(int device) {
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return ap;
}

CUmulticastObjectProp mc_prop(const XferState &x) {
  CUmulticastObjectProp p{};
  p.numDevices = (unsigned)x.world;
  p.size = x.mc_bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  p.flags = 0;
  return p;
}

// Region layout (identical on every rank) and its size rounded to both the
// multicast and the allocation granularity.
std::string plan_layout(XferState &x, int device) {
  const Drv &d = drv();
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = up(o + bytes, 256);
    return at;
  };
  x.mx_off = take((size_t)x.T_max * x.d_h * 2);
  x.mex_off = take((size_t)x.T_max * x.k * 4);
  x.mgw_off = take((size_t)x.T_max * x.k * 4);
  x.mpart_off = take((size_t)x.T_max * x.d_h * 2);
  x.mslot = o;  // kXferSlots slots: epoch % kXferSlots
  x.mc_bytes = kXferSlots * o;
  CUmulticastObjectProp mp = mc_prop(x);
  size_t g1 = 0, g2 = 0;
  CU_TRY(d.mcGranularity(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "granularity");
  CUmemAllocationProp ap = backing_prop(device);
  CU_TRY(d.memGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "alloc granularity");
  size_t g = g1 > g2 ? g1 : g2;
  if (g % g1 || g % g2) g = g1 * g2;
  x.mc_gran = g;
  x.mc_bytes = up(x.mc_bytes, g);
  return {};
}

}  // namespace

bool mc_supported(int device) {
  const Drv &d = drv();
  if (!d.ok) return false;
  CUdevice dev;
  if (d.deviceGet(&dev, device) != CUDA_SUCCESS) return false;
  int mc = 0, fd = 0;
  d.deviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  d.deviceGetAttribute(&fd, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  return mc && fd;
}

std::string mc_create(XferState &x, int device, int *fd) {
  const Drv &d = drv();
  if (!mc_supported(device)) return "xfer multicast: not supported on this device";
  std::string e = plan_layout(x, device);
  if (!e.empty()) return e;
  CUmulticastObjectProp mp = mc_prop(x);
  CUmemGenericAllocationHandle h;
  CU_TRY(d.mcCreate(&h, &mp), "cuMulticastCreate");
  x.mc_handle = h;
  int f = -1;
  CU_TRY(d.exportHandle(&f, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "export handle");
  CUdevice dev;
  CU_TRY(d.deviceGet(&dev, device), "cuDeviceGet");
  CU_TRY(d.mcAddDevice(h, dev), "cuMulticastAddDevice");
  *fd = f;
  return {};
}

std::string mc_join(XferState &x, int device, int fd) {
  const Drv &d = drv();
  if (!mc_supported(device)) return "xfer multicast: not supported on this device";
  std::string e = plan_layout(x, device);
  if (!e.empty()) return e;
  CUmemGenericAllocationHandle h;
  CU_TRY(d.importHandle(&h, reinterpret_cast<void *>(static_cast<intptr_t>(fd)),
                        CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
         "import handle");
  x.mc_handle = h;
  CUdevice dev;
  CU_TRY(d.deviceGet(&dev, device), "cuDeviceGet");
  CU_TRY(d.mcAddDevice(h, dev), "cuMulticastAddDevice");
  return {};
}

std::string mc_bind(XferState &x, int device) {
  const Drv &d = drv();
  if (!x.mc_handle) return "xfer multicast: create/join first";
  CUmemAllocationProp ap = backing_prop(device);
  CUmemGenericAllocationHandle mem;
  CU_TRY(d.memCreate(&mem, x.mc_bytes, &ap, 0), "cuMemCreate");
  x.mem_handle = mem;
  {
    CUresult r = d.mcBindMem(x.mc_handle, 0, mem, 0, x.mc_bytes, 0);
    if (r != CUDA_SUCCESS)
      return cu_err("cuMulticastBindMem", r) + " bytes=" + std::to_string(x.mc_bytes) +
             " gran=" + std::to_string(x.mc_gran);
  }
  x.mc_bound = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr va;
  CU_TRY(d.addressReserve(&va, x.mc_bytes, x.mc_gran, 0, 0), "reserve (multicast)");
  x.mc_va = va;
  CU_TRY(d.memMap(va, x.mc_bytes, 0, x.mc_handle, 0), "map (multicast)");
  CU_TRY(d.memSetAccess(va, x.mc_bytes, &acc, 1), "access (multicast)");
  CU_TRY(d.addressReserve(&va, x.mc_bytes, x.mc_gran, 0, 0), "reserve (unicast)");
  x.uc_va = va;
  CU_TRY(d.memMap(va, x.mc_bytes, 0, mem, 0), "map (unicast)");
  CU_TRY(d.memSetAccess(va, x.mc_bytes, &acc, 1), "access (unicast)");
  // partial-sum rows of ranks that never write them (attention ranks) must read 0
  if (cudaMemset(reinterpret_cast<void *>(x.uc_va), 0, x.mc_bytes) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return "xfer multicast: zeroing the backing failed";
  x.mc = true;
  return {};
}

void mc_free(XferState &x, int device) {
  const Drv &d = drv();
  if (!d.ok) return;
  cudaDeviceSynchronize();
  if (x.uc_va) {
    d.memUnmap(x.uc_va, x.mc_bytes);
    d.addressFree(x.uc_va, x.mc_bytes);
  }
  if (x.mc_va) {
    d.memUnmap(x.mc_va, x.mc_bytes);
    d.addressFree(x.mc_va, x.mc_bytes);
  }
  if (x.mc_bound) {
    CUdevice dev;
    if (d.deviceGet(&dev, device) == CUDA_SUCCESS) d.mcUnbind(x.mc_handle, dev, 0, x.mc_bytes);
  }
  if (x.mem_handle) d.memRelease(x.mem_handle);
  if (x.mc_handle) d.memRelease(x.mc_handle);
  x.mc = x.mc_bound = false;
  x.mc_va = x.uc_va = 0;
  x.mem_handle = x.mc_handle = 0;
}

}  // namespace janus
