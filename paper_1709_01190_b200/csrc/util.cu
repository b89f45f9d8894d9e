// util.cu — launch helpers shared by the kernel launchers of libflash.so.
#include <mutex>
#include <utility>
#include <map>

#include "flash_internal.cuh"

namespace flash {

// cudaFuncSetAttribute is per device: one process may drive several GPUs (one handle per
// device), so the largest dynamic shared-memory size set so far is cached per
// (kernel, device).  Returns false if the attribute could not be set.
bool ensure_smem_attr(const void* func, size_t bytes, bool carveout_max) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{func, dev}];
  if (bytes <= have && have) return true;
  if (bytes > 48 * 1024 &&
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (carveout_max) cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  have = bytes > have ? bytes : have;
  if (!have) have = 1;
  return true;
}

// Streaming-multiprocessor count of the current device (148 on B200), cached per device:
// persistent grids are sized as a multiple of it.
uint32_t device_sms() {
  static std::mutex mu;
  static std::map<int, uint32_t> sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 148;
  }
  sms[dev] = (uint32_t)n;
  return (uint32_t)n;
}

}  // namespace flash
