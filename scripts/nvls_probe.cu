// nvls_probe.cu -- does this box support CUDA multicast objects (NVLS)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
typedef CUresult (*GetAttr)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*McGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
int main() {
  int n = 0; cudaGetDeviceCount(&n);
  void* fa = nullptr; void* fg = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fa, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMulticastGetGranularity", &fg, cudaEnableDefault, &q);
  for (int d = 0; d < n; ++d) {
    int mc = -1, fabric = -1, posix = -1;
    ((GetAttr)fa)(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    ((GetAttr)fa)(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    ((GetAttr)fa)(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, d);
    printf("device %d multicast=%d fabric_handles=%d posix_fd_handles=%d\n", d, mc, fabric, posix);
  }
  CUmulticastObjectProp p = {}; p.numDevices = n; p.size = 64 << 20; p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0; CUresult r = ((McGran)fg)(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  printf("multicast granularity rc=%d recommended=%zu\n", (int)r, g);
  return 0;
}
