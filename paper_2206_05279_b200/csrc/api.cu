// Library identity and device check.
#include "common.cuh"

extern "C" const char *pilc_version(void) { return "pilc-sm100a 0.1.0"; }

extern "C" int pilc_device_arch(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return p.major * 10 + p.minor;
}
