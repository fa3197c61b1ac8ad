// Device-memory helpers of the C ABI, so that C / cgo / JNI callers need no CUDA headers.
#include "common.cuh"

extern "C" {

int stkg_device_alloc(void** ptr, size_t bytes) {
  return stkg::guarded([&] {
    STKG_REQUIRE(ptr, STKG_ARGUMENT, "stkg_device_alloc: null argument");
    STKG_CUDA_CHECK(cudaMalloc(ptr, bytes));
  });
}

int stkg_device_free(void* ptr) {
  return stkg::guarded([&] { STKG_CUDA_CHECK(cudaFree(ptr)); });
}

int stkg_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return stkg::guarded(
      [&] { STKG_CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); });
}

int stkg_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return stkg::guarded(
      [&] { STKG_CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}

int stkg_device_synchronize(void) {
  return stkg::guarded([&] { STKG_CUDA_CHECK(cudaDeviceSynchronize()); });
}

}  // extern "C"
