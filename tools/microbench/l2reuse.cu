// L2 write-back behaviour on B200 (design tool for the scratch footprint of the per-window kernels):
// kernel A writes an S-byte buffer (16-B stores), kernel B overwrites it, kernel C reads it; run under
//   ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum
// to see whether overwriting dirty L2-resident lines costs HBM writes, for S from 8 MB to 96 MB.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wr(uint4* p, size_t n, unsigned v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
__global__ void rd(const uint4* p, size_t n, unsigned* out) {
  unsigned a = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a ^= __ldcg(&p[i].x);
  if (a == 0x12345678) *out = a;
}
__global__ void discard(const char* p, size_t bytes) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes / 128; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p + i * 128) : "memory");
}
int main() {
  uint4* buf;
  unsigned* out;
  cudaMalloc(&buf, 256 << 20);
  cudaMalloc(&out, 4);
  for (size_t mb : {8, 16, 32, 48, 64, 96}) {
    size_t n = (mb << 20) / 16;
    wr<<<592, 256>>>(buf, n, 1);       // A: first write
    wr<<<592, 256>>>(buf, n, 2);       // B: overwrite
    rd<<<592, 256>>>(buf, n, out);     // C: read back
    discard<<<592, 256>>>((const char*)buf, mb << 20);
    wr<<<592, 256>>>(buf + (128 << 16), (64 << 20) / 16, 3);  // D: unrelated 64 MB write (evicts)
    cudaDeviceSynchronize();
    printf("size %zu MB done\n", mb);
  }
  return 0;
}
