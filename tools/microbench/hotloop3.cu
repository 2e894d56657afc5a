// The V3 (sphere-only) pair-test loop of hotloop2.cu alone, for an ncu capture.
#define HOTLOOP_ONLY_V3
#include "hotloop2.cu"
int main() {
  unsigned* d; cudaMalloc(&d, 64);
  k<3, 768><<<148, 768>>>(d, 0.5f, 0.2f, 10);
  k<3, 768><<<148, 768>>>(d, 0.5f, 0.2f, 200);
  cudaDeviceSynchronize();
  return 0;
}
