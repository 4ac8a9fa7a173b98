// tools/fp64_latency.cu — dependent-chain latency (cycles) of the fp64 primitives the
// phase-boundary solver uses (development tool).  One thread, clock64 around 256-long chains.
#include <cstdio>
#include <cmath>

#define CHAIN(NAME, EXPR)                                               \
  {                                                                     \
    double x = seed;                                                    \
    long long t0 = clock64();                                           \
    for (int i = 0; i < 256; ++i) { x = EXPR; }                         \
    long long t1 = clock64();                                           \
    if (threadIdx.x == 0) { out[k] = x; cyc[k] = (double)(t1 - t0) / 256; } \
    ++k;                                                                \
  }

__global__ void lat(double* out, double* cyc, double seed, double ca, double cb) {
  int k = 0;
  CHAIN("dfma", fma(x, ca, cb));
  CHAIN("ddiv", 1.0000001 / x);
  CHAIN("drcp_rn", __drcp_rn(x));
  CHAIN("dsqrt", sqrt(x + 1.0));
  CHAIN("dlog", log(x + 2.0));
  CHAIN("dlog1p", log1p(x * 1e-3));
  CHAIN("dexp", exp(x * 1e-3));
  float xf = (float)seed;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) xf = logf(xf + 2.0f);
  long long t1 = clock64();
  out[k] = xf; cyc[k] = (double)(t1 - t0) / 256; ++k;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) xf = 1.0f / xf + 1e-3f;
  t1 = clock64();
  out[k] = xf; cyc[k] = (double)(t1 - t0) / 256; ++k;
}

int main() {
  double *out, *cyc;
  cudaMallocManaged(&out, 64 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  lat<<<1, 1>>>(out, cyc, 1.5, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  lat<<<1, 1>>>(out, cyc, 1.5, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  const char* names[] = {"dfma", "ddiv", "drcp_rn", "dsqrt", "dlog", "dlog1p", "dexp", "logf", "fdiv"};
  printf("{");
  for (int i = 0; i < 9; ++i) printf("\"%s\": %.1f%s", names[i], cyc[i], i < 8 ? ", " : "");
  printf("}\n");
  return 0;
}
