// pdl_coresidency_probe.cu -- does a programmatic dependent launch start
// beside a running primary?  A: one 512-thread CTA per SM (NR live fp32
// registers, `smem` bytes of dynamic shared memory) that triggers
// griddepcontrol.launch_dependents at once and spins 100 us; B: the
// dependent (`bthreads` threads, NB registers) records its start time.
// B starting at ~1 us means co-resident; at ~100 us, it waited for A.
// (pipelined combine: why the early reducer gets its own SMs.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o pdl_probe tools/pdl_coresidency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int NR>
__global__ void __launch_bounds__(512, 1) A(unsigned long long* ts, float* sink, int spin_us) {
  extern __shared__ char smx[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0 = gt();
  if (threadIdx.x == 0) ts[blockIdx.x * 2] = t0;
  float acc[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) acc[i] = threadIdx.x * (i + 1);
  while (gt() - t0 < (unsigned long long)spin_us * 1000) {
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = acc[i] * 1.0001f + acc[(i + 1) % NR];
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NR; ++i) s += acc[i];
  sink[blockIdx.x * 512 + threadIdx.x] = s + smx[threadIdx.x];
  if (threadIdx.x == 0) ts[blockIdx.x * 2 + 1] = gt();
}
template <int NR>
__global__ void __launch_bounds__(512, 2) B(unsigned long long* ts, float* sink) {
  if (threadIdx.x == 0) ts[blockIdx.x] = gt();
  float acc[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) acc[i] = threadIdx.x * (i + 1);
  for (int r = 0; r < 10; ++r)
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[i] = acc[i] * 1.0001f + acc[(i + 1) % NR];
  float s = 0;
#pragma unroll
  for (int i = 0; i < NR; ++i) s += acc[i];
  sink[blockIdx.x * 512 + threadIdx.x] = s;
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
template <int NA, int NB>
void run(int sms, unsigned long long* ta, unsigned long long* tb, float* sink, cudaStream_t s, int smem, int bthreads) {
  cudaFuncAttributes fa, fb;
  cudaFuncGetAttributes(&fa, (void*)A<NA>); cudaFuncGetAttributes(&fb, (void*)B<NB>);
  cudaFuncSetAttribute((void*)A<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int spin = 100;
  for (int rep = 0; rep < 3; ++rep) {
    void* aargs[] = {&ta, &sink, &spin};
    cudaLaunchKernel((void*)A<NA>, dim3(sms), dim3(512), aargs, smem, s);
    cudaLaunchConfig_t lc{}; lc.gridDim = dim3(sms); lc.blockDim = dim3(bthreads); lc.stream = s;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1; lc.attrs = at; lc.numAttrs = 1;
    void* bargs[] = {&tb, &sink};
    cudaLaunchKernelExC(&lc, (void*)B<NB>, bargs);
  }
  cudaStreamSynchronize(s);
  unsigned long long ha[2 * 148], hb[148];
  cudaMemcpy(ha, ta, sms * 16, cudaMemcpyDeviceToHost); cudaMemcpy(hb, tb, sms * 8, cudaMemcpyDeviceToHost);
  unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b1 = 0;
  for (int i = 0; i < sms; ++i) { a0 = a0 < ha[2*i] ? a0 : ha[2*i]; a1 = a1 > ha[2*i+1] ? a1 : ha[2*i+1]; b0 = b0 < hb[i] ? b0 : hb[i]; b1 = b1 > hb[i] ? b1 : hb[i]; }
  printf("A regs %3d B regs %3d smem %6d bthreads %3d: A [0, %.1f] us, B start [%.1f, %.1f] us  err=%s\n", fa.numRegs, fb.numRegs, smem, bthreads,
         (a1 - a0) / 1e3, ((long long)(b0 - a0)) / 1e3, ((long long)(b1 - a0)) / 1e3, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *ta, *tb; cudaMalloc(&ta, sms * 16); cudaMalloc(&tb, sms * 8);
  float* sink; cudaMalloc(&sink, sms * 512 * 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int bt : {32, 128}) {
    run<101, 56>(sms, ta, tb, sink, s, 223744, bt);
    run<102, 56>(sms, ta, tb, sink, s, 223744, bt);
    run<103, 56>(sms, ta, tb, sink, s, 223744, bt);
    run<101, 62>(sms, ta, tb, sink, s, 223744, bt);
    run<102, 62>(sms, ta, tb, sink, s, 223744, bt);
    run<102, 64>(sms, ta, tb, sink, s, 223744, bt);
  }
  return 0;
}
