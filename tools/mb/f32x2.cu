#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){ u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
// MODE 0: scalar fmul+fadd (16 independent chains); 1: fma2(z)+add2 (8 chains x2); 2: plain ffma2 (8x2)
template<int MODE>
__global__ void k(float* out, int iters, float x, float y, float z){
  float acc[16]; u64 acc2[8];
  #pragma unroll
  for(int i=0;i<16;i++) acc[i]=threadIdx.x*i;
  #pragma unroll
  for(int i=0;i<8;i++) acc2[i]=pk(threadIdx.x*i, i);
  float a[16];
  #pragma unroll
  for(int i=0;i<16;i++) a[i]=x+threadIdx.x+i;
  u64 a2[8];
  #pragma unroll
  for(int i=0;i<8;i++) a2[i]=pk(a[2*i],a[2*i+1]);
  u64 b2 = pk(y, y*1.5f), z2 = pk(z, z);
  for(int it=0; it<iters; it++){
    if(MODE==0){
      #pragma unroll
      for(int i=0;i<16;i++){ float p = __fmul_rn(a[i], acc[(i+1)&15]); acc[i] = __fadd_rn(acc[i], p);} 
    } else if(MODE==1){
      #pragma unroll
      for(int i=0;i<8;i++){ u64 p = fma2(a2[i], acc2[(i+1)&7], z2); acc2[i] = add2(acc2[i], p);} 
    } else {
      #pragma unroll
      for(int i=0;i<8;i++){ acc2[i] = fma2(a2[i], acc2[(i+1)&7], acc2[i]);} 
    }
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<16;i++) s+=acc[i];
  #pragma unroll
  for(int i=0;i<8;i++){ float lo, hi; asm("mov.b64 {%0,%1}, %2;":"=f"(lo),"=f"(hi):"l"(acc2[i])); s+=lo+hi;}
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*256*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000;
  for(int mode=0; mode<3; mode++) for(int rep=0; rep<3; rep++){
    cudaEventRecord(e0);
    if(mode==0) k<0><<<148*8,256>>>(o, iters, 1.f, 2.f, -0.f); else if(mode==1) k<1><<<148*8,256>>>(o, iters, 1.f, 2.f, -0.f); else k<2><<<148*8,256>>>(o, iters, 1.f, 2.f, -0.f);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double prods = 148.0*8*256*iters*16;
    printf("mode %d: %.3f ms, %.2f Tprod/s\n", mode, ms, prods/ms/1e9);
  }
}
