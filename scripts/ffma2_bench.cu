#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk(float a, float b){uint64_t r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ float2 up(uint64_t r){float2 v; asm("mov.b64 {%0,%1}, %2;":"=f"(v.x),"=f"(v.y):"l"(r)); return v;}
// complex mul a*w with f32x2: (a.x,a.y)*(w.x,w.x) + (a.y,a.x)*(-w.y,w.y)
__global__ void cm(float2* a, const float2* w, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    float2 x = a[i], y = w[i];
    uint64_t xa = pk(x.x, x.y), xs = pk(x.y, x.x), wr = pk(y.x, y.x), wi = pk(-y.y, y.y), z;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(xa), "l"(wr));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(z) : "l"(xs), "l"(wi));
    a[i] = up(z);
}
template<int MODE>
__global__ void thr(float* out, float s, int iters) {
    float a0=threadIdx.x, a1=a0+1, a2=a0+2,a3=a0+3,a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
    float b0=a0*0.5f,b1=a1*0.5f,b2=a2*.5f,b3=a3*.5f,b4=a4*.5f,b5=a5*.5f,b6=a6*.5f,b7=a7*.5f;
    if (MODE==0) {
      for(int i=0;i<iters;i++){
        #pragma unroll
        for(int j=0;j<8;j++){ a0=a0*s+b0; b0=b0*s+a0; a1=a1*s+b1; b1=b1*s+a1; a2=a2*s+b2; b2=b2*s+a2; a3=a3*s+b3; b3=b3*s+a3;
          a4=a4*s+b4; b4=b4*s+a4; a5=a5*s+b5; b5=b5*s+a5; a6=a6*s+b6; b6=b6*s+a6; a7=a7*s+b7; b7=b7*s+a7;}
      }
    } else {
      uint64_t p0=pk(a0,a1),p1=pk(a2,a3),p2=pk(a4,a5),p3=pk(a6,a7),q0=pk(b0,b1),q1=pk(b2,b3),q2=pk(b4,b5),q3=pk(b6,b7),ss=pk(s,s);
      for(int i=0;i<iters;i++){
        #pragma unroll
        for(int j=0;j<8;j++){
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(p0):"l"(ss),"l"(q0));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(q0):"l"(ss),"l"(p0));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(p1):"l"(ss),"l"(q1));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(q1):"l"(ss),"l"(p1));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(p2):"l"(ss),"l"(q2));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(q2):"l"(ss),"l"(p2));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(p3):"l"(ss),"l"(q3));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;":"+l"(q3):"l"(ss),"l"(p3));
        }
      }
      float2 u0=up(p0),u1=up(p1),u2=up(p2),u3=up(p3),v0=up(q0),v1=up(q1),v2=up(q2),v3=up(q3);
      a0=u0.x;a1=u0.y;a2=u1.x;a3=u1.y;a4=u2.x;a5=u2.y;a6=u3.x;a7=u3.y;b0=v0.x;b1=v0.y;b2=v1.x;b3=v1.y;b4=v2.x;b5=v2.y;b6=v3.x;b7=v3.y;
    }
    out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7+b0+b1+b2+b3+b4+b5+b6+b7;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*1024*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=4096;
  for(int mode=0;mode<2;mode++) for(int rep=0;rep<3;rep++){
    cudaEventRecord(e0);
    if(mode==0) thr<0><<<148*8,1024/4*4>>>(o,0.999f,iters); else thr<1><<<148*8,1024>>>(o,0.999f,iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fmas = 148.0*8*1024*iters*8*16; // scalar fma count per thread: 8*16 per iter (both modes)
    printf("mode %d: %.3f ms, %.1f TFMA/s (scalar fma equivalents)\n", mode, ms, fmas/ms/1e9);
  }
  return 0;
}
