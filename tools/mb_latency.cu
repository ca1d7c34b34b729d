#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_pos(double b){double r=__longlong_as_double(0x7FE0000000000000LL-__double_as_longlong(b));
#pragma unroll
for(int i=0;i<5;i++) r=fma(r,fma(-b,r,1.0),r); return fma(r,fma(-b,r,1.0),r);}
__global__ void k(double *out, long long *cyc, double x0, int mode){
  double x=x0+threadIdx.x*1e-9, y=1.0000001; __shared__ double sm[1024];
  for(int i=threadIdx.x;i<1024;i+=blockDim.x) sm[i]=1.0+i*1e-9;
  __syncthreads();
  long long t0=clock64();
  const int N=1000;
  if(mode==0){ for(int i=0;i<N;i++) x=fma(x,y,1e-9); }
  else if(mode==1){ for(int i=0;i<N;i++) x=__drcp_rn(x+1.0); }
  else if(mode==2){ for(int i=0;i<N;i++) x=rcp_pos(x+1.0); }
  else if(mode==3){ int j=threadIdx.x; for(int i=0;i<N;i++){ double v=sm[j]; j=(int)(v*1e-12)+ (j+1)%1024; x+=v;} }
  else if(mode==4){ for(int i=0;i<N;i++) x=1.0/(x+1.0); }
  long long t1=clock64();
  out[threadIdx.x]=x; if(threadIdx.x==0) cyc[0]=t1-t0;
}
int main(){ double *o; long long *c; cudaMalloc(&o,8*1024); cudaMallocManaged(&c,8);
 const char* nm[]={"dfma chain","__drcp_rn chain","rcp_pos chain","lds chain","div chain"};
 for(int m=0;m<5;m++){ for(int w: {32, 1024}){ k<<<1,w>>>(o,c,1.0,m); cudaDeviceSynchronize(); k<<<1,w>>>(o,c,1.0,m); cudaDeviceSynchronize(); printf("%-18s threads %4d: %.1f cycles/op\n",nm[m],w,c[0]/1000.0);} }
 // full-GPU
 return 0;}
