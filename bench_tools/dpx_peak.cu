// Phase-0 microbenchmark: issue rate of the (min,+) candidate instruction mixes on sm_100a.
// SURVEY.md §8(d) "Establishing the DPX roofline (phase 0)". Not part of the product path.
// Each thread runs 16 independent accumulator chains over register operands that rotate
// every outer iteration, so no chain can be simplified. Reports (min,+) steps/s per mix,
// where one step = one add + one min on one 16-bit lane.
#include <cstdio>
#include <cstdint>
#define CHECK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ unsigned dpx(unsigned a, unsigned b, unsigned c){ return __viaddmin_u16x2(a,b,c); }
// packed add on the FMA pipe: IMAD d = a*one + b (one==1 at run time; ptxas cannot fold it)
__device__ __forceinline__ unsigned imad(unsigned a, unsigned one, unsigned b){ unsigned d; asm("mad.lo.u32 %0,%1,%2,%3;":"=r"(d):"r"(a),"r"(one),"r"(b)); return d; }
__device__ __forceinline__ unsigned iadd(unsigned a, unsigned b){ unsigned d; asm("add.u32 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d; }
__device__ __forceinline__ unsigned vmin(unsigned a, unsigned b){ unsigned d; asm("min.u16x2 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d; }
__device__ __forceinline__ unsigned hadd(unsigned a, unsigned b){ unsigned d; asm("add.rn.f16x2 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d; }
__device__ __forceinline__ unsigned hmin(unsigned a, unsigned b){ unsigned d; asm("min.f16x2 %0,%1,%2;":"=r"(d):"r"(a),"r"(b)); return d; }

// MODE 0: DPX only (2 steps / op)
// MODE 1: IMAD,IMAD,VIMNMX3 (4 steps / group)
// MODE 2: half DPX, half IMAD-group
// MODE 3: IADD,IADD,VIMNMX3 (adds on ALU)
// MODE 4: HADD2,HADD2,HMNMX2 x2 -> fp16 pipe probe (4 steps / group)
// MODE 5: 1/3 IMAD-group + 2/3 DPX
template<int MODE>
__global__ void __launch_bounds__(256) bench(const unsigned* __restrict__ in, unsigned* out, int iters){
  unsigned acc[16], xa[16], xb[16], ya[16], yb[16];
  const unsigned one = in[255] ;  // == 1
  #pragma unroll
  for(int i=0;i<16;i++){
    acc[i]=in[(i*7+threadIdx.x)&127];
    xa[i]=in[(i*13+threadIdx.x+5)&127]; xb[i]=in[(i*11+threadIdx.x+9)&127];
    ya[i]=in[(i*17+threadIdx.x+1)&127]; yb[i]=in[(i*19+threadIdx.x+3)&127];
  }
  for(int t=0;t<iters;t++){
    #pragma unroll
    for(int r=0;r<8;r++){
      #pragma unroll
      for(int i=0;i<16;i++){
        // every (a,b) pair is distinct within an outer iteration: no CSE possible
        unsigned a=xa[i], b=xb[(i+r)&15], a2=ya[i], b2=yb[(i+r)&15];
        bool g = (MODE==1)||(MODE==3)||(MODE==4)||(MODE==2 && (i&1))||(MODE==5 && (i%3)==0);
        if (!g) acc[i]=dpx(a,b,acc[i]);
        else if (MODE==3) acc[i]=vmin(vmin(acc[i],iadd(a,b)),iadd(a2,b2));
        else if (MODE==4) acc[i]=hmin(hmin(acc[i],hadd(a,b)),hadd(a2,b2));
        else acc[i]=vmin(vmin(acc[i],imad(a,one,b)),imad(a2,one,b2));
      }
    }
    #pragma unroll
    for(int r=0;r<16;r++){ xa[r] ^= ((unsigned)t & 0x00010001u); yb[r] ^= ((unsigned)t & 0x00010001u); }
  }
  unsigned s=0;
  #pragma unroll
  for(int i=0;i<16;i++) s^=acc[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

template<int MODE>
int run(const char* name, double steps_per_thread_iter, unsigned* din, unsigned* dout, int nsm, int occ){
  int grid=nsm*occ, block=256, iters=20000;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  bench<MODE><<<grid,block>>>(din,dout,100); CHECK(cudaDeviceSynchronize());
  float best=1e30f;
  for(int rep=0;rep<5;rep++){
    cudaEventRecord(e0);
    bench<MODE><<<grid,block>>>(din,dout,iters);
    cudaEventRecord(e1); CHECK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;
  }
  double steps=(double)grid*block*iters*steps_per_thread_iter;
  printf("{\"mode\":\"%s\",\"occ\":%d,\"ms\":%.3f,\"Tsteps_per_s\":%.3f}\n",name,occ,best,steps/(best*1e-3)/1e12);
  fflush(stdout);
  return 0;
}

int main(){
  int nsm; cudaDeviceGetAttribute(&nsm,cudaDevAttrMultiProcessorCount,0);
  unsigned *din,*dout; CHECK(cudaMalloc(&din,4096)); CHECK(cudaMalloc(&dout,(size_t)nsm*8*256*4));
  unsigned h[256]; for(int i=0;i<256;i++) h[i]=(0x0003u*(i%97+1))|((0x0005u*(i%89+1))<<16);
  h[255]=1;
  CHECK(cudaMemcpy(din,h,1024,cudaMemcpyHostToDevice));
  int clk; cudaDeviceGetAttribute(&clk,cudaDevAttrClockRate,0);
  printf("{\"sms\":%d,\"clock_khz\":%d}\n",nsm,clk);
  // steps per thread per outer iteration: 8 r * 16 acc * steps/acc-update
  for(int occ: {2,4,8}) run<0>("dpx_u16x2",8*16*2,din,dout,nsm,occ);
  run<1>("imad_imad_vimnmx3",8*16*4,din,dout,nsm,4);
  run<1>("imad_imad_vimnmx3",8*16*4,din,dout,nsm,8);
  run<2>("half_dpx_half_imadgrp",8*8*2+8*8*4,din,dout,nsm,4);
  run<2>("half_dpx_half_imadgrp",8*8*2+8*8*4,din,dout,nsm,8);
  run<5>("twothird_dpx_third_imadgrp",8*(6*4+10*2),din,dout,nsm,8);
  run<3>("iadd_iadd_vimnmx3",8*16*4,din,dout,nsm,8);
  run<4>("hadd2_hadd2_hmin3",8*16*4,din,dout,nsm,8);
  return 0;
}
