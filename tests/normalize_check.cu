// normalize_angle_2pi fast paths vs the reference form fmod / +2pi / reset
// (raycast.hpp:20-25), bit for bit on the device; run by tests/test_gpu_normalize.py.
#include <cstdio>
#include <cmath>
#include <cstdint>
#include "../paper_1705_01167_b200/csrc/cddt_device.cuh"
__device__ double ref_norm(double t){ t = fmod(t, rl::kTwoPi); if (t<0) t += rl::kTwoPi; if (t >= rl::kTwoPi) t = 0.0; return t; }
__global__ void k(unsigned long long* bad, uint64_t seed, int iters){
  uint64_t s = seed + blockIdx.x*blockDim.x + threadIdx.x;
  for (int i=0;i<iters;i++){
    s = s*6364136223846793005ull + 1442695040888963407ull;
    double u = double(s>>11)*0x1.0p-53;
    double t;
    int mode = (s>>3)&7;
    if (mode==0) t = (u-0.5)*8*rl::kTwoPi;
    else if (mode==1) t = rl::kTwoPi + (u-0.5)*1e-12;
    else if (mode==2) t = -rl::kTwoPi + (u-0.5)*1e-12;
    else if (mode==3) t = 2*rl::kTwoPi + (u-0.5)*1e-12;
    else if (mode==4) t = (u-0.5)*1e-300;
    else if (mode==5) t = __longlong_as_double((long long)(s ^ (s<<17)));
    else t = (u-0.5)*4*rl::kTwoPi;
    double a = rl::normalize_angle_2pi(t), b = ref_norm(t);
    if (__double_as_longlong(a) != __double_as_longlong(b) && !(isnan(a)&&isnan(b))) atomicAdd(bad,1ull);
  }
}
int main(){ unsigned long long* d; cudaMalloc(&d,8); cudaMemset(d,0,8); k<<<1184,256>>>(d, 12345, 4096); unsigned long long h; cudaMemcpy(&h,d,8,cudaMemcpyDeviceToHost); printf("normalize mismatches: %llu of %llu\n", h, 1184ull*256*4096); return h!=0; }
