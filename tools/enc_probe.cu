#include <cuda.h>
#include <cstdio>
int main(){
  CUresult r0 = cuInit(0); CUdevice dv; cuDeviceGet(&dv,0); CUcontext cx; cuDevicePrimaryCtxRetain(&cx,dv); cuCtxSetCurrent(cx); printf("init %d\n", r0);
  CUtensorMap m; cuuint32_t es[5]={1,1,1,1,1};
  long long maxc=66000, L=32, Hkv=8, T=16, D=128; long long chunk=4*T*L*Hkv*D, slab=chunk/L;
  for (int rot=0; rot<2; ++rot) for (int lg=0; lg<4; ++lg){
  cuuint64_t dims[5]={64,(cuuint64_t)T,2, rot? (cuuint64_t)(maxc*L*2*Hkv):(cuuint64_t)(L*2*Hkv), rot? 8ull:(cuuint64_t)maxc};
  cuuint64_t str[4]={(cuuint64_t)D*2,128,(cuuint64_t)(T*D*2),(cuuint64_t)(chunk+(rot?slab:0))};
  cuuint32_t box[5]={64,(cuuint32_t)T,1,1,1u<<lg};
  CUresult r=cuTensorMapEncodeTiled(&m,CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,5,(void*)0x7f0000000000ull,dims,str,box,es,CU_TENSOR_MAP_INTERLEAVE_NONE,CU_TENSOR_MAP_SWIZZLE_128B,CU_TENSOR_MAP_L2_PROMOTION_L2_256B,CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("rot %d lg %d -> %d\n",rot,lg,r);}
}
