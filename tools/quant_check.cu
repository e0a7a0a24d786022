#include <cstdio>
#include "quant.cuh"
using namespace mxp;
__global__ void k(const double* x, double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    out[4*i+0] = round_fp16(x[i]); out[4*i+1] = rne_format(x[i], 10, -14, 65504.0, false);
    out[4*i+2] = round_e4m3(x[i]); out[4*i+3] = rne_format(x[i], 3, -6, 448.0, true);
}
int main() {
    const int n = 1 << 22; double *x, *o; cudaMallocManaged(&x, n*8); cudaMallocManaged(&o, 4*n*8);
    unsigned long long s = 1;
    for (int i = 0; i < n; ++i) { s = s * 6364136223846793005ull + 1442695040888963407ull;
        int e = (int)((s >> 33) % 60) - 40; double m = 1.0 + (double)(s >> 11 & 0xFFFFF) / 1048576.0;
        if (i % 7 == 0) m = 1.0 + (double)((s >> 20) % 16) / 16.0 + ((i%14==0)? 1.0/32 : 0);  // ties for e4m3
        x[i] = ((s >> 63) ? -1 : 1) * ldexp(m, e); }
    k<<<(n+255)/256,256>>>(x,o,n); cudaDeviceSynchronize();
    int bad16=0, bad8=0; for (int i=0;i<n;++i){ if (o[4*i]!=o[4*i+1]) ++bad16; if (o[4*i+2]!=o[4*i+3]) ++bad8; }
    printf("fp16 mismatches %d, e4m3 mismatches %d of %d\n", bad16, bad8, n); return bad16+bad8;
}
