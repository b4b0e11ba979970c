// Probe: what cvt.rna.tf32.f32 (F2FP.TF32) returns on sm_100a -- rounded
// value with cleared low bits, or not?  Compare with integer RNE rounding.
#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k(const float* x, unsigned* a, unsigned* b, unsigned* c, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned r, q;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x[i]));
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(q) : "f"(x[i]));  // F2FP.TF32.F32 in SASS
    a[i] = r;
    c[i] = q;
    unsigned u = __float_as_uint(x[i]);
    b[i] = (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
}
int main() {
    const int n = 1 << 20;
    float* hx = new float[n];
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < n; ++i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        unsigned u = (unsigned)s;
        u = (u & 0x807FFFFFu) | (((u >> 23) % 60 + 100) << 23);
        if (i % 7 == 0) u = (u & ~0x1FFFu) | 0x1000u;  // exact ties
        memcpy(&hx[i], &u, 4);
    }
    float* dx; unsigned *da, *db, *dc;
    cudaMalloc(&dx, n * 4); cudaMalloc(&da, n * 4); cudaMalloc(&db, n * 4); cudaMalloc(&dc, n * 4);
    cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
    k<<<n / 256, 256>>>(dx, da, db, dc, n);
    unsigned *ha = new unsigned[n], *hb = new unsigned[n], *hc = new unsigned[n];
    cudaMemcpy(ha, da, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb, db, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, dc, n * 4, cudaMemcpyDeviceToHost);
    int rn_low = 0, rn_diff = 0;
    for (int i = 0; i < n; ++i) {
        if (hc[i] & 0x1FFFu) ++rn_low;
        if ((hc[i] & 0xFFFFE000u) != hb[i]) ++rn_diff;
    }
    printf("cvt.rn.tf32: %d/%d results with low 13 bits set; %d differ from integer RNE after masking\n", rn_low, n,
           rn_diff);
    int lowbits = 0, diff_masked = 0, diff_ties = 0;
    for (int i = 0; i < n; ++i) {
        if (ha[i] & 0x1FFFu) ++lowbits;
        if ((ha[i] & 0xFFFFE000u) != hb[i]) { ++diff_masked; if (i % 7 == 0) ++diff_ties; }
    }
    printf("cvt.rna.tf32: %d/%d results with low 13 bits set; %d differ from RNE after masking (%d of them ties)\n",
           lowbits, n, diff_masked, diff_ties);
    unsigned u; memcpy(&u, &hx[1], 4);
    printf("example x=%08x cvt=%08x rne=%08x\n", u, ha[1], hb[1]);
    return 0;
}
