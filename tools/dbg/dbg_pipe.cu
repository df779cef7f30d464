// Debug: run fwd0 -> top -> rev0 for MaternTraits<3>, n=2 single chunk, on device and host.
#ifdef HOSTEMU
#include "../../tests/emu/cuda_host_emu.h"
#endif
#include <cstdio>
#define SPINGP_DEBUG_PRINT 1
#include <vector>
#include "../../paper_1610_08035_b200/csrc/engine.cuh"
using namespace spingp_dev;
typedef MaternTraits<3> T;
int main() {
    ModelDesc md{};
    md.b = 3; md.nleaves = 1; md.nt = 2; md.rec_stride = 7; md.rec[0] = 4; md.H[0] = 1;
    double lam = 1.4907119849998598, var = 2.0;
    double tr = var * (1 + lam * lam / 3 + lam * lam * lam * lam);
    double dtrl = -(2.0 / 1.5) * var * lam * lam / 3 - (4.0 / 1.5) * var * lam * lam * lam * lam;
    double rp[7] = {0.3, 1e-10 * tr / 3, 1e-10 * tr / var / 3, 1e-10 * dtrl / 3, var, 1.5, lam};
    double t[2] = {0.1, 0.2}, y[2] = {0.5, -0.3};
    Geom g{};
    g.nlev = 1; g.S = 1; g.n[0] = 2; g.m[0] = 2; g.K[0] = 1; g.n[1] = 1;
    const int NF = Fac<3>::N * 2, NR = Rec<3>::N, NS = Sol<3>::N, NP = P_GRAD + 2;
    double hf[64], hr[64], hs[64], hp[16], htop[1];
    unsigned long long hst = ~0ULL;
    Outs o{nullptr, nullptr, 0, 1, 1};
#ifndef HOSTEMU
    double *dp, *dt, *dy, *df, *dr, *ds, *dpart, *dtop; unsigned long long* dst;
    cudaMalloc(&dp, 64); cudaMalloc(&dt, 16); cudaMalloc(&dy, 16); cudaMalloc(&df, 512); cudaMalloc(&dr, 512);
    cudaMalloc(&ds, 512); cudaMalloc(&dpart, 128); cudaMalloc(&dtop, 8); cudaMalloc(&dst, 8);
    cudaMemcpy(dp, rp, 56, cudaMemcpyHostToDevice); cudaMemcpy(dt, t, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y, 16, cudaMemcpyHostToDevice); cudaMemcpy(dst, &hst, 8, cudaMemcpyHostToDevice);
    k_fwd0<T><<<1, 128>>>(md, dp, dt, dy, g, df, dr, dpart, dst);
    k_top<3><<<1, 128>>>(g, dr, ds, dtop, dst);
    k_rev0<T><<<1, 128>>>(md, dp, dt, dy, g, df, ds, dpart, o, dst);
    cudaMemcpy(hf, df, NF * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hr, dr, NR * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs, ds, NS * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hp, dpart, NP * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hst, dst, 8, cudaMemcpyDeviceToHost);
    printf("DEVICE status %llx\n", hst);
#else
    emu_launch(1, 1, [&] { k_fwd0<T>(md, rp, t, y, g, hf, hr, hp, &hst); });
    emu_launch(1, 1, [&] { k_top<3>(g, hr, hs, htop, &hst); });
    emu_launch(1, 1, [&] { k_rev0<T>(md, rp, t, y, g, hf, hs, hp, o, &hst); });
    printf("HOST status %llx\n", hst);
#endif
    printf("fac: "); for (int i = 0; i < Fac<3>::N; ++i) printf("%.12g ", hf[i]); printf("\n");
    printf("rec: "); for (int i = 0; i < NR; ++i) printf("%.12g ", hr[i]); printf("\n");
    printf("sol: "); for (int i = 0; i < NS; ++i) printf("%.12g ", hs[i]); printf("\n");
    printf("part: "); for (int i = 0; i < NP; ++i) printf("%.12g ", hp[i]); printf("\n");
}
