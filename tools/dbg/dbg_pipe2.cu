// Debug: full level pipeline for a generic model (build_model) on device vs host emulation.
#ifdef HOSTEMU
#include "../../tests/emu/cuda_host_emu.h"
#endif
#include <cstdio>
#include <vector>
#include "../../paper_1610_08035_b200/csrc/engine.cuh"
#include "../../paper_1610_08035_b200/csrc/host_model.hpp"
using namespace spingp_dev;
using namespace spingp_host;
#ifndef GB
#define GB 3
#endif
typedef GenericTraits<GB> T;
int main(int argc, char** argv) {
    spingp_leaf lv[2] = {{1, 0}, {0, 0}};
    double th[4] = {1.0, 0.7, 0.5, 2.0};
    HostModel hm = build_model(lv, 2, 4);
    std::vector<double> rp(hm.rec_stride);
    fill_record(hm, th, 0.3, rp.data());
    ModelDesc md = hm.desc;
    md.eqconst = nullptr;
    double t[2] = {0.1, 0.2}, y[2] = {0.5, -0.3};
    Geom g{};
    g.nlev = 1; g.S = 1; g.n[0] = 2; g.m[0] = 2; g.K[0] = 1; g.n[1] = 1;
    const int NF = Fac<GB>::N * 2, NR = Rec<GB>::N, NS = Sol<GB>::N, NP = P_GRAD + 4;
    std::vector<double> hf(NF), hr(NR), hs(NS), hp(NP), top(1), mean(2), var(2);
    unsigned long long hst = ~0ULL;
#ifndef HOSTEMU
    double *dp, *dt, *dy, *df, *dr, *ds, *dpart, *dtop, *dm, *dv; unsigned long long* dst;
    cudaMalloc(&dp, 8 * rp.size()); cudaMalloc(&dt, 16); cudaMalloc(&dy, 16); cudaMalloc(&df, 8 * NF); cudaMalloc(&dr, 8 * NR);
    cudaMalloc(&ds, 8 * NS); cudaMalloc(&dpart, 8 * NP); cudaMalloc(&dtop, 8); cudaMalloc(&dst, 8); cudaMalloc(&dm, 16); cudaMalloc(&dv, 16);
    cudaMemcpy(dp, rp.data(), 8 * rp.size(), cudaMemcpyHostToDevice); cudaMemcpy(dt, t, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y, 16, cudaMemcpyHostToDevice); cudaMemcpy(dst, &hst, 8, cudaMemcpyHostToDevice);
    Outs o{dm, dv, 0, 1, 1};
    k_fwd0<T><<<1, 128>>>(md, dp, dt, dy, g, df, dr, dpart, dst);
    k_top<GB><<<1, 128>>>(g, dr, ds, dtop, dst);
    k_rev0<T><<<1, 128>>>(md, dp, dt, dy, g, df, ds, dpart, o, dst);
    cudaMemcpy(hf.data(), df, NF * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hr.data(), dr, NR * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), ds, NS * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hp.data(), dpart, NP * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(var.data(), dv, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hst, dst, 8, cudaMemcpyDeviceToHost);
    printf("DEVICE status %llx err %s\n", hst, cudaGetErrorString(cudaGetLastError()));
#else
    Outs o{mean.data(), var.data(), 0, 1, 1};
    emu_launch(1, 1, [&] { k_fwd0<T>(md, rp.data(), t, y, g, hf.data(), hr.data(), hp.data(), &hst); });
    emu_launch(1, 1, [&] { k_top<GB>(g, hr.data(), hs.data(), top.data(), &hst); });
    emu_launch(1, 1, [&] { k_rev0<T>(md, rp.data(), t, y, g, hf.data(), hs.data(), hp.data(), o, &hst); });
    printf("HOST status %llx\n", hst);
#endif
    printf("fac: "); for (int i = 0; i < Fac<GB>::N; ++i) printf("%.10g ", hf[i]); printf("\n");
    printf("rec: "); for (int i = 0; i < NR; ++i) printf("%.10g ", hr[i]); printf("\n");
    printf("sol: "); for (int i = 0; i < NS; ++i) printf("%.10g ", hs[i]); printf("\n");
    printf("part: "); for (int i = 0; i < NP; ++i) printf("%.10g ", hp[i]); printf("\n");
    printf("var: %.10g %.10g\n", var[0], var[1]);
}
