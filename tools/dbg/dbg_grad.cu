// Debug: run step_terms<MaternTraits<3>> on fixed inputs on device and host.
#ifdef HOSTEMU
#include "../../tests/emu/cuda_host_emu.h"
#endif
#include <cstdio>
#include "../../paper_1610_08035_b200/csrc/engine.cuh"
using namespace spingp_dev;
#ifndef HOSTEMU
#define HD __global__
#else
#define HD
#endif
HD void kern(double* out, ModelDesc md) {
    double rp[7] = {0.3, 1e-10, 1e-10, -1e-10, 2.0, 1.5, 1.4907119849998598};
    double Phi[9], Q[9], Qi[9], ld;
    MaternTraits<3>::step(md, rp, 0.1, Phi, Q);
    qt_inverse<3>(Q, 1e-10, 3, Qi, &ld);
    double xc[3] = {0.3, -0.2, 0.1}, xp[3] = {0.25, -0.1, 0.05};
    double Ccc[9] = {0.5, 0.1, 0.0, 0.1, 0.4, 0.05, 0.0, 0.05, 0.6};
    double Cpp[9] = {0.45, 0.05, 0.01, 0.05, 0.35, 0.02, 0.01, 0.02, 0.5};
    double Cpc[9] = {0.3, 0.02, 0.01, 0.01, 0.2, 0.01, 0.0, 0.01, 0.25};
    double fe = 0, g[4] = {0, 0, 0, 0};
    step_terms<MaternTraits<3>>(md, rp, 0.1, Phi, Q, Qi, xc, Ccc, xp, Cpp, Cpc, false, true, fe, g);
    out[0] = fe; out[1] = g[0]; out[2] = g[1];
    for (int i = 0; i < 9; ++i) { out[3 + i] = Phi[i]; out[12 + i] = Q[i]; out[21 + i] = Qi[i]; }
    double g2[4] = {0,0,0,0}, fe2 = 0;
    step_terms<MaternTraits<3>>(md, rp, -1.0, Phi, Q, Qi, xc, Ccc, xp, Cpp, Cpc, true, true, fe2, g2);
    out[30] = g2[0]; out[31] = g2[1];
}
int main() {
    ModelDesc md{};
    md.b = 3; md.nleaves = 1; md.nt = 2; md.rec_stride = 7; md.rec[0] = 4; md.H[0] = 1;
    double h[32];
#ifndef HOSTEMU
    double* d; cudaMalloc(&d, sizeof h);
    kern<<<1, 1>>>(d, md);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("device: ");
#else
    kern(h, md);
    printf("host:   ");
#endif
    for (int i = 0; i < 32; ++i) printf("%.15g ", h[i]);
    printf("\n");
}
