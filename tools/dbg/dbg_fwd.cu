// Debug: the first stages of k_fwd0 (step, qt_factor, chol_inv_solve, D, chol) for one
// generic-sum model, device vs host emulation, every intermediate dumped.
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
#define GB 8
#endif
typedef GenericTraits<GB> T;
constexpr int NO = 7 * GB * GB + 4;
__global__ void kstages(ModelDesc md_, const double* rp, double dt, double* out) {
    constexpr int B = GB;
#ifdef SMD
    __shared__ ModelDesc md;
    if (threadIdx.x == 0) md = md_;
    __syncthreads();
#else
    const ModelDesc& md = md_;
#endif
    double Phi[B * B], Q[B * B], Mq[B * B], Qinv[B * B], D[B * B], L[B * B];
    T::step(md, rp, dt, Phi, Q);
    const bool ok1 = qt_factor<B>(Q, rp[1], md.b, Mq, nullptr);
    chol_inv_solve<B>(Qinv, Mq);
    const double is2 = 1.0 / (rp[0] * rp[0]);
    for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j) D[i * B + j] = Qinv[i * B + j] + T::H(md, i) * T::H(md, j) * is2;
    double ld;
    const bool ok2 = chol<B>(L, D, ld);
    double PQP[B * B], U[B * B];
    step_assembly<B>(Phi, Mq, PQP, U);
    for (int i = 0; i < B * B; ++i) {
        out[i] = Phi[i]; out[B * B + i] = Q[i]; out[2 * B * B + i] = Mq[i]; out[3 * B * B + i] = Qinv[i];
        out[4 * B * B + i] = D[i]; out[5 * B * B + i] = L[i]; out[6 * B * B + i] = U[i];
    }
    out[7 * B * B] = ok1; out[7 * B * B + 1] = ok2; out[7 * B * B + 2] = ld;
}
int main(int argc, char** argv) {
    spingp_leaf lv[2] = {{4, 3}, {1, 0}};
    int nl = 1;
    std::vector<double> th = {1.0, 0.8, 1.3, 5.0};
    if (argc > 1 && argv[1][0] == 'e') { lv[0] = {3, 6}; th = {1.1, 1.4}; }
    if (argc > 1 && argv[1][0] == 's') { lv[0] = {1, 0}; lv[1] = {4, 2}; nl = 2; th = {1.0, 10.0, 1.0, 1.0, 1.0, 20.0}; }
    HostModel hm = build_model(lv, nl, static_cast<int>(th.size()));
    std::vector<double> rec(hm.rec_stride + hm.eqconst.size());
    fill_record(hm, th.data(), 0.3, rec.data());
    for (size_t i = 0; i < hm.eqconst.size(); ++i) rec[hm.rec_stride + i] = hm.eqconst[i];
    ModelDesc md = hm.desc;
    static double out[NO];
    for (double dt : {-1.0, 0.1}) {
#ifndef HOSTEMU
        double *drec, *dout;
        cudaMalloc(&drec, rec.size() * 8); cudaMalloc(&dout, sizeof out);
        cudaMemcpy(drec, rec.data(), rec.size() * 8, cudaMemcpyHostToDevice);
        md.eqconst = drec + hm.rec_stride;
        kstages<<<1, 1>>>(md, drec, dt, dout);
        cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
#else
        md.eqconst = rec.data() + hm.rec_stride;
        kstages(md, rec.data(), dt, out);
#endif
        const char* nm[7] = {"Phi", "Q", "Mq", "Qinv", "D", "L", "U"};
        printf("dt=%g ok1=%g ok2=%g ld=%.12g\n", dt, out[7 * GB * GB], out[7 * GB * GB + 1], out[7 * GB * GB + 2]);
        for (int a = 0; a < 7; ++a) {
            printf("%s\n", nm[a]);
            for (int i = 0; i < GB; ++i) { for (int j = 0; j < GB; ++j) printf("%12.6g ", out[a * GB * GB + i * GB + j]); printf("\n"); }
        }
    }
    return 0;
}
