// Debug: Generic<B> fwd0 + top for a QP(3) leaf, n=1, device vs host emulation.
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
#ifndef HOSTEMU
__global__ void kstep(ModelDesc md, const double* rp, double dt, double* out) {
    double Phi[GB * GB], Q[GB * GB], Qi[GB * GB];
    T::step(md, rp, dt, Phi, Q);
    bool ok = qt_factor<GB>(Q, rp[1], md.b, Qi, nullptr);
    for (int i = 0; i < GB * GB; ++i) { out[i] = Phi[i]; out[GB * GB + i] = Q[i]; }
    out[2 * GB * GB] = ok;
}
#endif
int main(int argc, char** argv) {
    spingp_leaf lv[1] = {{4, 3}};
    double th[4] = {1.0, 0.8, 1.3, 5.0};
    if (argc > 1) { lv[0].type = 3; lv[0].order = 6; th[0] = 1.0; th[1] = 1.0; }
    HostModel hm = build_model(lv, 1, argc > 1 ? 2 : 4);
    std::vector<double> rec(hm.rec_stride + hm.eqconst.size());
    fill_record(hm, th, 0.3, rec.data());
    for (size_t i = 0; i < hm.eqconst.size(); ++i) rec[hm.rec_stride + i] = hm.eqconst[i];
    ModelDesc md = hm.desc;
    double out[2 * GB * GB + 1];
    for (double dt : {-1.0, 0.1}) {
#ifndef HOSTEMU
        double *drec, *dout;
        cudaMalloc(&drec, rec.size() * 8); cudaMalloc(&dout, sizeof out);
        cudaMemcpy(drec, rec.data(), rec.size() * 8, cudaMemcpyHostToDevice);
        md.eqconst = drec + hm.rec_stride;
        kstep<<<1, 1>>>(md, drec, dt, dout);
        cudaMemcpy(out, dout, sizeof out, cudaMemcpyDeviceToHost);
        printf("DEV dt=%g ok=%g\n", dt, out[2 * GB * GB]);
#else
        md.eqconst = rec.data() + hm.rec_stride;
        double Qi[GB * GB];
        T::step(md, rec.data(), dt, out, out + GB * GB);
        out[2 * GB * GB] = qt_factor<GB>(out + GB * GB, rec[1], md.b, Qi, nullptr);
        printf("HOST dt=%g ok=%g\n", dt, out[2 * GB * GB]);
#endif
        for (int i = 0; i < GB; ++i) { for (int j = 0; j < GB; ++j) printf("%9.5f ", out[i * GB + j]); printf(" | "); for (int j = 0; j < GB; ++j) printf("%9.5f ", out[GB * GB + i * GB + j]); printf("\n"); }
    }
}
