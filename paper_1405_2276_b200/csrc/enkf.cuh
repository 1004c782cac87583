// enkf.cuh — the perturbed-observation ensemble Kalman filter (enkf.hpp:15-94) on the device.
#pragma once

#include "filter.cuh"

namespace fkb {

struct Enkf {
    Cov* cov = nullptr;
    cudaStream_t s = nullptr;
    long long n = 0;
    int m = 0, ne = 0;
    DevCsr H, HT;
    DBuf<double> X;  // members, n×ne column-major (Ensemble::members)
    DBuf<double> Xf, Xr, HXr, HX, mean, hmean, Z, Cyy, T, ybuf, ws, pws;
    DBuf<int> info;

    Enkf(Cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val, int n_members);
    void step(const double* y_host, double sigma2, uint64_t seed);  // enkf_step (enkf.hpp:49-94)
    void member_mean(double* out_dev);                             // Ensemble::mean (:20)
};

}  // namespace fkb
