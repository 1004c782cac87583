// host_linalg.h — host-side setup routines (H construction, small symmetric eigensolves).
#pragma once

#include <vector>

namespace fkb {

int trace_ray_into(int nx, int ny, double lx, double ly, double sx, double sy, double rx, double ry, int cap,
                   long long* cells, double* lengths);
void build_H(int nx, int ny, double lx, double ly, int ns, const double* src, int nr, const double* rec,
             std::vector<int>& rowptr, std::vector<int>& col, std::vector<double>& val);
void sym_eig_small(int n, const double* A, double* w, double* Z);

}  // namespace fkb
