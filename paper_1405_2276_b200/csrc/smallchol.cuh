// smallchol.cuh — cluster-resident SPD factor+solve for n ≤ 1024.
#pragma once

#include "common.cuh"

namespace fkb {

// K (n×n, column-major, lower triangle used) is overwritten by its Cholesky factor; b by
// K⁻¹b.  *info (device) is set to j+1 at the first non-positive pivot (must be 0 on entry).
// rdg: device scratch of n doubles (reciprocal pivots).
// gate (optional device flag): the kernel returns immediately when *gate == 0.
void chol_solve_small(int n, double* K, long long ld, double* b, double* rdg, int* info, cudaStream_t s,
                      unsigned long long* tdbg = nullptr, const int* gate = nullptr);
size_t chol_solve_smem(int n);
size_t chol_solve_scratch(int n);  // doubles of device scratch (diagonal-tile inverses)

}  // namespace fkb
