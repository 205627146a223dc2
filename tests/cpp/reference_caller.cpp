// A reference-style caller of the C++ wrapper (include/ihom_b200.hpp): the same calls a user of
// ihom::Homogenizer<float> (proj/include/ihom/homogenization.hpp) makes, with the namespace switched.
// Exit 0: solid C^H matches the reference's known answers (tests/test_homogenization.cpp:30-33);
// 3: no CUDA device (the library fails loudly); 2: wrong numbers.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ihom_b200.hpp"

int main() {
  using namespace ihom::gpu;
  const IVec3 reso{8, 8, 8};
  const BaseMaterial mat(1e6, 0.3);
  SolverOptions opts;
  opts.tol = 1e-10;
  opts.max_cycles = 100;
  try {
    BaseMaterial bad;
    try {
      bad = BaseMaterial(1e6, 0.7);
      return 4;  // the reference rejects nu >= 0.5
    } catch (const std::invalid_argument&) {
    }
    Homogenizer hom(reso, mat, 1.0, opts);
    hom.set_density(std::vector<double>(512, 1.0));
    const CellSolveStats st = hom.solve_cell_problems();
    const Matrix6 C = hom.effective_tensor();
    std::printf("converged %d cycles %d C00 %.9f C01 %.9f C33 %.9f\n", int(st.converged), st.total_cycles, C[0],
                C[1], C[21]);
    const bool ok = std::fabs(C[0] - 1346153.846153846) < 1e-4 && std::fabs(C[1] - 576923.0769230769) < 1e-4 &&
                    std::fabs(C[21] - 384615.3846153846) < 1e-4;
    return ok ? 0 : 2;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 3;
  }
}
