// The include-swap drop-in (include/sinkattn.hpp) used the way the reference's own callers use
// run_surrogate / r2_backward (inc/validation.hpp:102-114), on the reference's matrix type.
//   dropin_demo IN OUT half_band T R eps [direct]
// IN: int64 L, int64 d, then Q, K, V, G as L x d float32 (row-major); OUT: O, dQ, dK, dV, d_eps.
// With -DWITH_REFERENCE the reference's own sinktail::Matrix<float> (sinktail/types.hpp) is the
// matrix type; otherwise the same Eigen-API type from oracle/ref_shim.
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifdef WITH_REFERENCE
#include "sinktail/sinkhorn.hpp"  // the reference header: proves the types line up
using Mat = sinktail::Matrix<float>;
#else
#include <Eigen/Core>
using Mat = Eigen::Matrix<float, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
#endif
#include "sinkattn.hpp"

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s IN OUT half_band T R eps [direct]\n", argv[0]);
        return 2;
    }
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 3;
    int64_t L = 0, d = 0;
    if (std::fread(&L, 8, 1, f) != 1 || std::fread(&d, 8, 1, f) != 1) return 3;
    Mat Q(L, d), K(L, d), V(L, d), G(L, d);
    for (Mat* m : {&Q, &K, &V, &G})
        if (std::fread(m->data(), sizeof(float), (size_t)(L * d), f) != (size_t)(L * d)) return 3;
    std::fclose(f);
    try {
        sinkattn::Context ctx;
        auto run = sinkattn::run_surrogate(Q, K, V, std::atoll(argv[3]), std::atoll(argv[4]), std::atoll(argv[5]),
                                           std::atof(argv[6]), ctx);
        auto cot = sinkattn::r2_backward(run, G, Q, K, V,
                                         argc > 7 ? sinkattn::BackwardMode::DirectFourPlan
                                                  : sinkattn::BackwardMode::OneReference);
        FILE* o = std::fopen(argv[2], "wb");
        for (const Mat* m : {&run.output, &cot.grad_q, &cot.grad_k, &cot.grad_v})
            std::fwrite(m->data(), sizeof(float), (size_t)(m->rows() * m->cols()), o);
        std::fwrite(&cot.d_eps, sizeof(float), 1, o);
        std::fclose(o);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
