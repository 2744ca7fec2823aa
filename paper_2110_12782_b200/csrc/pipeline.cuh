// pipeline.cuh — NetMF+ stages on device blocks (pipeline.cu).
#pragma once
#include "common.cuh"

namespace netmfp {
void cholqr(Ctx &c, const Mat &Y, const Mat &out, const int32_t *deg, float rexp, int passes, const Mat *tmp,
            bool orthonormal = true);
// out_F: write F = D^(-1+α) U (Eq. 3) instead of U
void freigs(Ctx &c, const Graph &g, double alpha, int k, int s1, int q, uint64_t seed, const Mat &U,
            double *lam_dev, bool out_F = false);
void factor_pair(Ctx &c, const Graph &g, double alpha, int T, const Mat &U, const double *lam, int k,
                 const Mat &F, double *C,
                 bool u_is_F = false);
void sketch_svd(Ctx &c, const Mat &F, const double *C, int k, double scale, int d, int s2, int s3, int z,
                uint64_t seed, int logmode, const Mat *Uout, double *sigma_dev, const Mat *Eout,
                const Mat *Yout, double *Zout, int64_t row0 = 0, int64_t n_global = -1,
                const int32_t *comp_id = nullptr, const SketchA *preA = nullptr);
bool side_fork(Ctx &c);
void side_join_point(Ctx &c, cudaStream_t main);
void cheb_coeffs(int order, double mu, double theta, double *c);
void propagate(Ctx &c, const Graph &g, const Mat &E, int order, double mu, double theta);
}  // namespace netmfp
