// result.h - the opaque rhosvd_result handle (internal; shared by rhosvd.cu and t2c.cu).
#pragma once
#include "common.cuh"

struct rhosvd_result {
  int32_t ranks[3] = {0, 0, 0};
  int64_t n = 0, ldz = 0, Rl = 0, Rp = 0;
  double* Z[3] = {nullptr, nullptr, nullptr};      // n x r_l, col-major, ld ldz
  double* sigma[3] = {nullptr, nullptr, nullptr};  // r_l
  double* W[3] = {nullptr, nullptr, nullptr};      // r_l x Rp row-major (CP factors of the core)
  double* beta = nullptr;                          // r1 x r2 x r3, C order
  bool beta_valid = true;                          // false on ranks != 0 with RHOSVD_F_ROOT_ONLY_CORE
  // rhosvd_c2t_host: pinned host copies of Z (ld ldz), sigma and beta
  double* hZ[3] = {nullptr, nullptr, nullptr};
  double* hsigma[3] = {nullptr, nullptr, nullptr};
  double* hbeta = nullptr;
  rhosvd_report rep{};
};
