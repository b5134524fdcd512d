// SPDX-License-Identifier: Apache-2.0
// Built-in integrand factories of the C ABI (include/mcubes_b200.h
// mcb_integrand_id).  Each factory lives in its own translation unit
// (inst.cu compiled once per MCB_INST) so the kernel instantiations build in
// parallel.
#pragma once

#include <cstdint>

#include "mcubes_b200/mcubes.cuh"

namespace mcubes::gpu::abi {

struct BuiltinArgs {
  std::uint32_t dims;
  const double* dev_params;   ///< device copy of the params (table integrand)
  const double* host_params;  ///< host params (constants)
  std::uint32_t n_params;
};

#define MCB_FACTORIES(X) \
  X(F1) X(F2) X(F3) X(F4) X(F5) X(F6) X(FA) X(FB) X(Table) X(Tests)

#define MCB_DECLARE(name) IntegrandOps ops_##name(int id, RngKind rng, const BuiltinArgs& a);
MCB_FACTORIES(MCB_DECLARE)
#undef MCB_DECLARE

}  // namespace mcubes::gpu::abi
