// SPDX-License-Identifier: Apache-2.0
// Kernel instantiations for one built-in integrand, selected by -DMCB_INST=k
// (see Makefile).  Compiled with -fmad=false: the reference's
// -ffp-contract=off (proj/CMakeLists.txt:14-19).
#if MCB_INST == 9
#define MCB_DIMS_MAX 10  // the unit-test functors only need small dims
#endif
#include "registry.cuh"

namespace mcubes::gpu::abi {

template <class F>
static IntegrandOps both(RngKind rng, const F& f) {
  switch (rng) {
    case RngKind::philox: return make_ops<F, RngKind::philox>(f);
    case RngKind::philox_exact: return make_ops<F, RngKind::philox_exact>(f);
    default: return make_ops<F, RngKind::compat>(f);
  }
}

#if MCB_INST == 0
IntegrandOps ops_F1(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F1{}); }
#elif MCB_INST == 1
IntegrandOps ops_F2(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F2{}); }
#elif MCB_INST == 2
IntegrandOps ops_F3(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F3{}); }
#elif MCB_INST == 3
IntegrandOps ops_F4(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F4{}); }
#elif MCB_INST == 4
IntegrandOps ops_F5(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F5{}); }
#elif MCB_INST == 5
IntegrandOps ops_F6(int, RngKind r, const BuiltinArgs&) { return both(r, fn::F6{}); }
#elif MCB_INST == 6
IntegrandOps ops_FA(int, RngKind r, const BuiltinArgs&) { return both(r, fn::FA{}); }
#elif MCB_INST == 8
IntegrandOps ops_FB(int, RngKind r, const BuiltinArgs&) {
  // integrands.hpp:206-207, evaluated on the host exactly as the reference does
  const double sigma2 = 0.01;
  return both(r, fn::FB{std::pow(2.0 * 3.141592653589793 * sigma2, -4.5)});
}
#elif MCB_INST == 7
IntegrandOps ops_Table(int, RngKind r, const BuiltinArgs& a) {
  const auto n = static_cast<std::uint32_t>(a.host_params[0]);
  return both(r, fn::TableView{a.dev_params, a.dims, n});
}
#elif MCB_INST == 9
IntegrandOps ops_Tests(int id, RngKind, const BuiltinArgs& a) {
  switch (id) {
    case 32: return make_ops(fn::X0{});
    case 33: return make_ops(fn::Const{a.n_params ? a.host_params[0] : 0.0});
    case 34: return make_ops(fn::X0SqHalf{});
    case 35: return make_ops(fn::InfIfX0Pos{});
    case 36: return make_ops(fn::Inf{});
    case 38: return make_ops(fn::InfNearOrigin{a.n_params ? a.host_params[0] : 0.0});
    default: return make_ops(fn::Zero{});
  }
}
#endif

}  // namespace mcubes::gpu::abi
