// Narrow-line instance of the block-tridiagonal factor: ocp_block.cu compiled
// a second time, in its own namespace, with a 6-warp CTA (2 lookahead warps),
// two CTAs per SM and a 96-unknown shared-memory Schur block.
//
// On lines of <= 96 unknowns (config 5: 36 x 36 local grids, 72-unknown lines
// padded to 96) the factor of one subdomain is a short chain of dependent
// pivot steps that one 12-warp CTA per SM cannot hide; two independent chains
// per SM do (config-5 factor 19.7 -> 15 ms per launch, identical results).
// The host picks this instance when there are at least two subdomains per SM
// and nearly every line fits (ocp_abi.cu, bf_narrow).
#include <cstring>

#ifndef OCP_NW_THREADS
#define OCP_NW_THREADS 192
#endif
#ifndef OCP_NW_LAW
#define OCP_NW_LAW 2
#endif
#ifndef OCP_NW_MINB
#define OCP_NW_MINB 2
#endif
#ifdef OCP_NW_SERIAL
#define OCP_P1_SERIAL 1
#endif
#define OCP_BF_THREADS OCP_NW_THREADS
#define OCP_LAW OCP_NW_LAW
#define OCP_BF_MINB OCP_NW_MINB
#define OCP_BF_SMEM_MAX_NPB 96
#define OCP_NARROW_INSTANCE 1
#define ocp ocp_nw
#include "ocp_block.cu"
#undef ocp

namespace ocp {

struct SubInfo;
struct Phys;

int narrow_factor_max_npb() { return ocp_nw::BF_SMEM_MAX_NPB; }
int narrow_factor_ctas_per_sm() { return OCP_BF_MINB; }

cudaError_t narrow_set_factor_smem() {
  return raise_smem_limit((const void*)ocp_nw::k_block_factor, ocp_nw::block_factor_smem_bytes(0));
}

cudaError_t launch_narrow_factor(int grid, cudaStream_t st, const SubInfo* subs, const int* list,
                                 int cnt, const Phys* P, const double* JDpool, double* fac_pool,
                                 double* scratch, long long ws_stride, int* status) {
  ocp_nw::Phys p;   // same layout as ocp::Phys (one definition, two namespaces)
  std::memcpy(&p, P, sizeof p);
  ocp_nw::k_block_factor<<<grid, ocp_nw::BF_THREADS, ocp_nw::block_factor_smem_bytes(0), st>>>(
      reinterpret_cast<const ocp_nw::SubInfo*>(subs), list, cnt, p, JDpool, fac_pool, scratch,
      ws_stride, status);
  return cudaGetLastError();
}

}  // namespace ocp
