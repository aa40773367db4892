// Narrow-line instance of the block-tridiagonal factor: ocp_block.cu compiled
// a second time, in its own namespace, for decompositions of MANY SMALL
// subdomains (config 5: 4096 subdomains of 36 x 36 points, 72-unknown lines).
//
// There the factor of one subdomain is a short chain of dependent pivot
// steps that one 12-warp CTA per SM cannot hide; what helps is more
// independent chains per SM.  This instance runs 4-warp CTAs, three per SM:
//  * lines are padded to 16, not 32 (72 unknowns at NPB = 80 instead of 96):
//    the last panel is 16 wide (factor_one<.., HALF>), so the shared-memory
//    Schur block is 80 x 84 doubles and three CTAs fit an SM;
//  * every warp is a pivot warp and the schedule is the serial one (trailing
//    tiles by all warps, then the next pivot inverse): measured on wide lines,
//    overlapping the inverse with the tiles is nearly zero-sum anyway
//    (DESIGN.md 3.1).
// Round 1 ran 6-warp CTAs (2 lookahead warps), two per SM, NPB = 96
// (-DOCP_NW_THREADS=192 -DOCP_NW_LAW=2 -DOCP_NW_MINB=2 -DOCP_NW_MAX_NPB=96
// -DOCP_NW_OVERLAP rebuilds it).  The host picks this instance when there are
// at least two subdomains per SM and nearly every line fits (ocp_abi.cu,
// bf_narrow).
#include <cstring>

#ifndef OCP_NW_THREADS
#define OCP_NW_THREADS 128
#endif
#ifndef OCP_NW_LAW
#define OCP_NW_LAW 4
#endif
#ifndef OCP_NW_MINB
#define OCP_NW_MINB 3
#endif
#ifndef OCP_NW_MAX_NPB
#define OCP_NW_MAX_NPB 80
#endif
#if !defined(OCP_NW_OVERLAP) && !defined(OCP_P1_SERIAL)
#define OCP_P1_SERIAL 1
#endif
#define OCP_BF_THREADS OCP_NW_THREADS
#define OCP_LAW OCP_NW_LAW
#define OCP_BF_MINB OCP_NW_MINB
#define OCP_BF_SMEM_MAX_NPB OCP_NW_MAX_NPB
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
