// k_advance.cu -- decode-advance kernel (DESIGN.md §3.1 W6-W7, §3.2 B1-B8): one warp per
// instance; the per-instance procedure is advance_instance() in advance.cuh.
#include "advance.cuh"

namespace sf {

#ifndef SF_ADV_MINB
#define SF_ADV_MINB (16 / SF_ADV_WARPS)   // 16 warps per SM (128 registers, no spills)
#endif
__global__ void __launch_bounds__(32 * kWarpsPerBlock, SF_ADV_MINB) k_advance(GParams P, Dev D, int n_inst_total) {
  __shared__ AdvStage stage_all[kWarpsPerBlock];
  pdl_trigger();                                   // the ledger kernel may be scheduled now
  const int gi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gi >= n_inst_total) return;
  const int s = D.inst_scen[gi];
  const ScenConst C = D.sc[s];                     // constant: its load overlaps the wait
  // the scenario's previous window is complete: this instance's run list is final -- load it while
  // the coordinator runs, then wait for the coordinator
  if (P.pdl) warp_wait_geq(&D.f_led[s], P.epoch - 1);
  RunPre pre;
  preload_run(D, C, gi, pre);
  if (P.pdl) warp_wait_geq(&D.f_coord[s], P.epoch);     // this scenario's coordinator is done
  SF_TRACE_AT(4LL * P.n_scen + 2LL * gi);
  advance_instance(P, D, gi, stage_all[threadIdx.x >> 5], s, C, &pre);
  SF_TRACE_AT(4LL * P.n_scen + 2LL * gi + 1);
  fence_release();                                 // this lane's writes, device-wide
  __syncwarp();
  if ((threadIdx.x & 31) == 0) add_release(&D.f_adv[s], 1);
}

}  // namespace sf

void sf_launch_advance(const sf::GParams &P, const sf::Dev &D, int n_inst_total, cudaStream_t st) {
  const int blocks = (n_inst_total + sf::kWarpsPerBlock - 1) / sf::kWarpsPerBlock;
  sf_launch_pdl(sf::k_advance, blocks, 32 * sf::kWarpsPerBlock, st, P.pdl, P, D, n_inst_total);
}
