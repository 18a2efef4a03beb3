// k_coord.cu -- window begin + rollout coordinator kernel (DESIGN.md §3.1 W0-W5); the
// per-scenario procedure is coord_scenario() in coord.cuh.
#include "coord.cuh"

namespace sf {

template <int KS>
__global__ void __launch_bounds__(32 * kCoordWarps, KS == 1 ? SF_COORD_MINB : 8 / kCoordWarps) k_begin_coord(GParams P, Dev D) {
  __shared__ Stage stage_all[kCoordWarps];
  pdl_trigger();                                   // the advance kernel may be scheduled now
  const int s = blockIdx.x * kCoordWarps + (threadIdx.x >> 5);
  if (s >= P.n_scen) return;
  const ScenConst C = D.sc[s];                     // constant: its load overlaps the wait
  if (P.pdl) warp_wait_geq(&D.f_led[s], P.epoch - 1);   // this scenario's previous window is done
  SF_TRACE_AT(4LL * s);
  coord_scenario_fit<KS>(P, D, s, stage_all[threadIdx.x >> 5], C);
  SF_TRACE_AT(4LL * s + 1);
  fence_release();                                 // this lane's writes, device-wide
  __syncwarp();
  if ((threadIdx.x & 31) == 0) st_release(&D.f_coord[s], P.epoch);
}

}  // namespace sf

void sf_launch_begin_coord(const sf::GParams &P, const sf::Dev &D, int n_scen, int max_inst, cudaStream_t st) {
  const int blocks = (n_scen + sf::kCoordWarps - 1) / sf::kCoordWarps;
  const int thr = 32 * sf::kCoordWarps;
  if (max_inst <= 32) sf_launch_pdl(sf::k_begin_coord<1>, blocks, thr, st, P.pdl, P, D);
  else if (max_inst <= 64) sf_launch_pdl(sf::k_begin_coord<2>, blocks, thr, st, P.pdl, P, D);
  else sf_launch_pdl(sf::k_begin_coord<4>, blocks, thr, st, P.pdl, P, D);
}
