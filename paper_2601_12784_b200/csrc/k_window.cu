// k_window.cu -- fused window kernel for many small scenarios (DESIGN.md §8 "launch modes").
//
// Scenarios are independent, so one warp can run its scenario's whole window -- coordinator
// (W0-W5), the decode advance of each of its instances (W6-W7), then the reward ledger (W8-W9)
// -- with no grid-wide barrier between the phases.  Latency-bound coordinator work of one
// scenario then overlaps with other warps' decode steps on the same SM instead of every phase
// waiting for the slowest scenario, and several windows can run in one launch.  Used when every
// scenario has few instances (the per-warp serial advance stays short); the three-kernel path
// (k_begin_coord / k_advance / k_ledger) handles large instance counts.
#include "advance.cuh"
#include "coord.cuh"
#include "ledger.cuh"

namespace sf {

constexpr int kFusedWarps = 4;

union WinStage {
  Stage coord;
  AdvStage adv;
  EvStage led;
};

template <int KS>
__global__ void __launch_bounds__(32 * kFusedWarps) k_window(GParams P, Dev D, int n_windows) {
  __shared__ WinStage st_all[kFusedWarps];
  const int s = blockIdx.x * kFusedWarps + (threadIdx.x >> 5);
  if (s >= P.n_scen) return;
  WinStage &ws = st_all[threadIdx.x >> 5];
  const int inst_off = D.sc[s].inst_off, I = D.sc[s].I;
  for (int w = 0; w < n_windows; ++w) {
    coord_scenario<KS>(P, D, s, ws.coord, D.sc[s]);
    __syncwarp();
    for (int i = 0; i < I; ++i) advance_instance(P, D, inst_off + i, ws.adv, s, D.sc[s]);
    __syncwarp();
    ledger_scenario(P, D, s, ws.led, D.sc[s]);
    __syncwarp();
  }
}

}  // namespace sf

void sf_launch_window_fused(const sf::GParams &P, const sf::Dev &D, int n_scen, int max_inst, int n_windows,
                            cudaStream_t st) {
  const int blocks = (n_scen + sf::kFusedWarps - 1) / sf::kFusedWarps;
  (void)max_inst;                       // fused mode requires <= 32 instances (sf_api.cu)
  sf::k_window<1><<<blocks, 32 * sf::kFusedWarps, 0, st>>>(P, D, n_windows);
}

// ---------------------------------------------------------------------------------------------
// Block-per-scenario window kernel (SF_LAUNCH=block; the default for contexts with few scenarios,
// sf_api.cu): one block runs one scenario through all n_windows windows of the call -- warp 0 the
// coordinator (W0-W5), then every warp advances a share of the scenario's instances in parallel
// (W6-W7), then warp 0 the reward ledger (W8-W9) -- with __syncthreads() between the phases instead
// of kernel boundaries.  A single scenario (C1-C3) is one latency-bound chain per window, so the
// three launches and their hand-offs per window are what this removes.
namespace sf {

template <int KS, int NW>
__global__ void __launch_bounds__(32 * NW) k_window_block(GParams P, Dev D, int n_windows) {
  __shared__ union { Stage coord; EvStage led; } st0;
  __shared__ AdvStage adv[NW];
  const int s = blockIdx.x;
  const int w = threadIdx.x >> 5;
  const ScenConst C = D.sc[s];
  for (int win = 0; win < n_windows; ++win) {
    if (w == 0) coord_scenario_fit<KS>(P, D, s, st0.coord, C);
    __syncthreads();
    for (int i = w; i < C.I; i += NW) advance_instance(P, D, C.inst_off + i, adv[w], s, C);
    __syncthreads();
    if (w == 0) ledger_scenario(P, D, s, st0.led, C);
    __syncthreads();
  }
}

}  // namespace sf

void sf_launch_window_block(const sf::GParams &P, const sf::Dev &D, int n_scen, int max_inst, int n_windows,
                            cudaStream_t st) {
  if (max_inst <= 32) sf::k_window_block<1, 16><<<n_scen, 32 * 16, 0, st>>>(P, D, n_windows);
  else if (max_inst <= 64) sf::k_window_block<2, 8><<<n_scen, 32 * 8, 0, st>>>(P, D, n_windows);
  else sf::k_window_block<4, 8><<<n_scen, 32 * 8, 0, st>>>(P, D, n_windows);
}
