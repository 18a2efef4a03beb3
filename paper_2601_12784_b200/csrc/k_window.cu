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
// Block mode (SF_LAUNCH=block; the default for contexts with few scenarios, sf_api.cu): one block
// -- or one thread-block cluster for a scenario with many instances -- runs one scenario through all
// n_windows windows of the call: warp 0 the coordinator (W0-W5), then every warp advances a share of
// the scenario's instances in parallel (W6-W7), then warp 0 the reward ledger (W8-W9), with
// barriers between the phases instead of kernel boundaries.  A single scenario (C1-C3) is one
// latency-bound chain per window, so the three launches and their hand-offs per window are what
// this removes.
namespace sf {

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_idx() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster; release / acquire at cluster scope orders the global
// writes of one phase before the reads of the next (all global loads are L2 loads, -dlcm=cg)
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Cluster-per-scenario window kernel (block mode for scenarios with many instances): the CL CTAs
// of cluster k run scenario list[k] through all n_windows windows -- CTA 0's warp 0 the coordinator
// and the ledger, all CL * NW warps the advance of the scenario's instances (warp r * NW + w takes
// instances r * NW + w, + CL * NW, ...) -- with cluster barriers between the phases.  A large
// scenario's advance (I = 128: 16 instances per warp in one block) spreads over CL SMs.  CL = 1 is
// the plain block kernel over a scenario list.  Two barriers per window suffice: the ledger of window
// w and the coordinator of w + 1 run on the same warp, in order.
template <int KS, int NW, int CL>
__global__ void __launch_bounds__(32 * NW) k_window_cluster(GParams P, Dev D, const int *list, int n_windows) {
  __shared__ union { Stage coord; EvStage led; } st0;
  __shared__ AdvStage adv[NW];
  const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int s = list[CL > 1 ? (int)cluster_idx() : (int)blockIdx.x];
  const int w = threadIdx.x >> 5;
  const ScenConst C = D.sc[s];
  for (int win = 0; win < n_windows; ++win) {
    if (rank == 0 && w == 0) coord_scenario_fit<KS>(P, D, s, st0.coord, C);
    if constexpr (CL > 1) cluster_barrier(); else __syncthreads();
    for (int i = rank * NW + w; i < C.I; i += CL * NW) advance_instance(P, D, C.inst_off + i, adv[w], s, C);
    if constexpr (CL > 1) cluster_barrier(); else __syncthreads();
    if (rank == 0 && w == 0) ledger_scenario(P, D, s, st0.led, C);
    if constexpr (CL == 1) __syncthreads();     // not needed for ordering; keeps ptxas' 128-register
  }                                             // allocation of the 16-warp variant at its smallest spill
}

}  // namespace sf


template <int KS, int NW, int CL>
static cudaError_t launch_cluster(const sf::GParams &P, const sf::Dev &D, const int *list, int n, int n_windows,
                                  cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n * CL));
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CL > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, sf::k_window_cluster<KS, NW, CL>, P, D, list, n_windows);
}

// One scenario class of the block mode (sf_api.cu): ks instances per coordinator lane, cl CTAs per
// scenario.  Returns cudaErrorInvalidValue for an unsupported pair.
cudaError_t sf_launch_window_cluster(const sf::GParams &P, const sf::Dev &D, const int *list, int n, int ks, int cl,
                                     int n_windows, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (ks == 1 && cl == 1) return launch_cluster<1, 16, 1>(P, D, list, n, n_windows, st);
  if (ks == 1 && cl == 2) return launch_cluster<1, 8, 2>(P, D, list, n, n_windows, st);
  if (ks == 2 && cl == 1) return launch_cluster<2, 8, 1>(P, D, list, n, n_windows, st);
  if (ks == 2 && cl == 2) return launch_cluster<2, 8, 2>(P, D, list, n, n_windows, st);
  if (ks == 2 && cl == 4) return launch_cluster<2, 8, 4>(P, D, list, n, n_windows, st);
  if (ks == 4 && cl == 1) return launch_cluster<4, 8, 1>(P, D, list, n, n_windows, st);
  if (ks == 4 && cl == 2) return launch_cluster<4, 8, 2>(P, D, list, n, n_windows, st);
  if (ks == 4 && cl == 4) return launch_cluster<4, 8, 4>(P, D, list, n, n_windows, st);
  if (ks == 4 && cl == 8) return launch_cluster<4, 8, 8>(P, D, list, n, n_windows, st);
  return cudaErrorInvalidValue;
}

// Largest number of co-resident clusters of cl CTAs of the (ks, cl) kernel (cudaOccupancyMaxActiveClusters).
int sf_max_active_clusters(int ks, int cl) {
  cudaLaunchConfig_t cfg = {};
  const int nw = ks == 1 && cl == 1 ? 16 : 8;
  cfg.gridDim = dim3((unsigned)(cl * 64));
  cfg.blockDim = dim3(32 * nw);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaErrorInvalidValue;
  if (ks == 4 && cl == 8) e = cudaOccupancyMaxActiveClusters(&n, sf::k_window_cluster<4, 8, 8>, &cfg);
  else if (ks == 4 && cl == 4) e = cudaOccupancyMaxActiveClusters(&n, sf::k_window_cluster<4, 8, 4>, &cfg);
  else if (ks == 2 && cl == 4) e = cudaOccupancyMaxActiveClusters(&n, sf::k_window_cluster<2, 8, 4>, &cfg);
  else if (ks == 2 && cl == 2) e = cudaOccupancyMaxActiveClusters(&n, sf::k_window_cluster<2, 8, 2>, &cfg);
  return e == cudaSuccess ? n : 0;
}
