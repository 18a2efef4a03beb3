// k_dyn.cu -- dataflow window kernel (DESIGN.md §8.2 "launch modes"): one persistent launch per
// window whose warps run the window's tasks as soon as their inputs are ready.
//
// Tasks: the coordinator of every scenario (W0-W5), the advance of every instance (W6-W7) and the
// ledger of every scenario (W8-W9).  Warps first take coordinator tasks in scenario order from a
// counter; a finished coordinator appends its instances' advance tasks to a ready queue, and the
// last finished advance of a scenario appends that scenario's ledger task.  Once the coordinator
// tasks are exhausted, warps take queue positions in order and wait for the position's task to
// be published.  Every unpublished position belongs to a task whose producer is already running
// on some warp (producers never wait on the queue), so the kernel cannot deadlock, and no warp
// waits for the slowest scenario of the grid -- only for its own scenario's dependencies.  The
// per-scenario order (coordinator, then its advances, then its ledger) is exactly that of the
// three-kernel path, so results are identical.
#include "advance.cuh"
#include "coord.cuh"
#include "ledger.cuh"

namespace sf {

constexpr int kDynWarps = 4;
#ifndef SF_DYN_MAXSLEEP
#define SF_DYN_MAXSLEEP 4096
#endif

union DynStage {
  Stage coord;
  AdvStage adv;
  EvStage led;
};

template <int KS>
__global__ void __launch_bounds__(32 * kDynWarps, KS == 1 ? 16 / kDynWarps : 8 / kDynWarps) k_window_dyn(GParams P, Dev D, int n_scen) {
  __shared__ DynStage st_all[kDynWarps];
  DynStage &ws = st_all[threadIdx.x >> 5];
  const unsigned lane = lane_id();
  int *const q = D.q_tasks;                         // [n_inst + n_scen]: 0 = not yet published
  const int n_dyn = D.q_total;                      // advance + ledger tasks of the window
  bool coord_phase = true;
  for (;;) {
    if (coord_phase) {
      int s = 0;
      if (lane == 0) s = atomicAdd(&D.q_ctr[0], 1);
      s = __shfl_sync(0xffffffffu, s, 0);
      if (s < n_scen) {
        SF_TRACE_AT(4LL * s);
        coord_scenario_fit<KS>(P, D, s, ws.coord, D.sc[s]);
        SF_TRACE_AT(4LL * s + 1);
        __threadfence();
        __syncwarp();
        // publish this scenario's advance tasks (gi + 1)
        const int I = D.sc[s].I, off = D.sc[s].inst_off;
        int base = 0;
        if (lane == 0) base = atomicAdd(&D.q_ctr[1], I);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < I; i += 32) st_release32(&q[base + i], off + i + 1);
        __syncwarp();
        continue;
      }
      coord_phase = false;
    }
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&D.q_ctr[2], 1);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (pos >= n_dyn) break;
    int t = 0;
    if (lane == 0) {
      // exponential backoff: idle warps must not steal issue slots from the running tasks
      unsigned ns = 64;
      while ((t = ld_acquire32(&q[pos])) == 0) {
        __nanosleep(ns);
        ns = min(ns * 2, (unsigned)SF_DYN_MAXSLEEP);
      }
    }
    __syncwarp();
    t = ld_acquire32(&q[pos]);                      // every lane acquires the producer's writes
    if (t > 0) {                                    // advance of global instance gi
      const int gi = t - 1;
      SF_TRACE_AT(4LL * P.n_scen + 2LL * gi);
      {
        const int s = D.inst_scen[gi];
        advance_instance(P, D, gi, ws.adv, s, D.sc[s]);
      }
      SF_TRACE_AT(4LL * P.n_scen + 2LL * gi + 1);
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        const int s = D.inst_scen[gi];
        if (atomicAdd(&D.q_done[s], 1) + 1 == D.sc[s].I) {   // last instance: publish the ledger
          __threadfence();                          // (cumulative over the other instances' fences)
          const int b = atomicAdd(&D.q_ctr[1], 1);
          st_release32(&q[b], -(s + 1));
        }
      }
      __syncwarp();
    } else {                                        // ledger of scenario s
      const int s = -t - 1;
      SF_TRACE_AT(4LL * s + 2);
      ledger_scenario(P, D, s, ws.led, D.sc[s]);
      SF_TRACE_AT(4LL * s + 3);
    }
  }
}

}  // namespace sf

int sf_dyn_blocks(int max_inst) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (max_inst <= 32) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sf::k_window_dyn<1>, 32 * sf::kDynWarps, 0);
  else if (max_inst <= 64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sf::k_window_dyn<2>, 32 * sf::kDynWarps, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sf::k_window_dyn<4>, 32 * sf::kDynWarps, 0);
  return sms * (per_sm > 0 ? per_sm : 1);
}

void sf_launch_window_dyn(const sf::GParams &P, const sf::Dev &D, int n_scen, int max_inst, int blocks, cudaStream_t st) {
  if (max_inst <= 32) sf::k_window_dyn<1><<<blocks, 32 * sf::kDynWarps, 0, st>>>(P, D, n_scen);
  else if (max_inst <= 64) sf::k_window_dyn<2><<<blocks, 32 * sf::kDynWarps, 0, st>>>(P, D, n_scen);
  else sf::k_window_dyn<4><<<blocks, 32 * sf::kDynWarps, 0, st>>>(P, D, n_scen);
}
