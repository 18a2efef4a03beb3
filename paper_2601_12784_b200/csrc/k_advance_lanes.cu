// k_advance_lanes.cu -- decode-advance kernel with one lane per instance: one warp
// per block advances kLanes consecutive instances; the procedure is advance_lanes() in advance_lanes.cuh.
#include "advance_lanes.cuh"

namespace sf {

struct LaneBlockSmem {
  LaneSmem lanes;
  AdvStage stage;                                  // warp path for instances beyond kLS slots
};

__global__ void __launch_bounds__(32) k_advance_lanes(GParams P, Dev D, int n_inst_total) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LaneBlockSmem &sm = *reinterpret_cast<LaneBlockSmem *>(smem_raw);
  pdl_trigger();                                   // the ledger kernel may be scheduled now
  const int gi0 = blockIdx.x * kLanes;
  advance_lanes(P, D, gi0, n_inst_total, sm.lanes, sm.stage);
  // per instance: its writes, then the scenario's count of finished advances (release)
  const int gi = gi0 + (int)threadIdx.x;
  fence_release();                                 // this lane's writes, device-wide
  __syncwarp();
  if ((int)threadIdx.x < kLanes && gi < n_inst_total) add_release(&D.f_adv[D.inst_scen[gi]], 1);
}

}  // namespace sf

void sf_launch_advance_lanes(const sf::GParams &P, const sf::Dev &D, int n_inst_total, cudaStream_t st) {
  static unsigned long long attr_set = 0;           // per device (bit = device ordinal)
  const int bytes = (int)sizeof(sf::LaneBlockSmem);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_set >> (dev & 63)) & 1ULL)) {
    cudaFuncSetAttribute(sf::k_advance_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr_set |= 1ULL << (dev & 63);
  }
  const int blocks = (n_inst_total + sf::kLanes - 1) / sf::kLanes;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks > 0 ? blocks : 1);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, sf::k_advance_lanes, P, D, n_inst_total);
}
