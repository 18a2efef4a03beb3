// One-warp microbenchmark of the coordinator's versioned routing fast path (route_versioned_rep):
// cycles per decision with nothing else on the GPU, for ncu source-level stall analysis.
#include <cstdio>
#include <vector>
#include "../../paper_2601_12784_b200/csrc/coord.cuh"

using namespace sf;

__global__ void kbench(GParams P, Dev D, ScenConst C, int n_items, long long *out) {
  __shared__ Stage sg;
  const unsigned lane = lane_id();
  Cyc c;
  c.t = 1000; c.cu = 0; c.ps = 1; c.eta = 2; c.I = 4; c.G = 8; c.B = 64; c.n_v = n_items; c.n_vl = 0; c.vl_head = 0;
  c.n_ingested = 0; c.min_live_g = 0; c.window = 3; c.hash = 1469598103934665603ULL; c.cmd_n = 0; c.reserves = 0;
  c.mlq_err = 0; c.use_bits = 0; c.red_w = 4;
  InstRegs<1> S;
  S.v[0] = lane < 4 ? (int)(lane % 2) : 0; S.n[0] = lane < 4 ? 20 + 3 * (int)lane : 0; S.kv[0] = lane < 4 ? 30000 + 7000 * (long long)lane : 0;
  S.w[0] = 0;
  double Tcur = throughput_d(P, S.n[0], S.kv[0]);
  int acc = 0, arrn = 0, routed = 0;
  long long total = 0;
  int done_all = 0;
  for (int k0 = 0; k0 < n_items; k0 += 32) {
    const int kk = k0 + (int)lane;
    const int p_id = kk, p_vg = 0, p_l = 300 + (kk * 37) % 900;
    const long long p_ready = 0;
    const double p_thr = __dmul_rn(P.mu, ideal_gain_d(P, p_l));
    bool stop = false, hit = false;
    const int nbv = min(32, n_items - k0);
    const long long t0 = clock64();
    const int done = route_versioned_rep(P, D, C, c, S, Tcur, acc, arrn, sg, -1, nbv, p_id, p_vg, p_l, p_ready, p_thr,
                                         routed, stop, hit);
    total += clock64() - t0;
    done_all += done;
    if (stop) break;
  }
  if (lane == 0) { out[0] = total; out[1] = done_all; out[2] = routed; out[3] = (long long)c.hash; }
}

int main() {
  GParams P = {};
  P.B = 64; P.G = 8; P.Br = 64; P.Gr = 8;
  P.k1 = 72800; P.k2 = 1720000000LL; P.k3 = 125000000LL; P.k4 = 10700000000LL; P.k5 = 1; P.kp = 10000000; P.M = 1 << 20;
  P.k1i = (int)P.k1; P.k3i = (int)P.k3; P.kpi = (int)P.kp; P.gmag = ((1ULL << 40) + 7) / 8;
  P.mu = 0.3; P.phi_tp = 5.0; P.phi_wait = 3; P.delta = 1000000000000LL; P.r = 10000000000LL; P.q = 0; P.R = 0;
  P.cmdlog_cap = 0; P.n_scen = 1;
  const int n = 4096;
  Dev D = {};
  cudaMalloc(&D.loc, n); cudaMalloc(&D.tinst, 2 * n); cudaMalloc(&D.n_routes, 4 * n); cudaMalloc(&D.arr_id, 4 * 4 * n);
  cudaMalloc(&D.arr_t, 8 * 4 * n); cudaMalloc(&D.tsv_bits, n / 8); cudaMalloc(&D.cmdlog, 64);
  cudaMemset(D.n_routes, 0, 4 * n);
  ScenConst C = {};
  C.I = 4; C.eta = 2; C.cap = n; C.traj_off = 0; C.list_off = 0; C.bits_off = 0; C.cmd_off = 0;
  long long *out;
  cudaMalloc(&out, 64);
  for (int items : {32, 256, 1024}) {
    kbench<<<1, 32>>>(P, D, C, items, out);
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("items %5d decided %lld routed %lld: %.0f cycles per decision\n", items, h[1], h[2], (double)h[0] / (h[1] ? h[1] : 1));
  }
  return cudaDeviceSynchronize() != cudaSuccess;
}
