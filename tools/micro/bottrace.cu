// Per-phase cycle trace of the bottom kernel on a synthetic 63^2..1 hierarchy.
#define KC_BOT_TRACE 8192
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2010_00626_b200/csrc/kc_bottom.cuh"

int main(int argc, char** argv) {
  int kappa = argc > 1 ? atoi(argv[1]) : 3;
  const int cs = argc > 3 ? atoi(argv[3]) : 1;  // cluster size (16: entry 255^2, strips down to 31^2)
  const int m0 = argc > 4 ? atoi(argv[4]) : (cs > 1 ? 127 : 63), P = kc_pitch(m0);  // argv[4]: entry side
  int nlev = 0;
  while ((1 << nlev) - 1 < m0) ++nlev;
  int nstrip = 0;
  while (cs > 1 && nstrip < nlev && bot_m(m0, nstrip) >= KC_CLU_MIN_STRIP) ++nstrip;
  size_t el = (size_t)(m0 + 2) * P;
  std::vector<double> hf(el, 0.0);
  for (int y = 0; y < m0; ++y) for (int x = 0; x < m0; ++x) hf[kc_idx(P, y, x)] = ((y * 7 + x * 3) % 11) * 0.1;
  double *gv, *gf;
  cudaMalloc(&gv, el * 8); cudaMalloc(&gf, el * 8);
  cudaMemset(gv, 0, el * 8);
  cudaMemcpy(gf, hf.data(), el * 8, cudaMemcpyHostToDevice);
  BotParams bp{};
  bp.nlev = nlev;
  for (int d = 0; d < nlev; ++d) {
    for (int k = 0; k < 9; ++k) bp.st[d].w[k] = -0.1;
    bp.st[d].w[4] = 1.0; bp.st[d].center = 1.0; bp.st[d].c = 0.8;
  }
  BotBuilder b; b.m0 = m0; b.nlev = nlev; b.nu1 = 2; b.nu2 = 2; b.vz = 1;
  b.tiny = argc > 2 ? atoi(argv[2]) != 0 : true;
  b.nstrip = nstrip;
  // argv[5] = 1: side-15 frame operators (FMA build; dummy matrix values),
  // the five blocks B1, B2, A1, B3, A2 resident
  const bool mv = argc > 5 && atoi(argv[5]) != 0;
  // argv[6] = 1: deep halos on the 63^2 strips (PH_FRAME63; entry 127, 16 CTAs)
  bp.deep = (argc > 6 && atoi(argv[6]) != 0 && cs == 16 && m0 == 127 && nstrip == 2) ? 1 : -1;
  b.deep = bp.deep;
  // argv[7] = 1: deep halos on the 127^2 entry strips too (PH_FRAME127)
  bp.deep0 = (argc > 7 && atoi(argv[7]) != 0 && bp.deep == 1) ? 1 : 0;
  b.deep0 = bp.deep0 != 0;
  bp.nu1 = 2; bp.nu2 = 2; bp.nstrip = nstrip; bot_geometry(bp, m0, cs);
  if (mv) {
    double* mats; cudaMalloc(&mats, sizeof(double) * KC_MV_NBLK * KC_MV_N * KC_MV_LD);
    cudaMemset(mats, 0, sizeof(double) * KC_MV_NBLK * KC_MV_N * KC_MV_LD);
    const int R = (KC_MV_N + cs - 1) / cs, order[5] = {1, KC_MV_PAIR0, KC_MV_PAIR0 + 1, KC_MV_PAIR0 + 2, 3};
    bp.mv_mats = mats; bp.mv_rows = R; bp.mv_off = (bp.total + 1) & ~1;
    const int nres = bp.deep0 ? 4 : 5;  // the deeper 127^2 strips leave room for 4 blocks
    for (int i = 0; i < KC_MV_NBLK; ++i) bp.mv_slot[i] = -1;  // the others are read from global memory
    for (int i = 0; i < nres; ++i) bp.mv_slot[order[i]] = i;
    b.mv_mask = (1u << KC_MV_NBLK) - 1;
    bp.mv_avail = (1 << KC_MV_NBLK) - 1;

  }
  b.top(kappa, kappa > 1 ? kappa - 1 : 0);
  bp.mv_copy = (int)b.mv_used;
  if (mv) for (int i = 0; i < KC_MV_NBLK; ++i) if (bp.mv_slot[i] < 0) bp.mv_copy &= ~(1 << i);
  unsigned* ds; cudaMalloc(&ds, b.out.size() * 4);
  cudaMemcpy(ds, b.out.data(), b.out.size() * 4, cudaMemcpyHostToDevice);
  bp.gv = gv; bp.gf = gf; bp.gP = P; bp.v_zero = 1; bp.sched = ds; bp.nsched = (int)b.out.size(); bp.final_cur = b.cur & 1;
  if (mv) bp.mv_xin = bp.mv_off + (bp.deep0 ? 4 : 5) * ((KC_MV_N + cs - 1) / cs) * KC_MV_LD;
  size_t smem = sizeof(double) * (mv ? (size_t)(bp.mv_xin + 2 * KC_MV_N) : (size_t)bp.total);
  cudaFuncSetAttribute(k_bottom, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_bottom, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(KC_BOT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int zero = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpyToSymbol(kc_bot_trace_n, &zero, sizeof(int));
    cudaMemcpyToSymbol(kc_bot_sub_n, &zero, sizeof(int));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_bottom, bp, m0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep == 1) printf("kappa=%d+%d: %.1f us, %zu phases %s\n", kappa, kappa - 1, ms * 1e3, b.out.size(), cudaGetErrorString(err));
  }
  {
    unsigned long long st[8];
    cudaMemcpyFromSymbol(st, kc_bot_stamp, sizeof(st));
    printf("  CTA-0 timeline (us): init %.2f, entry load %.2f, phases %.2f, write-back %.2f; kernel body %.2f\n",
           (st[1] - st[0]) * 1e-3, (st[2] - st[1]) * 1e-3, (st[3] - st[2]) * 1e-3, (st[4] - st[3]) * 1e-3,
           (st[4] - st[0]) * 1e-3);
    printf("  init: zero %.2f, sched %.2f, setup %.2f\n", (st[5] - st[0]) * 1e-3, (st[6] - st[5]) * 1e-3, (st[1] - st[6]) * 1e-3);
    // in-graph: 20 back-to-back launches
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t g; cudaGraphExec_t ge;
    cfg.stream = s;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, k_bottom, bp, m0);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("  in-graph: %.2f us per launch\n", ms * 1e3 / 20);
    cfg.stream = 0;
  }
  int n; cudaMemcpyFromSymbol(&n, kc_bot_trace_n, sizeof(int));
  std::vector<long long> t(n); std::vector<int> op(n);
  cudaMemcpyFromSymbol(t.data(), kc_bot_trace, n * 8);
  cudaMemcpyFromSymbol(op.data(), kc_bot_trace_op, n * 4);
  std::vector<long long> te(n);
  cudaMemcpyFromSymbol(te.data(), kc_bot_trace_end, n * 8);
  double sum[16][8] = {}, cmp[16][8] = {}; int cnt[16][8] = {};
  for (int i = 0; i + 1 < n; ++i) {
    int o = op[i] / 16, d = op[i] % 16;
    sum[o][d] += t[i + 1] - t[i]; cmp[o][d] += te[i] - t[i]; cnt[o][d]++;
  }
  const char* nm[13] = {"jacobi", "resid", "restrict", "prolong", "join", "j2z", "rr", "pj", "tiny", "csync", "frame31",
                        "frame63", "frame127"};
  for (int o = 0; o < 13; ++o) for (int d = 0; d < nlev; ++d) if (cnt[o][d])
    printf("  %-9s level %d (m=%3d): %5d phases, %7.0f cycles avg (thread 0 to its barrier %5.0f), %9.0f total\n", nm[o], d,
           bot_m(m0, d), cnt[o][d], sum[o][d] / cnt[o][d], cmp[o][d] / cnt[o][d], sum[o][d]);
  printf("phases traced: %d, total cycles %lld\n", n, n > 1 ? t[n - 1] - t[0] : 0);
  {  // sub-phase stamps of the compiled deep frames: 1 pre127 | 2 ... pre63 | 3 frames31 | 4 post63 | 5 ... post127 | 6
    int ns = 0;
    cudaMemcpyFromSymbol(&ns, kc_bot_sub_n, sizeof(int));
    std::vector<long long> ts(ns);
    std::vector<int> cs(ns);
    cudaMemcpyFromSymbol(ts.data(), kc_bot_sub, ns * 8);
    cudaMemcpyFromSymbol(cs.data(), kc_bot_sub_code, ns * 4);
    const char* what[17] = {"", "pre127", "pre63", "frames31", "post63", "post127", "end", "f31 pre-sweeps",
                            "f31 residual", "f31 restrict", "f31 frame15", "f31 prolong", "f31 post-sweeps", "f31 end", "mv wait", "mv pack", "mv rows", };
    double acc[17] = {};
    int cnt[17] = {};
    for (int i = 0; i + 1 < ns; ++i) {
      acc[cs[i]] += ts[i + 1] - ts[i];
      cnt[cs[i]]++;
    }
    // codes 3 (frames31) now include the stamps 7..13 inside: sum them back
    for (int c = 7; c < 17; ++c) if (c != 13) acc[3] += acc[c];
    for (int c = 1; c < 17; ++c)
      if (acc[c] > 0 && c != 6) printf("  deep frames: %-16s %8.0f cycles in %d intervals (%.0f each)\n", what[c], acc[c],
                                       cnt[c], acc[c] / (cnt[c] ? cnt[c] : 1));
  }
  return 0;
}
