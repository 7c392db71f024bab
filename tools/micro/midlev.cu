// In-graph cost of one pre / post pass on a mid-size level (sides 255 ..
// 2047) for each kernel family: overlapped tiles (kc_tile.cuh), streaming
// (kc_stream.cuh) and the per-op kernels (kc_grid_kernels.cuh).  Each
// variant is captured N times back to back into one graph; us per pass.
//   ./midlev [nu]
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2010_00626_b200/csrc/kc_grid_kernels.cuh"
#include "../../paper_2010_00626_b200/csrc/kc_stream.cuh"
#include "../../paper_2010_00626_b200/csrc/kc_tile.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

static cudaStream_t s;
template <typename F>
static double time_graph(F body, int N = 40) {
  cudaGraph_t g; cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < N; ++i) body();
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
  return best * 1e3 / N;
}

int main(int argc, char** argv) {
  const int nu = argc > 1 ? atoi(argv[1]) : 2;
  if (nu != 2) { printf("nu=2 only\n"); return 1; }
  CK(cudaStreamCreate(&s));
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  St9 st{};
  const double w[9] = {0.249975, -0.50005, -0.249975, -0.50005, 2.0002, -0.50005, -0.249975, -0.50005, 0.249975};
  for (int k = 0; k < 9; ++k) st.w[k] = w[k];
  st.center = 2.0002; st.c = 0.8 / 2.0002;
  for (int m : {255, 511, 1023, 2047}) {
    const int mc = (m - 1) / 2, P = kc_pitch(m), Pc = kc_pitch(mc);
    const size_t el = (size_t)(m + 2) * P, elc = (size_t)(mc + 2) * Pc;
    double *u, *f, *uo, *fc, *vc;
    CK(cudaMalloc(&u, el * 8)); CK(cudaMalloc(&f, el * 8)); CK(cudaMalloc(&uo, el * 8));
    CK(cudaMalloc(&fc, elc * 8)); CK(cudaMalloc(&vc, elc * 8));
    std::vector<double> h(el, 0.0), hc(elc, 0.0);
    for (int y = 0; y < m; ++y) for (int x = 0; x < m; ++x) h[kc_idx(P, y, x)] = ((y * 7 + x * 3) % 11) * 0.1;
    for (int y = 0; y < mc; ++y) for (int x = 0; x < mc; ++x) hc[kc_idx(Pc, y, x)] = ((y * 5 + x) % 7) * 0.1;
    CK(cudaMemcpy(u, h.data(), el * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f, h.data(), el * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(uo, h.data(), el * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(vc, hc.data(), elc * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(fc, hc.data(), elc * 8, cudaMemcpyHostToDevice));
    // tiles
    TileParams tp{u, f, uo, fc, vc, m, P, mc, Pc, (m + KT_TX - 1) / KT_TX, st};
    const int tiles = tp.tiles_x * ((m + KT_TY - 1) / KT_TY);
    const int smp = 8 * kt_smem_doubles(3), smq = 8 * kt_smem_doubles(2);
    cudaFuncSetAttribute(k_tile_pre<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smp);
    cudaFuncSetAttribute(k_tile_post<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smq);
    const double t_tpre = time_graph([&] { k_tile_pre<2, false><<<tiles, KT_THREADS, smp, s>>>(tp); });
    // column tiles: bit-exact against k_tile_pre, then timed
    auto ctile = [&](auto kern, int ty, const char* name, int nwarp = KC_CT_NW) {
      TileParams cp = tp;
      cp.tiles_x = (m + KC_CT_TX - 1) / KC_CT_TX;
      const int nt = cp.tiles_x * ((m + ty - 1) / ty);
      std::vector<double> a(el), b(el), ac(elc), bc(elc);
      CK(cudaMemset(uo, 0, el * 8)); CK(cudaMemset(fc, 0, elc * 8));
      k_tile_pre<2, false><<<tiles, KT_THREADS, smp, s>>>(tp);
      CK(cudaStreamSynchronize(s));
      CK(cudaMemcpy(a.data(), uo, el * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(ac.data(), fc, elc * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemset(uo, 0, el * 8)); CK(cudaMemset(fc, 0, elc * 8));
      kern<<<nt, nwarp * 32, 0, s>>>(cp);
      CK(cudaStreamSynchronize(s));
      CK(cudaMemcpy(b.data(), uo, el * 8, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(bc.data(), fc, elc * 8, cudaMemcpyDeviceToHost));
      const bool same = memcmp(a.data(), b.data(), el * 8) == 0 && memcmp(ac.data(), bc.data(), elc * 8) == 0;
      const double t = time_graph([&] { kern<<<nt, nwarp * 32, 0, s>>>(cp); });
      printf("   m=%4d ctile pre %s: %6.2f us (%d blocks) %s\n", m, name, t, nt, same ? "bit-exact" : "MISMATCH");
    };
    ctile(k_ctile_pre<2, false, 16>, 16, "TY=16");
    ctile(k_ctile_pre<2, false, 32>, 32, "TY=32");
    ctile(k_ctile_pre<2, false, 48>, 48, "TY=48");
    ctile(k_ctile_pre<2, false, 32, 16>, 32, "TY=32 16w", 16);
    ctile(k_ctile_pre<2, false, 16, 4>, 16, "TY=16 4w", 4);
    {  // column-tile post: bit-exact against k_tile_post, then timed
      TileParams cp = tp;
      cp.tiles_x = (m + KC_CT_TX - 1) / KC_CT_TX;
      for (int ty : {16, 32}) {
        const int nt = cp.tiles_x * ((m + ty - 1) / ty);
        std::vector<double> a(el), b(el);
        CK(cudaMemcpy(uo, h.data(), el * 8, cudaMemcpyHostToDevice));
        k_tile_post<2, false><<<tiles, KT_THREADS, smq, s>>>(tp);
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpy(a.data(), uo, el * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(uo, h.data(), el * 8, cudaMemcpyHostToDevice));
        auto kern = ty == 16 ? k_ctile_post<2, false, 16> : k_ctile_post<2, false, 32>;
        kern<<<nt, KC_CT_NW * 32, 0, s>>>(cp);
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpy(b.data(), uo, el * 8, cudaMemcpyDeviceToHost));
        const bool same = memcmp(a.data(), b.data(), el * 8) == 0;
        const double t = time_graph([&] { kern<<<nt, KC_CT_NW * 32, 0, s>>>(cp); });
        printf("   m=%4d ctile post TY=%d: %6.2f us (%d blocks) %s\n", m, ty, t, nt, same ? "bit-exact" : "MISMATCH");
      }
    }
    const double t_tpost = time_graph([&] { k_tile_post<2, false><<<tiles, KT_THREADS, smq, s>>>(tp); });
    // streaming (kc_engine.cu ks_params / ks_choose_nq)
    auto sparams = [&](int D, const void* fn, int* nw) {
      StreamParams p{};
      p.u = u; p.f = f; p.uo = uo; p.fc = fc; p.vc = vc; p.m = m; p.P = P; p.mc = mc; p.Pc = Pc; p.s = st;
      p.rows = m; p.gy0 = 0; p.mg = m; p.hb = 1; p.mcr = mc; p.hbc = 1;
      const int npb = (KS_BAND - 1 - D - 2 * ((D + 2) / 2)) / 2;
      p.nbands = (mc + 1 + npb - 1) / npb;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ks_smem_bytes(D));
      int blocks = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, 128, ks_smem_bytes(D));
      int slots = std::max(blocks, 1) * 4 * nsm;
      auto choose = [&](int sl) { int k = std::max(sl / p.nbands, 1); return std::max((mc + 1 + k - 1) / k, 2); };
      p.nq = choose(slots);
      if (10 * (2 * D + 1) > 2 * p.nq) p.nq = choose(std::min(slots, 16 * nsm));
      *nw = p.nbands * ((mc + 1 + p.nq - 1) / p.nq);
      return p;
    };
    int nw1, nw2;
    StreamParams sp1 = sparams(3, (const void*)k_pre<2, false>, &nw1);
    StreamParams sp2 = sparams(2, (const void*)k_post<2, false, 0>, &nw2);
    const double t_spre = time_graph([&] { k_pre<2, false><<<(nw1 + 3) / 4, 128, ks_smem_bytes(3), s>>>(sp1); });
    const double t_spost = time_graph([&] { k_post<2, false, 0><<<(nw2 + 3) / 4, 128, ks_smem_bytes(2), s>>>(sp2); });
    // per-op
    const dim3 gj((m + KC_BX - 1) / KC_BX, (m + KC_BY * KC_RY - 1) / (KC_BY * KC_RY));
    const dim3 gr((mc + KC_BX - 1) / KC_BX, (mc + KC_BY - 1) / KC_BY);
    const dim3 gp((m + KC_BX - 1) / KC_BX, (m + KC_BY - 1) / KC_BY);
    const dim3 bl(KC_BX, KC_BY);
    const double t_opre = time_graph([&] {
      k_jacobi<false><<<gj, bl, 0, s>>>(u, f, uo, m, m, P, st);
      k_jacobi<false><<<gj, bl, 0, s>>>(uo, f, u, m, m, P, st);
      k_resid_restrict<false><<<gr, bl, 0, s>>>(u, f, fc, mc, mc, P, Pc, st);
    });
    const double t_opost = time_graph([&] {
      k_prolong_add<false><<<gp, bl, 0, s>>>(u, vc, m, m, P, Pc);
      k_jacobi<false><<<gj, bl, 0, s>>>(u, f, uo, m, m, P, st);
      k_jacobi<false><<<gj, bl, 0, s>>>(uo, f, u, m, m, P, st);
    });
    const double t_j = time_graph([&] { k_jacobi<false><<<gj, bl, 0, s>>>(u, f, uo, m, m, P, st); });
    printf("m=%4d  tile pre %6.2f post %6.2f | stream pre %6.2f post %6.2f (warps %d/%d) | per-op pre %6.2f post %6.2f (jacobi %5.2f) us\n",
           m, t_tpre, t_tpost, t_spre, t_spost, nw1, nw2, t_opre, t_opost, t_j);
    cudaFree(u); cudaFree(f); cudaFree(uo); cudaFree(fc); cudaFree(vc);
  }
  return 0;
}
