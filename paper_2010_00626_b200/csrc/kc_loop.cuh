// kc_loop.cuh — the stand-alone solve's device-resident loop state and stop
// test (cycle.py:332-353), shared by k_stop_check (kc_engine.cu) and the
// norm reduction that ends a loop iteration (k_norms_lanes, kc_stream.cuh).
#pragma once
#include <cuda_runtime.h>

#include "../../include/kcb200.h"

// advanced once per cycle inside the conditional WHILE graph of the solve
struct SolveState {
  double target, prev, reduction;
  int it, max_it, streak, status, stop_mode, pad;
  double* err_hist;
  double* res_hist;
};

// the conditional handles a stop test sets (set_rest: also an IF node's)
struct LoopCheck {
  cudaGraphConditionalHandle h_loop, h_rest;
  int set_rest;
  SolveState* st;
};

// one thread: record the norms e = ||v_it||, r = ||f - A v_it||, decide
// whether the loop goes on (cycle.py:338-353)
__device__ __forceinline__ void kc_stop_test(const LoopCheck& ck, double e, double r) {
  SolveState* st = ck.st;
  const int it = st->it;  // cycles completed
  st->err_hist[it] = e;
  st->res_hist[it] = r;
  const double cur = st->stop_mode == KC_STOP_ERROR ? e : r;
  if (it == 0) st->target = cur / st->reduction;  // cycle.py:338-341
  unsigned go = 1u;
  if (cur <= st->target) {  // cycle.py:347
    st->status = KC_STATUS_CONVERGED;
    go = 0u;
  } else if (it > 0) {  // cycle.py:350-353: five consecutive growth steps
    const int streak = cur > st->prev ? st->streak + 1 : 0;
    st->streak = streak;
    if (streak >= 5) {
      st->status = KC_STATUS_DIVERGED;
      go = 0u;
    }
  }
  st->prev = cur;
  if (go && it >= st->max_it) go = 0u;  // status stays MAX_CYCLES
  if (go) st->it = it + 1;
  cudaGraphSetConditional(ck.h_loop, go);
  if (ck.set_rest) cudaGraphSetConditional(ck.h_rest, go);
}
