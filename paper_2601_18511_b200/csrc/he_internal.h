// he_internal.h -- private definitions shared by the C-ABI translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "../../include/he_b200.h"
#include "he_kernels.h"

struct he_context {
  he_params p;
  he::RingDims R;
  he::NttTable ntt[3];     // degree N: q0, q1, P
  he::NttTable ntt_rh[3];  // degree rhombus_degree: q0, q1, P
  int sm_count = 148;
};

struct he_pcmm_plan {
  const he_context* ctx;
  uint32_t n_out, n_in, d_w, d0, d1, width;
  const int8_t* digits;
  CUtensorMap tmA;
  he::GemmEpiConst epi;
  // K7 spectral a-part (he_pcmm_spectral_prepare); algo 0 = K1 over every GEMM column
  int algo = 0;
  uint32_t L = 0, r_pad = 0, kg = 0, dsp[2] = {0, 0};   // kg: G^ row bytes (16 ceil(R / 16)), r_pad: A^ row bytes
  uint32_t ob = 0, nblk = 0, nbp = 0;  // outputs per block (L - k), blocks, blocks padded to 32
  uint64_t spec_off[2] = {0, 0};       // S3 recombination offsets (multiples of q_i)
  const int8_t* spec_w = nullptr;  // caller-owned: G^ limb 0 [L][D0][n_out][kg], then limb 1
  CUtensorMap tmSA[2];
  he::SpecTable st[2];
  // he_pcmm_profile: per-stage CUDA events recorded on the launching stream (profiling state only)
  static constexpr int kStages = 6;
  mutable bool prof_on = false;
  mutable std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[kStages];
  cudaEvent_t prof_begin(int stage, cudaStream_t s) const {
    if (!prof_on) return nullptr;
    cudaEvent_t e0 = nullptr;
    cudaEventCreate(&e0);
    cudaEventRecord(e0, s);
    prof_ev[stage].emplace_back(e0, nullptr);
    return e0;
  }
  void prof_end(int stage, cudaStream_t s) const {
    if (!prof_on || prof_ev[stage].empty()) return;
    cudaEvent_t e1 = nullptr;
    cudaEventCreate(&e1);
    cudaEventRecord(e1, s);
    prof_ev[stage].back().second = e1;
  }
  void prof_clear() const {
    for (auto& v : prof_ev) {
      for (auto& pr : v) {
        if (pr.first) cudaEventDestroy(pr.first);
        if (pr.second) cudaEventDestroy(pr.second);
      }
      v.clear();
    }
  }
  ~he_pcmm_plan() {
    prof_clear();
    he::spec_table_free(st[0]);
    he::spec_table_free(st[1]);
  }
};

he_status fail(he_status s, const char* fmt, ...);
he_status cuda_fail(cudaError_t e, const char* what);
#define HE_CUDA(call, what)                              \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, what);   \
  } while (0)
