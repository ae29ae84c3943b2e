// sgm_codegen.h — planner + CUDA code generator for instantiated sGraph candidates.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/sgm.h"

namespace sgmcg {

// One TMA tensor map the launch must encode: the whole input tensor `slot`
// (rank-4, row-major, dims d[0..3] outermost first), box {box0 (innermost),
// box1, 1, 1}.
struct TmaSpec {
  int slot = 0;
  int elem_bytes = 2;   // 2: bf16, 4: fp32 / u32
  int u32 = 0;          // 4-byte finite-field residues: UINT32 tensor map (bits copied as they are)
  int box0 = 64, box1 = 64, box2 = 1, box3 = 1;
  int swizzle128 = 0;
  int64_t dims[4] = {1, 1, 1, 1};
};

struct GenResult {
  int status = SGM_OK;
  std::string error;
  std::string source;       // CUDA C++ for NVRTC
  std::string kernel_name;  // extern "C" entry
  int64_t logical_blocks = 1;
  int64_t ctas = 1;
  int cluster = 1;
  int threads = 256;
  int smem_bytes = 0;
  int loop_parts = 1;
  int64_t free_parts = 1;
  int64_t scratch_bytes = 0;   // total global scratch (all CTAs)
  int64_t scratch_per_cta = 0;
  int64_t trace_off = -1;      // byte offset of the trace region inside each CTA's scratch
  int n_tcgen05 = 0;
  int n_tma = 0;               // streamed matmuls fed by the TMA producer warp
  int ring_slots = 0;
  int ctas_per_sm = 1;         // the plan counts on this many co-resident CTAs per SM
  std::vector<TmaSpec> tmaps;
  std::string summary;
};

// Validate the descriptor, derive tile shapes from the mapping exactly as the
// reference interpreter slices (interp.py:90-125), plan the CTA/cluster
// decomposition and emit the kernel source.
GenResult generate(const sgm_plan_desc& desc, int num_sms);

// Helpers shared with the runtime.
uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull);
uint32_t ff_const(int64_t num, int64_t den);  // num * den^-1 mod 2^31-1

}  // namespace sgmcg
