// sgm_codegen.cpp — planner + CUDA code generator for instantiated sGraph candidates.
//
// Input: an sgm_plan_desc (the POD lowering of a symfuse ConcreteGraph).
// Output: CUDA C++ source of ONE kernel that executes every logical block of the
// candidate, for NVRTC (sm_100a).
//
// Execution model (B200-first):
//  * A logical block (one grid coordinate, interp.py:156-158) is executed by
//    FREE x CLUSTER CTAs.  Free parts split an axis class that no node reduces
//    (independent CTAs, no communication); cluster parts split a reduced axis
//    class or the for-loop iterations (interp.py:162) and combine partial tiles
//    through DSMEM (cluster all-reduce), so the IR's "no inter-block reduction"
//    rule (graph.py:311-320) is kept while a logical block can still use many SMs.
//  * Tiles are materialised in shared memory (dense rank-4, compute type) with
//    liveness-based reuse; loader tiles consumed only as the large operand of a
//    matmul stay *views* of HBM and are streamed once (ld.global.nc, 16-byte
//    vectors, unrolled for memory-level parallelism).
//  * Loop-invariant body nodes are hoisted; accumulators are zeroed once and
//    summed per iteration (interp.py:171-176); the epilogue runs after the loop
//    with loop-split loaders on their last tile (interp.py:182-189).
//  * Savers write each output cell from exactly one CTA; write conflicts are
//    detected statically with the reference's outcome (interp.py:200-203).

#include "sgm_codegen.h"

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>

namespace sgmcg {

typedef int64_t i64;
typedef uint32_t u32;

uint64_t fnv1a(const std::string& s, uint64_t h) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

static const uint32_t kP = 0x7FFFFFFFu;
static uint32_t ffmul(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) % kP); }
static uint32_t ffpow(uint32_t a, uint32_t e) {
  uint32_t r = 1;
  while (e) {
    if (e & 1) r = ffmul(r, a);
    a = ffmul(a, a);
    e >>= 1;
  }
  return r;
}
uint32_t ff_const(int64_t num, int64_t den) {
  int64_t n = num % (int64_t)kP;
  if (n < 0) n += kP;
  int64_t d = den % (int64_t)kP;
  if (d < 0) d += kP;
  return ffmul((uint32_t)n, ffpow((uint32_t)d, kP - 2));
}

namespace {

// ST_XG: a bf16 input used only as the A operand of streamed tcgen05 matmuls; no
// tile, its A^T buffer is built straight from global memory (bf16 is exact: no
// fp32 staging tile, no residual rows)
enum Store { ST_NONE = 0, ST_VIEW, ST_SMEM, ST_GLOBAL, ST_XG };

struct Node {
  int kind = 0, nin = 0, in[2] = {-1, -1}, slot = -1, axis = -1;
  i64 cnum = 0, cden = 1;
  int rank = 0;
  i64 sh[4] = {1, 1, 1, 1};   // full per-block tile (rank-4, left padded)
  i64 sl[4] = {1, 1, 1, 1};   // per-CTA slice
  u32 gmask[4] = {0, 0, 0, 0};
  int lsplit[4] = {0, 0, 0, 0};
  int cls[4] = {-1, -1, -1, -1};
  bool body = false, hoist = false, loopdep = false;
  int store = ST_NONE;
  int off = 0;                 // smem offset or scratch offset
  std::vector<int> cons;
  u32 pend = 0;                // pending cluster bits (partial over these CTAs)
  bool gpend = false;          // partial over gsplit work items (reduced at the tail)
  bool lin = false;            // linear in its pending operands: computes on partials, reduced later
  bool deferred = false;
  // matmul realisation
  bool gemv = false;
  int vn = 1, ks = 1, unr = 4;
  bool shfl = false;
  i64 red_bytes = 0;
  int red_off = 0;
  i64 at_bytes = 0;  // k-major copy of the gemv A operand
  int at_off = 0;
  bool tc = false;   // tcgen05 realisation (bf16)
  int tc_kc = 16, tc_s = 4, tc_cols = 32;
  bool tma = false;  // B streamed by the TMA producer warp through the smem ring
  int tma_id = -1;
  int kc = 64;       // rows of B per ring stage
  int bw = 64;       // columns of B per TMA box (fp32 path)
  int acc = 1;       // TMEM accumulators per 128-column tile (tcgen05 path)
  bool staged = false;     // loader tile fetched by the producer (TMA) into a staging buffer
  int stage_id = -1, stage_off = 0, sbox = 0;
  bool inv = false;        // item-invariant: computed once per CTA, before the item loop
  bool xc = false;         // x-cached: independent of the grid coordinate; recomputed only when the
                           // item's other coordinates change (items run gx-fastest, contiguous per CTA)
  bool xb_shared = false;  // tcgen05 A^T buffer shared per A node (batch 1)
  bool xb_build = true;    // this consumer (re)builds the shared A^T buffer
};

struct Class {
  i64 extent = 1;
  bool reduced = false;
  bool twice = false;
  int parts = 1;
  bool cluster = false;  // split across the cluster (reduced) or free CTAs
  bool gsplit = false;   // reduced class split over work items, reduced at the tail through global memory
  int bit_shift = 0;     // cluster rank bit field
  i64 radix = 1;         // free-part / gsplit-part mixed radix
};

struct Ev {
  enum { NODE, FLUSH, GFLUSH, LOOP_BEGIN, LOOP_END } type;
  int node = -1;
  std::vector<int> flush;
};

struct Interval {
  int id;       // node id, or -(1+k) for transient k
  int start, end;
  i64 bytes;
};

struct Gen {
  const sgm_plan_desc& d;
  int num_sms;
  GenResult R;
  int ns = 0;      // number system
  int es = 4;      // storage element size
  int ec = 4;      // compute element size
  int ea = 4;      // accumulator element size
  int vecw = 4;    // elements per 16-byte vector (storage)
  int NT = 256;
  std::vector<Node> nodes;
  std::vector<Class> cls;
  i64 grid[3] = {1, 1, 1};
  int ngrid = 1;
  i64 nloop = 1;
  i64 LB = 1;
  int LP = 1;            // loop parts
  bool loop_gs = false;  // loop parts are gsplit work items (else cluster ranks)
  i64 GP = 1;            // gsplit parts per reduction group
  int loop_shift = 0;
  int CL = 1;            // cluster size
  i64 FP = 1;            // free parts
  bool loop_split_ok = false;
  i64 in_strides[SGM_MAX_SLOTS][4];
  i64 in_dims[SGM_MAX_SLOTS][4];
  i64 out_strides[SGM_MAX_SLOTS][4];
  i64 out_dims[SGM_MAX_SLOTS][4];
  int in_rank[SGM_MAX_SLOTS];
  int out_rank[SGM_MAX_SLOTS];
  std::vector<Ev> sched;
  int loop_begin_pos = -1, loop_end_pos = -1;
  std::vector<i64> flush_tmp_bytes;   // per schedule position
  std::map<std::pair<int, int>, int> flush_tmp_off;  // (pos,node) -> smem offset
  int smem_peak = 0;
  i64 scratch_per_cta = 0;
  i64 trace_off = -1;
  int budget = 200 * 1024;
  // TMA producer warp + ring (any tma matmul)
  bool prod = false;
  int nstaged = 0;
  i64 stage_total = 0;   // bytes of staging buffers (after the ring)
  bool no_tma_forced = false;
  double est_us = 0;     // planner's time estimate
  int ringS = 0;
  int ring_off = 0;
  // interleave: the big stream `ilv_big` issues k-chunks [0, ilv_kc) before the small
  // chain that starts at schedule position ilv_pos, the rest at its own position;
  // chain MMAs use TMEM columns from ilv_tmem (after the big stream's accumulators)
  int ilv_big = -1, ilv_pos = -1, ilv_kc = 0, ilv_tmem = 0;
  std::set<int> ilv_chain;
  bool emit_seg1 = false;  // emit_node(ilv_big) emits the first segment (build + MMAs only)
  // elementwise fusion: fused[n] = n is computed in registers inside its single
  // elementwise consumer's map (no smem tile write, no barrier)
  std::vector<char> fused;
  // accumulate-into: acc_first's MMAs land in acc_second's TMEM accumulators (no
  // read-back of its own), so acc_second's read-back is acc_first + acc_second and
  // the add node acc_add becomes a copy (LoRA: O = X@W + (X@A)@B)
  int acc_first = -1, acc_second = -1, acc_add = -1, acc_pre = 0;
  // finite field: a broadcast divisor tile consumed only by one div is inverted in
  // place once (Fermat inverse, ~60 modular products) and the div becomes a mul,
  // instead of one inverse per numerator element (QK-norm's [128, L] / [1, L])
  std::vector<char> inv_first;
  // x-cache: some nodes (>= one matmul) do not depend on the grid coordinate gx
  // (e.g. attention scores when only the head dim of V/O is split, LoRA's X@A when
  // only output columns are): each CTA runs a contiguous range of items gx-fastest
  // and recomputes those nodes only when the item's other coordinates change
  bool xcache = false, xcache_loop = false;
  static constexpr int kSlot = 32768;  // largest ring slot; plan_ring may pick 16 KB
  int slotB = 32768;
  static constexpr int kSmemCap = 225 * 1024;  // dynamic smem incl. ring alignment slack

  Gen(const sgm_plan_desc& desc, int sms) : d(desc), num_sms(sms) {}

  bool fail(int st, const std::string& msg) {
    if (R.status == SGM_OK) {
      R.status = st;
      R.error = msg;
    }
    return false;
  }

  // ------------------------------------------------------------------ setup
  bool load() {
    if (d.abi_version != SGM_ABI_VERSION) return fail(SGM_ERR_INVALID, "abi version mismatch");
    ns = d.numsys;
    switch (ns) {
      case SGM_F64: es = 8; ec = 8; ea = 8; break;
      case SGM_F32: es = 4; ec = 4; ea = 4; break;
      case SGM_BF16: es = 2; ec = 4; ea = 4; break;
      case SGM_FF: es = 4; ec = 4; ea = 8; break;
      default: return fail(SGM_ERR_INVALID, "unknown number system");
    }
    vecw = 16 / es;
    NT = d.hints.threads > 0 ? d.hints.threads : 256;
    if (NT % 32 || NT > 1024) return fail(SGM_ERR_INVALID, "threads must be a multiple of 32 <= 1024");
    if (d.hints.smem_budget > 0) budget = d.hints.smem_budget;
    if (d.n_grid < 1 || d.n_grid > 3) return fail(SGM_ERR_INVALID, "n_grid must be 1..3");
    ngrid = d.n_grid;
    for (int g = 0; g < ngrid; ++g) {
      if (d.grid[g] < 1) return fail(SGM_ERR_DIVISIBILITY, "grid size must be positive");
      grid[g] = d.grid[g];
      LB *= grid[g];
    }
    if (d.n_loop < 1) return fail(SGM_ERR_DIVISIBILITY, "loop size must be positive");
    nloop = d.n_loop;
    if (d.n_inputs < 0 || d.n_inputs > SGM_MAX_SLOTS || d.n_outputs < 0 || d.n_outputs > SGM_MAX_SLOTS)
      return fail(SGM_ERR_INVALID, "bad slot count");
    auto slot_setup = [&](const sgm_slot_desc& s, i64* dims, i64* strides, int& rank) -> bool {
      if (s.rank < 1 || s.rank > 4) return fail(SGM_ERR_INVALID, "slot rank must be 1..4");
      rank = s.rank;
      int pad = 4 - s.rank;
      for (int k = 0; k < 4; ++k) dims[k] = 1;
      for (int k = 0; k < s.rank; ++k) {
        if (s.dims[k] < 1) return fail(SGM_ERR_INVALID, "slot dims must be positive");
        dims[pad + k] = s.dims[k];
      }
      i64 st = 1;
      for (int k = 3; k >= 0; --k) {
        strides[k] = st;
        st *= dims[k];
      }
      return true;
    };
    for (int k = 0; k < d.n_inputs; ++k)
      if (!slot_setup(d.inputs[k], in_dims[k], in_strides[k], in_rank[k])) return false;
    for (int k = 0; k < d.n_outputs; ++k)
      if (!slot_setup(d.outputs[k], out_dims[k], out_strides[k], out_rank[k])) return false;
    if (d.n_nodes < 1 || d.n_nodes > SGM_MAX_NODES) return fail(SGM_ERR_INVALID, "bad node count");
    nodes.resize(d.n_nodes);
    for (int n = 0; n < d.n_nodes; ++n) {
      const sgm_node_desc& s = d.nodes[n];
      Node& x = nodes[n];
      x.kind = s.kind;
      x.nin = s.n_inputs;
      if (x.nin < 0 || x.nin > 2) return fail(SGM_ERR_INVALID, "bad input count");
      for (int k = 0; k < x.nin; ++k) {
        x.in[k] = s.inputs[k];
        if (x.in[k] < 0 || x.in[k] >= n) return fail(SGM_ERR_SHAPE, "forward edge in block graph");
        nodes[x.in[k]].cons.push_back(n);
      }
      x.slot = s.slot;
      x.axis = s.axis;
      x.cnum = s.const_num;
      x.cden = s.const_den;
      int want = 0;
      switch (x.kind) {
        case SGM_INPUT: want = 0; break;
        case SGM_OUTPUT: case SGM_EXP: case SGM_SILU: case SGM_SQUARE: case SGM_SQRT:
        case SGM_SUM: case SGM_ACCUM: case SGM_SCALE: want = 1; break;
        case SGM_MATMUL: case SGM_DIV: case SGM_MUL: case SGM_ADD: want = 2; break;
        default: return fail(SGM_ERR_UNSUPPORTED, "unknown op kind");
      }
      if (x.nin != want) return fail(SGM_ERR_INVALID, "wrong number of inputs for op");
      if (x.kind == SGM_INPUT && (x.slot < 0 || x.slot >= d.n_inputs)) return fail(SGM_ERR_INVALID, "bad input slot");
      if (x.kind == SGM_OUTPUT && (x.slot < 0 || x.slot >= d.n_outputs)) return fail(SGM_ERR_INVALID, "bad output slot");
      if (x.kind == SGM_SCALE && x.cden == 0) return fail(SGM_ERR_INVALID, "scale with zero denominator");
      for (int k = 0; k < 4; ++k) {
        x.gmask[k] = 0;
        x.lsplit[k] = 0;
      }
      if (x.kind == SGM_INPUT || x.kind == SGM_OUTPUT) {
        int r = x.kind == SGM_INPUT ? in_rank[x.slot] : out_rank[x.slot];
        int pad = 4 - r;
        for (int k = 0; k < r; ++k) {
          x.gmask[pad + k] = s.grid_mask[k] & ((1u << ngrid) - 1u);
          x.lsplit[pad + k] = (x.kind == SGM_INPUT) ? (s.loop_split[k] != 0) : 0;
        }
      }
    }
    return true;
  }

  // Tile shapes from the mapping, as the reference slices (interp.py:90-125);
  // op shapes with numpy semantics (interp.py:45-66).
  bool shapes() {
    char buf[256];
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      if (x.kind == SGM_INPUT) {
        x.rank = in_rank[x.slot];
        for (int k = 0; k < 4; ++k) {
          i64 w = in_dims[x.slot][k];
          if (w > 1) {
            for (int g = 0; g < ngrid; ++g)
              if (x.gmask[k] >> g & 1u) {
                if (w % grid[g]) {
                  snprintf(buf, sizeof buf, "extent %" PRId64 " not divisible by %" PRId64, w, grid[g]);
                  return fail(SGM_ERR_SHAPE, buf);
                }
                w /= grid[g];
              }
            if (x.lsplit[k]) {
              if (w % nloop) {
                snprintf(buf, sizeof buf, "extent %" PRId64 " not divisible by %" PRId64, w, nloop);
                return fail(SGM_ERR_SHAPE, buf);
              }
              w /= nloop;
            }
          } else {
            x.gmask[k] = 0;
            x.lsplit[k] = 0;
          }
          x.sh[k] = w;
        }
        continue;
      }
      const Node& a = nodes[x.in[0]];
      switch (x.kind) {
        case SGM_OUTPUT: case SGM_EXP: case SGM_SILU: case SGM_SQUARE: case SGM_SQRT:
        case SGM_ACCUM: case SGM_SCALE:
          x.rank = a.rank;
          for (int k = 0; k < 4; ++k) x.sh[k] = a.sh[k];
          break;
        case SGM_SUM: {
          x.rank = a.rank;
          if (x.axis < 0 || x.axis >= a.rank) return fail(SGM_ERR_INVALID, "axis out of bounds for sum");
          int ax = x.axis + 4 - a.rank;
          for (int k = 0; k < 4; ++k) x.sh[k] = (k == ax) ? 1 : a.sh[k];
          break;
        }
        case SGM_DIV: case SGM_MUL: case SGM_ADD: {
          const Node& b = nodes[x.in[1]];
          x.rank = std::max(a.rank, b.rank);
          for (int k = 0; k < 4; ++k) {
            if (a.sh[k] == b.sh[k] || b.sh[k] == 1) x.sh[k] = a.sh[k];
            else if (a.sh[k] == 1) x.sh[k] = b.sh[k];
            else return fail(SGM_ERR_INVALID, "operands could not be broadcast together");
          }
          break;
        }
        case SGM_MATMUL: {
          const Node& b = nodes[x.in[1]];
          if (a.rank < 2 || b.rank < 2) return fail(SGM_ERR_INVALID, "matmul operands need rank >= 2");
          if (a.sh[3] != b.sh[2]) return fail(SGM_ERR_INVALID, "matmul: mismatch in its core dimension");
          x.rank = std::max(a.rank, b.rank);
          for (int k = 0; k < 2; ++k) {
            if (a.sh[k] == b.sh[k] || b.sh[k] == 1) x.sh[k] = a.sh[k];
            else if (a.sh[k] == 1) x.sh[k] = b.sh[k];
            else return fail(SGM_ERR_INVALID, "matmul: batch dims could not be broadcast");
          }
          x.sh[2] = a.sh[2];
          x.sh[3] = b.sh[3];
          break;
        }
        default: return fail(SGM_ERR_UNSUPPORTED, "unknown op");
      }
    }
    // Saver regions must match their tiles (interp.py:196-199).
    for (auto& x : nodes) {
      if (x.kind != SGM_OUTPUT) continue;
      i64 reg[4];
      for (int k = 0; k < 4; ++k) {
        i64 w = out_dims[x.slot][k];
        if (w > 1) {
          for (int g = 0; g < ngrid; ++g)
            if (x.gmask[k] >> g & 1u) {
              if (w % grid[g]) return fail(SGM_ERR_SHAPE, "saver region not divisible");
              w /= grid[g];
            }
        } else {
          x.gmask[k] = 0;
        }
        reg[k] = w;
      }
      bool same = (x.rank == out_rank[x.slot]);
      for (int k = 0; k < 4; ++k) same = same && reg[k] == x.sh[k];
      if (!same) {
        std::ostringstream os;
        os << "saver slot " << x.slot << ": tile (";
        for (int k = 4 - x.rank; k < 4; ++k) os << x.sh[k] << (k < 3 ? "," : "");
        os << ") vs region (";
        for (int k = 4 - out_rank[x.slot]; k < 4; ++k) os << reg[k] << (k < 3 ? "," : "");
        os << ")";
        return fail(SGM_ERR_SHAPE, os.str());
      }
    }
    // Static write-conflict detection: two logical blocks write the same cell iff
    // some grid dim with size > 1 is absent from the saver's output map, or two
    // savers target one output (interp.py:200-203 raises on the second write).
    std::vector<int> writers(d.n_outputs, 0);
    for (auto& x : nodes) {
      if (x.kind != SGM_OUTPUT) continue;
      writers[x.slot]++;
      for (int g = 0; g < ngrid; ++g) {
        if (grid[g] <= 1) continue;
        bool used = false;
        for (int k = 0; k < 4; ++k) used = used || (x.gmask[k] >> g & 1u);
        if (!used) return fail(SGM_ERR_WRITE_CONFLICT, "output slot " + std::to_string(x.slot) +
                                                        ": blocks overwrite cells (grid dim " +
                                                        std::to_string(g) + " not in output map)");
      }
    }
    for (int s = 0; s < d.n_outputs; ++s) {
      if (writers[s] > 1 && LB >= 1)
        return fail(SGM_ERR_WRITE_CONFLICT, "output slot " + std::to_string(s) + " written by two savers");
    }
    return true;
  }

  // ------------------------------------------------------------ structure
  void structure() {
    // body = accumulators and their ancestors (graph.py:242-254)
    for (int n = (int)nodes.size() - 1; n >= 0; --n) {
      Node& x = nodes[n];
      if (x.kind == SGM_ACCUM) x.body = true;
      if (x.body)
        for (int k = 0; k < x.nin; ++k) nodes[x.in[k]].body = true;
    }
    for (auto& x : nodes) {
      bool dep = false;
      if (x.kind == SGM_INPUT)
        for (int k = 0; k < 4; ++k) dep = dep || x.lsplit[k];
      if (x.kind == SGM_ACCUM) dep = true;
      for (int k = 0; k < x.nin; ++k) dep = dep || nodes[x.in[k]].loopdep;
      x.loopdep = dep;
      x.hoist = x.body && !dep && !d.hints.no_hoist;
    }
    // loop split legality
    bool any_accum = false;
    for (auto& x : nodes) any_accum = any_accum || x.kind == SGM_ACCUM;
    loop_split_ok = nloop > 1 && any_accum && !d.hints.no_loop_split;
    for (auto& x : nodes) {
      for (int k = 0; k < x.nin; ++k) {
        const Node& p = nodes[x.in[k]];
        if (x.body && !x.hoist && p.kind == SGM_ACCUM && x.kind != SGM_ACCUM) loop_split_ok = false;
        if (x.body && p.kind == SGM_ACCUM) loop_split_ok = false;  // running totals consumed in-loop
        if (!x.body && p.body && !p.hoist && p.kind != SGM_ACCUM) loop_split_ok = false;
      }
    }
    // axis classes
    int N = (int)nodes.size();
    std::vector<int> par(N * 4);
    for (int i = 0; i < N * 4; ++i) par[i] = i;
    std::function<int(int)> find = [&](int v) { return par[v] == v ? v : par[v] = find(par[v]); };
    auto unite = [&](int a, int b) {
      a = find(a);
      b = find(b);
      if (a != b) par[a] = b;
    };
    auto id = [](int n, int k) { return n * 4 + k; };
    for (int n = 0; n < N; ++n) {
      Node& x = nodes[n];
      if (x.kind == SGM_INPUT) continue;
      if (x.kind == SGM_MATMUL) {
        const Node& a = nodes[x.in[0]];
        const Node& b = nodes[x.in[1]];
        for (int k = 0; k < 2; ++k) {
          if (x.sh[k] > 1 && a.sh[k] == x.sh[k]) unite(id(n, k), id(x.in[0], k));
          if (x.sh[k] > 1 && b.sh[k] == x.sh[k]) unite(id(n, k), id(x.in[1], k));
        }
        if (x.sh[2] > 1) unite(id(n, 2), id(x.in[0], 2));
        if (x.sh[3] > 1) unite(id(n, 3), id(x.in[1], 3));
        if (a.sh[3] > 1) unite(id(x.in[0], 3), id(x.in[1], 2));
      } else if (x.kind == SGM_SUM) {
        int ax = x.axis + 4 - nodes[x.in[0]].rank;
        for (int k = 0; k < 4; ++k)
          if (k != ax && x.sh[k] > 1) unite(id(n, k), id(x.in[0], k));
      } else {
        for (int j = 0; j < x.nin; ++j) {
          const Node& a = nodes[x.in[j]];
          for (int k = 0; k < 4; ++k)
            if (x.sh[k] > 1 && a.sh[k] == x.sh[k]) unite(id(n, k), id(x.in[j], k));
        }
      }
    }
    std::map<int, int> root2cls;
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < 4; ++k) {
        if (nodes[n].sh[k] <= 1) continue;
        int r = find(id(n, k));
        auto it = root2cls.find(r);
        int c;
        if (it == root2cls.end()) {
          c = (int)cls.size();
          root2cls[r] = c;
          Class C;
          C.extent = nodes[n].sh[k];
          cls.push_back(C);
        } else {
          c = it->second;
        }
        nodes[n].cls[k] = c;
        if (cls[c].extent != nodes[n].sh[k]) cls[c].twice = true;  // inconsistent: never split
      }
    for (int n = 0; n < N; ++n) {
      Node& x = nodes[n];
      for (int k = 0; k < 4; ++k)
        for (int j = k + 1; j < 4; ++j)
          if (x.cls[k] >= 0 && x.cls[k] == x.cls[j]) cls[x.cls[k]].twice = true;
      if (x.kind == SGM_MATMUL) {
        int c = nodes[x.in[0]].cls[3];
        if (c >= 0) cls[c].reduced = true;
      }
      if (x.kind == SGM_SUM) {
        int c = nodes[x.in[0]].cls[x.axis + 4 - nodes[x.in[0]].rank];
        if (c >= 0) cls[c].reduced = true;
      }
    }
  }

  // ------------------------------------------------------------ planning
  static i64 prod4(const i64* s) { return s[0] * s[1] * s[2] * s[3]; }

  i64 loader_traffic(const Node& x) const {
    i64 b = prod4(x.sh) * es;
    if (x.body && x.loopdep) b *= nloop;
    return b;
  }
  bool has_cls(const Node& x, int c) const {
    for (int k = 0; k < 4; ++k)
      if (x.cls[k] == c) return true;
    return false;
  }
  bool loader_loop_split(const Node& x) const {
    for (int k = 0; k < 4; ++k)
      if (x.lsplit[k]) return true;
    return false;
  }

  void decide_views() {
    for (auto& x : nodes) {
      if (x.kind == SGM_OUTPUT) { x.store = ST_NONE; continue; }
      x.store = ST_SMEM;
    }
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      if (x.kind != SGM_INPUT || x.cons.empty()) continue;
      bool view = true;
      for (int c : x.cons) {
        const Node& m = nodes[c];
        if (m.kind != SGM_MATMUL) { view = false; break; }
        int other = m.in[0] == n ? m.in[1] : m.in[0];
        if (m.in[0] == n && m.in[1] == n) { view = false; break; }
        const Node& o = nodes[other];
        // stream the larger operand; the smaller one is reused from smem
        if (prod4(x.sh) < prod4(o.sh) || (prod4(x.sh) == prod4(o.sh) && m.in[1] != n)) { view = false; break; }
        // ... unless it is loop-invariant and its consumer runs every loop iteration:
        // a view would be re-read from L2 on each of the n_loop iterations (A's split-KV
        // candidates re-read Q per key), a small smem tile is loaded once per item
        if (nloop > 1 && m.body && m.loopdep && !x.loopdep && prod4(x.sh) * ec <= 64 * 1024) { view = false; break; }
      }
      if (view) x.store = ST_VIEW;
    }
  }

  void slices() {
    for (auto& x : nodes)
      for (int k = 0; k < 4; ++k) {
        int c = x.cls[k];
        x.sl[k] = (c >= 0) ? x.sh[k] / cls[c].parts : x.sh[k];
      }
  }

  // ---- split planning: greedy search on a cost model of the persistent kernel.
  // A state assigns each axis class a power-of-two part count and a mode (free
  // CTAs / cluster ranks / gsplit work items) and the for-loop a part count
  // (cluster or gsplit).  Time model (calibrated on B200, tools/bench_tma_ring.cu,
  // tools/gemv_probe.py): HBM-unique bytes at ~5.9 TB/s, redundant re-reads at L2
  // speed, per-CTA stream rate <= ~60 GB/s, wave quantisation of work items over
  // co-resident clusters, and fixed per-item costs for cluster flushes (~5 us)
  // and gsplit tail reductions (~1.5 us).
  struct PlanState {
    std::vector<int> parts, mode;  // mode: 0 free, 1 cluster, 2 gsplit
    int lp = 1, lmode = 1;
  };

  void apply_state(const PlanState& st) {
    for (int c = 0; c < (int)cls.size(); ++c) {
      cls[c].parts = st.parts[c];
      cls[c].cluster = st.parts[c] > 1 && st.mode[c] == 1;
      cls[c].gsplit = st.parts[c] > 1 && st.mode[c] == 2;
    }
    LP = st.lp;
    loop_gs = st.lp > 1 && st.lmode == 2;
    finalize_layout();
  }

  static i64 resident_ctas(int cl, int sms) {
    // co-resident CTAs at one CTA per SM under GPC placement of clusters
    switch (cl) {
      case 1: case 2: return sms;
      case 4: return sms * 132 / 148;
      case 8: return sms * 120 / 148;
      default: return sms * 112 / 148;
    }
  }

  double plan_cost(bool* valid) {
    *valid = true;
    if (GP > 1 && CL > 1) { *valid = false; return 1e30; }
    slices();
    schedule();
    if (GP > 1 && !gs_tail_ok()) { *valid = false; return 1e30; }
    // shared-memory feasibility of this split (tiles + A^T buffers + a minimal ring)
    invariants();
    matmul_choices();
    plan_xcache();
    const int peak = allocate();
    const int cap = prod ? std::min(budget, kSmemCap - (3 * 16384 + 1024) - (int)stage_total) : budget;
    // soft penalty (10 us per KB over) so the search can walk out of infeasible splits
    const double over = peak > cap ? (double)(peak - cap) / 1024.0 * 1e-5 : 0.0;
    // residency: two CTAs per SM when the tiles leave room for a 3 x 16 KB ring in half an SM
    // measured: the occupancy of kernels that use tcgen05 (TMEM) is one CTA per SM
    // whatever their shared memory, so only CUDA-core kernels can pair up
    const bool two = prod && pairable() && !d.hints.one_cta && peak + 3 * 16384 + 1024 + stage_total <= 110 * 1024;
    const int cps = two ? 2 : 1;
    const i64 items = LB * FP * GP;
    const i64 slots = std::max<i64>(1, resident_ctas(CL, num_sms) * cps / CL);
    const i64 rounds = (items + slots - 1) / slots;
    const i64 active = std::min(items, slots) * CL;
    const double active_sms = std::max(1.0, std::min<double>(num_sms, (double)active / cps));
    // bytes in flight per SM bound its stream rate (Little's law, ~3 us loaded latency)
    const double inflight = prod ? (two ? cps * std::min<double>(6 * 16384, 110 * 1024 - peak - 1024 - stage_total)
                                        : std::min<double>(6 * 32768, kSmemCap - peak - 1024 - stage_total))
                                 : 64.0 * 1024;
    const double bw_sm = std::min(60e9, std::max(32768.0, inflight) / 3e-6);
    u32 gdep = 0;
    for (int g = 0; g < ngrid; ++g)
      if (grid[g] > 1) gdep |= 1u << g;
    double unique = 0, total = 0;
    for (auto& x : nodes) {
      if (x.kind != SGM_INPUT || x.cons.empty()) continue;
      unique += (double)prod4(in_dims[x.slot]) * es;
      double per = (double)prod4(x.sl) * es;
      double reps = (x.body && x.loopdep) ? (double)nloop / LP : 1.0;
      bool item_dep = x.body;
      for (int k = 0; k < 4; ++k) {
        item_dep = item_dep || (x.gmask[k] & gdep) || x.lsplit[k];
        int c = x.cls[k];
        item_dep = item_dep || (c >= 0 && cls[c].parts > 1 && !cls[c].cluster);
      }
      double execs = item_dep ? (double)items * CL : (double)active;
      // x-cached loaders are re-read only when a CTA's item moves to other coordinates
      if (xcache && x.xc) execs = std::min(execs, (double)items / (double)grid[0] + (double)active);
      total += per * reps * execs;
    }
    double redundant = std::max(0.0, total - unique);
    // gsplit partial tiles: written by every item, read back by the group's last one
    double gs_bytes = 0;
    for (auto& e : sched)
      if (e.type == Ev::GFLUSH)
        for (int f : e.flush) gs_bytes += 2.0 * (double)prod4(nodes[f].sl) * ec * items;
    redundant += gs_bytes;
    total += gs_bytes;
    // streamed operands that lose the TMA ring (misaligned / unsupported) stream at about half speed
    double slow = 0;
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && !x.tma && (ns == SGM_BF16 || ns == SGM_F32)) {
        const Node& b = nodes[x.in[1]];
        if (b.store == ST_VIEW) slow += (double)prod4(in_dims[b.slot]) * es;
      }
    double t_mem = (unique + slow) / 5.9e12 + redundant / 8e12;
    double t_sm = (total / active_sms) / bw_sm;
    double t_stream = std::max(t_mem, t_sm) * ((double)rounds * slots / std::max<i64>(1, items));
    int cflush = 0, gflush = 0;
    for (auto& e : sched) cflush += e.type == Ev::FLUSH, gflush += e.type == Ev::GFLUSH;
    // fixed per-item work (activation loads, A^T builds, epilogues; measured 2-6 us) is
    // largely hidden when two CTAs share an SM
    // fixed per-item costs measured with trace mode (tools/trace_one.py): ring refill
    // + activation staging + epilogue ~4 us, cluster flush ~5 us, gsplit tail ~2 us
    const double base = d.hints.item_cost_ns > 0 ? d.hints.item_cost_ns * 1e-9 : 4.0e-6;
    double t_item = (base + cflush * 5.0e-6 + gflush * 2.0e-6 * (base / 4.0e-6)) * (two ? 0.4 : 1.0);
    double loop_iters = loop_begin_pos >= 0 ? (double)nloop / LP : 0.0;
    // x-cached work runs only when a CTA's item moves to other coordinates: the
    // loop, and (a guess, without a compute term in this model) half of the
    // fixed per-item work, which the cached matmuls dominate
    if (xcache) {
      const double miss = std::min(1.0, ((double)items / (double)grid[0] + (double)active) / (double)items);
      if (xcache_loop) loop_iters *= miss;
      t_item *= miss + 0.5 * (1.0 - miss);
    }
    static const double iter_s = getenv("SGM_ITER_NS") ? atof(getenv("SGM_ITER_NS")) * 1e-9 : 0.6e-6;  // A/B experiments
    t_item += loop_iters * iter_s;
    return t_stream + (double)rounds * t_item + over;
  }

  // Beam search from no split (width 4): each step doubles one class (in an
  // allowed mode) or the loop; `policy` restricts the mode of reduced classes and
  // the loop (0: either, 1: cluster only, 2: gsplit only, 3: not split).  A plain greedy
  // descent gets trapped by early shared-memory-driven choices (e.g. splitting a
  // GEMV's rows, which multiplies the weight stream).
  double greedy(int policy, PlanState& out) {
    const int max_cluster = d.hints.max_cluster > 0 ? std::min(16, d.hints.max_cluster) : 8;
    const bool dbg = getenv("SGM_PLAN_DEBUG") != nullptr;
    PlanState root;
    root.parts.assign(cls.size(), 1);
    root.mode.assign(cls.size(), 0);
    apply_state(root);
    bool valid;
    double root_cost = plan_cost(&valid);
    if (d.hints.min_gsplit > 1) root_cost += d.hints.min_gsplit;
    std::vector<std::pair<double, PlanState>> beam = {{root_cost, root}};
    std::set<std::vector<int>> seen;
    auto key = [&](const PlanState& st) {
      std::vector<int> k = st.parts;
      k.insert(k.end(), st.mode.begin(), st.mode.end());
      k.push_back(st.lp);
      k.push_back(st.lmode);
      return k;
    };
    seen.insert(key(root));
    double best = root_cost;
    PlanState best_st = root;
    const std::vector<int> rmodes = policy == 1   ? std::vector<int>{1}
                                    : policy == 2 ? std::vector<int>{2}
                                    : policy == 3 ? std::vector<int>{}
                                                  : std::vector<int>{1, 2};
    for (int iter = 0; iter < 40; ++iter) {
      std::vector<std::pair<double, PlanState>> next;
      auto consider = [&](const PlanState& st) {
        if (!seen.insert(key(st)).second) return;
        apply_state(st);
        if (LB * FP * GP > (1LL << 22) || CL > max_cluster) return;
        if (d.hints.max_gsplit > 0 && GP > d.hints.max_gsplit) return;
        bool ok;
        double c = plan_cost(&ok);
        // below the requested gsplit count a state is only a stepping stone
        if (ok && d.hints.min_gsplit > 0 && GP < d.hints.min_gsplit) c += (double)d.hints.min_gsplit / GP;
        if (dbg)
          fprintf(stderr, "  plan p%d iter %d: LB=%lld FP=%lld GP=%lld CL=%d LP=%d%s ok=%d cost=%.2fus\n", policy, iter,
                  (long long)LB, (long long)FP, (long long)GP, CL, LP, loop_gs ? "g" : "", (int)ok, c * 1e6);
        if (ok) next.push_back({c, st});
      };
      for (auto& bs : beam) {
        const PlanState& cur = bs.second;
        for (int c = 0; c < (int)cls.size(); ++c) {
          const Class& C = cls[c];
          if (C.twice || C.extent % (cur.parts[c] * 2)) continue;
          std::vector<int> modes;
          if (!C.reduced) modes = {0};
          else if (cur.parts[c] > 1) modes = {cur.mode[c]};
          else modes = rmodes;
          for (int m : modes) {
            PlanState st = cur;
            st.parts[c] *= 2;
            st.mode[c] = m;
            consider(st);
          }
        }
        if (loop_split_ok && policy != 3 && nloop % (cur.lp * 2) == 0) {
          std::vector<int> modes = cur.lp > 1 ? std::vector<int>{cur.lmode} : rmodes;
          for (int m : modes) {
            PlanState st = cur;
            st.lp *= 2;
            st.lmode = m;
            consider(st);
          }
        }
      }
      if (next.empty()) break;
      std::sort(next.begin(), next.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (auto& ns : next) pool.push_back(ns);
      if (next.size() > 4) next.resize(4);
      const bool improved = next.front().first < best * 0.99;
      if (next.front().first < best) { best = next.front().first; best_st = next.front().second; }
      // keep descending while any beam state is still (nearly) competitive
      if (!improved && next.front().first > best * 1.5) break;
      beam = next;
    }
    out = best_st;
    return best;
  }

  // every state the searches evaluated, for plan variants
  std::vector<std::pair<double, PlanState>> pool;

  void split_plan() {
    PlanState best_st;
    double best = 1e30;
    pool.clear();
    // free splits only, then gsplit-only: cluster plans must win by 10% (their flush and
    // GPC-placement costs are the least well modelled, measured 3-7 us per item).  The
    // free-only descent matters when splitting the reductions first pulls the other beams
    // away from a many-item plan that only the x-cache makes cheap (Q's head-dim splits)
    static const bool no_free = getenv("SGM_NO_FREE_POLICY") != nullptr;  // A/B experiments
    for (int policy : {3, 2, 1, 0}) {
      if (policy == 3 && no_free) continue;
      PlanState st;
      double c = greedy(policy, st);
      if (c < best * (policy >= 2 ? 1.0 : 0.9)) { best = c; best_st = st; }
    }
    // hints.variant = v > 0: the v-th best distinct split the searches scored instead
    // (the profiler auto-tunes the physical plan of the best candidates over variants)
    if (d.hints.variant > 0) {
      std::sort(pool.begin(), pool.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      std::vector<std::pair<double, PlanState>> uniq;
      for (auto& ps : pool) {
        bool dup = false;
        for (auto& u : uniq) dup = dup || (u.second.parts == ps.second.parts && u.second.mode == ps.second.mode &&
                                           u.second.lp == ps.second.lp && u.second.lmode == ps.second.lmode);
        if (!dup) uniq.push_back(ps);
        if ((int)uniq.size() > d.hints.variant) break;
      }
      if ((int)uniq.size() > d.hints.variant) { best = uniq[d.hints.variant].first; best_st = uniq[d.hints.variant].second; }
    }
    apply_state(best_st);
    bool valid;
    plan_cost(&valid);
    est_us = best * 1e6;
  }

  void finalize_layout() {
    // cluster rank bit fields: loop first (unless gsplit), then cluster classes;
    // free parts and gsplit parts as mixed radices
    int shift = 0;
    loop_shift = 0;
    i64 gradix = 1;
    if (LP > 1 && !loop_gs) { loop_shift = 0; while ((1 << shift) < LP) ++shift; }
    if (LP > 1 && loop_gs) gradix = LP;
    i64 radix = 1;
    for (auto& C : cls) {
      if (C.parts <= 1) { C.cluster = C.gsplit = false; continue; }
      if (C.cluster) {
        C.bit_shift = shift;
        int b = 0;
        while ((1 << b) < C.parts) ++b;
        shift += b;
      } else if (C.gsplit) {
        C.radix = gradix;
        gradix *= C.parts;
      } else {
        C.radix = radix;
        radix *= C.parts;
      }
    }
    FP = radix;
    GP = gradix;
    CL = 1 << shift;
  }

  u32 class_bits(int c) const {
    const Class& C = cls[c];
    if (!C.cluster || C.parts <= 1) return 0;
    return (u32)(C.parts - 1) << C.bit_shift;
  }
  u32 loop_bits() const { return (LP > 1 && !loop_gs) ? (u32)(LP - 1) << loop_shift : 0; }
  bool class_gs(int c) const { return c >= 0 && cls[c].gsplit && cls[c].parts > 1; }
  bool uses_tc() const {
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && x.gemv && x.tc) return true;
    return false;
  }
  // Two TMEM-using CTAs share an SM when each allocates at most half of TMEM
  // (256 columns): measured on B200 (tools/tmem_occ_probe.cu) the hardware
  // co-schedules them although the occupancy API reports one CTA per SM.
  // Streamed tiles (ntl <= 16) fit with fewer accumulators; the cp.async GEMV
  // path needs ntl * 16 columns.
  // Which producer kernels pair up.  Measured on a plain fp32 GEMV (64 MB,
  // tools/gemv_probe.py): paired 23.8 us vs one CTA per SM 16.8 us -- the
  // CUDA-core fp32 consumer (2 FMA per streamed byte) does not gain from a
  // second CTA and loses registers to the 2-CTA launch bound; the tcgen05
  // kernels gain (G 73% -> 82% of the roofline).
  bool pairable() const { return uses_tc() && tc_pairable(); }
  bool tc_pairable() const {
    for (auto& x : nodes) {
      if (!(x.kind == SGM_MATMUL && x.gemv && x.tc)) continue;
      const i64 ntl = (x.sl[3] + 127) / 128;
      if (ntl * 16 > 256) return false;
    }
    return true;
  }

  // pending partials + schedule
  // Partial values.  A node reducing a split class (matmul K, sum axis) yields a
  // partial over that split.  Ops linear in the partial operands that are still
  // unreduced when they run propagate the partial (sum(x_p) @ B = sum(x_p @ B),
  // sum x_p + sum y_p = sum(x_p + y_p), ...), and accumulators absorb partials of
  // loop-body values they alone consume; any other consumer first flushes every
  // pending partial.  So e.g. LoRA's X@W + (X@A)@B reduces once, at the tail.
  bool linear_now(const Node& x, const std::set<int>& pending) const {
    auto pd = [&](int k) { return pending.count(x.in[k]) > 0; };
    switch (x.kind) {
      case SGM_SCALE: case SGM_SUM: return pd(0);
      case SGM_MATMUL: case SGM_MUL: return pd(0) != pd(1);
      case SGM_DIV: return pd(0) && !pd(1);
      case SGM_ADD: {
        const Node& a = nodes[x.in[0]];
        const Node& b = nodes[x.in[1]];
        return pd(0) && pd(1) && a.pend == b.pend && a.gpend == b.gpend;
      }
      default: return false;
    }
  }

  // bytes a node streams from HBM (view operands of a matmul)
  i64 stream_bytes(const Node& x) const {
    if (x.kind != SGM_MATMUL) return 0;
    i64 b = 0;
    for (int k = 0; k < 2; ++k)
      if (nodes[x.in[k]].store == ST_VIEW) b += prod4(nodes[x.in[k]].sl) * es;
    return b;
  }

  void reduce_bits(Node& x) const {
    if (x.kind == SGM_MATMUL) {
      int c = nodes[x.in[0]].cls[3];
      if (c >= 0) { x.pend |= class_bits(c); x.gpend = x.gpend || class_gs(c); }
    } else if (x.kind == SGM_SUM) {
      int c = nodes[x.in[0]].cls[x.axis + 4 - nodes[x.in[0]].rank];
      if (c >= 0) { x.pend |= class_bits(c); x.gpend = x.gpend || class_gs(c); }
    }
  }

  void schedule() {
    for (auto& x : nodes) { x.pend = 0; x.gpend = false; x.deferred = false; x.lin = false; }
    sched.clear();
    std::set<int> pending;
    auto flush_all = [&]() {
      std::vector<int> cf, gf;
      for (int p : pending) {
        if (nodes[p].pend) cf.push_back(p);
        if (nodes[p].gpend) gf.push_back(p);
      }
      pending.clear();
      if (!cf.empty()) {
        Ev e;
        e.type = Ev::FLUSH;
        e.flush = cf;
        sched.push_back(e);
      }
      if (!gf.empty()) {
        Ev e;
        e.type = Ev::GFLUSH;
        e.flush = gf;
        sched.push_back(e);
      }
    };
    auto push_node = [&](int n) {
      Node& x = nodes[n];
      bool any = false;
      for (int k = 0; k < x.nin; ++k) any = any || pending.count(x.in[k]);
      if (x.kind == SGM_ACCUM) {
        const int p = x.in[0];
        bool absorb = pending.count(p) && nodes[p].body && !d.hints.no_hoist;
        for (int c : nodes[p].cons) absorb = absorb && nodes[c].kind == SGM_ACCUM;
        if (absorb) {
          nodes[p].deferred = true;
          x.pend = nodes[p].pend;
          x.gpend = nodes[p].gpend;
          pending.erase(p);
        } else if (any) {
          flush_all();
        }
        x.pend |= loop_bits();
        x.gpend = x.gpend || (LP > 1 && loop_gs);
      } else if (any && x.kind != SGM_OUTPUT && !d.hints.no_hoist && linear_now(x, pending)) {
        x.lin = true;
        for (int k = 0; k < x.nin; ++k)
          if (pending.count(x.in[k])) {
            x.pend |= nodes[x.in[k]].pend;
            x.gpend = x.gpend || nodes[x.in[k]].gpend;
          }
      } else if (any) {
        flush_all();
      }
      reduce_bits(x);
      Ev e;
      e.type = Ev::NODE;
      e.node = n;
      sched.push_back(e);
      if (x.pend || x.gpend) pending.insert(n);
      if (x.lin)  // partial operands whose every consumer is linear never need the reduced value
        for (int k = 0; k < x.nin; ++k) {
          const int p = x.in[k];
          bool all_lin = true;
          for (int c : nodes[p].cons) all_lin = all_lin && (nodes[c].lin || c == n);
          if (all_lin && pending.count(p)) pending.erase(p);
        }
    };
    // Within each region nodes are list-scheduled (see the priority in push_region).
    std::vector<int> height(nodes.size(), 0);
    for (int n = (int)nodes.size() - 1; n >= 0; --n)
      for (int c : nodes[n].cons) height[n] = std::max(height[n], height[c] + 1);
    // would scheduling n now force a flush of pending partials?
    auto would_flush = [&](int n) {
      const Node& x = nodes[n];
      bool any = false;
      for (int k = 0; k < x.nin; ++k) any = any || pending.count(x.in[k]);
      if (!any || x.kind == SGM_ACCUM) return false;
      return !(x.kind != SGM_OUTPUT && !d.hints.no_hoist && linear_now(x, pending));
    };
    auto push_region = [&](auto in_region) {
      std::vector<char> done(nodes.size(), 0);
      for (int n = 0; n < (int)nodes.size(); ++n) done[n] = !in_region(n);
      for (;;) {
        int pick = -1;
        for (int n = 0; n < (int)nodes.size(); ++n) {
          if (done[n]) continue;
          bool ready = true;
          for (int k = 0; k < nodes[n].nin; ++k) ready = ready && (done[nodes[n].in[k]] || !in_region(nodes[n].in[k]));
          // in-region inputs must already be scheduled (done marks both out-of-region and scheduled)
          if (!ready) continue;
          // nodes that need reduced values wait while anything else is ready, so
          // one flush (one round of cluster barriers) reduces every partial at once
          // (streamed views emit no code: take them at once so their consumers are ready)
          const bool vn = nodes[n].kind == SGM_INPUT && nodes[n].store == ST_VIEW;
          const bool vp = pick >= 0 && nodes[pick].kind == SGM_INPUT && nodes[pick].store == ST_VIEW;
          if (vp) continue;
          if (vn) { pick = n; continue; }
          // Then the longest chain to a sink: a short chain of small matmuls (LoRA's
          // X@A -> T@B) runs before an independent big stream (X@W) while the ring
          // pre-fills with the big stream's boxes (measured: W first is ~5% slower
          // on L).  Ties: the smaller stream first.
          const bool fn = would_flush(n), fp = pick >= 0 && would_flush(pick);
          const i64 sn = stream_bytes(nodes[n]), sp = pick >= 0 ? stream_bytes(nodes[pick]) : 0;
          const bool big = d.hints.big_first && fn == fp && pick >= 0 && sn != sp && (sn > 0 || sp > 0);
          if (big) {
            if (sn > sp) pick = n;
          } else if (pick < 0 || (!fn && fp) ||
                     (fn == fp && (height[n] > height[pick] || (height[n] == height[pick] && sn < sp))))
            pick = n;
        }
        if (pick < 0) break;
        done[pick] = 1;
        push_node(pick);
      }
    };
    push_region([&](int n) { return (bool)nodes[n].hoist; });
    bool has_loop = false;
    for (auto& x : nodes) has_loop = has_loop || (x.body && !x.hoist);
    if (has_loop) {
      if (!pending.empty()) flush_all();  // hoisted partials must be complete before the loop re-reads them
      Ev b;
      b.type = Ev::LOOP_BEGIN;
      loop_begin_pos = (int)sched.size();
      sched.push_back(b);
      push_region([&](int n) { return nodes[n].body && !nodes[n].hoist; });
      Ev en;
      en.type = Ev::LOOP_END;
      loop_end_pos = (int)sched.size();
      sched.push_back(en);
    } else {
      loop_begin_pos = loop_end_pos = -1;
    }
    push_region([&](int n) { return !nodes[n].body; });
  }

  // A gsplit plan is legal iff its partials are reduced by a single GFLUSH after
  // which only the group's last work item continues: nothing after it may depend
  // on a gsplit part (slices of gsplit classes), stream (views), loop or flush again.
  bool gs_tail_ok() const {
    int g = -1;
    for (int p = 0; p < (int)sched.size(); ++p)
      if (sched[p].type == Ev::GFLUSH) {
        if (g >= 0) return false;
        g = p;
      }
    if (g < 0) return GP <= 1;
    for (int p = g + 1; p < (int)sched.size(); ++p) {
      const Ev& e = sched[p];
      if (e.type != Ev::NODE) return false;
      const Node& x = nodes[e.node];
      if (x.gpend || x.pend) return false;
      for (int k = 0; k < 4; ++k)
        if (class_gs(x.cls[k])) return false;
      for (int k = 0; k < x.nin; ++k)
        if (nodes[x.in[k]].store == ST_VIEW) return false;
    }
    return true;
  }

  // matmul realisation choices (depend on slices)
  void matmul_choices() {
    int ntma = 0;
    for (auto& t : nodes)
      if (t.store == ST_XG) t.store = ST_SMEM;
    // a small stream (e.g. LoRA's X@A, 32 KB per item) queued in the ring ahead of a
    // large one holds slots and delays the large stream's start by its whole
    // dependency chain; hint small_plain = 1 reads it with plain loads instead (measured
    // on L: plain loads queue behind the producer's TMA traffic, 12.0 -> 15.2 us, so
    // the ring stays the default)
    i64 max_stream = 0;
    for (auto& t : nodes) max_stream = std::max(max_stream, stream_bytes(t));
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      if (x.kind != SGM_MATMUL) continue;
      const Node& a = nodes[x.in[0]];
      const Node& b = nodes[x.in[1]];
      x.gemv = false;
      x.tc = false;
      x.tma = false;
      x.xb_shared = false;
      x.xb_build = true;
      x.red_bytes = 0;
      x.at_bytes = 0;
      i64 M = x.sl[2], K = a.sl[3], NN = x.sl[3];
      if (b.store == ST_VIEW && a.store != ST_VIEW && M <= 16 && NN >= 1) {
        // B stride along n must be 1 (row-major view), alignment for vectors
        int accw = ea / 4;  // 32-bit registers per accumulator
        int vn = 1;
        for (int cand : {16 / es, 8 / es, 4 / es, 2 / es, 1}) {
          if (cand < 1) continue;
          if (NN % cand) continue;
          if (M * cand * accw > 64 && cand > 1) continue;
          bool ok = true;
          const i64* st = in_strides[b.slot];
          for (int k = 0; k < 3; ++k)
            if (in_dims[b.slot][k] > 1 && st[k] % cand) ok = false;
          // all offset coefficients along dim 3 are multiples of the slice width
          if (b.sl[3] % cand) ok = false;
          if (!ok) continue;
          vn = cand;
          break;
        }
        x.gemv = true;
        x.vn = vn;
        i64 NV = NN / vn;
        i64 items = x.sl[0] * x.sl[1] * NV;
        i64 ks = 1;
        while (items * ks * 2 <= NT && ks * 2 <= K) ks *= 2;
        x.ks = (int)ks;
        i64 per_thread = (K + ks - 1) / ks;
        int umax = (M * vn * accw <= 32) ? 16 : 8;
        x.unr = per_thread >= umax ? umax : per_thread >= 8 ? 8 : (per_thread >= 4 ? 4 : (per_thread >= 2 ? 2 : 1));
        bool nv_pow2 = (NV & (NV - 1)) == 0;
        i64 work = items * ks;
        x.shfl = nv_pow2 && ((work % NT == 0) || (work < NT && work % 32 == 0));
        i64 kin = (!x.shfl || NV >= 32) ? 1 : std::min<i64>(32 / NV, ks);
        i64 kout = ks / kin;
        if (kout > 1) x.red_bytes = kout * items * M * vn * ea;
        i64 a0 = (a.sl[0] > 1) ? x.sl[0] : 1, a1 = (a.sl[1] > 1) ? x.sl[1] : 1;
        x.at_bytes = a0 * a1 * K * M * ec;
        // tcgen05 path: bf16 weights, <= 16 rows, K in multiples of 16, 16-byte row alignment
        x.tc = false;
        bool row16 = true;
        for (int k = 0; k < 3; ++k)
          if (in_dims[b.slot][k] > 1 && (in_strides[b.slot][k] * es) % 16) row16 = false;
        i64 ntl = (NN + 127) / 128;
        if (ns == SGM_BF16 && d.hints.use_tcgen05 >= 0 && M <= 16 && K % 16 == 0 && NN % 8 == 0 && NN >= 64 &&
            ntl <= 32 && row16 && x.sl[0] * x.sl[1] <= 8) {
          i64 kc = 16;
          while (kc * 2 <= K && K % (kc * 2) == 0 && (kc * 2 / 8) * 2048 <= 16 * 1024) kc *= 2;
          i64 nst = (K / kc) * ntl;
          int S = (int)std::min<i64>(8, std::max<i64>(3, nst + 2));
          i64 bytes = S * (kc / 8) * 2048 + 32 * K + 8 * S;
          x.tc = true;
          x.tc_kc = (int)kc;
          x.tc_s = S;
          int cols = 32;
          while (cols < ntl * 16) cols *= 2;
          x.tc_cols = cols;
          x.red_bytes = 0;
          x.at_bytes = bytes;  // the tcgen05 work area re-uses the transient slot
        }
        // TMA-fed streaming (producer warp + ring): bf16 on tcgen05, fp32 on CUDA cores
        x.tma = false;
        x.xb_shared = false;
        const i64 d3 = in_dims[b.slot][3];
        // every box starts 16-byte aligned iff the slice width along n is a multiple of 16 bytes
        // (all start terms are multiples of it); TMA faults on misaligned box starts
        const bool batch_ok = x.sl[0] * x.sl[1] <= 8 && b.sl[3] == NN && b.sl[2] == K && (NN * es) % 16 == 0 && !x.inv;
        const i64 sb = stream_bytes(x);
        const bool small = d.hints.small_plain && sb <= 64 * 1024 && sb * 8 <= max_stream;
        // the finite-field checker can stream its 4-byte residues through the same ring
        // into the CUDA-core consumer (u64 lazy-reduced accumulators, hints.ff_tma):
        // measured on the sweep it lost overall (A's FF checks 1.66 -> 3.17 s per step,
        // L 0.26 -> 0.34; Q 0.76 -> 0.72, R 49 -> 43 ms), so plain loads stay the default
        static const bool ff_tma_env = getenv("SGM_FF_TMA") != nullptr;  // A/B experiments
        const bool ff_ok = ns == SGM_FF && (d.hints.ff_tma || ff_tma_env);
        if (!d.hints.no_tma && !no_tma_forced && batch_ok && ntma < 4 &&
            (ns == SGM_BF16 || ns == SGM_F32 || ff_ok) && !small) {
          if (ns == SGM_BF16 && d.hints.use_tcgen05 >= 0 && M <= 16 && K % 16 == 0 && (d3 * 2) % 16 == 0 &&
              ntl * 16 <= 512) {
            x.tma = true;
            ++ntma;
            x.tc = true;
            x.kc = K % 128 == 0 ? 128 : (K % 64 == 0 ? 64 : (K % 32 == 0 ? 32 : 16));
            // narrow tiles (NN <= 64, one 64-column box per stage) take up to 256 k-rows
            // per stage: a 16-column LoRA X@A stage otherwise held a whole slot for 4 KB
            if (NN <= 64 && K % 256 == 0) x.kc = 256;
            x.xb_shared = x.sl[0] * x.sl[1] == 1;
            x.at_bytes = x.xb_shared ? 0 : 32 * K;
            x.red_bytes = 0;
            // independent accumulators (up to 4 per tile, TMEM permitting): consecutive MMAs
            // of a stage rotate over them instead of serialising on one
            x.acc = 4;
            while (x.acc > 1 && ntl * x.acc * 16 > 512) x.acc /= 2;
            int cols = 32;
            while (cols < ntl * x.acc * 16) cols *= 2;
            x.tc_cols = cols;
          } else if ((ns == SGM_F32 || ns == SGM_FF) && M <= 8 && K % 8 == 0 && NN % 8 == 0 && (d3 * 4) % 16 == 0) {
            x.tma = true;
            ++ntma;
            x.tc = false;
            x.bw = NN >= 64 ? 64 : (NN >= 32 ? 32 : (NN >= 16 ? 16 : 8));
            while (x.bw > 8 && NN % x.bw) x.bw /= 2;
            i64 kmax = std::min<i64>(256, kSlot / (x.bw * 4));  // plan_ring halves it for 16 KB slots
            x.kc = 8;
            while (x.kc * 2 <= kmax && K % (x.kc * 2) == 0) x.kc *= 2;
            i64 a0 = (a.sl[0] > 1) ? x.sl[0] : 1, a1 = (a.sl[1] > 1) ? x.sl[1] : 1;
            // mm_stream_f32 reads a single-batch row-major A in place (DIRECT)
            const bool direct = a0 * a1 == 1 && a.store != ST_VIEW;
            x.at_bytes = direct ? 0 : a0 * a1 * K * M * 4;
            x.red_bytes = (i64)(NT / 32) * M * 64 * ea;
          }
        }
      }
    }
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& t = nodes[n];
      if (t.kind != SGM_INPUT || t.store != ST_SMEM || t.body || t.cons.empty() || ns != SGM_BF16) continue;
      const i64* st = in_strides[t.slot];
      bool ok = st[3] == 1 && (st[2] * 2) % 16 == 0 && t.sl[3] % 8 == 0 && t.sl[2] <= 16 && t.sl[0] * t.sl[1] == 1;
      for (int c : t.cons) {
        const Node& m = nodes[c];
        ok = ok && m.kind == SGM_MATMUL && m.tma && m.tc && m.xb_shared && m.in[0] == n && m.in[1] != n;
      }
      if (ok && !d.hints.no_tma) t.store = ST_XG;
    }
    prod = false;
    int id = 0;
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && x.tma) {
        prod = true;
        x.tma_id = id++;
      }
    // per-item loader tiles of producer kernels come through TMA too, issued by the
    // producer ahead of the item's streamed boxes (plain loads would queue behind them)
    nstaged = 0;
    stage_total = 0;
    // loaders after a gsplit tail reduction run only in the group's last item: the
    // producer cannot know which, so they keep plain loads
    int gpos = (int)sched.size();
    std::vector<int> npos(nodes.size(), -1);
    for (int q = 0; q < (int)sched.size(); ++q) {
      if (sched[q].type == Ev::GFLUSH) gpos = std::min(gpos, q);
      if (sched[q].type == Ev::NODE) npos[sched[q].node] = q;
    }
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      x.staged = false;
      x.stage_id = -1;
      if (!prod || d.hints.no_tma || x.kind != SGM_INPUT || x.store != ST_SMEM || x.inv || x.body || x.cons.empty())
        continue;
      if (npos[n] > gpos) continue;
      if (id >= 4) break;
      const i64 d3 = in_dims[x.slot][3];
      if ((x.sl[3] * es) % 16 || (d3 * es) % 16 || x.sl[0] > 256 || x.sl[1] > 256 || x.sl[2] > 256) continue;
      i64 b3 = x.sl[3];
      while (b3 > 256) b3 /= 2;
      if (x.sl[3] % b3 || (b3 * es) % 16) continue;
      const i64 bytes = prod4(x.sl) * es;
      if (bytes > 64 * 1024) continue;
      x.staged = true;
      x.stage_id = nstaged++;
      x.tma_id = id++;
      x.sbox = (int)b3;
      x.stage_off = (int)stage_total;
      stage_total += (bytes + 127) / 128 * 128;
    }
  }

  // Item-invariant nodes (persistent kernels): values that depend only on the
  // CTA's cluster parts, not on the work item (grid coordinates / free parts),
  // e.g. the activation tile of a column-split GEMV.  Computed once per CTA.
  void invariants() {
    u32 gdep = 0;
    for (int g = 0; g < ngrid; ++g)
      if (grid[g] > 1) gdep |= 1u << g;
    auto free_split = [&](const Node& x) {
      for (int k = 0; k < 4; ++k) {
        int c = x.cls[k];
        if (c >= 0 && cls[c].parts > 1 && !cls[c].cluster) return true;
      }
      return false;
    };
    // a view (HBM-resident loader) whose slice does not depend on the work item
    auto view_inv = [&](const Node& v) {
      if (v.kind != SGM_INPUT || v.store != ST_VIEW || v.body || free_split(v)) return false;
      for (int k = 0; k < 4; ++k)
        if ((v.gmask[k] & gdep) || v.lsplit[k]) return false;
      return true;
    };
    for (auto& x : nodes) {
      x.inv = false;
      if (d.hints.no_hoist || LB * FP * GP <= 1) continue;
      if (x.body || x.pend || x.gpend || x.kind == SGM_OUTPUT || x.kind == SGM_ACCUM) continue;
      if (x.store != ST_SMEM && x.store != ST_GLOBAL && x.store != ST_XG) continue;
      if (free_split(x)) continue;
      if (x.kind == SGM_INPUT) {
        bool dep = false;
        for (int k = 0; k < 4; ++k) dep = dep || (x.gmask[k] & gdep) || x.lsplit[k];
        x.inv = !dep;
      } else if (x.kind == SGM_MATMUL) {
        // e.g. LoRA's X @ A when only the output columns are split: once per CTA,
        // reading the (L2-resident) view directly; matmul_choices keeps it off the TMA ring
        const Node& a = nodes[x.in[0]];
        const Node& b = nodes[x.in[1]];
        const bool va = a.store == ST_VIEW, vb = b.store == ST_VIEW;
        x.inv = !(va && vb) && (va ? view_inv(a) : a.inv) && (vb ? view_inv(b) : b.inv);
      } else {
        bool all = true;
        for (int k = 0; k < x.nin; ++k) all = all && nodes[x.in[k]].inv;
        x.inv = all;
      }
    }
  }

  // liveness-based smem allocation; returns peak bytes
  int allocate() {
    int S = (int)sched.size();
    std::vector<int> pos_of(nodes.size(), -1);
    for (int p = 0; p < S; ++p)
      if (sched[p].type == Ev::NODE) pos_of[sched[p].node] = p;
    std::vector<Interval> iv;
    std::vector<int> last(nodes.size(), -1);
    for (int p = 0; p < S; ++p) {
      const Ev& e = sched[p];
      if (e.type == Ev::NODE) {
        const Node& x = nodes[e.node];
        for (int k = 0; k < x.nin; ++k) last[x.in[k]] = std::max(last[x.in[k]], p);
      } else if (e.type == Ev::FLUSH || e.type == Ev::GFLUSH) {
        for (int f : e.flush) last[f] = std::max(last[f], p);
      }
    }
    int tcount = 0;
    flush_tmp_off.clear();
    std::vector<std::pair<std::pair<int, int>, int>> flush_ids;
    // in-place elementwise ops: the output reuses its first operand's tile when that
    // operand has the same slice and dies at this node (each element is read and
    // written by the same thread)
    std::vector<int> rep(nodes.size());
    for (int n = 0; n < (int)nodes.size(); ++n) rep[n] = n;
    for (int p = 0; p < S; ++p) {
      if (sched[p].type != Ev::NODE) continue;
      const int n = sched[p].node;
      const Node& x = nodes[n];
      const bool ew = x.kind == SGM_EXP || x.kind == SGM_SILU || x.kind == SGM_SQUARE || x.kind == SGM_SQRT ||
                      x.kind == SGM_SCALE || x.kind == SGM_DIV || x.kind == SGM_MUL || x.kind == SGM_ADD;
      if (!ew || x.store != ST_SMEM || x.inv || x.xc || d.hints.no_hoist) continue;
      const Node& a = nodes[x.in[0]];
      bool same = a.store == ST_SMEM && a.kind != SGM_ACCUM && a.kind != SGM_INPUT && !a.inv && !a.xc &&
                  last[x.in[0]] == p;
      for (int k = 0; k < 4 && same; ++k) same = a.sl[k] == x.sl[k];
      if (x.nin == 2 && x.in[1] != x.in[0] && rep[x.in[1]] == rep[x.in[0]]) same = false;
      if (same) rep[n] = rep[x.in[0]];
    }
    std::map<int, Interval> groups;
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      if (x.store != ST_SMEM || x.kind == SGM_OUTPUT) continue;
      int st = pos_of[n];
      if (x.kind == SGM_ACCUM) st = loop_begin_pos;
      int en = std::max(last[n], pos_of[n]);
      if (loop_begin_pos >= 0 && st < loop_begin_pos && en > loop_begin_pos) en = std::max(en, loop_end_pos);
      if (x.kind == SGM_ACCUM) en = std::max(en, loop_end_pos);
      if (x.inv || x.xc) { st = 0; en = S; }  // lives across items
      auto it = groups.find(rep[n]);
      if (it == groups.end()) {
        Interval I;
        I.id = rep[n];
        I.start = st;
        I.end = en;
        I.bytes = prod4(x.sl) * ec;
        groups[rep[n]] = I;
      } else {
        it->second.start = std::min(it->second.start, st);
        it->second.end = std::max(it->second.end, en);
        it->second.bytes = std::max<i64>(it->second.bytes, prod4(x.sl) * ec);
      }
    }
    for (auto& kv : groups) iv.push_back(kv.second);
    // shared tcgen05 A^T buffers, one per A node: [first, last consumer], or the
    // whole kernel when A is item-invariant (built once before the item loop)
    std::map<int, std::vector<int>> xb_users;
    for (int p = 0; p < S; ++p)
      if (sched[p].type == Ev::NODE) {
        const Node& x = nodes[sched[p].node];
        if (x.kind == SGM_MATMUL && x.tma && x.tc && x.xb_shared) xb_users[x.in[0]].push_back(sched[p].node);
      }
    std::map<int, int> xb_iv;  // A node -> interval id
    for (auto& kv : xb_users) {
      const Node& a = nodes[kv.first];
      Interval I;
      I.id = -(1 + tcount++);
      I.start = a.inv ? 0 : pos_of[kv.second.front()];
      I.end = a.inv ? S : pos_of[kv.second.back()];
      I.bytes = 32 * a.sl[3];
      iv.push_back(I);
      xb_iv[kv.first] = I.id;
    }
    std::map<int, int> red_iv, at_iv;  // matmul node -> transient interval id
    for (int n = 0; n < (int)nodes.size(); ++n)
      if (nodes[n].kind == SGM_MATMUL && nodes[n].red_bytes > 0) {
        Interval I;
        I.id = -(1 + tcount++);
        I.start = I.end = pos_of[n];
        I.bytes = nodes[n].red_bytes;
        iv.push_back(I);
        red_iv[n] = I.id;
      }
    for (int n = 0; n < (int)nodes.size(); ++n)
      if (nodes[n].kind == SGM_MATMUL && nodes[n].at_bytes > 0) {
        Interval I;
        I.id = -(1 + tcount++);
        I.start = I.end = pos_of[n];
        I.bytes = nodes[n].at_bytes;
        iv.push_back(I);
        at_iv[n] = I.id;
      }
    for (int p = 0; p < S; ++p)
      if (sched[p].type == Ev::FLUSH) {
        const bool push = push_flush(sched[p].flush);
        for (int f : sched[p].flush) {
          Interval I;
          I.id = -(1 + tcount++);
          if (push) {  // receive buffers: written by peers at any time, live for the whole kernel
            I.start = 0;
            I.end = S;
            I.bytes = 2 * CL * pad4(prod4(nodes[f].sl)) * ec;
          } else {
            I.start = I.end = p;
            I.bytes = prod4(nodes[f].sl) * ec;
          }
          iv.push_back(I);
          flush_ids.push_back({{p, f}, I.id});
        }
      }
    std::sort(iv.begin(), iv.end(), [](const Interval& a, const Interval& b) {
      if (a.start != b.start) return a.start < b.start;
      return a.bytes > b.bytes;
    });
    std::vector<std::pair<Interval, i64>> placed;
    i64 peak = 0;
    std::map<int, i64> off_of;
    for (auto& I : iv) {
      std::vector<std::pair<i64, i64>> busy;
      for (auto& pl : placed)
        if (!(pl.first.end < I.start || pl.first.start > I.end)) busy.push_back({pl.second, pl.second + pl.first.bytes});
      std::sort(busy.begin(), busy.end());
      i64 off = 0;
      for (auto& b : busy) {
        if (off + I.bytes <= b.first) break;
        off = std::max(off, (b.second + 15) / 16 * 16);
      }
      placed.push_back({I, off});
      off_of[I.id] = off;
      if (getenv("SGM_ALLOC_DEBUG"))
        fprintf(stderr, "  alloc id=%d [%d,%d] bytes=%lld off=%lld\n", I.id, I.start, I.end, (long long)I.bytes,
                (long long)off);
      peak = std::max(peak, off + I.bytes);
    }
    for (auto& x : nodes) x.off = 0;
    for (int n = 0; n < (int)nodes.size(); ++n)
      if (nodes[n].store == ST_SMEM && nodes[n].kind != SGM_OUTPUT && off_of.count(rep[n]))
        nodes[n].off = (int)off_of[rep[n]];
    for (auto& kv : red_iv) nodes[kv.first].red_off = (int)off_of[kv.second];
    for (auto& kv : at_iv) nodes[kv.first].at_off = (int)off_of[kv.second];
    for (auto& fi : flush_ids) flush_tmp_off[fi.first] = (int)off_of[fi.second];
    for (auto& kv : xb_users) {
      const bool pre = nodes[kv.first].inv;
      for (size_t u = 0; u < kv.second.size(); ++u) {
        Node& x = nodes[kv.second[u]];
        x.at_off = (int)off_of[xb_iv[kv.first]];
        x.xb_build = !pre && u == 0;
      }
    }
    // global scratch for tiles that did not fit
    scratch_per_cta = 0;
    for (auto& x : nodes)
      if (x.store == ST_GLOBAL) {
        x.off = (int)scratch_per_cta;
        scratch_per_cta += (prod4(x.sl) * ec + 255) / 256 * 256;
      }
    return (int)peak;
  }

  // Loop-body loaders prefetched one iteration ahead into registers (TilePf):
  // j-dependent plain tile loads of at most 8 loads per thread, 32 registers in all.
  std::vector<char> pf;
  void plan_prefetch() {
    pf.assign(nodes.size(), 0);
    if (getenv("SGM_NO_PREFETCH") || d.hints.no_prefetch || loop_begin_pos < 0 || nloop / LP < 2) return;
    int regs = 0;
    for (int p = loop_begin_pos; p < loop_end_pos; ++p) {
      const Ev& e = sched[p];
      if (e.type != Ev::NODE) continue;
      const Node& x = nodes[e.node];
      if (x.kind != SGM_INPUT || !x.body || x.hoist || !x.loopdep || x.inv || x.staged || x.store == ST_VIEW ||
          x.store == ST_XG || e.node == ilv_big)
        continue;
      if (strip_ok(x)) {
        const i64 it = (x.sl[0] * x.sl[1] * x.sl[2] + NT - 1) / NT;
        if (it <= 8 && regs + 4 * it <= 40) {
          regs += 4 * (int)it;
          pf[e.node] = 2;
          continue;
        }
      }
      const int vec = io_vec(x, true);
      const i64 tot = prod4(x.sl) / (vec > 1 ? vec : 1);
      const i64 it = (tot + NT - 1) / NT;
      const int r = (int)it * (vec > 1 ? 4 : (es + 3) / 4);
      if (it > 8 || regs + r > 40) continue;
      regs += r;
      pf[e.node] = 1;
    }
  }

  // A loader whose loop steps its contiguous innermost dim T elements per iteration
  // with a T-element tile along it (T columns per iteration, T | 16 / es): TileStrip
  // reads the next 16 bytes of every row once per 16 / es / T iterations.  Every other offset term
  // must keep 16-byte alignment (sgm_plan_run requires 16-byte aligned base pointers).
  bool strip_ok(const Node& x) const {
    if (getenv("SGM_NO_STRIP")) return false;
    const i64 G = 16 / es;
    const i64* dims = in_dims[x.slot];
    const i64* st = in_strides[x.slot];
    const i64 T = x.sl[3];
    if (G % T || st[3] != 1 || !x.lsplit[3] || (nloop / LP) % (G / T)) return false;
    i64 w = dims[3];
    for (int g = 0; g < ngrid; ++g)
      if (x.gmask[3] >> g & 1u) {
        w /= grid[g];
        if (grid[g] > 1 && w % G) return false;
      }
    if (w / nloop != T) return false;
    const int c = x.cls[3];
    if (c >= 0 && cls[c].parts > 1 && (x.sh[3] / cls[c].parts) % G) return false;
    for (int k = 0; k < 3; ++k)
      if (dims[k] > 1 && st[k] % G) return false;
    return true;
  }

  std::string pf_type(const Node& x) const {
    const i64* st = in_strides[x.slot];
    std::ostringstream t;
    t << "sgm::TilePf<N, " << x.sl[0] << ", " << x.sl[1] << ", " << x.sl[2] << ", " << x.sl[3] << ", " << st[0]
      << "LL, " << st[1] << "LL, " << st[2] << "LL, " << st[3] << "LL, " << io_vec(x, true) << ", NT>";
    return t.str();
  }

  bool any_tc() const {
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && x.tc) return true;
    return false;
  }

  // Loops over small tiles (L's one-k-per-iteration LoRA candidates: every body tile
  // <= 128 elements, 4096 iterations) are barrier-latency chains; 256 threads leave
  // most lanes idle and cap residency (registers).  Fewer threads per CTA -- at least
  // a quarter of the largest body tile, a 64th of the largest other tile -- put more
  // CTAs (independent chains) on each SM.  CUDA-core plans without a producer only.
  int small_loop_threads() const {
    if (d.hints.threads > 0 || prod || CL > 1 || any_tc() || getenv("SGM_NO_SMALL_NT")) return 0;
    if (loop_begin_pos < 0 || nloop / LP < 16) return 0;
    i64 wb = 0, wa = 0;
    for (auto& x : nodes) {
      if (x.store == ST_VIEW || x.store == ST_XG || x.kind == SGM_OUTPUT) continue;
      const i64 w = prod4(x.sl);
      if (x.body && !x.hoist) wb = std::max(wb, w);
      else wa = std::max(wa, w);
    }
    int nt = 32;
    while (nt < NT && (nt * 4 < wb || nt * 64 < wa)) nt *= 2;
    return nt < NT ? nt : 0;
  }

  void plan_xcache() {
    for (auto& x : nodes) x.xc = false;
    xcache = xcache_loop = false;
    if (getenv("SGM_NO_XCACHE") || d.hints.no_xcache || d.hints.interleave || CL != 1 || ngrid != 1 ||
        grid[0] <= 1)
      return;
    std::vector<char> dep(nodes.size(), 0);
    for (int n = 0; n < (int)nodes.size(); ++n) {
      const Node& x = nodes[n];
      if (x.kind == SGM_INPUT) {
        for (int k = 0; k < 4; ++k) dep[n] = dep[n] || (x.gmask[k] & 1u);
      } else if (x.kind == SGM_OUTPUT) {
        dep[n] = 1;
      } else {
        for (int k = 0; k < x.nin; ++k) dep[n] = dep[n] || dep[x.in[k]];
      }
    }
    bool loop_inv = true, has_body = false;
    for (int n = 0; n < (int)nodes.size(); ++n)
      if (nodes[n].body && !nodes[n].hoist) { has_body = true; loop_inv = loop_inv && !dep[n]; }
    std::set<int> flushed;
    for (auto& e : sched)
      if (e.type == Ev::FLUSH || e.type == Ev::GFLUSH)
        for (int f : e.flush) flushed.insert(f);
    int mm = 0;
    for (int n = 0; n < (int)nodes.size(); ++n) {
      Node& x = nodes[n];
      if (dep[n] || x.inv || x.kind == SGM_OUTPUT || x.staged || x.pend || x.gpend || flushed.count(n)) continue;
      if (x.body && !x.hoist && !loop_inv) continue;
      if (x.store == ST_GLOBAL) continue;
      x.xc = true;
      if (x.kind == SGM_MATMUL) ++mm;
    }
    if (!mm) {
      for (auto& x : nodes) x.xc = false;
      return;
    }
    xcache = true;
    xcache_loop = has_body && loop_inv;
  }

  // item loop header: the default round-robin order, or (x-cache) a contiguous
  // range of items per CTA run gx-fastest, with xc_miss = the other coordinates changed
  void emit_item_loop(const char* ind, const char* counter) {
    const i64 T = LB * FP * GP;
    if (!xcache) {
      os << ind << "for (long long item = cid; item < " << T << "LL; item += ncl, ++" << counter << ") {\n";
      emit_item_vars(ind);
      return;
    }
    os << ind << "long long xc_f = -1, xc_g = -1;\n";
    os << ind << "const long long xc_lo = cid * " << T << "LL / ncl, xc_hi = (cid + 1) * " << T << "LL / ncl;\n";
    os << ind << "for (long long xc_t = xc_lo; xc_t < xc_hi; ++xc_t, ++" << counter << ") {\n";
    os << ind << "const long long xc_gx = xc_t % " << grid[0] << "LL, xc_r = xc_t / " << grid[0] << "LL;\n";
    os << ind << "const long long item = (xc_r % " << GP << "LL) + " << GP << "LL * ((xc_r / " << GP << "LL) + " << FP
       << "LL * xc_gx);\n";
    emit_item_vars(ind);
    os << ind << "const bool xc_miss = fpart != xc_f || gpart != xc_g; xc_f = fpart; xc_g = gpart;\n";
  }

  bool fit() {
    // grow splits on the largest tile while over budget, then spill to global
    for (int iter = 0; iter < 64; ++iter) {
      slices();
      schedule();
      invariants();
      matmul_choices();
      plan_xcache();
      smem_peak = allocate();
      const int tile_budget = prod ? std::min(budget, kSmemCap - (3 * 16384 + 1024) - (int)stage_total) : budget;
      if (smem_peak <= tile_budget) return true;
      // largest smem tile
      int big = -1;
      i64 bb = 0;
      for (int n = 0; n < (int)nodes.size(); ++n) {
        const Node& x = nodes[n];
        if (x.store != ST_SMEM || x.kind == SGM_OUTPUT) continue;
        i64 b = prod4(x.sl) * ec;
        if (b > bb) { bb = b; big = n; }
      }
      if (big < 0) break;
      // try a split of one of its classes (more CTAs share the tile)
      int max_cluster = d.hints.max_cluster > 0 ? std::min(16, d.hints.max_cluster) : 8;
      int bestc = -1;
      i64 bestrem = 0;
      for (int k = 0; k < 4; ++k) {
        int c = nodes[big].cls[k];
        if (c < 0 || cls[c].twice) continue;
        if (cls[c].extent % (cls[c].parts * 2)) continue;
        if (cls[c].reduced && GP == 1 && CL * 2 > max_cluster) continue;
        i64 rem = cls[c].extent / cls[c].parts;
        if (rem > bestrem) { bestrem = rem; bestc = c; }
      }
      if (bestc >= 0 && bestrem >= 2) {
        Class& B = cls[bestc];
        const bool was_c = B.cluster, was_g = B.gsplit;
        B.parts *= 2;
        // a new reduction split: gsplit when one is open already, or when the plan
        // is x-cached (cluster plans cannot keep nodes across items), else cluster
        const bool keep_xc = xcache && !getenv("SGM_NO_XC_FIT");
        if (B.reduced && B.parts == 2) {
          if (GP > 1 || keep_xc) B.gsplit = true;
          else B.cluster = true;
        }
        finalize_layout();
        if (B.gsplit) {  // the reduction must still be a tail reduction
          slices();
          schedule();
          if (!gs_tail_ok()) {
            B.gsplit = was_g;
            if (B.reduced && B.parts == 2 && GP == 1 && keep_xc && CL * 2 <= max_cluster) {
              B.cluster = true;  // no tail reduction: the cluster split after all
              finalize_layout();
            } else {
              B.parts /= 2;
              B.cluster = was_c;
              finalize_layout();
              bestc = -1;
            }
          }
        }
        if (bestc >= 0) continue;
      }
      // spill the largest tile that never takes part in a DSMEM reduction
      int sp = -1;
      i64 sb = 0;
      for (int n = 0; n < (int)nodes.size(); ++n) {
        const Node& x = nodes[n];
        if (x.store != ST_SMEM || x.kind == SGM_OUTPUT || x.pend || x.kind == SGM_ACCUM) continue;
        i64 b = prod4(x.sl) * ec;
        if (b > sb) { sb = b; sp = n; }
      }
      if (sp < 0) break;
      nodes[sp].store = ST_GLOBAL;
    }
    return smem_peak <= (prod ? std::min(budget, kSmemCap - (3 * 16384 + 1024) - (int)stage_total) : budget);
  }

  // ring geometry after the tile plan: as many 16 KB slots as fit (<= 12), capped so
  // that two CTAs share an SM when the grid exceeds one wave
  // Measured on B200 (tools/bench_tma_ring.cu): TMA streaming reaches ~6.3 TB/s with
  // 32 KB stages at one CTA per SM, or 16 KB stages at two CTAs per SM; 8 KB
  // stages stall near 3.8 TB/s whatever the ring depth.
  bool paired = false;  // the ring plan counts on two CTAs per SM
  void plan_ring() {
    paired = false;
    if (!prod) { ringS = 0; return; }
    int base = (smem_peak + 1023) / 1024 * 1024;
    const int stg = (int)stage_total;
    i64 ctas = LB * FP * GP * CL;
    slotB = 32768;
    int S = std::min(6, (kSmemCap - base - 1024 - stg) / slotB);
    if (ctas > num_sms && pairable() && !d.hints.one_cta) {  // two CTAs per SM if 3+ 16 KB slots fit in half the SM
      int S2 = (110 * 1024 - base - 1024 - stg) / 16384;
      if (S2 >= 3) { slotB = 16384; S = std::min(6, S2); paired = true; }
    }
    // 16 KB slots at one CTA per SM (hint): twice the slots for the same bytes, so
    // small boxes (LoRA's 16-column X@A stages) do not each hold a 32 KB slot
    // while the big stream waits behind them
    if (S < 3 || (!paired && d.hints.slot_kb == 16)) {
      slotB = 16384;
      S = std::min(12, (kSmemCap - base - 1024 - stg) / slotB);
    }
    for (auto& x : nodes) {
      if (x.kind != SGM_MATMUL || !x.tma) continue;
      if (x.tc) while (x.kc * (x.sl[3] <= 64 ? 128 : 256) > slotB) x.kc /= 2;
      else while (x.kc * x.bw * 4 > slotB) x.kc /= 2;
    }
    if (paired)  // half of TMEM per CTA: fewer independent accumulators
      for (auto& x : nodes) {
        if (!(x.kind == SGM_MATMUL && x.gemv && x.tc)) continue;
        const i64 ntl = (x.sl[3] + 127) / 128;
        if (x.tma)
          while (x.acc > 1 && ntl * x.acc * 16 > 256) x.acc /= 2;
        int cols = 32;
        while (cols < ntl * (x.tma ? x.acc : 1) * 16) cols *= 2;
        x.tc_cols = cols;
      }
    ringS = S;
    ring_off = base;
    smem_peak = base + 1024 + S * slotB + stg;
  }

  // ------------------------------------------------------------ emission
  std::ostringstream os;

  std::string tile_ptr(int n) const { return "t" + std::to_string(n); }

  const char* nstruct() const {
    switch (ns) {
      case SGM_F64: return "sgm::NF64";
      case SGM_F32: return "sgm::NF32";
      case SGM_BF16: return "sgm::NBF16";
      default: return "sgm::NFF";
    }
  }

  std::string part_var(int c) const { return "p" + std::to_string(c); }

  // global element offset of a loader/saver tile slice (interp.py:90-125 nesting)
  std::string offset_expr(const Node& x, bool loader, const std::string& jexpr) const {
    const i64* dims = loader ? in_dims[x.slot] : out_dims[x.slot];
    const i64* st = loader ? in_strides[x.slot] : out_strides[x.slot];
    std::ostringstream e;
    e << "0LL";
    static const char* gv[3] = {"gx", "gy", "gz"};
    for (int k = 0; k < 4; ++k) {
      i64 w = dims[k];
      if (w <= 1) continue;
      std::ostringstream dim;
      bool any = false;
      for (int g = 0; g < ngrid; ++g)
        if (x.gmask[k] >> g & 1u) {
          w /= grid[g];
          if (grid[g] == 1) continue;  // coordinate always 0
          dim << (any ? " + " : "") << gv[g] << " * " << w << "LL";
          any = true;
        }
      if (loader && x.lsplit[k]) {
        w /= nloop;
        dim << (any ? " + " : "") << "(long long)(" << jexpr << ") * " << w << "LL";
        any = true;
      }
      int c = x.cls[k];
      if (c >= 0 && cls[c].parts > 1) {
        dim << (any ? " + " : "") << part_var(c) << " * " << (x.sh[k] / cls[c].parts) << "LL";
        any = true;
      }
      if (any) e << " + (" << dim.str() << ") * " << st[k] << "LL";
    }
    return e.str();
  }

  // start index along padded dim k of a loader tile slice (same nesting as offset_expr)
  std::string coord_expr(const Node& x, int k, const std::string& jexpr) const {
    const i64* dims = in_dims[x.slot];
    static const char* gv[3] = {"gx", "gy", "gz"};
    i64 w = dims[k];
    std::ostringstream e;
    e << "0";
    if (w <= 1) return e.str();
    for (int g = 0; g < ngrid; ++g)
      if (x.gmask[k] >> g & 1u) {
        w /= grid[g];
        if (grid[g] > 1) e << " + (int)" << gv[g] << " * " << w;
      }
    if (x.lsplit[k]) {
      w /= nloop;
      e << " + (int)(" << jexpr << ") * " << w;
    }
    int c = x.cls[k];
    if (c >= 0 && cls[c].parts > 1) e << " + " << part_var(c) << " * " << (x.sh[k] / cls[c].parts);
    return e.str();
  }

  // producer-side stage sequence of one streamed matmul (mirrors mm_stream_tc / mm_stream_f32)
  void emit_producer_node(int n, bool in_loop, int kb = 0, int ke = -1) {
    const Node& x = nodes[n];
    const Node& a = nodes[x.in[0]];
    const Node& b = nodes[x.in[1]];
    std::string J = in_loop ? "j" : std::to_string(nloop - 1);
    i64 K = a.sl[3], NN = x.sl[3];
    os << "      SGM_TRP(" << 4000 + n << ");\n";
    os << "      { // stream for node " << n << "\n";
    os << "        const int c0 = " << coord_expr(b, 3, J) << ", c1 = " << coord_expr(b, 2, J) << ", c2 = "
       << coord_expr(b, 1, J) << ", c3 = " << coord_expr(b, 0, J) << ";\n";
    os << "        for (int bi = 0; bi < " << x.sl[0] * x.sl[1] << "; ++bi) {\n";
    os << "          const int d2 = c2 + " << (b.sl[1] > 1 ? "bi % " + std::to_string(x.sl[1]) : std::string("0"))
       << ", d3 = c3 + " << (b.sl[0] > 1 ? "bi / " + std::to_string(x.sl[1]) : std::string("0")) << ";\n";
    if (x.tc) {
      i64 ntl = (NN + 127) / 128;
      if (ke < 0) ke = (int)(K / x.kc);
      os << "          for (int kc = " << kb << "; kc < " << ke << "; ++kc)\n";
      os << "            for (int t = 0; t < " << ntl << "; ++t) {\n";
      os << "              const unsigned slot = sgm::ring_acquire<" << ringS << ">(empty, pq++);\n";
      os << "              const int nb = (" << NN << " - t * 128 > 64) ? 2 : 1;\n";
      os << "              sgm::mbar_expect_tx(&full[slot], nb * " << x.kc * 128 << ");\n";
      os << "              unsigned char* dst = ring + slot * " << slotB << ";\n";
      os << "              sgm::tma_load_4d(dst, &a.tm[" << x.tma_id << "], c0 + t * 128, c1 + kc * " << x.kc
         << ", d2, d3, &full[slot]);\n";
      os << "              if (nb == 2) sgm::tma_load_4d(dst + " << x.kc * 128 << ", &a.tm[" << x.tma_id
         << "], c0 + t * 128 + 64, c1 + kc * " << x.kc << ", d2, d3, &full[slot]);\n";
      os << "            }\n";
    } else {
      i64 ntb = (NN + x.bw - 1) / x.bw;
      os << "          for (int t = 0; t < " << ntb << "; ++t)\n";
      os << "            for (int kc = 0; kc < " << K / x.kc << "; ++kc) {\n";
      os << "              const unsigned slot = sgm::ring_acquire<" << ringS << ">(empty, pq++);\n";
      os << "              sgm::mbar_expect_tx(&full[slot], " << x.kc * x.bw * 4 << ");\n";
      os << "              sgm::tma_load_4d(ring + slot * " << slotB << ", &a.tm[" << x.tma_id << "], c0 + t * " << x.bw
         << ", c1 + kc * "
         << x.kc << ", d2, d3, &full[slot]);\n";
      os << "            }\n";
    }
    os << "        }\n      }\n";
  }

  void emit_producer() {
    // the producer fills the ring while the compute warps run the item-invariant
    // prologue (measured: a few % faster than holding it back so the prologue's
    // loads do not queue behind TMA traffic; SGM_LATE_STREAM=1 restores the wait)
    os << "    if (tid == NT) {\n      unsigned pq = 0;\n";
    if (d.hints.wd_test) os << "      return;  // wd_test: nothing is streamed, every ring wait must time out\n";
    if (getenv("SGM_LATE_STREAM")) os << "      sgm::mbar_wait(go, 0);\n";
    os << "      unsigned pit = 0;\n";
    emit_item_loop("      ", "pit");
    os << "      SGM_TRP(3);\n";
    for (auto& x : nodes) {
      if (!x.staged) continue;
      const std::string J = std::to_string(nloop - 1);
      os << "      { // staged loader tile\n";
      os << "        if (pit > 0u) sgm::mbar_wait(&sempty[" << x.stage_id << "], (pit - 1u) & 1u);\n";
      os << "        sgm::mbar_expect_tx(&sfull[" << x.stage_id << "], " << prod4(x.sl) * es << "u);\n";
      os << "        const int c0 = " << coord_expr(x, 3, J) << ", c1 = " << coord_expr(x, 2, J) << ", c2 = "
         << coord_expr(x, 1, J) << ", c3 = " << coord_expr(x, 0, J) << ";\n";
      os << "        for (int b = 0; b < " << x.sl[3] / x.sbox << "; ++b) sgm::tma_load_4d(stg + " << x.stage_off << " + b * "
         << (i64)x.sbox * x.sl[0] * x.sl[1] * x.sl[2] * es << ", &a.tm[" << x.tma_id << "], c0 + b * " << x.sbox
         << ", c1, c2, c3, &sfull[" << x.stage_id << "]);\n      }\n";
    }
    bool in_loop = false;
    for (int p = 0; p < (int)sched.size(); ++p) {
      const Ev& e = sched[p];
      if (e.type == Ev::LOOP_BEGIN) {
        if (xcache_loop) os << "      if (xc_miss) {\n";
        os << "      for (int j = jp * " << nloop / LP << "; j < (jp + 1) * " << nloop / LP << "; ++j) {\n";
        in_loop = true;
      } else if (e.type == Ev::LOOP_END) {
        os << "      }\n";
        if (xcache_loop) os << "      }\n";
        in_loop = false;
      } else if (e.type == Ev::NODE) {
        if (p == ilv_pos) emit_producer_node(ilv_big, in_loop, 0, ilv_kc);
        if (nodes[e.node].kind == SGM_MATMUL && nodes[e.node].tma) {
          const bool wrap = nodes[e.node].xc && !(in_loop && xcache_loop);
          if (wrap) os << "      if (xc_miss) {\n";
          emit_producer_node(e.node, in_loop, e.node == ilv_big ? ilv_kc : 0);
          if (wrap) os << "      }\n";
        }
      }
    }
    os << "      }\n      SGM_TRP(6);\n    }\n    return;\n";
  }

  // vector width for a loader (x) or a saver (x = saver node, sl = its input's slice)
  int io_vec(const Node& x, bool loader, const i64* sl = nullptr) const {
    const i64* dims = loader ? in_dims[x.slot] : out_dims[x.slot];
    const i64* st = loader ? in_strides[x.slot] : out_strides[x.slot];
    if (!sl) sl = x.sl;
    int v = vecw;
    if (sl[3] % v) return 1;
    for (int k = 0; k < 3; ++k)
      if (dims[k] > 1 && st[k] % v) return 1;
    return v;
  }

  std::string const_literal(const Node& x) const {
    char buf[64];
    if (ns == SGM_FF) {
      snprintf(buf, sizeof buf, "%uu", ff_const(x.cnum, x.cden));
    } else if (ns == SGM_F64) {
      double v = (double)x.cnum / (double)x.cden;
      snprintf(buf, sizeof buf, "%a", v);
    } else {
      double v = (double)x.cnum / (double)x.cden;
      snprintf(buf, sizeof buf, "%af", (double)(float)v);
    }
    return buf;
  }

  // dense strides of a slice with broadcast zeros where the consumer needs it
  void dense_strides(const i64* sl, i64* out) const {
    i64 s = 1;
    for (int k = 3; k >= 0; --k) {
      out[k] = sl[k] > 1 ? s : 0;
      s *= sl[k];
    }
  }

  std::string saver_pred(const Node& x) const {
    std::ostringstream p;
    p << "true";
    const Node& src = nodes[x.in[0]];
    for (int c = 0; c < (int)cls.size(); ++c) {
      if (cls[c].parts <= 1 || cls[c].gsplit) continue;  // gsplit parts: only the group's last item gets here
      if (has_cls(src, c)) continue;
      p << " && " << part_var(c) << " == 0";
    }
    if (LP > 1 && !loop_gs) p << " && jp == 0";
    return p.str();
  }

  std::string cl_sync() const {
    if (prod) return "    sgm::cl_barrier<NT, " + std::to_string(CL) + ">(clbar, sclph);\n";
    return "    sgm::cluster_sync();\n";
  }

  // one-barrier push flush for small tiles (two receive buffers of CL slots each)
  static constexpr i64 kPushBudget = 32 * 1024;
  static i64 pad4(i64 n) { return (n + 3) / 4 * 4; }
  bool push_flush(const std::vector<int>& fl) const {
    if (CL <= 1) return false;
    i64 b = 0;
    for (int f : fl) b += 2 * CL * pad4(prod4(nodes[f].sl)) * ec;
    return b <= kPushBudget;
  }

  void emit_flush(const std::vector<int>& fl, int pos) {
    if (push_flush(fl)) {
      for (int f : fl) {
        const Node& x = nodes[f];
        const u32 keep = (u32)(CL - 1) & ~x.pend;
        const i64 szp = pad4(prod4(x.sl));
        os << "    sgm::cl_push<N, " << prod4(x.sl) << ", " << szp << ", " << CL << ", " << keep << "u, NT>("
           << tile_ptr(f) << ", (C*)(sm + " << flush_tmp_off.at({pos, f}) << ") + (cit & 1u) * " << CL * szp
           << ", crank);\n";
      }
      os << cl_sync();
      os << "  SGM_TR(" << 3000 + 4 * pos + 1 << ");\n";
      for (int f : fl) {
        const Node& x = nodes[f];
        const u32 keep = (u32)(CL - 1) & ~x.pend;
        const i64 szp = pad4(prod4(x.sl));
        os << "    sgm::cl_gather<N, " << prod4(x.sl) << ", " << szp << ", " << CL << ", " << keep << "u, NT>("
           << tile_ptr(f) << ", (const C*)(sm + " << flush_tmp_off.at({pos, f}) << ") + (cit & 1u) * " << CL * szp
           << ", crank);\n";
      }
      os << "    sgm::csync<NT>();\n";
      os << "  SGM_TR(" << 3000 + 4 * pos + 3 << ");\n";
      return;
    }
    // reduce-scatter (DSMEM loads into tmp) + all-gather (DSMEM stores)
    os << cl_sync();
    os << "  SGM_TR(" << 3000 + 4 * pos + 1 << ");\n";
    for (int f : fl) {
      const Node& x = nodes[f];
      u32 keep = (u32)(CL - 1) & ~x.pend;
      os << "    sgm::cl_rs_phase1<N, " << prod4(x.sl) << ", " << CL << ", " << keep << "u, NT>(" << tile_ptr(f)
         << ", (C*)(sm + " << flush_tmp_off.at({pos, f}) << "), crank);\n";
    }
    os << cl_sync();
    os << "  SGM_TR(" << 3000 + 4 * pos + 2 << ");\n";
    for (int f : fl) {
      const Node& x = nodes[f];
      u32 keep = (u32)(CL - 1) & ~x.pend;
      os << "    sgm::cl_rs_phase2<N, " << prod4(x.sl) << ", " << CL << ", " << keep << "u, NT>(" << tile_ptr(f)
         << ", (const C*)(sm + " << flush_tmp_off.at({pos, f}) << "), crank);\n";
    }
    os << cl_sync();
    os << "  SGM_TR(" << 3000 + 4 * pos + 3 << ");\n";
  }

  // gsplit tail reduction: every work item of a group stores its partial tiles to
  // the global workspace and counts itself in; the last one sums the partials in
  // part order (bit-identical whatever the arrival order), resets the counter
  // and runs the rest of the item; the others go on to their next item.
  i64 gws_off = 0, gcnt_off = 0, gws_tile = 0, gws_end = 0;
  void emit_gflush(const std::vector<int>& fl, int gpos) {
    i64 fo[SGM_MAX_NODES];
    i64 tot = 0;
    for (int f : fl) { fo[f] = tot; tot += (prod4(nodes[f].sl) + 3) / 4 * 4; }  // 16-byte aligned slots
    gws_tile = tot;
    os << "    {\n      C* gw = (C*)((unsigned char*)a.scratch + " << gws_off << "LL);\n";
    os << "      unsigned* gcnt = (unsigned*)((unsigned char*)a.scratch + " << gcnt_off << "LL);\n";
    for (int f : fl)
      os << "      sgm::gws_store<N, " << prod4(nodes[f].sl) << ", NT>(gw + (grp * " << GP << " + gpart) * " << tot
         << "LL + " << fo[f] << ", " << tile_ptr(f) << ");\n";
    // the CTA barrier orders every thread's partial stores before thread 0's
    // acq_rel counter update (cumulativity), so one gpu-scope RMW replaces a
    // fence per thread; the last arrival's acquire covers all groups' partials
    os << "      sgm::csync<NT>();\n";
    os << "      if (tid == 0) sgm_last = (sgm::atom_add_acq_rel(&gcnt[grp], 1u) == " << GP - 1 << "u);\n";
    os << "      sgm::csync<NT>();\n    }\n";
    os << "  SGM_TR(" << 3000 + 4 * gpos + 1 << ");\n";
    os << "  if (sgm_last) {\n";
    os << "    {\n      const C* gw = (const C*)((unsigned char*)a.scratch + " << gws_off << "LL);\n";
    for (int f : fl)
      os << "      sgm::gws_reduce<N, " << prod4(nodes[f].sl) << ", " << GP << ", " << tot << "LL, NT>(" << tile_ptr(f)
         << ", gw + grp * " << GP * tot << "LL + " << fo[f] << ");\n";
    os << "      if (tid == 0) ((unsigned*)((unsigned char*)a.scratch + " << gcnt_off << "LL))[grp] = 0u;\n";
    os << "      sgm::csync<NT>();\n    }\n";
    os << "  SGM_TR(" << 3000 + 4 * gpos + 2 << ");\n";
  }

  // Elementwise map over node n's tile: each thread computes 4 elements into
  // registers before storing any.  In-place ops (output aliasing an operand)
  // otherwise serialise every iteration's loads behind the previous store.
  static bool elementwise(int k) {
    return k == SGM_EXP || k == SGM_SILU || k == SGM_SQUARE || k == SGM_SQRT || k == SGM_SCALE || k == SGM_DIV ||
           k == SGM_MUL || k == SGM_ADD;
  }
  bool same_slice(const Node& a, const Node& b) const {
    for (int k = 0; k < 4; ++k)
      if (a.sl[k] != b.sl[k]) return false;
    return true;
  }
  i64 tile_end(const Node& x) const { return x.off + prod4(x.sl) * ec; }

  // Elementwise chains fused in registers: node k is evaluated inside the map of
  // its only consumer y when both are elementwise over the same slice, y comes
  // right after k in the schedule (same region, no flush or loop boundary in
  // between), k is not a pending partial, and y's output tile does not overlap
  // the tiles the fused expression reads (the allocator freed k's operands at k).
  void plan_fusion() {
    fused.assign(nodes.size(), 0);
    if (getenv("SGM_NO_FUSE")) return;
    std::set<int> flushed;
    for (auto& e : sched)
      if (e.type == Ev::FLUSH || e.type == Ev::GFLUSH)
        for (int f : e.flush) flushed.insert(f);
    for (int p = 0; p + 1 < (int)sched.size(); ++p) {
      if (sched[p].type != Ev::NODE || sched[p + 1].type != Ev::NODE) continue;
      const int k = sched[p].node, y = sched[p + 1].node;
      const Node& K = nodes[k];
      const Node& Y = nodes[y];
      if (!elementwise(K.kind) || !elementwise(Y.kind) || K.cons.size() != 1 || K.cons[0] != y) continue;
      if (k == acc_add || y == acc_add) continue;
      if (K.store != ST_SMEM || Y.store != ST_SMEM || !same_slice(K, Y) || K.pend || K.gpend || flushed.count(k)) continue;
      if (K.inv != Y.inv || K.hoist != Y.hoist || K.body != Y.body) continue;
      // leaves the fused expression reads (k's operands, recursively through fused ones)
      std::vector<int> leaves, stack = {k};
      while (!stack.empty()) {
        const int q = stack.back();
        stack.pop_back();
        for (int i = 0; i < nodes[q].nin; ++i) {
          const int in = nodes[q].in[i];
          if (fused[in]) stack.push_back(in);
          else leaves.push_back(in);
        }
      }
      bool ok = true;
      for (int l : leaves) {
        const Node& L = nodes[l];
        if (L.store != ST_SMEM) { ok = false; break; }
        // y's output over an operand of the fused expression: only element-wise
        // aliasing (same slice: each element read and written by one thread) is safe
        if (L.off < tile_end(Y) && Y.off < tile_end(L) && !(same_slice(L, Y) && L.off == Y.off)) { ok = false; break; }
      }
      if (ok) fused[k] = 1;
    }
  }

  void plan_accfuse() {
    acc_first = acc_second = acc_add = -1;
    if (getenv("SGM_NO_ACCFUSE") || !prod || ilv_big >= 0) return;
    std::vector<int> pos(nodes.size(), -1);
    for (int p = 0; p < (int)sched.size(); ++p)
      if (sched[p].type == Ev::NODE) pos[sched[p].node] = p;
    for (int n = 0; n < (int)nodes.size(); ++n) {
      const Node& ad = nodes[n];
      if (ad.kind != SGM_ADD || ad.inv || ad.body) continue;
      int a = ad.in[0], b = ad.in[1];
      if (a == b) continue;
      const Node& A = nodes[a];
      const Node& B = nodes[b];
      auto ok = [&](const Node& m) {
        return m.kind == SGM_MATMUL && m.tma && m.tc && !m.inv && !m.body && m.cons.size() == 1 &&
               m.sl[0] * m.sl[1] == 1 && same_slice(m, ad);
      };
      if (!ok(A) || !ok(B) || A.acc != B.acc || A.tc_cols != B.tc_cols || A.xc || B.xc) continue;
      if (pos[a] < 0 || pos[b] < 0) continue;
      int f = pos[a] < pos[b] ? a : b, sec = f == a ? b : a;
      // adjacent, nothing in between (measured: X@W first with X@A -> T@B in their own
      // TMEM columns after it was 9% slower on L -- the chain's stream queues behind W)
      if (pos[sec] != pos[f] + 1 || pos[n] < pos[sec]) continue;
      const Node& F = nodes[f];
      const int nmma = (int)(nodes[F.in[0]].sl[3] / 16);
      acc_first = f;
      acc_second = sec;
      acc_add = n;
      acc_pre = std::min(F.acc, nmma);
      return;
    }
  }

  void plan_inv() {
    inv_first.assign(nodes.size(), 0);
    if (ns != SGM_FF || getenv("SGM_NO_INVFIRST")) return;
    for (auto& d : nodes) {
      if (d.kind != SGM_DIV) continue;
      const int bi = d.in[1];
      const Node& b = nodes[bi];
      if (d.in[0] == bi || b.store != ST_SMEM || b.cons.size() != 1 || fused[bi] || b.pend || b.gpend) continue;
      if (prod4(b.sl) >= prod4(d.sl) || b.inv != d.inv || b.hoist != d.hoist || b.body != d.body) continue;
      if (b.kind == SGM_INPUT && b.staged) continue;
      inv_first[bi] = 1;
    }
  }

  // value of elementwise node n at flat element e (index decomposition i0..i3 of
  // the slice in scope), with fused operands inlined
  std::string val_expr(int n) const {
    const Node& x = nodes[n];
    auto idx = [&](const Node& a) {
      i64 sa[4];
      dense_strides(a.sl, sa);
      std::ostringstream q;
      q << "0";
      const char* iv[4] = {"i0", "i1", "i2", "i3"};
      for (int k = 0; k < 4; ++k)
        if (a.sl[k] > 1) q << " + " << iv[k] << " * " << sa[k];
      return q.str();
    };
    auto arg = [&](int k, bool unary) {
      if (fused[k]) return "(" + val_expr(k) + ")";
      return tile_ptr(k) + "[" + (unary ? std::string("e") : idx(nodes[k])) + "]";
    };
    switch (x.kind) {
      case SGM_EXP: return "N::ex(" + arg(x.in[0], true) + ")";
      case SGM_SILU: return "N::silu(" + arg(x.in[0], true) + ")";
      case SGM_SQUARE: return "N::sq(" + arg(x.in[0], true) + ")";
      case SGM_SQRT: return "N::sqr(" + arg(x.in[0], true) + ")";
      case SGM_SCALE: return "N::scale(" + arg(x.in[0], true) + ", (C)" + const_literal(x) + ")";
      default: {
        const char* fn = x.kind == SGM_DIV ? (inv_first[x.in[1]] ? "N::mul" : "N::div")
                         : x.kind == SGM_MUL ? "N::mul" : "N::add";
        return std::string(fn) + "(" + arg(x.in[0], false) + ", " + arg(x.in[1], false) + ")";
      }
    }
  }

  void emit_map(int n, const std::string& pre, const std::string& expr) {
    const i64 sz = prod4(nodes[n].sl);
    os << "    for (int e0 = tid; e0 < " << sz << "; e0 += 4 * NT) {\n      C v_[4];\n";
    // guarded (not clamped) reads: a clamped index made out-of-range lanes re-read the
    // last element while its owner wrote it in place (a benign but real smem race,
    // compute-sanitizer racecheck)
    os << "#pragma unroll\n      for (int j = 0; j < 4; ++j) {\n        const int e = e0 + j * NT;\n";
    os << "        if (e < " << sz << ") { " << pre << "v_[j] = " << expr << "; }\n      }\n";
    os << "#pragma unroll\n      for (int j = 0; j < 4; ++j) {\n        const int e = e0 + j * NT;\n";
    os << "        if (e < " << sz << ") " << tile_ptr(n) << "[e] = v_[j];\n      }\n    }\n";
  }

  void emit_node(int n, bool in_loop) {
    Node& x = nodes[n];
    std::string J = in_loop ? "j" : std::to_string(nloop - 1);
    os << "    // node " << n << " kind " << x.kind << " slice [" << x.sl[0] << "," << x.sl[1] << "," << x.sl[2] << ","
       << x.sl[3] << "]\n";
    switch (x.kind) {
      case SGM_INPUT: {
        if (x.store == ST_VIEW || x.store == ST_XG) return;  // read by its consumer (pointer built there)
        if (x.staged) {
          os << "    sgm::mbar_wait(&sfull[" << x.stage_id << "], cit & 1u);\n";
          os << "    sgm::stage_convert<N, " << x.sl[0] << ", " << x.sl[1] << ", " << x.sl[2] << ", " << x.sl[3] << ", "
             << x.sbox << ", NT>(" << tile_ptr(n) << ", (const S*)(stg + " << x.stage_off << "));\n";
          os << "    sgm::csync<NT>();\n    if (tid == 0) sgm::mbar_arrive(&sempty[" << x.stage_id << "]);\n";
          return;
        }
        if (in_loop && !pf.empty() && pf[n] == 2) {  // column strip: a 16-byte load per row every G iterations
          const i64 G = 16 / es / x.sl[3];  // iterations per strip
          const std::string j0 = "(jp * " + std::to_string(nloop / LP) + ")";
          // the next strip is loaded right after the last column of this one is written
          os << "    st" << n << ".store(" << tile_ptr(n) << ", (j - " << j0 << ") & " << G - 1 << ");\n";
          os << "    if (((j - " << j0 << ") & " << G - 1 << ") == " << G - 1 << " && j + 1 < (jp + 1) * " << nloop / LP
             << ") st" << n << ".load((const S*)a.in[" << x.slot << "] + (" << offset_expr(x, true, "(j + 1)") << "));\n";
          break;
        }
        if (in_loop && !pf.empty() && pf[n] == 1) {  // this iteration's tile from registers, the next one's loads issued
          os << "    pf" << n << ".store(" << tile_ptr(n) << ");\n";
          os << "    if (j + 1 < (jp + 1) * " << nloop / LP << ") pf" << n << ".load((const S*)a.in[" << x.slot << "] + ("
             << offset_expr(x, true, "(j + 1)") << "));\n";
          break;
        }
        std::string off = offset_expr(x, true, J);
        const i64* st = in_strides[x.slot];
        os << "    sgm::load_tile<N, " << x.sl[0] << ", " << x.sl[1] << ", " << x.sl[2] << ", " << x.sl[3] << ", "
           << st[0] << "LL, " << st[1] << "LL, " << st[2] << "LL, " << st[3] << "LL, " << io_vec(x, true)
           << ", NT>(" << tile_ptr(n) << ", (const S*)a.in[" << x.slot << "] + (" << off << "));\n";
        break;
      }
      case SGM_OUTPUT: {
        const Node& src = nodes[x.in[0]];
        std::string off = offset_expr(x, false, "0");
        const i64* st = out_strides[x.slot];
        os << "    if (" << saver_pred(x) << ") sgm::store_tile<N, " << src.sl[0] << ", " << src.sl[1] << ", "
           << src.sl[2] << ", " << src.sl[3] << ", " << st[0] << "LL, " << st[1] << "LL, " << st[2] << "LL, "
           << st[3] << "LL, " << io_vec(x, false, src.sl) << ", NT>((S*)a.out[" << x.slot << "] + (" << off << "), "
           << tile_ptr(x.in[0]) << ");\n";
        return;  // no barrier needed after a global store
      }
      case SGM_EXP: case SGM_SILU: case SGM_SQUARE: case SGM_SQRT: case SGM_SCALE:
      case SGM_DIV: case SGM_MUL: case SGM_ADD: {
        if (x.kind == SGM_DIV && inv_first[x.in[1]]) {  // invert the divisor tile once, in place
          const i64 sz = prod4(nodes[x.in[1]].sl);
          os << "    for (int e = tid; e < " << sz << "; e += NT) " << tile_ptr(x.in[1]) << "[e] = N::inv("
             << tile_ptr(x.in[1]) << "[e]);\n    sgm::csync<NT>();\n";
        }
        if (fused[n]) return;  // evaluated inside its consumer's map
        if (n == acc_add) {  // the sum was formed in TMEM by the accumulate-into pair
          emit_map(n, "", tile_ptr(acc_second) + "[e]");
          break;
        }
        std::ostringstream pre;
        pre << "int r = e; const int i3 = r % " << x.sl[3] << "; r /= " << x.sl[3] << "; const int i2 = r % " << x.sl[2]
            << "; r /= " << x.sl[2] << "; const int i1 = r % " << x.sl[1] << "; const int i0 = r / " << x.sl[1]
            << "; (void)i0; (void)i1; (void)i2; (void)i3; ";
        emit_map(n, pre.str(), val_expr(n));
        break;
      }
      case SGM_ACCUM: {
        emit_map(n, "", "N::add(" + tile_ptr(n) + "[e], " + tile_ptr(x.in[0]) + "[e])");
        break;
      }
      case SGM_SUM: {
        const Node& a = nodes[x.in[0]];
        int ax = x.axis + 4 - a.rank;
        os << "    sgm::sum_axis<N, " << a.sl[0] << ", " << a.sl[1] << ", " << a.sl[2] << ", " << a.sl[3] << ", " << ax
           << ", NT>(" << tile_ptr(n) << ", " << tile_ptr(x.in[0]) << ");\n";
        break;
      }
      case SGM_MATMUL: {
        const Node& a = nodes[x.in[0]];
        const Node& b = nodes[x.in[1]];
        i64 M = x.sl[2], K = a.sl[3], NN = x.sl[3];
        auto strides_of = [&](const Node& t, i64* s) {
          if (t.store == ST_VIEW) {
            const i64* st = in_strides[t.slot];
            for (int k = 0; k < 4; ++k) s[k] = t.sl[k] > 1 ? st[k] : 0;
          } else {
            dense_strides(t.sl, s);
          }
        };
        i64 sa[4], sb[4];
        strides_of(a, sa);
        strides_of(b, sb);
        auto view_ptr = [&](const Node& t) {
          return "((const S*)a.in[" + std::to_string(t.slot) + "] + (" + offset_expr(t, true, J) + "))";
        };
        std::string pa = a.store == ST_VIEW ? view_ptr(a) : tile_ptr(x.in[0]);
        std::string pb = b.store == ST_VIEW ? view_ptr(b) : tile_ptr(x.in[1]);
        bool build = x.xb_build;
        const bool chain_node = ilv_big >= 0 && ilv_chain.count(n);
        const bool prebuilt = chain_node && x.in[0] == nodes[ilv_big].in[0] && x.at_off == nodes[ilv_big].at_off;
        if (x.tma && x.tc && a.store == ST_XG) {
          const bool big_build = n == ilv_big ? emit_seg1 : x.xb_build;
          if (big_build && !prebuilt) {
            os << "    sgm::build_xb_g<" << M << ", " << K << ", " << in_strides[a.slot][2] << "LL, NT>((u16*)(sm + "
               << x.at_off << "), (const u16*)" << view_ptr(a) << ");\n";
            os << "    sgm::fence_async_smem();\n    sgm::csync<NT>();\n";
            os << "  SGM_TR(" << 600 + n << ");  // A^T built\n";
          }
          pa = "(const float*)nullptr";
          build = false;
        }
        if (x.tma && x.tc) {
          // interleaved big stream: its first ilv_kc k-chunks were issued before the chain
          std::string seg =
              n != ilv_big ? std::string()
                           : emit_seg1 ? ", 0, " + std::to_string(ilv_kc) + ", false"
                                       : ", " + std::to_string(ilv_kc) + ", " + std::to_string(K / x.kc) + ", true";
          if (n == acc_first) seg = ", 0, " + std::to_string(K / x.kc) + ", false";
          if (n == acc_second) seg = ", 0, " + std::to_string(K / x.kc) + ", true, " + std::to_string(acc_pre);
          const std::string tm = chain_node ? "tmem_base + " + std::to_string(ilv_tmem) + "u" : std::string("tmem_base");
          os << "    sgm::mm_stream_tc<" << x.sl[0] << ", " << x.sl[1] << ", " << M << ", " << K << ", " << NN << ", "
             << sa[0] << "LL, " << sa[1] << "LL, " << sa[2] << "LL, " << sa[3] << "LL, " << x.kc << ", " << ringS << ", "
             << slotB << ", NT, " << (build ? "true" : "false") << ", " << x.acc << seg << ">(" << tile_ptr(n) << ", " << pa
             << ", sm + " << x.at_off << ", " << tm << ", ring, full, empty, done, sq, sdph);\n";
        } else if (x.tma) {
          os << "    sgm::mm_stream_f32<N, " << x.sl[0] << ", " << x.sl[1] << ", " << M << ", " << K << ", " << NN << ", "
             << sa[0] << "LL, " << sa[1] << "LL, " << sa[2] << "LL, " << sa[3] << "LL, " << x.kc << ", " << x.bw << ", "
             << ringS << ", " << slotB << ", NT>(" << tile_ptr(n) << ", " << pa << ", (C*)(sm + " << x.at_off << "), (A*)(sm + "
             << x.red_off << "), ring, full, empty, sq);\n";
        } else if (x.gemv && x.tc) {
          os << "    sgm::mm_gemv_tc<" << x.sl[0] << ", " << x.sl[1] << ", " << M << ", " << K << ", " << NN << ", "
             << sa[0] << "LL, " << sa[1] << "LL, " << sa[2] << "LL, " << sa[3] << "LL, " << sb[0] << "LL, " << sb[1]
             << "LL, " << sb[2] << "LL, " << x.tc_kc << ", " << x.tc_s << ", NT>(" << tile_ptr(n) << ", " << pa
             << ", " << pb << ", sm + " << x.at_off << ", tmem_base);\n";
        } else if (x.gemv) {
          os << "    sgm::mm_gemv<N, S, " << x.sl[0] << ", " << x.sl[1] << ", " << M << ", " << K << ", " << NN << ", "
             << sa[0] << "LL, " << sa[1] << "LL, " << sa[2] << "LL, " << sa[3] << "LL, " << sb[0] << "LL, " << sb[1]
             << "LL, " << sb[2] << "LL, " << x.vn << ", " << x.ks << ", " << x.unr << ", "
             << (x.shfl ? "true" : "false") << ", NT>(" << tile_ptr(n) << ", " << pa << ", " << pb << ", (A*)(sm + "
             << x.red_off << "), (C*)(sm + " << x.at_off << "));\n";
        } else {
          std::string ta = a.store == ST_VIEW ? "S" : "C";
          std::string tb = b.store == ST_VIEW ? "S" : "C";
          os << "    sgm::mm_generic<N, " << ta << ", " << tb << ", " << x.sl[0] << ", " << x.sl[1] << ", " << M << ", "
             << K << ", " << NN << ", " << sa[0] << "LL, " << sa[1] << "LL, " << sa[2] << "LL, " << sa[3] << "LL, "
             << sb[0] << "LL, " << sb[1] << "LL, " << sb[2] << "LL, " << sb[3] << "LL, NT>(" << tile_ptr(n) << ", "
             << pa << ", " << pb << ");\n";
        }
        break;
      }
      default: break;
    }
    os << "    sgm::csync<NT>();\n";
  }

  // per-item coordinates: free part, grid coordinates, free-part split indices
  void emit_item_vars(const char* ind) {
    static const char* gv[3] = {"gx", "gy", "gz"};
    os << ind << "long long rest = item;\n";
    os << ind << "const long long gpart = rest % " << GP << "; rest /= " << GP << "; (void)gpart;\n";
    os << ind << "const long long grp = rest; (void)grp;  // reduction group (gsplit)\n";
    os << ind << "const long long fpart = rest % " << FP << "; rest /= " << FP << "; (void)fpart;\n";
    for (int g = 0; g < ngrid; ++g)
      os << ind << "const long long " << gv[g] << " = rest % " << grid[g] << "; rest /= " << grid[g] << "; (void)"
         << gv[g] << ";\n";
    for (int c = 0; c < (int)cls.size(); ++c) {
      if (cls[c].parts <= 1 || cls[c].cluster) continue;
      os << ind << "const int " << part_var(c) << " = (int)((" << (cls[c].gsplit ? "gpart" : "fpart") << " / "
         << cls[c].radix << "LL) % " << cls[c].parts << "LL);\n";
    }
    if (LP > 1 && loop_gs) os << ind << "const int jp = (int)(gpart % " << LP << "LL);\n";
  }

  void emit() {
    plan_prefetch();
    if (d.hints.no_wd) os << "#define SGM_WD_MODE 0  // canonical unbounded waits (no watchdog)\n";
    os << "#include \"sgm_dev.cuh\"\n";
    os << "// generated by sgm_codegen.cpp: logical blocks " << LB << ", free parts " << FP << ", cluster " << CL
       << ", loop parts " << LP << "\n";
    os << "typedef " << nstruct() << " N;\ntypedef N::S S;\ntypedef N::C C;\ntypedef N::A A;\n";
    os << "#define NT " << NT << "\n";
    // a paired plan must get its two CTAs per SM: cap registers at 64K / (2 x threads)
    // (the fp32 consumer otherwise compiled to ~116 and ran one CTA per SM at 3x the time)
    os << "extern \"C\" __global__ void __launch_bounds__(" << (prod ? NT + 32 : NT) << (paired ? ", 2" : "") << ")";
    if (CL > 1) os << " __cluster_dims__(" << CL << ", 1, 1)";
    os << " @KNAME@(const __grid_constant__ sgm::Args a) {\n";
    os << "  extern __shared__ __align__(1024) unsigned char sm[];\n";
    os << "  const int tid = threadIdx.x;\n";
    os << "  const long long bid = blockIdx.x;\n";
    if (CL > 1) os << "  const unsigned crank = sgm::cluster_rank();\n";
    else os << "  const unsigned crank = 0u; (void)crank;\n";
    // persistent: cluster `cid` of `ncl` processes work items cid, cid + ncl, ... (item = logical
    // block x free part); the cluster-split parts and loop part are fixed per CTA
    os << "  const long long cid = bid / " << CL << ", ncl = (long long)gridDim.x / " << CL << ";\n";
    for (int c = 0; c < (int)cls.size(); ++c) {
      if (cls[c].parts <= 1 || !cls[c].cluster) continue;
      os << "  const int " << part_var(c) << " = (int)((crank >> " << cls[c].bit_shift << ") & " << (cls[c].parts - 1)
         << "u);\n";
    }
    if (LP > 1 && !loop_gs) os << "  const int jp = (int)((crank >> " << loop_shift << ") & " << (LP - 1) << "u);\n";
    else if (LP == 1) os << "  const int jp = 0; (void)jp;\n";
    if (scratch_per_cta > 0 || GP > 1)
      os << "  unsigned char* scr = (unsigned char*)a.scratch + bid * " << scratch_per_cta << "LL;\n";
    if (d.hints.trace) {
      os << "  unsigned long long* trc = (unsigned long long*)(scr + " << trace_off << ");\n";
      os << "  unsigned tpos = 0, ppos = " << SGM_TRACE_N / 2 << ";\n";
      os << "#define SGM_TR(ev) do { if (tid == 0 && tpos < " << SGM_TRACE_N / 2
         << "u) { trc[2 * tpos] = sgm::gtimer(); trc[2 * tpos + 1] = (ev); ++tpos; } } while (0)\n";
      os << "#define SGM_TRP(ev) do { if (ppos < " << SGM_TRACE_N
         << "u) { trc[2 * ppos] = sgm::gtimer(); trc[2 * ppos + 1] = (ev); ++ppos; } } while (0)\n";
    } else {
      os << "#define SGM_TR(ev) do {} while (0)\n#define SGM_TRP(ev) do {} while (0)\n";
    }
    // programmatic dependent launch: the next launch in the stream may start its
    // CTAs as ours retire; it waits (griddepcontrol.wait) for our completion and
    // memory before touching global memory.  No-ops without the launch attribute.
    os << "  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");\n";
    if (!prod) os << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
    os << "  SGM_TR(0);  // entry\n";
    for (int n = 0; n < (int)nodes.size(); ++n) {
      const Node& x = nodes[n];
      if (x.store == ST_SMEM && x.kind != SGM_OUTPUT)
        os << "  C* " << tile_ptr(n) << " = (C*)(sm + " << x.off << ");\n";
      else if (x.store == ST_GLOBAL)
        os << "  C* " << tile_ptr(n) << " = (C*)(scr + " << x.off << ");\n";
    }
    if (prod) {
      // ring barriers; the producer warp (threads NT..NT+31) runs ahead of the compute warps
      os << "  __shared__ __align__(8) unsigned long long sgm_bars[" << 2 * ringS + 3 + 2 * std::max(nstaged, 1) << "];\n";
      os << "  unsigned long long* full = sgm_bars;\n  unsigned long long* empty = sgm_bars + " << ringS
         << ";\n  unsigned long long* done = sgm_bars + " << 2 * ringS << ";\n  unsigned long long* clbar = sgm_bars + "
         << 2 * ringS + 1 << ";\n  unsigned long long* go = sgm_bars + " << 2 * ringS + 2
         << ";\n  unsigned long long* sfull = sgm_bars + " << 2 * ringS + 3 << ";\n  unsigned long long* sempty = sfull + "
         << std::max(nstaged, 1) << ";\n  (void)done; (void)clbar; (void)go; (void)sfull; (void)sempty;\n";

      os << "  unsigned char* ring = sm + " << ring_off << ";\n";
      os << "  ring += (1024u - (sgm::smem_u32(ring) & 1023u)) & 1023u;\n";
      os << "  unsigned char* stg = ring + " << ringS * slotB << "; (void)stg;  // staged loader tiles\n";
      bool any_tc = false;
      for (auto& x : nodes) any_tc = any_tc || (x.kind == SGM_MATMUL && x.tma && x.tc);
      os << "  if (tid == 0) {\n";
      os << "    for (int q = 0; q < " << ringS << "; ++q) { sgm::mbar_init(&full[q], 1); sgm::mbar_init(&empty[q], "
         << (any_tc ? 1 : NT / 32) << "); }\n";
      os << "    sgm::mbar_init(done, 1);\n    sgm::mbar_init(clbar, " << CL << ");\n    sgm::mbar_init(go, 1);\n";
      if (nstaged) os << "    for (int q = 0; q < " << nstaged << "; ++q) { sgm::mbar_init(&sfull[q], 1); sgm::mbar_init(&sempty[q], 1); }\n";
      os << "    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n  }\n";
      os << "  if (tid == NT) {\n";
      for (auto& x : nodes)
        if ((x.kind == SGM_MATMUL && x.tma) || x.staged) os << "    sgm::tma_prefetch_desc(&a.tm[" << x.tma_id << "]);\n";
      os << "  }\n";
      os << "  __syncthreads();\n";
      if (CL > 1) os << "  sgm::cluster_sync();\n";
      // barrier init and descriptor prefetch (kernel parameters only) overlapped the
      // previous grid's tail; inputs, outputs and scratch wait for its completion
      os << "  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");\n";
      os << "  if (tid >= NT) {\n";
      emit_producer();
      os << "  }\n";
      os << "  unsigned sq = 0, sdph = 0, sclph = 0; (void)sq; (void)sdph; (void)sclph;\n";
    }
    int tmem_cols = 0;
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && x.gemv && x.tc) tmem_cols = std::max(tmem_cols, x.tc_cols);
    if (ilv_big >= 0) {  // big-stream accumulators + the chain's, side by side
      int c = 0;
      for (int n : ilv_chain) c = std::max(c, nodes[n].tc_cols);
      tmem_cols = 32;
      while (tmem_cols < ilv_tmem + c) tmem_cols *= 2;
    }
    if (tmem_cols) {
      os << "  __shared__ unsigned tmem_slot;\n";
      os << "  const unsigned tmem_base = sgm::tmem_alloc<NT>(&tmem_slot, " << tmem_cols << "u);\n";
    }
    os << "  SGM_TR(8);\n";
    {
      bool any = false;
      for (int p = 0; p < (int)sched.size(); ++p)
        if (sched[p].type == Ev::NODE && nodes[sched[p].node].inv) {
          if (!any) os << "  // item-invariant values, once per CTA\n";
          any = true;
          emit_node(sched[p].node, false);
        }
      if (any) os << "  SGM_TR(9);\n";
      for (auto& x : nodes) {
        if (!(x.kind == SGM_MATMUL && x.tma && x.tc && x.xb_shared)) continue;
        const Node& a = nodes[x.in[0]];
        if (!a.inv) continue;
        bool first = true;  // one build per A node
        for (auto& y : nodes)
          if (&y == &x) break;
          else if (y.kind == SGM_MATMUL && y.tma && y.tc && y.xb_shared && y.in[0] == x.in[0]) first = false;
        if (!first) continue;
        i64 sa[4];
        dense_strides(a.sl, sa);
        if (a.store == ST_XG)
          os << "  sgm::build_xb_g<" << x.sl[2] << ", " << a.sl[3] << ", " << in_strides[a.slot][2]
             << "LL, NT>((u16*)(sm + " << x.at_off << "), (const u16*)((const S*)a.in[" << a.slot << "] + ("
             << offset_expr(a, true, std::to_string(nloop - 1)) << ")));\n";
        else
          os << "  sgm::build_xb<" << x.sl[2] << ", " << a.sl[3] << ", " << sa[2] << "LL, " << sa[3]
             << "LL, NT>((u16*)(sm + " << x.at_off << "), " << tile_ptr(x.in[0]) << ");\n";
        os << "  sgm::fence_async_smem();\n  sgm::csync<NT>();\n";
      }
    }
    if (prod) os << "  if (tid == 0) sgm::mbar_arrive(go);  // the producer starts streaming now\n";
    os << "  SGM_TR(1);\n";
    bool gs_open = false;
    if (GP > 1) os << "  __shared__ unsigned sgm_last;\n";
    os << "  unsigned cit = 0; (void)cit;\n";
    emit_item_loop("  ", "cit");
    os << "  SGM_TR(2);\n";
    bool in_loop = false;
    for (int p = 0; p < (int)sched.size(); ++p) {
      const Ev& e = sched[p];
      if (e.type == Ev::LOOP_BEGIN) {
        if (xcache_loop) os << "  if (xc_miss) {  // the whole loop is independent of gx\n";
        for (int n = 0; n < (int)nodes.size(); ++n)
          if (nodes[n].kind == SGM_ACCUM)
            os << "  for (int e = tid; e < " << prod4(nodes[n].sl) << "; e += NT) " << tile_ptr(n) << "[e] = N::zero();\n";
        os << "  sgm::csync<NT>();\n";
        // loop part jp runs a CONTIGUOUS range of iterations: a loop-split loader's
        // consecutive tiles are adjacent in memory, so a strided column tile's
        // sectors serve the next iterations from L1/L2 (interleaved parts re-fetched
        // every sector; A's split-KV candidates read Kt one column per iteration)
        for (int n = 0; n < (int)pf.size(); ++n) {
          const Node& x = nodes[n];
          if (pf[n] == 1)
            os << "  " << pf_type(x) << " pf" << n << ";\n  pf" << n << ".load((const S*)a.in[" << x.slot << "] + ("
               << offset_expr(x, true, "(jp * " + std::to_string(nloop / LP) + ")") << "));\n";
          if (pf[n] == 2) {
            const i64* st = in_strides[x.slot];
            os << "  sgm::TileStrip<N, " << x.sl[0] << ", " << x.sl[1] << ", " << x.sl[2] << ", " << x.sl[3] << ", "
               << st[0] << "LL, "
               << st[1] << "LL, " << st[2] << "LL, NT> st" << n << ";\n  st" << n << ".load((const S*)a.in["
               << x.slot << "] + (" << offset_expr(x, true, "(jp * " + std::to_string(nloop / LP) + ")") << "));\n";
          }
        }
        os << "  for (int j = jp * " << nloop / LP << "; j < (jp + 1) * " << nloop / LP << "; ++j) {\n";
        in_loop = true;
      } else if (e.type == Ev::LOOP_END) {
        os << "  }\n";
        if (xcache_loop) os << "  }\n";
        in_loop = false;
      } else if (e.type == Ev::FLUSH) {
        os << "  SGM_TR(" << 2000 + p << ");\n";
        emit_flush(e.flush, p);
      } else if (e.type == Ev::GFLUSH) {
        os << "  SGM_TR(" << 2000 + p << ");\n";
        emit_gflush(e.flush, p);
        gs_open = true;
      } else if (!nodes[e.node].inv) {
        if (p == ilv_pos) {  // the big stream's first ring-full, ahead of the small chain
          os << "  SGM_TR(" << 1700 + ilv_big << ");\n";
          emit_seg1 = true;
          emit_node(ilv_big, in_loop);
          emit_seg1 = false;
        }
        if (nodes[e.node].kind == SGM_MATMUL || nodes[e.node].kind == SGM_SUM) os << "  SGM_TR(" << 1000 + e.node << ");\n";
        const bool xwrap = nodes[e.node].xc && !(in_loop && xcache_loop);
        if (xwrap) os << "  if (xc_miss) {  // independent of gx: kept from the previous item\n";
        if (d.hints.trace) {  // thread 0's own share done (before the node's closing barrier)
          std::ostringstream keep;
          keep << os.str();
          os.str("");
          emit_node(e.node, in_loop);
          std::string body = os.str();
          const std::string tail = "    sgm::csync<NT>();\n";
          if (body.size() > tail.size() && body.compare(body.size() - tail.size(), tail.size(), tail) == 0)
            body.insert(body.size() - tail.size(), "  SGM_TR(" + std::to_string(1500 + e.node) + ");\n");
          os.str("");
          os << keep.str() << body;
        } else {
          emit_node(e.node, in_loop);
        }
        if (xwrap) os << "  }\n";
      }
    }
    if (gs_open) os << "  }  // last work item of the reduction group\n";
    os << "  SGM_TR(5);\n";
    os << "  sgm::csync<NT>();  // tiles are reused by the next item\n  }\n";
    os << "  SGM_TR(7);  // exit\n";
    // no CTA of a cluster leaves while a peer may still touch its shared memory
    // (DSMEM pushes / remote barrier arrivals of the last item)
    if (CL > 1) os << cl_sync();
    if (tmem_cols) os << "  sgm::tmem_free<NT>(tmem_base, " << tmem_cols << "u);\n";
    os << "}\n";
  }

  // ---- interleave (hint, one CTA per SM): see the members.  Measured on L
  // (x=2/8/32): 12.5-13.1 us against 12.0 us in the schedule order -- with W's
  // boxes first, the X^T build's plain loads queue behind the TMA burst (2.5 us
  // instead of 1.0 us).  Kept as an opt-in physical variant.  Legal when the big stream is a
  // single-batch tcgen05 TMA matmul outside the loop whose A operand is built
  // straight from global bf16 (ST_XG), the nodes scheduled right before it are
  // tcgen05 TMA matmuls it does not consume (and views), and none of their
  // shared-memory regions overlaps the big stream's A^T buffer.
  void plan_interleave() {
    ilv_big = ilv_pos = -1;
    ilv_chain.clear();
    if (!d.hints.interleave || !prod || paired) return;
    int big = -1;
    i64 best = 0;
    for (int n = 0; n < (int)nodes.size(); ++n) {
      const Node& x = nodes[n];
      if (x.kind == SGM_MATMUL && x.tma && x.tc && stream_bytes(x) > best) { best = stream_bytes(x); big = n; }
    }
    if (big < 0) return;
    const Node& B = nodes[big];
    const Node& BA = nodes[B.in[0]];
    if (B.body || B.inv || B.sl[0] * B.sl[1] != 1 || BA.store != ST_XG) return;
    int pb = -1;
    for (int p = 0; p < (int)sched.size(); ++p)
      if (sched[p].type == Ev::NODE && sched[p].node == big) pb = p;
    if (pb < 0) return;
    int ps = pb;
    std::set<int> chain;
    for (int p = pb - 1; p >= 0; --p) {
      const Ev& e = sched[p];
      if (e.type != Ev::NODE) break;
      const Node& y = nodes[e.node];
      if (y.kind == SGM_INPUT && y.store == ST_VIEW) { ps = p; continue; }
      if (y.kind != SGM_MATMUL || !y.tma || !y.tc || y.inv || y.body || y.sl[0] * y.sl[1] != 1) break;
      if (B.in[0] == e.node || B.in[1] == e.node) break;
      chain.insert(e.node);
      ps = p;
    }
    if (chain.empty()) return;
    const i64 K = BA.sl[3];
    const int nkc = (int)(K / B.kc), ntl = (int)((B.sl[3] + 127) / 128);
    if (nkc < 2 || ringS / ntl < 1) return;
    // shared-memory hazards: the big stream's A^T buffer must survive the chain
    const i64 xb0 = B.at_off, xb1 = B.at_off + 32 * K;
    auto overlaps = [&](i64 a0, i64 a1) { return a0 < xb1 && xb0 < a1; };
    for (int c : chain) {
      const Node& y = nodes[c];
      const bool same_xb = y.in[0] == B.in[0] && y.at_off == B.at_off;
      if (!same_xb && y.at_bytes && overlaps(y.at_off, y.at_off + y.at_bytes)) return;
      if (y.store == ST_SMEM && overlaps(y.off, y.off + prod4(y.sl) * ec)) return;
    }
    int cols = 0;
    for (int c : chain) cols = std::max(cols, nodes[c].tc_cols);
    int total = 32;
    while (total < B.tc_cols + cols) total *= 2;
    if (total > (paired ? 256 : 512)) return;  // two CTAs per SM share the 512 TMEM columns
    ilv_big = big;
    ilv_pos = ps;
    ilv_chain = chain;
    ilv_kc = std::max(1, std::min(nkc - 1, ringS / ntl));
    ilv_tmem = B.tc_cols;
  }

  GenResult run() {
    if (!load() || !shapes()) return R;
    structure();
    decide_views();
    split_plan();
    bool ok = fit();
    if (!ok && prod) {  // the ring does not fit next to the tiles: plain streamed loads
      no_tma_forced = true;
      ok = fit();
    }
    if (const int nt = small_loop_threads()) {  // re-plan with fewer threads per CTA
      const int keep = NT;
      const bool keep_forced = no_tma_forced;
      NT = nt;
      split_plan();
      ok = fit();
      if (!ok || prod || any_tc()) {
        NT = keep;
        no_tma_forced = keep_forced;
        split_plan();
        ok = fit();
        if (!ok && prod) {
          no_tma_forced = true;
          ok = fit();
        }
      }
    }
    plan_ring();
    plan_interleave();
    plan_accfuse();
    plan_fusion();
    plan_inv();
    if (d.hints.trace) {
      trace_off = scratch_per_cta;
      scratch_per_cta += SGM_TRACE_N * 16;
    }
    {
      // gsplit workspace after the per-CTA scratch: partial tiles [group][part][tile], then counters
      i64 gt = 0;
      for (auto& e : sched)
        if (e.type == Ev::GFLUSH)
          for (int f : e.flush) gt += (prod4(nodes[f].sl) + 3) / 4 * 4;  // 16-byte aligned slots
      const i64 work_ctas = LB * FP * GP * CL;
      gws_off = (work_ctas * scratch_per_cta + 255) / 256 * 256;
      gcnt_off = gws_off + (LB * FP * GP * gt * ec + 255) / 256 * 256;
      gws_end = GP > 1 ? gcnt_off + LB * FP * 4 : work_ctas * scratch_per_cta;
    }
    if (!ok) {
      // still over budget after spilling everything spillable; the hard cap leaves
      // room for the templates' static smem under the 227 KB opt-in limit
      if (smem_peak > 224 * 1024) {
        fail(SGM_ERR_RESOURCE, "shared memory plan exceeds 224 KB");
        return R;
      }
    }
    emit();
    std::string src = os.str();
    uint64_t h = fnv1a(src);
    char name[64];
    snprintf(name, sizeof name, "sgm_cand_%016" PRIx64, h);
    R.kernel_name = name;
    size_t at = src.find("@KNAME@");
    if (at != std::string::npos) src.replace(at, 7, name);
    R.source = src;
    R.logical_blocks = LB;
    R.cluster = CL;
    R.free_parts = FP;
    R.ctas = LB * FP * GP * CL;
    R.threads = prod ? NT + 32 : NT;
    R.ring_slots = ringS;
    R.ctas_per_sm = paired ? 2 : 1;
    std::vector<TmaSpec> specs(4);
    int nspec = 0;
    for (auto& x : nodes) {
      if (!x.staged) continue;
      TmaSpec t;
      t.slot = x.slot;
      t.elem_bytes = es;
      t.u32 = ns == SGM_FF;
      t.box0 = x.sbox;
      t.box1 = (int)x.sl[2];
      t.box2 = (int)x.sl[1];
      t.box3 = (int)x.sl[0];
      t.swizzle128 = 0;
      for (int k = 0; k < 4; ++k) t.dims[k] = in_dims[x.slot][k];
      specs[x.tma_id] = t;
      nspec = std::max(nspec, x.tma_id + 1);
    }
    for (auto& x : nodes) {
      if (x.kind != SGM_MATMUL || !x.tma) continue;
      R.n_tma++;
      const Node& b = nodes[x.in[1]];
      TmaSpec t;
      t.slot = b.slot;
      t.elem_bytes = es;
      t.u32 = ns == SGM_FF;
      t.box0 = x.tc ? 64 : x.bw;
      t.box1 = x.kc;
      t.swizzle128 = x.tc ? 1 : 0;
      for (int k = 0; k < 4; ++k) t.dims[k] = in_dims[b.slot][k];
      specs[x.tma_id] = t;
      nspec = std::max(nspec, x.tma_id + 1);
    }
    specs.resize(nspec);
    R.tmaps = specs;
    R.smem_bytes = smem_peak;
    R.loop_parts = LP;
    R.scratch_bytes = gws_end;
    R.scratch_per_cta = scratch_per_cta;
    R.trace_off = trace_off;
    for (auto& x : nodes)
      if (x.kind == SGM_MATMUL && x.gemv && x.tc) R.n_tcgen05++;
    std::ostringstream s;
    if (NT != 256) s << "NT=" << NT << " ";
    s << "LB=" << LB << " FP=" << FP << " GP=" << GP << " CL=" << CL << " LP=" << LP << (loop_gs ? "g" : "")
      << " ring=" << ringS << "x" << slotB / 1024 << "K est=" << (int)est_us << "us smem=" << smem_peak
      << " scratch/cta=" << scratch_per_cta << " classes:";
    for (int c = 0; c < (int)cls.size(); ++c)
      s << " c" << c << "(" << cls[c].extent << (cls[c].reduced ? "r" : "f") << "/" << cls[c].parts
        << (cls[c].parts > 1 ? (cls[c].cluster ? "c" : cls[c].gsplit ? "g" : "") : "") << ")";
    s << " mm:";
    for (int n = 0; n < (int)nodes.size(); ++n)
      if (nodes[n].kind == SGM_MATMUL) s << " n" << n << (nodes[n].tma ? (nodes[n].tc ? "tma-tc" : "tma-f32") : nodes[n].gemv ? (nodes[n].tc ? "tc" : "gemv") : "gen") << (nodes[n].gemv ? "/vn" + std::to_string(nodes[n].vn) + "ks" + std::to_string(nodes[n].ks) : "");
    R.summary = s.str();
    return R;
  }
};

}  // namespace

GenResult generate(const sgm_plan_desc& desc, int num_sms) {
  Gen g(desc, num_sms > 0 ? num_sms : 148);
  return g.run();
}

}  // namespace sgmcg
