// plan_format.h -- binary plan layout shared by the planner (planner.cpp) and the runtime
// (runtime.cu).  Host- and device-visible POD records; little endian; version-checked.
//
// A plan is the lowered form of bucket elimination (§4.2) with
// step-dependent slicing (§5.3):
//   phase A  -- the shared prefix: bucket steps over the first s indices of the order, run once,
//               with the sliced indices still present (they are the TOP bits of every tensor);
//   phase B  -- per slice j (Eq. 1): the residual bucket steps; tensors that
//               contain sliced indices are addressed at offset pext(j, slice_mask) << rank.
// Elimination-order layout: the indices of every tensor are ordered by their layout key, the
// earliest key being the MOST significant bit.  Keys: sliced index with slice bit b -> -1-b;
// prefix / residual index -> its position in the elimination order.  Hence the summed index of
// a bucket is the top non-sliced bit of every input and every input is a monotone sub-embedding
// of the output (no transposes).
#pragma once
#include <stdint.h>

namespace tnb {

constexpr uint32_t kPlanMagic = 0x32424E54u;  // "TNB2"
constexpr uint32_t kPlanVersion = 8;
constexpr int kMaxIn = 8;     // inputs per bucket step
constexpr int kMaxP = 16;     // QAOA depth supported by the materializer
constexpr int kMaxFactors = 4;
constexpr uint64_t kAlign = 32;  // element alignment of every tensor in the arena

// leaf gate codes (values are per element of the layout-ordered leaf; all rank-2 gates are
// symmetric matrices, so the axis order of a rank-2 leaf does not matter)
enum LeafCode : uint8_t {
  LC_PLUS = 0,     // |+> without 1/sqrt2: [1, 1]                 (rank 1)
  LC_ZOBS = 1,     // Z diagonal: [1, -1]                          (rank 1)
  LC_RXROW0 = 2,   // <0| e^{-i b X}: [cos b, -i sin b]            (rank 1, layer l)
  LC_ZZ = 3,       // [[1, e^{-i g}], [e^{-i g}, 1]]               (rank 2, layer l)
  LC_RX = 4,       // e^{-i b X} = [[cos b, -i sin b], [-i sin b, cos b]]   (rank 2, layer l)
};

struct LeafRec {
  uint64_t off;            // arena element offset
  int32_t rank;            // 0..2
  int32_t nfact;           // 1..kMaxFactors (tensors with identical index sets are pre-merged)
  uint8_t code[kMaxFactors];
  uint8_t layer[kMaxFactors];  // 0-based layer (gamma/beta index)
  uint8_t conj[kMaxFactors];   // complex-conjugate the factor (bra side of a light cone)
  uint8_t pad[4];
};

struct InRec {
  uint64_t off;        // arena element offset (slice 0 for tensors holding sliced indices)
  uint64_t out_mask;   // output bits present in this input
  uint32_t rank;       // bits of this input in the current phase (excl. sliced bits in phase B)
  uint32_t slice_mask; // phase B: which slice bits this tensor holds (its top bits); else 0
  uint32_t pv;         // bit position of the summed index in the input
  uint32_t flags;      // bit0: streamed (read once, large); bit2: F_REL -- a per-slice tensor
                       // (relocated into the slice's window when slices run batched)
};
constexpr uint32_t F_REL = 4u;

struct StepRec {
  uint64_t out_off;
  int32_t out_rank;
  int32_t n_in;
  int32_t inplace;     // output aliases in[0]'s lower half
  int32_t phase;       // 0 = A (prefix), 1 = B (per slice)
  int32_t label;       // eliminated index label
  int32_t degree;      // N_{G_i}(v_i) = out_rank (+ sliced bits in phase A)
  InRec in[kMaxIn];
};

enum OpType : int32_t { OP_BIG = 0, OP_RUN = 1, OP_CHAIN = 2, OP_GROUP = 3, OP_PRUN = 4, OP_GROUP_FEED = 5 };
constexpr int kMaxGroupPlan = 5;    // summed indices of one fused merge group (k_group_t, M <= 5)
constexpr int kMaxChain = 8;        // summed indices of one fused reduce chain (W table 2^8)
constexpr int kMaxChainW = 3;       // x-only weights per chained step
struct OpRec {
  int32_t type;   // OP_BIG: one standalone bucket-kernel launch of step `begin`;
                  // OP_RUN: steps [begin, end) in one CTA of the interpreter kernel;
                  // OP_CHAIN: steps [begin, end) -- a run of reduce steps whose only other
                  //   inputs are rank-1 weights on the summed index -- as ONE streaming pass
                  //   out[o] = sum_{x < 2^m} W[x] A[o + x 2^{R_A - m}] (exact re-association);
                  // OP_GROUP: steps [begin, end) -- any step followed by in-place reduce steps with
                  //   rank-1 weights -- as ONE k_group_t launch summing M = end-begin indices;
                  // OP_PRUN: steps [begin, end) -- independent small steps of one dependency level
                  //   of the prefix -- in one interpreter launch, one CTA per step;
                  // OP_GROUP_FEED: an OP_GROUP whose output is a full input of the next op (an
                  //   OP_GROUP) and read by nothing else: the two may run as ONE launch that computes
                  //   the output tile by tile and consumes it without writing it (k_gemm_fc), else
                  //   as the two groups
  int32_t begin;
  int32_t end;
  int32_t phase;
};

struct ScalarRec {       // per-slice final factors: tensors holding no eliminated index -- rank 0,
  uint64_t off;          // or only sliced and open indices.  Element of batch entry o in slice j:
  uint32_t slice_mask;   //   off + (pext(j, slice_mask) << popcount(open_mask)) + pext(o, open_mask)
  int32_t program;
  uint32_t flags;        // F_REL: produced per slice
  uint32_t open_mask;    // open indices held (bit b = the b-th open index, §6 amplitude batch)
};

struct ProgramRec {      // amplitude: one program; energy: one per edge (light cone)
  int32_t stepA_begin, stepA_end, opA_begin, opA_end;
  int32_t stepB_begin, stepB_end, opB_begin, opB_end;
  int32_t scal_begin, scal_end;
  int32_t edge_u, edge_v;
  double log2_scale;     // the dropped 1/sqrt2 of every |+>: result *= 2^{log2_scale}
  uint64_t arena_begin;  // first arena element owned by this program
  uint64_t arena_end;
};

struct PlanHeader {
  uint32_t magic, version;
  int32_t kind, n_qubits, p, n_edges;
  int32_t width, unsliced_width, k, slice_step;
  int32_t orderer, r, small_log2, n_labels;
  int32_t n_programs, n_leaves, n_steps, n_ops, n_scalars;
  int32_t n_prefix, n_residual, n_degrees;
  uint64_t arena_elems;
  uint64_t persistent_elems;
  double pred_elems_slice;     // algorithmic elements moved per slice (phase B)
  double pred_elems_prefix;    // phase A
  double pred_elems_big_slice; // part of pred_elems_slice in OP_BIG launches
  uint64_t big_launches_slice;
  uint64_t launches_prefix, launches_slice;
  int32_t n_open;              // open output indices a: every result is a batch of 2^a amplitudes
  int32_t pad0;
  uint64_t reserved[3];
};
// Buffer = PlanHeader | ProgramRec[n_programs] | LeafRec[n_leaves] | StepRec[n_steps]
//          | OpRec[n_ops] | ScalarRec[n_scalars] | int32 prefix[n_prefix] | int32 sliced[k]
//          | int32 residual[n_residual] | int32 degrees[n_degrees]

}  // namespace tnb
