// planner.h -- host-side planner internals (network builder, line graph, orderers,
// step-dependent slicing, lowering).  Product code; the oracle shares none of it.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "plan_format.h"

namespace tnb {

struct Factor {
  uint8_t code, layer, conj;
};

struct NetTensor {
  std::vector<int> labels;       // sorted ascending, distinct
  std::vector<Factor> factors;   // elementwise product of gate tensors on `labels`
};

struct Network {
  int n_labels = 0;
  std::vector<NetTensor> tensors;
  double log2_scale = 0.0;       // -(#|+> factors)/2
  int edge_u = -1, edge_v = -1;
  std::vector<int> open_labels;  // never-eliminated output indices (§6 amplitude batch); bit b of
                                 // a batch index <-> open_labels[b] (ascending qubit)
};

// PAPER.md:199-235 (§4.1) + Fig. 1 with the CNOT-Z-CNOT gadget fused into a
// diagonal ZZ(gamma): live indices w(q,l) = l*N + q, l = 0..p-1 (reading A6).
// open_qubits: output wires left open (§6): the network evaluates the batch
// <x_open 0_rest|U|0^N>; open wire of the b-th open qubit (ascending) -> label n*p + b.
Network build_amplitude_network(int n, const std::vector<int>& edges, int p,
                                const std::vector<int>& open_qubits = {});
// <psi|Z_u Z_v|psi> restricted to the reverse light cone of edge (u, v).
Network build_cone_network(int n, const std::vector<int>& edges, int p, int u, int v);

// ---------------------------------------------------------------- line graph
class BitGraph {
 public:
  BitGraph() = default;
  explicit BitGraph(int n);
  static BitGraph from_network(const Network& net);
  int size() const { return n_; }
  bool alive(int v) const { return alive_[v] != 0; }
  int degree(int v) const { return deg_[v]; }
  int n_alive() const { return n_alive_; }
  // kept vertices (open indices, §6) are never eliminated, sliced or chosen by an orderer
  bool kept(int v) const { return !keep_.empty() && keep_[v] != 0; }
  void keep(int v);
  int n_kept() const { return n_kept_; }
  int n_free() const { return n_alive_ - n_kept_; }   // vertices an orderer may still eliminate
  void add_edge(int a, int b);
  // elimination of vertex v: remove it and make its neighbourhood a clique
  void eliminate(int v);
  // slicing: remove v and its edges, no fill-in
  void remove(int v);
  bool adjacent(int a, int b) const { return (row(a)[b >> 6] >> (b & 63)) & 1; }
  const uint64_t* row(int v) const { return &adj_[(size_t)v * W_]; }
  int words() const { return W_; }
  int64_t fill_in(int v) const;  // non-adjacent neighbour pairs of v
  std::vector<int> neighbours(int v) const;

 private:
  uint64_t* rowm(int v) { return &adj_[(size_t)v * W_]; }
  int n_ = 0, W_ = 0, n_alive_ = 0, n_kept_ = 0;
  std::vector<uint64_t> adj_;
  std::vector<uint8_t> alive_, keep_;
  std::vector<int> deg_;
};

struct Ordering {
  std::vector<int> order;
  std::vector<int> degrees;   // N_{G_i}(v_i)
  int width = 0;              // max degree
  double cost = 0.0;          // sum_i 2^{degree_i} ("C ~ 2^c")
};

// orderer + rgreedy parameters
struct OrderSpec {
  int orderer = 0;       // TN_ORDER_*
  int q = 1;             // rgreedy runs
  double tau = 0.5;      // rgreedy temperature
  uint64_t seed = 0;
};

// greedy orderers: TN_ORDER_MIN_FILL / TN_ORDER_MIN_DEGREE;
// rgreedy: best of the deterministic greedy run and q Boltzmann-sampled runs
Ordering greedy_order(BitGraph g, int orderer);
Ordering order_graph(const BitGraph& g, const OrderSpec& spec, uint64_t salt = 0);

struct Schedule {
  std::vector<int> prefix;    // phase A order (first slicing round's prefix, s indices)
  std::vector<int> sliced;    // ascending labels; bit b of a slice id <-> sliced[b]
  std::vector<int> residual;  // phase B order (later rounds' prefixes + final residual)
  int width = 0, unsliced_width = 0;
  double cost = 0.0;
};

// one candidate of the first slicing round: slicing after s steps of the full order
struct SliceCandidate {
  int s;          // candidate slice step (reading A8: s in [0, peak])
  int width;      // max(prefix width, residual width) of the plan slicing at s
  double cost;    // predicted sum 2^degree over the plan (prefix once + 2^n x residual)
};

// step-dependent slicing (Fig. slice_algo): n indices in rounds of r.
// scan (optional): every candidate s of the first round (Fig. hist_of_cost)
Schedule slice_search(const BitGraph& g0, int n, int r, const OrderSpec& spec,
                      std::vector<SliceCandidate>* scan = nullptr, int* peak_out = nullptr);

struct LoweredProgram {
  std::vector<LeafRec> leaves;
  std::vector<StepRec> steps;
  std::vector<ScalarRec> scalars;
  std::vector<OpRec> ops;
  ProgramRec prog{};
  uint64_t arena_elems = 0, persistent_elems = 0;
  double elems_slice = 0, elems_prefix = 0, elems_big_slice = 0;
  uint64_t big_launches_slice = 0, launches_prefix = 0, launches_slice = 0;
  int width = 0;
  std::vector<int> degrees;   // executed step degrees (phase A then phase B)
};

LoweredProgram lower(const Network& net, const Schedule& sch, int small_log2, std::string* err);

}  // namespace tnb
