// planner.cpp -- host planner: QAOA network builder, bitset line graph, greedy min-fill /
// min-degree orderers, step-dependent slicing and lowering to a bucket program.
//
//   PAPER.md:199-235, 350-359  circuit -> tensor expression -> line graph (indices = vertices,
//                              tensors = cliques, diagonal gates share one index per wire)
//   PAPER.md:361-368           elimination of vertex i (neighbourhood becomes a clique)
//   PAPER.md:384-401           contraction width c = max_i N_{G_i}(v_i)
//   PAPER.md:459-463           greedy ordering (lowest degree first)
//   PAPER.md:509-527, Eq. (1)  slicing n indices -> 2^n independent networks
//   PAPER.md:545-567           step-dependent slicing (Fig. slice_algo)
#include "planner.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>

#include "../../include/tn_b200.h"

namespace tnb {

// ============================================================== network builders
namespace {

struct NetBuilder {
  Network net;
  std::map<std::vector<int>, int> index;
  int n_plus = 0;
  void add(std::vector<int> labels, Factor f) {
    std::sort(labels.begin(), labels.end());
    if (std::adjacent_find(labels.begin(), labels.end()) != labels.end())
      throw std::runtime_error("tensor with repeated index");
    if (f.code == LC_PLUS) n_plus++;
    auto it = index.find(labels);
    if (it == index.end()) {
      index.emplace(labels, (int)net.tensors.size());
      net.tensors.push_back(NetTensor{labels, {f}});
    } else {
      auto& t = net.tensors[it->second];
      if ((int)t.factors.size() >= kMaxFactors) throw std::runtime_error("too many merged factors");
      t.factors.push_back(f);
    }
  }
};

void check_edges(int n, const std::vector<int>& edges) {
  std::vector<std::pair<int, int>> seen;
  for (size_t e = 0; e + 1 < edges.size(); e += 2) {
    int a = edges[e], b = edges[e + 1];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b) throw std::invalid_argument("bad edge");
    seen.emplace_back(std::min(a, b), std::max(a, b));
  }
  std::sort(seen.begin(), seen.end());
  if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
    throw std::invalid_argument("duplicate edge");
}

}  // namespace

Network build_amplitude_network(int n, const std::vector<int>& edges, int p,
                                const std::vector<int>& open_qubits) {
  check_edges(n, edges);
  std::vector<int> opened(open_qubits);
  std::sort(opened.begin(), opened.end());
  if (std::adjacent_find(opened.begin(), opened.end()) != opened.end() ||
      (!opened.empty() && (opened.front() < 0 || opened.back() >= n)))
    throw std::invalid_argument("bad open qubit list");
  std::vector<int> open_rank(n, -1);
  for (size_t b = 0; b < opened.size(); ++b) open_rank[opened[b]] = (int)b;
  NetBuilder b;
  auto w = [n](int q, int l) { return l * n + q; };
  for (int q = 0; q < n; ++q) b.add({w(q, 0)}, {LC_PLUS, 0, 0});
  for (int l = 1; l <= p; ++l) {
    for (size_t e = 0; e + 1 < edges.size(); e += 2)
      b.add({w(edges[e], l - 1), w(edges[e + 1], l - 1)}, {LC_ZZ, (uint8_t)(l - 1), 0});
    for (int q = 0; q < n; ++q) {
      if (l < p)
        b.add({w(q, l - 1), w(q, l)}, {LC_RX, (uint8_t)(l - 1), 0});
      else if (open_rank[q] >= 0)  // open output wire (§6): e^{-i b X} between w(q, p-1) and it
        b.add({w(q, p - 1), n * p + open_rank[q]}, {LC_RX, (uint8_t)(l - 1), 0});
      else  // output wire fixed to 0: <0| e^{-i b X} is a vector on w(q, p-1)
        b.add({w(q, p - 1)}, {LC_RXROW0, (uint8_t)(l - 1), 0});
    }
  }
  b.net.n_labels = n * p + (int)opened.size();
  for (size_t k = 0; k < opened.size(); ++k) b.net.open_labels.push_back(n * p + (int)k);
  b.net.log2_scale = -0.5 * b.n_plus;
  return b.net;
}

Network build_cone_network(int n, const std::vector<int>& edges, int p, int u, int v) {
  check_edges(n, edges);
  // reverse light cone (reading A17): L_p = {u, v}; E_l = edges touching L_l;
  // L_{l-1} = L_l U endpoints(E_l); m_q = max{l : q in L_l}
  std::vector<std::vector<char>> L(p + 1, std::vector<char>(n, 0));
  std::vector<std::vector<int>> E(p + 1);
  L[p][u] = L[p][v] = 1;
  for (int l = p; l >= 1; --l) {
    L[l - 1] = L[l];
    for (size_t e = 0; e + 1 < edges.size(); e += 2) {
      int a = edges[e], c = edges[e + 1];
      if (L[l][a] || L[l][c]) {
        E[l].push_back((int)e);
        L[l - 1][a] = L[l - 1][c] = 1;
      }
    }
  }
  std::vector<int> m(n, -1);
  for (int q = 0; q < n; ++q)
    for (int l = 0; l <= p; ++l)
      if (L[l][q]) m[q] = l;
  // labels: per cone qubit ascending: ket levels 0..m-1, shared top t, bra levels 0..m-1
  std::vector<std::vector<int>> kl(n), bl(n);
  int next = 0;
  for (int q = 0; q < n; ++q) {
    if (m[q] < 0) continue;
    kl[q].resize(m[q] + 1);
    bl[q].resize(m[q] + 1);
    for (int a = 0; a < m[q]; ++a) kl[q][a] = next++;
    int t = next++;
    kl[q][m[q]] = bl[q][m[q]] = t;
    for (int a = 0; a < m[q]; ++a) bl[q][a] = next++;
  }
  NetBuilder b;
  for (int q = 0; q < n; ++q) {
    if (m[q] < 0) continue;
    b.add({kl[q][0]}, {LC_PLUS, 0, 0});
    b.add({bl[q][0]}, {LC_PLUS, 0, 1});
  }
  for (int l = 1; l <= p; ++l) {
    for (int e : E[l]) {
      int a = edges[e], c = edges[e + 1];
      b.add({kl[a][l - 1], kl[c][l - 1]}, {LC_ZZ, (uint8_t)(l - 1), 0});
      b.add({bl[a][l - 1], bl[c][l - 1]}, {LC_ZZ, (uint8_t)(l - 1), 1});
    }
    for (int q = 0; q < n; ++q) {
      if (m[q] >= l) {
        b.add({kl[q][l - 1], kl[q][l]}, {LC_RX, (uint8_t)(l - 1), 0});
        b.add({bl[q][l - 1], bl[q][l]}, {LC_RX, (uint8_t)(l - 1), 1});
      }
    }
  }
  b.add({kl[u][m[u]]}, {LC_ZOBS, 0, 0});
  b.add({kl[v][m[v]]}, {LC_ZOBS, 0, 0});
  b.net.n_labels = next;
  b.net.log2_scale = -0.5 * b.n_plus;
  b.net.edge_u = u;
  b.net.edge_v = v;
  return b.net;
}

// ============================================================== bitset line graph
static inline int popc(uint64_t x) { return __builtin_popcountll(x); }

BitGraph::BitGraph(int n) : n_(n), W_((n + 63) / 64), n_alive_(n) {
  adj_.assign((size_t)n * W_, 0);
  alive_.assign(n, 1);
  deg_.assign(n, 0);
}

BitGraph BitGraph::from_network(const Network& net) {
  BitGraph g(net.n_labels);
  for (const auto& t : net.tensors)
    for (size_t i = 0; i < t.labels.size(); ++i)
      for (size_t j = i + 1; j < t.labels.size(); ++j) g.add_edge(t.labels[i], t.labels[j]);
  // the batch result is a tensor over the open indices: "a clique on left-out indices"
  // (PAPER.md:603-605), and they are never eliminated
  const auto& o = net.open_labels;
  for (size_t i = 0; i < o.size(); ++i)
    for (size_t j = i + 1; j < o.size(); ++j) g.add_edge(o[i], o[j]);
  for (int v : o) g.keep(v);
  return g;
}

void BitGraph::keep(int v) {
  if (keep_.empty()) keep_.assign(n_, 0);
  if (!keep_[v]) {
    keep_[v] = 1;
    n_kept_++;
  }
}

void BitGraph::add_edge(int a, int b) {
  if (a == b || adjacent(a, b)) return;
  rowm(a)[b >> 6] |= 1ull << (b & 63);
  rowm(b)[a >> 6] |= 1ull << (a & 63);
  deg_[a]++;
  deg_[b]++;
}

std::vector<int> BitGraph::neighbours(int v) const {
  std::vector<int> out;
  const uint64_t* r = row(v);
  for (int w = 0; w < W_; ++w) {
    uint64_t x = r[w];
    while (x) {
      int b = __builtin_ctzll(x);
      out.push_back(w * 64 + b);
      x &= x - 1;
    }
  }
  return out;
}

void BitGraph::eliminate(int v) {
  std::vector<int> nb = neighbours(v);
  const uint64_t* rv = row(v);
  for (int a : nb) {
    uint64_t* ra = rowm(a);
    ra[v >> 6] &= ~(1ull << (v & 63));
    int d = 0;
    for (int w = 0; w < W_; ++w) {
      ra[w] |= rv[w];
      if (w == (a >> 6)) ra[w] &= ~(1ull << (a & 63));
      if (w == (v >> 6)) ra[w] &= ~(1ull << (v & 63));
      d += popc(ra[w]);
    }
    deg_[a] = d;
  }
  std::fill(rowm(v), rowm(v) + W_, 0ull);
  deg_[v] = 0;
  alive_[v] = 0;
  n_alive_--;
}

void BitGraph::remove(int v) {
  for (int a : neighbours(v)) {
    rowm(a)[v >> 6] &= ~(1ull << (v & 63));
    deg_[a]--;
  }
  std::fill(rowm(v), rowm(v) + W_, 0ull);
  deg_[v] = 0;
  alive_[v] = 0;
  n_alive_--;
}

int64_t BitGraph::fill_in(int v) const {
  const uint64_t* rv = row(v);
  int64_t missing = 0;
  for (int a : neighbours(v)) {
    const uint64_t* ra = row(a);
    int c = 0;
    for (int w = 0; w < W_; ++w) c += popc(rv[w] & ~ra[w]);
    missing += c - 1;  // a itself is in N(v) but not in N(a)
  }
  return missing / 2;
}

// ============================================================== greedy orderers
Ordering greedy_order(BitGraph g, int orderer) {
  const int n = g.size();
  Ordering o;
  std::vector<int64_t> fill(n, 0);
  const bool minfill = orderer == TN_ORDER_MIN_FILL;
  if (minfill)
    for (int v = 0; v < n; ++v)
      if (g.alive(v)) fill[v] = g.fill_in(v);
  std::vector<char> dirty(n, 0);
  while (g.n_free() > 0) {
    int best = -1;
    for (int v = 0; v < n; ++v) {
      if (!g.alive(v) || g.kept(v)) continue;
      if (best < 0) { best = v; continue; }
      if (minfill) {
        if (fill[v] < fill[best] || (fill[v] == fill[best] && g.degree(v) < g.degree(best))) best = v;
      } else if (g.degree(v) < g.degree(best)) {
        best = v;
      }
    }
    const int d = g.degree(best);
    o.order.push_back(best);
    o.degrees.push_back(d);
    o.width = std::max(o.width, d);
    o.cost += std::ldexp(1.0, d);
    if (!minfill) {
      g.eliminate(best);
      continue;
    }
    std::vector<int> nb = g.neighbours(best);
    g.eliminate(best);
    // fill values change only within distance 2 of the eliminated vertex
    std::vector<int> touched;
    for (int a : nb) {
      if (!dirty[a]) { dirty[a] = 1; touched.push_back(a); }
      for (int c : g.neighbours(a))
        if (!dirty[c]) { dirty[c] = 1; touched.push_back(c); }
    }
    for (int a : touched) {
      fill[a] = g.fill_in(a);
      dirty[a] = 0;
    }
  }
  return o;
}

// ============================================================== rgreedy
namespace {
inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
struct Rng {
  uint64_t s;
  double uniform() {
    s = mix64(s);
    return (s >> 11) * (1.0 / 9007199254740992.0);
  }
};

// one randomized elimination: vertex v is chosen with probability ~ exp(-key(v)/tau), key =
// degree (rgreedy) or fill-in (rgreedy-fill)
Ordering boltzmann_run(BitGraph g, bool by_fill, double tau, uint64_t seed) {
  const int n = g.size();
  Ordering o;
  Rng rng{seed};
  std::vector<double> w(n);
  while (g.n_free() > 0) {
    int64_t kmin = INT64_MAX;
    std::vector<int64_t> key(n, 0);
    for (int v = 0; v < n; ++v) {
      if (!g.alive(v) || g.kept(v)) continue;
      key[v] = by_fill ? g.fill_in(v) : g.degree(v);
      kmin = std::min(kmin, key[v]);
    }
    double tot = 0.0;
    for (int v = 0; v < n; ++v) {
      w[v] = (g.alive(v) && !g.kept(v)) ? std::exp(-(double)(key[v] - kmin) / tau) : 0.0;
      tot += w[v];
    }
    double u = rng.uniform() * tot;
    int pick = -1;
    for (int v = 0; v < n; ++v) {
      if (!g.alive(v) || g.kept(v)) continue;
      pick = v;
      u -= w[v];
      if (u <= 0.0) break;
    }
    const int d = g.degree(pick);
    o.order.push_back(pick);
    o.degrees.push_back(d);
    o.width = std::max(o.width, d);
    o.cost += std::ldexp(1.0, d);
    g.eliminate(pick);
  }
  return o;
}
}  // namespace

Ordering order_graph(const BitGraph& g, const OrderSpec& spec, uint64_t salt) {
  if (spec.orderer == TN_ORDER_MIN_FILL || spec.orderer == TN_ORDER_MIN_DEGREE)
    return greedy_order(g, spec.orderer);
  const bool by_fill = spec.orderer == TN_ORDER_RGREEDY_FILL;
  Ordering best = greedy_order(g, by_fill ? TN_ORDER_MIN_FILL : TN_ORDER_MIN_DEGREE);
  for (int i = 0; i < spec.q; ++i) {
    Ordering o = boltzmann_run(g, by_fill, spec.tau, mix64(spec.seed ^ mix64(salt * 1000003ull + i)));
    if (o.width < best.width || (o.width == best.width && o.cost < best.cost)) best = std::move(o);
  }
  return best;
}

// ============================================================== step-dependent slicing
Schedule slice_search(const BitGraph& g0, int n, int r, const OrderSpec& spec,
                      std::vector<SliceCandidate>* scan, int* peak_out) {
  Schedule sch;
  Ordering full0 = order_graph(g0, spec, 0);
  sch.unsliced_width = full0.width;
  if (n <= 0) {
    sch.residual = full0.order;
    sch.width = full0.width;
    sch.cost = full0.cost;
    return sch;
  }
  if (r <= 0 || r > n) r = n;
  if (n > g0.n_free()) throw std::invalid_argument("n exceeds the live vertex count");
  BitGraph g = g0;
  int prefix_width = 0;
  double prefix_cost = 0.0;
  int n_done = 0;
  bool first_round = true;
  std::vector<int> phaseB_prefix;
  while (n_done < n) {
    const int rr = std::min(r, n - n_done);
    Ordering full = first_round ? full0 : order_graph(g, spec, 1000 + n_done);
    int peak = 0;
    for (size_t i = 0; i < full.degrees.size(); ++i)
      if (full.degrees[i] > full.degrees[peak]) peak = (int)i;
    if (first_round && peak_out) *peak_out = peak;
    // candidate steps s in [0, peak] (reading A8)
    BitGraph gs = g;
    int pmax = prefix_width;
    double pcost = 0.0;
    int best_s = -1, best_w = 1 << 30;
    double best_cost = 0.0;
    std::vector<int> best_S;
    BitGraph best_g;
    for (int s = 0; s <= peak && s <= (int)full.order.size(); ++s) {
      if (s > 0) {
        pmax = std::max(pmax, full.degrees[s - 1]);
        pcost += std::ldexp(1.0, full.degrees[s - 1]) * std::ldexp(1.0, n_done);
        gs.eliminate(full.order[s - 1]);
      }
      if (gs.n_free() < rr) break;
      // the rr vertices with the most neighbours in G_s, ties -> smaller label (reading A9);
      // open (kept) indices are never sliced
      std::vector<int> cand;
      for (int v = 0; v < gs.size(); ++v)
        if (gs.alive(v) && !gs.kept(v)) cand.push_back(v);
      std::stable_sort(cand.begin(), cand.end(),
                       [&](int a, int b) { return gs.degree(a) > gs.degree(b); });
      std::vector<int> S(cand.begin(), cand.begin() + rr);
      BitGraph gr = gs;
      for (int v : S) gr.remove(v);
      Ordering res = order_graph(gr, spec, 1 + s + 7919ull * n_done);
      const int w = std::max(pmax, res.width);
      const double cost = prefix_cost + pcost + std::ldexp(res.cost, n_done + rr);
      if (first_round && scan) scan->push_back(SliceCandidate{s, w, cost});
      // best: smaller width, then fewer predicted operations, then smaller s (reading A10)
      if (w < best_w || (w == best_w && cost < best_cost)) {
        best_w = w;
        best_cost = cost;
        best_s = s;
        best_S = S;
        best_g = gr;
      }
    }
    if (best_s < 0) throw std::invalid_argument("n exceeds the live vertex count");
    std::vector<int> pre(full.order.begin(), full.order.begin() + best_s);
    for (int i = 0; i < best_s; ++i) {
      prefix_width = std::max(prefix_width, full.degrees[i]);
      prefix_cost += std::ldexp(1.0, full.degrees[i]) * std::ldexp(1.0, n_done);
    }
    if (first_round)
      sch.prefix = pre;
    else
      phaseB_prefix.insert(phaseB_prefix.end(), pre.begin(), pre.end());
    sch.sliced.insert(sch.sliced.end(), best_S.begin(), best_S.end());
    g = best_g;
    n_done += rr;
    first_round = false;
  }
  Ordering res = order_graph(g, spec, 999983);
  sch.residual = phaseB_prefix;
  sch.residual.insert(sch.residual.end(), res.order.begin(), res.order.end());
  std::sort(sch.sliced.begin(), sch.sliced.end());
  sch.width = std::max(prefix_width, res.width);
  sch.cost = prefix_cost + std::ldexp(res.cost, n);
  return sch;
}

// ============================================================== lowering
namespace {

struct Sym {
  std::vector<int> idx;   // layout order: ascending key = most significant first
  int leaf = -1;
  int birth = 0;          // time of production (0 = materialization)
  int death = -1;         // last use
  bool persistent = false;
  bool scalar_ref = false;
  uint64_t off = 0;
  uint64_t size = 0;      // allocated elements (aligned)
  bool phaseB_born = false;
};

uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Arena {
  std::map<uint64_t, uint64_t> holes;  // off -> size
  uint64_t top = 0;
  uint64_t alloc(uint64_t need) {
    for (auto it = holes.begin(); it != holes.end(); ++it) {
      if (it->second >= need) {
        uint64_t off = it->first, sz = it->second;
        holes.erase(it);
        if (sz > need) holes[off + need] = sz - need;
        return off;
      }
    }
    // extend at the top, absorbing a trailing hole
    if (!holes.empty()) {
      auto last = std::prev(holes.end());
      if (last->first + last->second == top) {
        uint64_t off = last->first;
        holes.erase(last);
        top = off + need;
        return off;
      }
    }
    uint64_t off = top;
    top += need;
    return off;
  }
  void release(uint64_t off, uint64_t sz) {
    if (sz == 0) return;
    auto it = holes.emplace(off, sz).first;
    auto nx = std::next(it);
    if (nx != holes.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      holes.erase(nx);
    }
    if (it != holes.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        holes.erase(it);
      }
    }
  }
};

}  // namespace

LoweredProgram lower(const Network& net, const Schedule& sch, int small_log2, std::string* err) {
  LoweredProgram out;
  const int NL = net.n_labels;
  const int k = (int)sch.sliced.size();
  std::vector<int64_t> key(NL, INT64_MIN);
  std::vector<int> slice_bit(NL, -1);
  for (int b = 0; b < k; ++b) {
    key[sch.sliced[b]] = -1 - b;
    slice_bit[sch.sliced[b]] = b;
  }
  const int sA = (int)sch.prefix.size();
  for (int i = 0; i < sA; ++i) key[sch.prefix[i]] = i;
  for (size_t i = 0; i < sch.residual.size(); ++i) key[sch.residual[i]] = sA + (int64_t)i;
  const int total_pos = sA + (int)sch.residual.size();
  // open indices (§6): after every eliminated position; the b-th open label is bit b of every
  // tensor holding open labels (b = 0 least significant), so a final tensor's element for batch
  // index o is pext(o, its open mask)
  const int n_open = (int)net.open_labels.size();
  std::vector<int> open_bit(NL, -1);
  for (int b = 0; b < n_open; ++b) {
    const int l = net.open_labels[b];
    if (key[l] != INT64_MIN) {
      *err = "an open index is in the elimination order";
      return out;
    }
    key[l] = total_pos + (n_open - 1 - b);
    open_bit[l] = b;
  }
  for (int l = 0; l < NL; ++l)
    if (key[l] == INT64_MIN) {
      *err = "order misses live label " + std::to_string(l);
      return out;
    }
  auto by_key = [&](int a, int b) { return key[a] < key[b]; };

  std::vector<Sym> syms;
  for (size_t t = 0; t < net.tensors.size(); ++t) {
    Sym s;
    s.idx = net.tensors[t].labels;
    std::sort(s.idx.begin(), s.idx.end(), by_key);
    s.leaf = (int)t;
    syms.push_back(s);
  }
  auto home = [&](const Sym& s) -> int64_t {  // min key over eliminated (non-sliced, non-open)
    for (int l : s.idx)                        // indices; -1 if none (a final factor)
      if (slice_bit[l] < 0) return key[l] < total_pos ? key[l] : -1;
    return -1;
  };
  std::vector<std::vector<int>> bucket(total_pos);
  std::vector<int> scalars;
  auto route = [&](int id) {
    int64_t h = home(syms[id]);
    if (h < 0) {
      syms[id].scalar_ref = true;
      scalars.push_back(id);
    } else {
      bucket[h].push_back(id);
    }
  };
  for (size_t i = 0; i < syms.size(); ++i) route((int)i);

  struct PendingStep {
    StepRec rec;
    std::vector<int> ins;
    int outsym;
    int orig = 0;    // position in the elimination order (before the level sort of phase A)
  };
  std::vector<PendingStep> pend;
  for (int pos = 0; pos < total_pos; ++pos) {
    const int v = pos < sA ? sch.prefix[pos] : sch.residual[pos - sA];
    const bool phaseB = pos >= sA;
    std::vector<int> ins = bucket[pos];
    if (ins.empty()) continue;  // an index of no tensor (cannot happen for connected networks)
    if ((int)ins.size() > kMaxIn) {
      *err = "bucket with more than 8 tensors at label " + std::to_string(v);
      return out;
    }
    const int t_now = (int)pend.size() + 1;
    Sym o;
    for (int id : ins)
      for (int l : syms[id].idx)
        if (l != v && !(phaseB && slice_bit[l] >= 0)) o.idx.push_back(l);  // phase B: sliced fixed
    std::sort(o.idx.begin(), o.idx.end(), by_key);
    o.idx.erase(std::unique(o.idx.begin(), o.idx.end()), o.idx.end());
    o.birth = t_now;
    o.phaseB_born = phaseB;
    // bits of the output in this phase (phase B: sliced indices are fixed, not bits)
    std::vector<int> obits;
    for (int l : o.idx)
      if (!(phaseB && slice_bit[l] >= 0)) obits.push_back(l);
    if (phaseB && obits.size() != o.idx.size()) {
      *err = "internal: phase-B output holds a sliced index";
      return out;
    }
    const int R = (int)obits.size();
    if (R > 62) {
      *err = "output rank above 62";
      return out;
    }
    StepRec rec;
    std::memset(&rec, 0, sizeof(rec));
    rec.out_rank = R;
    rec.n_in = (int)ins.size();
    rec.phase = phaseB ? 1 : 0;
    rec.label = v;
    rec.degree = R;
    // largest input first (in-place candidate)
    std::stable_sort(ins.begin(), ins.end(),
                     [&](int a, int b) { return syms[a].idx.size() > syms[b].idx.size(); });
    for (size_t t = 0; t < ins.size(); ++t) {
      const Sym& s = syms[ins[t]];
      std::vector<int> bits;
      uint32_t smask = 0;
      for (int l : s.idx) {
        if (phaseB && slice_bit[l] >= 0)
          smask |= 1u << slice_bit[l];
        else
          bits.push_back(l);
      }
      InRec& in = rec.in[t];
      in.rank = (uint32_t)bits.size();
      in.slice_mask = smask;
      uint64_t mask = 0;
      int pv = -1;
      for (size_t i = 0; i < bits.size(); ++i) {
        const int pos_in = (int)bits.size() - 1 - (int)i;
        if (bits[i] == v) {
          pv = pos_in;
          continue;
        }
        auto it = std::find(obits.begin(), obits.end(), bits[i]);
        const int pos_out = R - 1 - (int)(it - obits.begin());
        mask |= 1ull << pos_out;
      }
      in.out_mask = mask;
      in.pv = (uint32_t)pv;
      // monotone check: the non-v bits of the input must be the selected output bits in order
      if (pv < 0 || popc(mask) + 1 != (int)bits.size()) {
        *err = "internal: bad embedding";
        return out;
      }
      in.flags = (in.rank + 2 >= (uint32_t)R && R >= 16) ? 1u : 0u;
      if (phaseB && s.phaseB_born) in.flags |= F_REL;
    }
    // in-place: in[0] is an intermediate of this phase holding every output bit with v on top
    {
      const Sym& s0 = syms[ins[0]];
      const InRec& i0 = rec.in[0];
      const uint64_t full = R == 64 ? ~0ull : ((1ull << R) - 1);
      const bool same_phase_interm = s0.leaf < 0 && s0.phaseB_born == phaseB;
      rec.inplace = (same_phase_interm && i0.slice_mask == 0 && i0.rank == (uint32_t)R + 1 &&
                     i0.out_mask == full && i0.pv == (uint32_t)R && s0.idx.size() == (size_t)R + 1)
                        ? 1
                        : 0;
    }
    for (int id : ins) syms[id].death = t_now;
    const int oid = (int)syms.size();
    syms.push_back(o);
    pend.push_back(PendingStep{rec, ins, oid, (int)pend.size()});
    route(oid);
  }
  for (size_t i = 0; i < syms.size(); ++i) {
    if (syms[i].death < 0 && !syms[i].scalar_ref) {
      *err = "internal: dangling tensor";
      return out;
    }
  }
  const int nsteps = (int)pend.size();
  const int T_end = nsteps + 1;
  struct FeedPair {
    int consumer_out;         // output sym of the consumer step c
    std::vector<int> inputs;  // syms the producer block reads (not its in-place chain)
  };
  std::vector<FeedPair> feed_pairs;
  int nA = 0;
  for (auto& ps : pend)
    if (ps.rec.phase == 0) nA++;
  // ---- phase B: a merge block (a merge step and the in-place reduce steps after it) whose output
  // is a full input of a later merge step c (it holds every output bit of c and c's summed index)
  // moves down to just before c, so that the runtime can compute the block's output tile by tile
  // inside c's launch instead of writing and re-reading it (OP_GROUP_FEED, k_gemm_fc).  Legal: the
  // block's inputs exist before it, its output has exactly one consumer (c), and the steps it
  // moves past neither read its output nor produce its inputs -- the arithmetic is unchanged; only
  // the block's inputs live longer.  TNB_NO_FEED=1 keeps the elimination order.
  if (!(std::getenv("TNB_NO_FEED") && std::getenv("TNB_NO_FEED")[0] == '1')) {
    std::vector<int> consumer(syms.size(), -1);
    for (int si = nA; si < nsteps; ++si)
      for (int id : pend[si].ins) consumer[id] = si;
    std::vector<std::vector<std::pair<int, int>>> attach(nsteps);   // blocks emitted right before c
    std::vector<char> moved(nsteps, 0);
    feed_pairs.clear();
    int si = nA;
    while (si < nsteps) {
      if (pend[si].rec.inplace) { ++si; continue; }
      int e = si + 1;
      while (e < nsteps && pend[e].rec.inplace && pend[e].ins[0] == pend[e - 1].outsym) ++e;
      const int T = pend[e - 1].outsym;
      const int c = consumer[T];
      bool ok = c > e && e - si >= 2 && e - si <= kMaxGroupPlan && pend[c].rec.out_rank > small_log2 &&
                pend[e - 1].rec.out_rank > small_log2;
      if (ok) {
        const StepRec& cr = pend[c].rec;
        int t = -1;
        for (size_t k2 = 0; k2 < pend[c].ins.size(); ++k2)
          if (pend[c].ins[k2] == T) t = (int)k2;
        const uint64_t full = (1ull << cr.out_rank) - 1;
        ok = t >= 0 && cr.in[t].out_mask == full && cr.in[t].pv == (uint32_t)cr.out_rank &&
             cr.in[t].slice_mask == 0;
      }
      if (std::getenv("TNB_PLAN_DEBUG"))
        std::fprintf(stderr, "feed? block [%d,%d) R=%d -> consumer %d (inplace %d R %d) ok=%d\n", si, e,
                     pend[e - 1].rec.out_rank, c, c >= 0 ? pend[c].rec.inplace : -1, c >= 0 ? pend[c].rec.out_rank : -1, (int)ok);
      if (ok) {
        attach[c].push_back({si, e});
        for (int k2 = si; k2 < e; ++k2) moved[k2] = 1;
        // the fused launch reads the block's inputs while it writes c's output: they must stay
        // allocated until c (see the lifetime extension before the arena)
        FeedPair fp;
        fp.consumer_out = pend[c].outsym;
        for (int k2 = si; k2 < e; ++k2)
          for (size_t t2 = 0; t2 < pend[k2].ins.size(); ++t2)
            if (!(k2 > si && t2 == 0 && pend[k2].rec.inplace)) fp.inputs.push_back(pend[k2].ins[t2]);
        feed_pairs.push_back(fp);
      }
      si = e;
    }
    std::vector<PendingStep> re(pend.begin(), pend.begin() + nA);
    re.reserve(nsteps);
    std::vector<int> stack;
    std::function<void(int)> emit = [&](int s2) {
      for (const auto& b : attach[s2])
        for (int k2 = b.first; k2 < b.second; ++k2) emit(k2);
      re.push_back(pend[s2]);
    };
    for (int s2 = nA; s2 < nsteps; ++s2)
      if (!moved[s2]) emit(s2);
    if ((int)re.size() != nsteps) {
      *err = "internal: phase-B reorder lost steps";
      return out;
    }
    pend.swap(re);
    for (auto& sy : syms) sy.death = -1;
    for (int s2 = 0; s2 < nsteps; ++s2) {
      for (int id : pend[s2].ins) syms[id].death = s2 + 1;
      syms[pend[s2].outsym].birth = s2 + 1;
    }
  }
  // ---- the prefix (phase A) in dependency levels: its buckets form a shallow DAG (C5a: 143
  // steps, depth 5), so the steps of one level run side by side, one CTA each (OP_PRUN).  Phase A
  // is stably sorted by (level, big step); the memory a level frees is released only when the
  // level ends, so no output of a level overwrites an input another step of the level still reads.
  std::vector<int> lend(nsteps + 1, 0);   // per step (new order): time at which its level ends
  std::vector<int> level(nsteps, 0);
  // unsliced plans (k = 0, one "slice"): a phase-B run of small steps that forms a shallow DAG
  // (C2: 62-68 steps in 3-5 levels) is level-sorted like the prefix and runs as one OP_PRUN per
  // level; sliced plans keep their runs (slice lanes / batching already overlap them)
  std::vector<char> parB(nsteps, 0);
  {
    std::vector<int> producer(syms.size(), -1);
    for (int si = 0; si < nsteps; ++si) producer[pend[si].outsym] = si;
    std::vector<int> lev(nsteps, 0);
    for (int si = 0; si < nsteps; ++si) {
      int l = 0;
      for (int id : pend[si].ins)
        if (producer[id] >= 0) l = std::max(l, lev[producer[id]]);
      lev[si] = l + 1;
    }
    std::vector<int> idx(nA);
    for (int i = 0; i < nA; ++i) idx[i] = i;
    auto big = [&](int si) { return pend[si].rec.out_rank > small_log2 ? 1 : 0; };
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
      if (lev[a] != lev[b]) return lev[a] < lev[b];
      return big(a) < big(b);
    });
    std::vector<PendingStep> re;
    re.reserve(nsteps);
    for (int i = 0; i < nA; ++i) { re.push_back(pend[idx[i]]); level[i] = lev[idx[i]]; }
    {
      int si = nA;
      while (si < nsteps) {
        if (k != 0 || pend[si].rec.out_rank > small_log2) {
          level[re.size()] = 0;
          re.push_back(pend[si]);
          ++si;
          continue;
        }
        int e = si;
        std::map<int, int> per;
        while (e < nsteps && pend[e].rec.out_rank <= small_log2) { per[lev[e]]++; ++e; }
        const int len = e - si;
        const bool go = len >= 8 && (int)per.size() * 4 <= len;
        std::vector<int> ix;
        for (int q = si; q < e; ++q) ix.push_back(q);
        if (go) std::stable_sort(ix.begin(), ix.end(), [&](int a, int b) { return lev[a] < lev[b]; });
        for (int q : ix) {
          level[re.size()] = go ? lev[q] : 0;
          parB[re.size()] = go ? 1 : 0;
          re.push_back(pend[q]);
        }
        si = e;
      }
    }
    pend.swap(re);
    for (auto& sy : syms) sy.death = -1;
    for (int si = 0; si < nsteps; ++si) {
      for (int id : pend[si].ins) syms[id].death = si + 1;
      syms[pend[si].outsym].birth = si + 1;
    }
    for (int si = 0; si < nsteps; ++si) {
      int e = si;
      if (si < nA)
        while (e + 1 < nA && level[e + 1] == level[si]) ++e;
      else if (parB[si])
        while (e + 1 < nsteps && parB[e + 1] && level[e + 1] == level[si]) ++e;
      lend[si + 1] = e + 1;
    }
    for (auto& sy : syms)   // inputs of a level-parallel step live until its level ends
      if (sy.death >= 1 && (sy.death <= nA || parB[sy.death - 1])) sy.death = lend[sy.death];
    if (std::getenv("TNB_PLAN_DEBUG")) {   // phase-B runs of small steps: length and depth
      int si = nA;
      while (si < nsteps) {
        if (pend[si].rec.out_rank > small_log2) { ++si; continue; }
        int e = si;
        std::map<int, int> per;
        while (e < nsteps && pend[e].rec.out_rank <= small_log2) { per[lev[e]]++; ++e; }
        int wmax = 0;
        for (auto& kv : per) wmax = std::max(wmax, kv.second);
        std::fprintf(stderr, "phase-B run [%d,%d): %d steps, %zu levels, widest %d\n", si, e, e - si, per.size(), wmax);
        si = e;
      }
    }
  }
  // producer -> consumer candidates (OP_GROUP_FEED): every input of the producer block lives until
  // the consumer step, so the first-fit arena never places the consumer's output over memory the
  // fused launch (k_gemm_fc) still reads in other CTAs
  {
    std::vector<int> at(syms.size(), -1);
    for (int si = 0; si < nsteps; ++si) at[pend[si].outsym] = si;
    for (const auto& fp : feed_pairs) {
      const int c = at[fp.consumer_out];
      if (c < 0) continue;
      for (int id : fp.inputs) syms[id].death = std::max(syms[id].death, c + 1);
    }
  }
  // lifetimes: tensors used in phase B but born before it persist across slices
  for (auto& s : syms) {
    if (s.scalar_ref) s.death = T_end;
    const bool usedB = s.death > nA;
    if (usedB && !s.phaseB_born) {
      s.persistent = true;
      s.death = T_end + 1;
    }
    s.size = align_up(1ull << s.idx.size());
  }
  // ---- arena: interval allocation in time order; leaves at t = 0
  Arena ar;
  for (auto& s : syms)
    if (s.leaf >= 0) s.off = ar.alloc(s.size);
  // free dead leaves / tensors at step t after allocating the step's output
  std::vector<std::vector<int>> dies(T_end + 2);
  for (size_t i = 0; i < syms.size(); ++i)
    if (syms[i].death <= T_end) dies[syms[i].death].push_back((int)i);
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> deferred(T_end + 2);
  for (int si = 0; si < nsteps; ++si) {
    const int t = si + 1;
    PendingStep& ps = pend[si];
    Sym& o = syms[ps.outsym];
    if (ps.rec.inplace) {
      Sym& a = syms[ps.ins[0]];
      o.off = a.off;
      deferred[lend[t]].push_back({a.off + o.size, a.size - o.size});   // the upper half
      a.size = 0;  // its lower part now belongs to the output
    } else {
      o.off = ar.alloc(o.size);
    }
    for (auto& d : deferred[t]) ar.release(d.first, d.second);
    for (int id : dies[t]) {
      if (syms[id].persistent) continue;
      ar.release(syms[id].off, syms[id].size);
      syms[id].size = 0;
    }
  }
  out.arena_elems = ar.top;
  uint64_t pers = 0;
  for (auto& s : syms)
    if (s.persistent) pers = std::max(pers, s.off + align_up(1ull << s.idx.size()));
  out.persistent_elems = pers;

  // ---- records
  for (size_t t = 0; t < net.tensors.size(); ++t) {
    LeafRec lr;
    std::memset(&lr, 0, sizeof(lr));
    lr.off = syms[t].off;
    lr.rank = (int32_t)net.tensors[t].labels.size();
    lr.nfact = (int32_t)net.tensors[t].factors.size();
    for (int f = 0; f < lr.nfact; ++f) {
      lr.code[f] = net.tensors[t].factors[f].code;
      lr.layer[f] = net.tensors[t].factors[f].layer;
      lr.conj[f] = net.tensors[t].factors[f].conj;
    }
    out.leaves.push_back(lr);
  }
  out.degrees.assign(nsteps, 0);
  for (int si = 0; si < nsteps; ++si) {
    PendingStep& ps = pend[si];
    ps.rec.out_off = syms[ps.outsym].off;
    for (int t = 0; t < ps.rec.n_in; ++t) ps.rec.in[t].off = syms[ps.ins[t]].off;
    const Sym& o = syms[ps.outsym];
    ps.rec.degree = (int)o.idx.size();
    out.degrees[ps.orig] = ps.rec.degree;    // reported in elimination order (tn_plan_schedule)
    out.width = std::max(out.width, ps.rec.degree);
    out.steps.push_back(ps.rec);
  }
  for (int id : scalars) {
    ScalarRec sr;
    std::memset(&sr, 0, sizeof(sr));
    sr.off = syms[id].off;
    uint32_t m = 0, om = 0;
    for (int l : syms[id].idx) {
      if (slice_bit[l] >= 0) m |= 1u << slice_bit[l];
      else if (open_bit[l] >= 0) om |= 1u << open_bit[l];
    }
    sr.slice_mask = m;
    sr.open_mask = om;
    sr.flags = syms[id].phaseB_born ? F_REL : 0u;
    out.scalars.push_back(sr);
  }
  // ---- ops: runs of small steps go to the interpreter, the rest are standalone launches
  for (int phase = 0; phase < 2; ++phase) {
    int i = 0;
    while (i < nsteps) {
      if (out.steps[i].phase != phase) { ++i; continue; }
      const StepRec& st = out.steps[i];
      double elems = std::ldexp(1.0, st.out_rank);
      for (int t = 0; t < st.n_in; ++t) elems += std::ldexp(1.0, (int)st.in[t].rank);
      if (phase == 0) out.elems_prefix += elems; else out.elems_slice += elems;
      if (st.out_rank > small_log2 && st.out_rank >= 1) {
        out.ops.push_back(OpRec{OP_BIG, i, i + 1, phase});
        if (phase == 1) { out.elems_big_slice += elems; out.big_launches_slice++; }
        ++i;
        continue;
      }
      int j = i;
      while (j < nsteps && out.steps[j].phase == phase && out.steps[j].out_rank <= small_log2 &&
             parB[j] == parB[i] && ((phase == 1 && !parB[i]) || level[j] == level[i])) {
        if (j > i) {
          const StepRec& s2 = out.steps[j];
          double e2 = std::ldexp(1.0, s2.out_rank);
          for (int t = 0; t < s2.n_in; ++t) e2 += std::ldexp(1.0, (int)s2.in[t].rank);
          if (phase == 0) out.elems_prefix += e2; else out.elems_slice += e2;
        }
        ++j;
      }
      // a phase-A run lies inside one dependency level: its steps are independent (OP_PRUN)
      out.ops.push_back(OpRec{(phase == 0 || parB[i]) ? OP_PRUN : OP_RUN, i, j, phase});
      i = j;
    }
  }
  // ---- fusion (phase B).  A reduce step holds every output bit in its first input with the
  // summed bit on top and has only rank-1 weights on the summed index as other inputs; a follower
  // is the in-place reduce of the previous step's output.
  //   reduce head + followers      -> OP_CHAIN (k_chain, up to kMaxChain summed indices)
  //   other head + g followers     -> OP_GROUP (k_group_t, M = g + 1 <= kMaxGroupPlan) when the
  //                                   time model says it pays; remaining followers form a chain
  {
    auto is_reduce = [&](const StepRec& st) {
      if (st.out_rank < 1 || st.n_in - 1 > kMaxChainW) return false;
      const uint64_t full = (1ull << st.out_rank) - 1;
      if (st.in[0].out_mask != full || st.in[0].pv != (uint32_t)st.out_rank ||
          st.in[0].rank != (uint32_t)st.out_rank + 1)
        return false;
      for (int t = 1; t < st.n_in; ++t)
        if (st.in[t].out_mask != 0 || st.in[t].rank != 1) return false;
      return true;
    };
    auto step_elems = [&](const StepRec& st) {
      double e = std::ldexp(1.0, st.out_rank);
      for (int t = 0; t < st.n_in; ++t) e += std::ldexp(1.0, (int)st.in[t].rank);
      return e;
    };
    // time model (c64, seconds): HBM-bound streams at kBW; fused groups also pay per-output work
    const double kBW = 5.5e12, kOps = 2.0e13;
    auto t_elems = [&](double e) { return e * 8.0 / kBW; };
    auto t_chain = [&](int RA, int m) {   // m reduce steps starting from a rank-RA input
      if (m <= 0) return 0.0;
      return t_elems(std::ldexp(1.0, RA) + std::ldexp(1.0, RA - m));
    };
    auto t_group = [&](int s0, int g) {   // head s0 + g followers
      const StepRec& h = out.steps[s0];
      const int M = g + 1;
      const int Rf = out.steps[s0 + g].out_rank;
      double e = std::ldexp(1.0, Rf);
      int nv = 0;
      for (int t = 0; t < h.n_in; ++t) {
        e += std::ldexp(1.0, (int)h.in[t].rank);
        if ((h.in[t].out_mask & ((1ull << Rf) - 1)) != 0) ++nv;
      }
      const double ops = std::ldexp(1.0, Rf + M) * (nv + 1) * 10.0;
      return std::max(t_elems(e), ops / kOps);
    };
    std::vector<OpRec> fused;
    for (size_t oi = 0; oi < out.ops.size(); ++oi) {
      const OpRec& op = out.ops[oi];
      if (op.phase != 1 || op.type != OP_BIG) {
        fused.push_back(op);
        continue;
      }
      const int s0 = op.begin;
      int f = 0;
      while (oi + 1 + f < out.ops.size()) {
        const OpRec& nx = out.ops[oi + 1 + f];
        if (nx.phase != 1 || nx.type != OP_BIG || nx.begin != s0 + 1 + f) break;
        const StepRec& st = out.steps[nx.begin];
        const StepRec& pv = out.steps[nx.begin - 1];
        if (!st.inplace || !is_reduce(st) || st.in[0].off != pv.out_off) break;
        ++f;
      }
      if (f == 0) {
        fused.push_back(op);
        continue;
      }
      double unf = 0.0;
      if (is_reduce(out.steps[s0])) {
        const int take = std::min(f, kMaxChain - 1);
        const int end = s0 + 1 + take;
        for (int k = s0; k < end; ++k) unf += step_elems(out.steps[k]);
        const StepRec& h = out.steps[s0];
        const int m = end - s0;
        double fz = std::ldexp(1.0, (int)h.in[0].rank) + std::ldexp(1.0, (int)h.in[0].rank - m);
        for (int k = s0; k < end; ++k) fz += 2.0 * (out.steps[k].n_in - 1);
        out.elems_slice += fz - unf;
        out.elems_big_slice += fz - unf;
        out.big_launches_slice -= (uint64_t)(m - 1);
        fused.push_back(OpRec{OP_CHAIN, s0, end, 1});
        oi += take;
        continue;
      }
      // merge head: choose the number of followers g to fuse
      const StepRec& h = out.steps[s0];
      int best_g = 0;
      double best_t = t_elems(step_elems(h)) + t_chain(h.out_rank + 0, f) * 1.0;
      int n_inputs = h.n_in;
      for (int g = 1; g <= std::min(f, kMaxGroupPlan - 1); ++g) {
        n_inputs += out.steps[s0 + g].n_in - 1;
        if (n_inputs > kMaxIn) break;
        const int rest = f - g;
        const double t = t_group(s0, g) + t_chain(out.steps[s0 + g].out_rank, rest);
        if (t < best_t) { best_t = t; best_g = g; }
      }
      if (best_g == 0) {
        fused.push_back(op);
        continue;
      }
      const int end = s0 + 1 + best_g;
      for (int k = s0; k < end; ++k) unf += step_elems(out.steps[k]);
      double fz = std::ldexp(1.0, out.steps[end - 1].out_rank);
      for (int t = 0; t < h.n_in; ++t) fz += std::ldexp(1.0, (int)h.in[t].rank);
      for (int k = s0 + 1; k < end; ++k) fz += 2.0 * (out.steps[k].n_in - 1);
      out.elems_slice += fz - unf;
      out.elems_big_slice += fz - unf;
      out.big_launches_slice -= (uint64_t)best_g;
      fused.push_back(OpRec{OP_GROUP, s0, end, 1});
      oi += best_g;
    }
    out.ops.swap(fused);
    // reduce chains among the small steps of phase-B interpreter runs (e.g. the final reduction of
    // a slice to its scalar) run as streaming chain launches too -- unless every per-slice op is
    // an interpreter run (then slices run batched, one CTA each, and stay that way)
    bool all_runs = true;
    for (const auto& op : out.ops)
      if (op.phase == 1 && op.type != OP_RUN) all_runs = false;
    if (!all_runs) {
      std::vector<OpRec> ops2;
      for (const auto& op : out.ops) {
        if (op.phase != 1 || op.type != OP_RUN) {
          ops2.push_back(op);
          continue;
        }
        // only chains on inputs of >= 2^run_chain_min elements pay for their own launch; shorter
        // ones stay in the interpreter run (TNB_RUN_CHAIN_MIN, default 10: C5a's 2^13 -> 2^5 chain
        // keeps its launch (9 us; 41 us in the one-CTA interpreter), the 2^5 -> 1 tail joins the run)
        static const int run_chain_min = [] {
          const char* e = std::getenv("TNB_RUN_CHAIN_MIN");
          return e ? std::atoi(e) : 10;
        }();
        int i = op.begin, run_start = op.begin;
        while (i < op.end) {
          if (is_reduce(out.steps[i]) && (int)out.steps[i].in[0].rank >= run_chain_min) {
            int j = i + 1;
            while (j < op.end && j - i < kMaxChain && out.steps[j].inplace && is_reduce(out.steps[j]) &&
                   out.steps[j].in[0].off == out.steps[j - 1].out_off)
              ++j;
            if (j - i >= 2) {
              if (run_start < i) ops2.push_back(OpRec{OP_RUN, run_start, i, 1});
              ops2.push_back(OpRec{OP_CHAIN, i, j, 1});
              run_start = i = j;
              continue;
            }
          }
          ++i;
        }
        if (run_start < op.end) ops2.push_back(OpRec{OP_RUN, run_start, op.end, 1});
      }
      out.ops.swap(ops2);
    }
  }
  // ---- producer -> consumer pairs (phase B): an OP_GROUP whose output is a full input of the
  // next op's head (an OP_GROUP) becomes OP_GROUP_FEED; its output is then never written or read
  // when the fused launch takes the pair (predicted bytes / launches assume it does)
  for (size_t oi = 0; oi + 1 < out.ops.size(); ++oi) {
    OpRec& a = out.ops[oi];
    const OpRec& b = out.ops[oi + 1];
    if (std::getenv("TNB_PLAN_DEBUG") && a.phase == 1 && b.phase == 1)
      std::fprintf(stderr, "op pair %zu: [%d,%d) type %d -> [%d,%d) type %d\n", oi, a.begin, a.end, a.type, b.begin,
                   b.end, b.type);
    if (a.phase != 1 || b.phase != 1 || a.type != OP_GROUP || (b.type != OP_GROUP && b.type != OP_GROUP_FEED)) continue;
    const StepRec& last = out.steps[a.end - 1];
    const StepRec& head = out.steps[b.begin];
    const uint64_t full = (1ull << head.out_rank) - 1;
    bool feed = false;
    for (int t = 0; t < head.n_in; ++t)
      if (head.in[t].off == last.out_off && head.in[t].out_mask == full && head.in[t].pv == (uint32_t)head.out_rank &&
          head.in[t].rank == (uint32_t)last.out_rank && (head.in[t].flags & F_REL))
        feed = true;
    if (std::getenv("TNB_PLAN_DEBUG"))
      std::fprintf(stderr, "feed mark: ops %zu [%d,%d) type %d -> [%d,%d) type %d: %d\n", oi, a.begin, a.end, a.type,
                   b.begin, b.end, b.type, (int)feed);
    // the fused launch reads every producer input while other CTAs write the consumer's output:
    // an in-place producer head (its output aliases its own input) or any overlap of the
    // consumer's output with a producer input rules the pair out
    if (feed && out.steps[a.begin].inplace) feed = false;
    if (feed) {
      const uint64_t olo = head.out_off, ohi = head.out_off + align_up(1ull << head.out_rank);
      for (int si2 = a.begin; si2 < a.end && feed; ++si2) {
        const StepRec& st2 = out.steps[si2];
        for (int t = 0; t < st2.n_in; ++t) {
          if (si2 > a.begin && t == 0 && st2.inplace) continue;   // the producer's own chain
          const InRec& in = st2.in[t];
          const uint64_t ilo = in.off, ihi = in.off + align_up(1ull << (in.rank + popc(in.slice_mask)));
          if (ilo < ohi && olo < ihi) feed = false;
        }
      }
    }
    if (!feed) continue;
    a.type = OP_GROUP_FEED;
    const double t_elems = 2.0 * std::ldexp(1.0, last.out_rank);
    out.elems_slice -= t_elems;
    out.elems_big_slice -= t_elems;
    out.big_launches_slice -= 1;
  }
  for (auto& op : out.ops) (op.phase == 0 ? out.launches_prefix : out.launches_slice)++;
  out.launches_slice += 1;  // per-slice finalize
  ProgramRec& pr = out.prog;
  std::memset(&pr, 0, sizeof(pr));
  pr.stepA_begin = 0;
  pr.stepA_end = nA;
  pr.stepB_begin = nA;
  pr.stepB_end = nsteps;
  int oa = 0;
  while (oa < (int)out.ops.size() && out.ops[oa].phase == 0) ++oa;
  pr.opA_begin = 0;
  pr.opA_end = oa;
  pr.opB_begin = oa;
  pr.opB_end = (int)out.ops.size();
  pr.scal_begin = 0;
  pr.scal_end = (int)out.scalars.size();
  pr.edge_u = net.edge_u;
  pr.edge_v = net.edge_v;
  pr.log2_scale = net.log2_scale;
  pr.arena_begin = 0;
  pr.arena_end = out.arena_elems;
  (void)T_end;
  return out;
}

}  // namespace tnb
