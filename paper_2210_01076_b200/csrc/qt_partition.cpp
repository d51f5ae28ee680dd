// qt_partition.cpp -- host model of the reference's partition DAG (see
// qt_partition.hpp). Citations are to /root/reference/proj.
#include "qt_partition.hpp"

#include <algorithm>
#include <cmath>

#include "qt_gates.hpp"

namespace qtb {

namespace {

constexpr uint64_t kOutput = 0;  // the permanent sink node (graph.hpp:32)

// bit insertion of element_ops.cpp:11-14: x spread at `pos`, `bit` there
inline uint64_t spread(uint64_t x, int pos, uint64_t bit) {
  const uint64_t low = x & ((uint64_t{1} << pos) - 1);
  return ((x >> pos) << (pos + 1)) | (bit << pos) | low;
}

// Element-op stream of a non-superposition gate (element_ops.cpp:24-133):
// only what partitioning needs -- the count and op k's (i, j) indices.
struct OpStream {
  enum Form { Empty, PairBit, PairCnot, PairSwap, ScaleSet, ScaleClear, ScaleAll, ScaleBoth };
  Form form = Empty;
  int lo = 0, hi = 0;
  uint64_t count = 0;

  OpStream(const qt_gate& g, int n) {
    const uint64_t dim = uint64_t{1} << n;
    if (g.kind == QT_CNOT) {  // swap (i, i | 2^t) where control = 1, t = 0
      form = PairCnot;
      lo = g.target;
      hi = g.control;
      count = dim >> 2;
      return;
    }
    if (g.kind == QT_SWAP) {
      form = PairSwap;
      lo = std::min(g.target, g.control);
      hi = std::max(g.target, g.control);
      count = dim >> 2;
      return;
    }
    if (g.kind == QT_CZ) {  // additive kind: a -1 on the indices with both bits set
      form = ScaleBoth;
      lo = std::min(g.target, g.control);
      hi = std::max(g.target, g.control);
      count = dim >> 2;
      return;
    }
    const Mat2 m = g.kind == QT_U3 ? u3_matrix(g.theta, g.phi, g.lambda) : gate_matrix_1q(g.kind, g.theta);
    auto zero = [](cplx c) { return std::hypot(c.re, c.im) <= kZeroThreshold; };
    auto one = [](cplx c) { return std::hypot(c.re - 1.0, c.im) <= kZeroThreshold; };
    lo = g.target;
    if (zero(m[1]) && zero(m[2])) {
      const bool k0 = !one(m[0]), k1 = !one(m[3]);
      form = k0 && k1 ? ScaleAll : k1 ? ScaleSet : k0 ? ScaleClear : Empty;
      count = form == ScaleAll ? dim : form == Empty ? 0 : dim >> 1;
      return;
    }
    form = PairBit;  // anti-diagonal: a scaled bit flip
    count = dim >> 1;
  }

  void op(uint64_t k, uint64_t* i, uint64_t* j) const {
    switch (form) {
      case PairBit:
        *i = spread(k, lo, 0);
        *j = *i | (uint64_t{1} << lo);
        return;
      case PairCnot: {
        const int p0 = std::min(lo, hi), p1 = std::max(lo, hi);
        uint64_t x = spread(k, p0, p0 == hi ? 1 : 0);
        x = spread(x, p1, p1 == hi ? 1 : 0);
        *i = x;
        *j = x | (uint64_t{1} << lo);
        return;
      }
      case PairSwap: {
        const uint64_t x = spread(spread(k, lo, 1), hi, 0);
        *i = x;
        *j = x + (uint64_t{1} << hi) - (uint64_t{1} << lo);
        return;
      }
      case ScaleBoth:
        *i = *j = spread(spread(k, lo, 1), hi, 1);
        return;
      case ScaleSet:
        *i = *j = spread(k, lo, 1);
        return;
      case ScaleClear:
        *i = *j = spread(k, lo, 0);
        return;
      case ScaleAll:
      case Empty:
        *i = *j = k;
        return;
    }
  }
};

// Sorted disjoint inclusive block intervals with subtraction (the masking of
// graph.cpp's edge discovery).
class Cover {
 public:
  explicit Cover(PmRange r) { iv_.push_back(r); }
  bool empty() const { return iv_.empty(); }
  bool hits(PmRange r) const {
    for (const PmRange& x : iv_)
      if (std::max(x.first, r.first) <= std::min(x.last, r.last)) return true;
    return false;
  }
  void remove(PmRange r) {
    std::vector<PmRange> keep;
    keep.reserve(iv_.size() + 1);
    for (const PmRange& x : iv_) {
      if (r.last < x.first || x.last < r.first) {
        keep.push_back(x);
        continue;
      }
      if (x.first < r.first) keep.push_back(PmRange{x.first, r.first - 1});
      if (r.last < x.last) keep.push_back(PmRange{r.last + 1, x.last});
    }
    iv_.swap(keep);
  }

 private:
  std::vector<PmRange> iv_;
};

inline bool overlap(PmRange a, PmRange b) { return std::max(a.first, b.first) <= std::min(a.last, b.last); }

}  // namespace

PartitionModel::PartitionModel(int nqubits, uint64_t block_size)
    : n_(nqubits), cfg_bs_(block_size) {
  const uint64_t dim = uint64_t{1} << n_;
  bs_ = block_size < dim ? block_size : dim;
  nblocks_ = dim / bs_;
  Node out;
  out.is_output = true;
  out.read = PmRange{0, nblocks_ - 1};
  nodes_.emplace(kOutput, std::move(out));
}

// ---- circuit mirror --------------------------------------------------------

void PartitionModel::insert_net(uint32_t net, uint32_t after) {
  size_t at = 0;
  if (after) at = static_cast<size_t>(std::find(order_.begin(), order_.end(), after) - order_.begin()) + 1;
  order_.insert(order_.begin() + static_cast<std::ptrdiff_t>(at), net);
  net_gates_[net];
  net_stages_[net];
}

void PartitionModel::insert_net_back(uint32_t net) {
  order_.push_back(net);
  net_gates_[net];
  net_stages_[net];
}

void PartitionModel::remove_net(uint32_t net) {
  const std::vector<uint32_t> gs = net_gates_[net];
  for (uint32_t g : gs) remove_gate(g);
  order_.erase(std::find(order_.begin(), order_.end(), net));
  net_gates_.erase(net);
  net_stages_.erase(net);
}

void PartitionModel::insert_gate(uint32_t gate, const qt_gate& g, uint32_t net) {
  const bool sup = is_superposition_gate(g);
  gates_.emplace(gate, GateRec{g, net, sup});
  net_gates_[net].push_back(gate);
  // engine.cpp:93-111: superposition gates rebuild the net's MxV stage
  if (sup) rebuild_mxv(net);
  else add_permute_stage(net, gate);
}

void PartitionModel::remove_gate(uint32_t gate) {
  auto it = gates_.find(gate);
  if (it == gates_.end()) return;
  const GateRec rec = it->second;
  auto erase_from_net = [&] {
    std::vector<uint32_t>& gs = net_gates_[rec.net];
    gs.erase(std::find(gs.begin(), gs.end(), gate));
    gates_.erase(gate);
  };
  // engine.cpp:113-124
  if (rec.superposition) {
    erase_from_net();
    rebuild_mxv(rec.net);
  } else {
    drop_stage(gate_stage_.at(gate), true);
    gate_stage_.erase(gate);
    erase_from_net();
  }
}

// ---- stages ----------------------------------------------------------------

size_t PartitionModel::exec_index(uint32_t net, size_t local) const {
  size_t idx = 0;
  for (uint32_t m : order_) {
    if (m == net) return idx + local;
    auto it = net_stages_.find(m);
    if (it != net_stages_.end()) idx += it->second.size();
  }
  return idx + local;
}

std::vector<PmPart> PartitionModel::permute_parts(const qt_gate& g) const {
  // chunk_tasks (plan.cpp:26-36): runs of cfg block_size ops, hull
  // [op(first).i, op(last).j]; form_partitions (plan.cpp:53-74): greedy
  // merge of tasks overlapping the running hull, blocks at granularity bs
  const OpStream s(g, n_);
  std::vector<PmPart> parts;
  uint64_t h0 = 0, h1 = 0;
  for (uint64_t first = 0; first < s.count; first += cfg_bs_) {
    const uint64_t last = std::min(first + cfg_bs_, s.count) - 1;
    uint64_t i0 = 0, j0 = 0, i1 = 0, j1 = 0;
    s.op(first, &i0, &j0);
    s.op(last, &i1, &j1);
    const PmTask t{first, last, i0, j1};
    if (!parts.empty() && t.lo <= h1 && h0 <= t.hi) {
      parts.back().tasks.push_back(t);
      h0 = std::min(h0, t.lo);
      h1 = std::max(h1, t.hi);
    } else {
      parts.push_back(PmPart{0, 0, {t}});
      h0 = t.lo;
      h1 = t.hi;
    }
    parts.back().first_block = h0 / bs_;
    parts.back().last_block = h1 / bs_;
  }
  return parts;
}

uint32_t PartitionModel::make_stage(Stage&& st, uint32_t net, size_t local) {
  st.id = next_stage_++;
  st.net = net;
  st.block_count = 0;
  for (const PmPart& p : st.parts) st.block_count += p.last_block - p.first_block + 1;
  if (st.kind != PmKind::Sync) st.materialized.assign(nblocks_, 0);
  // read / write ranges per stage kind (engine.cpp:159-171)
  const PmRange full{0, nblocks_ - 1};
  std::vector<PmRange> reads, writes;
  std::vector<bool> has_write;
  for (const PmPart& p : st.parts) {
    const PmRange own{p.first_block, p.last_block};
    reads.push_back(st.kind == PmKind::PermuteScale ? own : full);
    writes.push_back(st.kind == PmKind::Sync ? full : own);
    has_write.push_back(true);
  }
  const size_t at = exec_index(net, local);
  st.nodes = connect(st.id, st.kind, reads, writes, has_write, at);
  exec_.insert(exec_.begin() + static_cast<std::ptrdiff_t>(at), st.id);
  reposition();
  std::vector<uint32_t>& list = net_stages_[net];
  list.insert(list.begin() + static_cast<std::ptrdiff_t>(local), st.id);
  const uint32_t id = st.id;
  stages_.emplace(id, std::move(st));
  return id;
}

void PartitionModel::drop_stage(uint32_t sid, bool frontier_succs) {
  const Removal rm = disconnect(sid);
  for (uint64_t n : rm.removed) frontiers_.erase(n);
  if (frontier_succs)
    for (const auto& succ : rm.successors) frontiers_.insert(succ.begin(), succ.end());
  const Stage& st = stages_.at(sid);
  exec_.erase(std::find(exec_.begin(), exec_.end(), sid));
  reposition();
  std::vector<uint32_t>& list = net_stages_[st.net];
  list.erase(std::find(list.begin(), list.end(), sid));
  stages_.erase(sid);
}

void PartitionModel::add_permute_stage(uint32_t net, uint32_t gate) {
  Stage st;
  st.kind = PmKind::PermuteScale;
  st.gate = gate;
  st.parts = permute_parts(gates_.at(gate).g);
  uint64_t blocks = 0;
  for (const PmPart& p : st.parts) blocks += p.last_block - p.first_block + 1;
  // permute stages of a net: ascending total block count, ties by gate id,
  // after the net's Sync / MxV stages (engine.cpp:217-233)
  const std::vector<uint32_t>& list = net_stages_[net];
  size_t local = 0;
  while (local < list.size() && stages_.at(list[local]).kind != PmKind::PermuteScale) ++local;
  while (local < list.size()) {
    const Stage& s = stages_.at(list[local]);
    if (s.block_count < blocks || (s.block_count == blocks && s.gate < gate)) ++local;
    else break;
  }
  const uint32_t id = make_stage(std::move(st), net, local);
  const Stage& made = stages_.at(id);
  frontiers_.insert(made.nodes.begin(), made.nodes.end());
  gate_stage_[gate] = id;
}

void PartitionModel::rebuild_mxv(uint32_t net) {
  // engine.cpp:241-285: the net's superposition gates fuse into one MxV
  // stage (one single-block partition per block) behind a Sync barrier
  bool any = false;
  for (uint32_t g : net_gates_[net]) any = any || gates_.at(g).superposition;
  auto have = [&] {
    const std::vector<uint32_t>& l = net_stages_[net];
    return !l.empty() && stages_.at(l.front()).kind == PmKind::Sync;
  };
  if (!any) {
    if (have()) {
      drop_stage(net_stages_[net][1], true);
      drop_stage(net_stages_[net][0], true);
    }
    return;
  }
  if (have()) {
    drop_stage(net_stages_[net][1], true);
  } else {
    Stage sync;
    sync.kind = PmKind::Sync;
    sync.parts.push_back(PmPart{0, nblocks_ - 1, {}});
    const uint32_t sid = make_stage(std::move(sync), net, 0);
    const Stage& made = stages_.at(sid);
    frontiers_.insert(made.nodes.begin(), made.nodes.end());
  }
  Stage mxv;
  mxv.kind = PmKind::MatrixVector;
  mxv.parts.reserve(nblocks_);
  for (uint64_t k = 0; k < nblocks_; ++k)  // plan.cpp:76-89
    mxv.parts.push_back(PmPart{k, k, {PmTask{k * bs_, (k + 1) * bs_ - 1, k * bs_, (k + 1) * bs_ - 1}}});
  const uint32_t id = make_stage(std::move(mxv), net, 1);
  const Stage& made = stages_.at(id);
  frontiers_.insert(made.nodes.begin(), made.nodes.end());
}

// ---- graph -----------------------------------------------------------------

void PartitionModel::link(uint64_t a, uint64_t b) {
  nodes_.at(a).succs.insert(b);
  nodes_.at(b).preds.insert(a);
}

void PartitionModel::unlink(uint64_t a, uint64_t b) {
  nodes_.at(a).succs.erase(b);
  nodes_.at(b).preds.erase(a);
}

void PartitionModel::reposition() {
  pos_.clear();
  for (size_t i = 0; i < exec_.size(); ++i) pos_[exec_[i]] = i;
}

size_t PartitionModel::position(uint32_t stage) const { return pos_.at(stage); }

bool PartitionModel::justified(uint64_t from, uint64_t to) const {
  // graph.cpp:93-114: some block of write(from) n read(to) that no stage
  // strictly between them writes
  const Node& a = nodes_.at(from);
  const Node& b = nodes_.at(to);
  if (!a.has_write) return false;
  const PmRange common{std::max(a.write.first, b.read.first), std::min(a.write.last, b.read.last)};
  if (common.first > common.last) return false;
  Cover left(common);
  const size_t lo = position(a.stage);
  const size_t hi = b.is_output ? exec_.size() : position(b.stage);
  for (size_t s = lo + 1; s < hi && !left.empty(); ++s)
    for (uint64_t q : stages_.at(exec_[s]).nodes) {
      const Node& qn = nodes_.at(q);
      if (qn.has_write) left.remove(qn.write);
    }
  return !left.empty();
}

std::vector<uint64_t> PartitionModel::connect(uint32_t stage, PmKind kind,
                                              const std::vector<PmRange>& reads,
                                              const std::vector<PmRange>& writes,
                                              const std::vector<bool>& has_write, size_t at) {
  // graph.cpp:116-189. The new stage is not yet in exec_ / stages_: the
  // scans walk the stages before `at` and from `at` on.
  std::vector<uint64_t> ids;
  for (size_t k = 0; k < reads.size(); ++k) {
    Node nd;
    nd.stage = stage;
    nd.index = static_cast<uint32_t>(k);
    nd.kind = kind;
    nd.read = reads[k];
    nd.write = writes[k];
    nd.has_write = has_write[k];
    const uint64_t id = next_node_++;
    nodes_.emplace(id, std::move(nd));
    ids.push_back(id);
  }
  std::set<uint64_t> before, after;
  for (uint64_t pid : ids) {
    const Node& p = nodes_.at(pid);
    // backward: the nearest writers of every block read
    Cover need(p.read);
    for (size_t s = at; s-- > 0 && !need.empty();)
      for (uint64_t q : stages_.at(exec_[s]).nodes) {
        const Node& qn = nodes_.at(q);
        if (qn.has_write && need.hits(qn.write)) {
          link(q, pid);
          before.insert(q);
          need.remove(qn.write);
        }
      }
    // forward: the nearest readers of every block written
    if (p.has_write) {
      Cover left(p.write);
      for (size_t s = at; s < exec_.size() && !left.empty(); ++s)
        for (uint64_t q : stages_.at(exec_[s]).nodes) {
          const Node& qn = nodes_.at(q);
          if (left.hits(qn.read)) {
            link(pid, q);
            after.insert(q);
            if (qn.has_write) left.remove(qn.write);
          }
        }
      if (!left.empty()) {
        link(pid, kOutput);
        after.insert(kOutput);
      }
    }
  }
  // transitive pruning needs the new stage in the execution order
  exec_.insert(exec_.begin() + static_cast<std::ptrdiff_t>(at), stage);
  Stage placeholder;
  placeholder.id = stage;
  placeholder.nodes = ids;
  const bool temp = stages_.count(stage) == 0;
  if (temp) stages_.emplace(stage, placeholder);
  reposition();
  for (uint64_t a : before)
    for (uint64_t b : after)
      if (nodes_.at(a).succs.count(b) && !justified(a, b)) unlink(a, b);
  if (temp) stages_.erase(stage);
  exec_.erase(exec_.begin() + static_cast<std::ptrdiff_t>(at));
  reposition();
  return ids;
}

PartitionModel::Removal PartitionModel::disconnect(uint32_t stage) {
  // graph.cpp:191-232: predecessors reconnect to successors where blocks
  // meet; surviving successors are returned (they become frontiers)
  Removal rm;
  const std::vector<uint64_t> parts = stages_.at(stage).nodes;
  for (uint64_t pid : parts) {
    Node& p = nodes_.at(pid);
    rm.removed.push_back(pid);
    rm.successors.emplace_back(p.succs.begin(), p.succs.end());
    for (uint64_t a : p.preds)
      for (uint64_t b : p.succs) {
        const Node& an = nodes_.at(a);
        const Node& bn = nodes_.at(b);
        if (an.has_write && overlap(an.write, bn.read) && !an.succs.count(b)) link(a, b);
      }
    for (uint64_t a : std::set<uint64_t>(p.preds)) unlink(a, pid);
    for (uint64_t b : std::set<uint64_t>(p.succs)) unlink(pid, b);
  }
  for (uint64_t pid : parts) nodes_.erase(pid);
  for (auto& list : rm.successors)
    list.erase(std::remove_if(list.begin(), list.end(), [&](uint64_t id) { return !nodes_.count(id); }),
               list.end());
  return rm;
}

std::set<uint64_t> PartitionModel::affected(const std::set<uint64_t>& from) const {
  std::set<uint64_t> seen;
  std::vector<uint64_t> stack(from.begin(), from.end());
  while (!stack.empty()) {
    const uint64_t id = stack.back();
    stack.pop_back();
    if (!seen.insert(id).second) continue;
    for (uint64_t s : nodes_.at(id).succs)
      if (!seen.count(s)) stack.push_back(s);
  }
  return seen;
}

// ---- update accounting (engine.cpp:392-504) ---------------------------------

void PartitionModel::update() {
  std::set<uint64_t> run;
  if (!ran_full_) {
    for (const auto& kv : stages_) run.insert(kv.second.nodes.begin(), kv.second.nodes.end());
    run.insert(kOutput);
  } else {
    run = affected(frontiers_);
  }
  PmAccount acc;
  acc.valid = true;
  acc.full = !ran_full_;
  std::set<uint64_t> blocks;
  for (uint64_t id : run) {
    const Node& nd = nodes_.at(id);
    if (nd.is_output || nd.kind == PmKind::Sync) continue;
    Stage& st = stages_.at(nd.stage);
    const PmPart& part = st.parts[nd.index];
    acc.executed_partitions += 1;
    acc.materialized_blocks += part.last_block - part.first_block + 1;
    for (uint64_t b = part.first_block; b <= part.last_block; ++b) {
      blocks.insert(b);
      st.materialized[b] = 1;
    }
  }
  acc.rewritten_blocks.assign(blocks.begin(), blocks.end());
  acc.rewritten_amplitudes = static_cast<uint64_t>(blocks.size()) * bs_;
  last_ = std::move(acc);
  frontiers_.clear();
  ran_full_ = true;
}

// ---- introspection -----------------------------------------------------------

std::vector<PartitionModel::StageInfo> PartitionModel::stages() const {
  std::vector<StageInfo> out;
  out.reserve(exec_.size());
  for (uint32_t sid : exec_) {
    const Stage& s = stages_.at(sid);
    StageInfo v;
    v.id = s.id;
    v.net = s.net;
    v.gate = s.gate;
    v.kind = s.kind;
    v.parts = &s.parts;
    v.nodes = &s.nodes;
    v.materialized = &s.materialized;
    out.push_back(v);
  }
  return out;
}

std::vector<std::pair<uint64_t, uint64_t>> PartitionModel::edges() const {
  std::vector<std::pair<uint64_t, uint64_t>> out;
  for (const auto& kv : nodes_)
    for (uint64_t s : kv.second.succs) out.emplace_back(kv.first, s);
  std::sort(out.begin(), out.end());
  return out;
}

std::string PartitionModel::node_name(uint64_t node) const {
  // engine.cpp:570-586
  if (node == kOutput) return "output";
  auto it = nodes_.find(node);
  if (it == nodes_.end()) return "?";
  const Stage& s = stages_.at(it->second.stage);
  const size_t pos = static_cast<size_t>(std::find(order_.begin(), order_.end(), s.net) - order_.begin()) + 1;
  switch (s.kind) {
    case PmKind::Sync: return "sync_" + std::to_string(pos);
    case PmKind::MatrixVector: return "MxV" + std::to_string(pos) + "_" + std::to_string(it->second.index);
    case PmKind::PermuteScale:
      return "g" + std::to_string(s.gate) + "_p" + std::to_string(it->second.index);
  }
  return "?";
}

void PartitionModel::dump_dot(std::ostream& os) const {
  // graph.cpp:302-327 with the engine's node names
  if (exec_.empty()) {
    os << "digraph qtask { output; }\n";
    return;
  }
  os << "digraph qtask {\n";
  for (uint32_t sid : exec_)
    for (uint64_t id : stages_.at(sid).nodes) {
      const Node& nd = nodes_.at(id);
      const std::string nm = node_name(id);
      os << "  " << nm << " [label=\"" << nm << " [" << nd.read.first << ".." << nd.read.last << "]\"];\n";
    }
  os << "  output;\n";
  std::vector<std::pair<std::string, std::string>> named;
  for (const auto& e : edges()) named.emplace_back(node_name(e.first), node_name(e.second));
  std::sort(named.begin(), named.end());
  for (const auto& e : named) os << "  " << e.first << " -> " << e.second << ";\n";
  os << "}\n";
}

}  // namespace qtb
