// qt_netindex.hpp -- order index of a circuit's nets (host only).
//
// The reference keeps its nets in a std::list and walks it to turn a net or a
// gate into a circuit position (circuit.cpp:67-120). Modifiers arrive one per
// update in the incremental workloads, so every such walk is on the latency
// path. Here the nets sit in an implicit treap (randomised balanced tree keyed
// by their order) whose nodes carry subtree net and gate counts:
//   rank of a net, gates before a net, net holding gate position p,
//   insert / erase of a net at a rank, change of a net's gate count
// are all O(log nets) expected.
#pragma once

#include <cstdint>
#include <unordered_map>
#include <vector>

namespace qtb {

class NetIndex {
 public:
  NetIndex() = default;
  NetIndex(const NetIndex&) = delete;
  NetIndex& operator=(const NetIndex&) = delete;
  ~NetIndex() { clear(); }

  size_t nets() const { return cnt(root_); }
  uint64_t gates() const { return sum(root_); }
  bool has(uint32_t net) const { return by_id_.count(net) != 0; }

  // insert a new (empty) net so that `rank` nets precede it
  void insert(uint32_t net, size_t rank) {
    Node* n = new Node{};
    n->id = net;
    n->pri = next_pri();
    n->nets = 1;
    by_id_.emplace(net, n);
    Node *a = nullptr, *b = nullptr;
    split(root_, rank, &a, &b);
    root_ = merge(merge(a, n), b);
    if (root_) root_->parent = nullptr;
  }

  void erase(uint32_t net) {
    auto it = by_id_.find(net);
    if (it == by_id_.end()) return;
    const size_t r = rank(net);
    Node *a = nullptr, *b = nullptr, *c = nullptr;
    split(root_, r, &a, &b);
    split(b, 1, &b, &c);
    delete b;
    by_id_.erase(it);
    root_ = merge(a, c);
    if (root_) root_->parent = nullptr;
  }

  // gate count of a net changes by delta
  void add_gates(uint32_t net, int64_t delta) {
    Node* const n0 = by_id_.at(net);
    n0->own = static_cast<uint64_t>(static_cast<int64_t>(n0->own) + delta);
    for (Node* n = n0; n; n = n->parent) n->gsum = static_cast<uint64_t>(static_cast<int64_t>(n->gsum) + delta);
  }

  // number of nets before `net`
  size_t rank(uint32_t net) const {
    const Node* n = by_id_.at(net);
    size_t r = cnt(n->left);
    for (; n->parent; n = n->parent)
      if (n->parent->right == n) r += cnt(n->parent->left) + 1;
    return r;
  }

  // number of gates in the nets before `net`
  uint64_t gates_before(uint32_t net) const {
    const Node* n = by_id_.at(net);
    uint64_t g = sum(n->left);
    for (; n->parent; n = n->parent)
      if (n->parent->right == n) g += sum(n->parent->left) + n->parent->own;
    return g;
  }

  uint64_t gates_of(uint32_t net) const { return by_id_.at(net)->own; }

  // the net holding gate position pos (< gates()): its id, and the position
  // of its first gate in *first
  uint32_t net_at_gate(uint64_t pos, uint64_t* first) const {
    const Node* n = root_;
    uint64_t base = 0;
    while (n) {
      const uint64_t l = sum(n->left);
      if (pos < base + l) {
        n = n->left;
      } else if (pos < base + l + n->own) {
        if (first) *first = base + l;
        return n->id;
      } else {
        base += l + n->own;
        n = n->right;
      }
    }
    if (first) *first = base;
    return 0;
  }

  // net ids in order, starting at rank `from`
  void order(std::vector<uint32_t>* out, size_t from = 0) const {
    out->clear();
    out->reserve(nets() > from ? nets() - from : 0);
    walk(root_, from, out);
  }

  void clear() {
    std::vector<Node*> stack;
    if (root_) stack.push_back(root_);
    while (!stack.empty()) {
      Node* n = stack.back();
      stack.pop_back();
      if (n->left) stack.push_back(n->left);
      if (n->right) stack.push_back(n->right);
      delete n;
    }
    root_ = nullptr;
    by_id_.clear();
  }

 private:
  struct Node {
    uint32_t id = 0;
    uint32_t pri = 0;
    uint64_t own = 0;   // gates of this net
    uint64_t gsum = 0;  // gates of the subtree
    size_t nets = 0;    // nets of the subtree
    Node *left = nullptr, *right = nullptr, *parent = nullptr;
  };
  static size_t cnt(const Node* n) { return n ? n->nets : 0; }
  static uint64_t sum(const Node* n) { return n ? n->gsum : 0; }
  static void pull(Node* n) {
    n->nets = 1 + cnt(n->left) + cnt(n->right);
    n->gsum = n->own + sum(n->left) + sum(n->right);
    if (n->left) n->left->parent = n;
    if (n->right) n->right->parent = n;
  }
  uint32_t next_pri() {
    // xorshift32: a fixed sequence, so every run builds the same tree
    rng_ ^= rng_ << 13;
    rng_ ^= rng_ >> 17;
    rng_ ^= rng_ << 5;
    return rng_;
  }
  // first `k` nets of t go to *a, the rest to *b
  static void split(Node* t, size_t k, Node** a, Node** b) {
    if (!t) {
      *a = *b = nullptr;
      return;
    }
    t->parent = nullptr;
    if (cnt(t->left) >= k) {
      Node* l = nullptr;
      split(t->left, k, &l, &t->left);
      pull(t);
      if (l) l->parent = nullptr;
      *a = l;
      *b = t;
    } else {
      Node* r = nullptr;
      split(t->right, k - cnt(t->left) - 1, &t->right, &r);
      pull(t);
      if (r) r->parent = nullptr;
      *a = t;
      *b = r;
    }
  }
  static Node* merge(Node* a, Node* b) {
    if (!a) return b;
    if (!b) return a;
    if (a->pri >= b->pri) {
      a->right = merge(a->right, b);
      pull(a);
      a->parent = nullptr;
      return a;
    }
    b->left = merge(a, b->left);
    pull(b);
    b->parent = nullptr;
    return b;
  }
  // in-order from rank `from` (explicit stack)
  static void walk(const Node* n, size_t from, std::vector<uint32_t>* out) {
    std::vector<const Node*> stack;
    size_t skip = from;
    while (n || !stack.empty()) {
      while (n) {
        if (skip > cnt(n->left)) {  // n and its left subtree are skipped
          skip -= cnt(n->left) + 1;
          n = n->right;
          continue;
        }
        stack.push_back(n);
        if (skip == cnt(n->left)) {  // the left subtree is skipped, n is kept
          skip = 0;
          break;
        }
        n = n->left;
      }
      if (stack.empty()) break;
      const Node* top = stack.back();
      stack.pop_back();
      out->push_back(top->id);
      n = top->right;
    }
  }

  Node* root_ = nullptr;
  std::unordered_map<uint32_t, Node*> by_id_;
  uint32_t rng_ = 0x2545f491u;
};

}  // namespace qtb
