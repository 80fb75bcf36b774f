// Schedule validator of the product loader (docs/SCHEDULE.md "Check order"). A second,
// independent implementation of the rules the oracle checks (oracle/validate.py,
// oracle/simulate.py); verdicts are compared on a mutation corpus in tests.
//  structure  PAPER.md:742-744 (equal chunks), 750 (<=1 send peer, <=1 recv peer per tb),
//             751-752 (deps name steps); input read-only
//  match      k-th send on (A->B, chan) pairs with k-th receive (reading G1)
//  cycle      sequential tbs + deps + matching must be acyclic
//  race       conflicting accesses ordered by happens-before; direct-store single assignment
//  uninit / postcondition   symbolic execution against App. B pre/postconditions
//             (PAPER.md:1324-1330), AR contribution multisets
#include <algorithm>
#include <deque>
#include <map>
#include <queue>
#include <set>
#include <tuple>

#include "taccl_internal.h"

namespace taccl {
namespace {

[[noreturn]] void fail(const char* kind, const std::string& m) { throw SchedError{kind, m}; }

std::string where(int r, int t, int k) {
  return "rank " + std::to_string(r) + " tb" + std::to_string(t) + ":s" + std::to_string(k);
}

const char* bufname(BufId b) { return b == B_I ? "i" : b == B_O ? "o" : "s"; }

void check_structure(const Program& P) {
  int n_in, n_out;
  buffer_chunks(P.coll, P.nranks, P.p, &n_in, &n_out);
  const int n = P.nranks;
  for (const Gpu& g : P.gpus) {
    const int r = g.id;
    if (g.i_chunks != n_in || g.o_chunks != n_out)
      fail("structure", "rank " + std::to_string(r) + ": i_chunks/o_chunks do not match the collective (V5)");
    std::set<std::pair<int, int>> sends, recvs;
    for (const TB& tb : g.tbs) {
      for (int peer : {tb.send, tb.recv}) {
        if (peer != -1 && (peer < 0 || peer >= n))
          fail("structure", "rank " + std::to_string(r) + " tb " + std::to_string(tb.id) + ": peer out of range (V1)");
        if (peer == r) fail("structure", "rank " + std::to_string(r) + " tb " + std::to_string(tb.id) + ": peer is itself (V1)");
      }
      if (tb.chan < 0) fail("structure", "negative chan");
      if (tb.send != -1 && !sends.insert({tb.send, tb.chan}).second)
        fail("structure", "rank " + std::to_string(r) + ": two tbs send to " + std::to_string(tb.send) + " on one chan (V3)");
      if (tb.recv != -1 && !recvs.insert({tb.recv, tb.chan}).second)
        fail("structure", "rank " + std::to_string(r) + ": two tbs receive from " + std::to_string(tb.recv) + " on one chan (V3)");
      for (const Step& st : tb.steps) {
        std::string w = where(r, tb.id, st.s);
        if (st.type == ST_S && tb.send == -1) fail("structure", w + ": send in a tb with no send peer (V2)");
        if ((st.type == ST_R || st.type == ST_RRC) && tb.recv == -1) fail("structure", w + ": receive in a tb with no recv peer (V2)");
        if (st.type != ST_NOP && st.cnt < 1) fail("structure", w + ": cnt < 1");
        if (st.type == ST_MR && (tb.send != -1 || tb.recv != -1))
          fail("structure", w + ": multicast reduce in a tb with a peer (its peer is the switch)");
        if (st.type == ST_MR && P.coll != C_AR && P.coll != C_RS)
          fail("structure", w + ": multicast reduce in a non-reducing collective");
        if (st.dstbuf == B_I) fail("structure", w + ": writes the input buffer (read-only)");
        if (st.srcbuf != B_NONE && (long long)st.srcoff + st.cnt > g.nchunks(st.srcbuf))
          fail("structure", w + ": source range exceeds buffer (V4)");
        if (st.dstbuf != B_NONE && (long long)st.dstoff + st.cnt > g.nchunks(st.dstbuf))
          fail("structure", w + ": destination range exceeds buffer (V4)");
        for (auto [dt, dk] : st.deps) {
          if (dt >= (int)g.tbs.size() || dk >= (int)g.tbs[dt].steps.size())
            fail("structure", w + ": dependency " + std::to_string(dt) + ":" + std::to_string(dk) + " does not exist (V6)");
          if (dt == tb.id && dk == st.s) fail("structure", w + ": depends on itself (V6)");
        }
      }
    }
  }
}

struct Graph {
  std::vector<std::tuple<int, int, int>> nodes;   // (rank, tb, step)
  std::map<std::tuple<int, int, int>, int> id;
  std::vector<std::vector<int>> succ;
  std::vector<int> match;                         // recv node -> send node, else -1
  std::vector<std::vector<int>> groups;           // mr group k -> member nodes (rank order)
  std::map<std::tuple<int, int, int>, std::vector<std::pair<int, int>>> conns;  // (A,B,c)->(send,recv)
};

Graph build(const Program& P) {
  Graph G;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        G.id[{g.id, tb.id, st.s}] = (int)G.nodes.size();
        G.nodes.emplace_back(g.id, tb.id, st.s);
      }
  G.succ.assign(G.nodes.size(), {});
  G.match.assign(G.nodes.size(), -1);
  std::map<std::tuple<int, int, int>, std::vector<int>> S, R;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        int v = G.id[{g.id, tb.id, st.s}];
        if (st.s > 0) G.succ[G.id[{g.id, tb.id, st.s - 1}]].push_back(v);
        for (auto [dt, dk] : st.deps) G.succ[G.id[{g.id, dt, dk}]].push_back(v);
        if (st.type == ST_S) S[{g.id, tb.send, tb.chan}].push_back(v);
        if (st.type == ST_R || st.type == ST_RRC) R[{tb.recv, g.id, tb.chan}].push_back(v);
      }
  std::set<std::tuple<int, int, int>> keys;
  for (auto& kv : S) keys.insert(kv.first);
  for (auto& kv : R) keys.insert(kv.first);
  for (auto& key : keys) {
    auto& ss = S[key];
    auto& rr = R[key];
    auto [a, b, c] = key;
    std::string cn = "connection " + std::to_string(a) + "->" + std::to_string(b) + " chan " + std::to_string(c);
    if (ss.size() != rr.size())
      fail("match", cn + ": " + std::to_string(ss.size()) + " sends vs " + std::to_string(rr.size()) + " receives");
    auto& pairs = G.conns[key];
    for (size_t q = 0; q < ss.size(); ++q) {
      auto [sr, st_, sk] = G.nodes[ss[q]];
      auto [rr_, rt, rk] = G.nodes[rr[q]];
      int cs = P.gpus[sr].tbs[st_].steps[sk].cnt, cr = P.gpus[rr_].tbs[rt].steps[rk].cnt;
      if (cs != cr) fail("match", cn + " message " + std::to_string(q) + ": send cnt " + std::to_string(cs) + " vs receive cnt " + std::to_string(cr));
      G.succ[ss[q]].push_back(rr[q]);
      G.match[rr[q]] = ss[q];
      pairs.emplace_back(ss[q], rr[q]);
    }
  }
  // multicast reduce groups: the k-th mr step of every rank (tb, step order) is a barrier —
  // every predecessor of a member precedes every member, every member precedes every successor
  std::vector<std::vector<int>> mrs(P.nranks);
  bool any = false;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps)
        if (st.type == ST_MR) {
          mrs[g.id].push_back(G.id[{g.id, tb.id, st.s}]);
          any = true;
        }
  if (any) {
    for (int r = 1; r < P.nranks; ++r)
      if (mrs[r].size() != mrs[0].size()) fail("match", "multicast reduce: ranks have different numbers of mr steps");
    const int N = (int)G.nodes.size();
    std::vector<std::vector<int>> pred(N), out = G.succ;
    for (int u = 0; u < N; ++u)
      for (int v : G.succ[u]) pred[v].push_back(u);
    for (size_t k = 0; k < mrs[0].size(); ++k) {
      std::vector<int> mem;
      for (int r = 0; r < P.nranks; ++r) mem.push_back(mrs[r][k]);
      auto cnt_of = [&](int v) { auto [r, t, s] = G.nodes[v]; return P.gpus[r].tbs[t].steps[s].cnt; };
      for (int v : mem)
        if (cnt_of(v) != cnt_of(mem[0])) fail("match", "multicast reduce group " + std::to_string(k) + ": cnt differs across ranks");
      auto member = [&](int x) { return std::find(mem.begin(), mem.end(), x) != mem.end(); };
      for (int q : mem)
        for (int r : mem) {
          if (r == q) continue;
          for (int x : out[q])
            if (!member(x)) G.succ[r].push_back(x);
          for (int x : pred[q])
            if (!member(x)) G.succ[x].push_back(r);
        }
      G.groups.push_back(mem);
    }
  }
  return G;
}

std::vector<int> topo(const Graph& G) {
  const int N = (int)G.nodes.size();
  std::vector<int> indeg(N, 0);
  for (auto& vs : G.succ)
    for (int v : vs) ++indeg[v];
  // min-heap on (rank, tb, step): deterministic like the oracle's Kahn order
  std::priority_queue<std::pair<std::tuple<int, int, int>, int>,
                      std::vector<std::pair<std::tuple<int, int, int>, int>>, std::greater<>> pq;
  for (int v = 0; v < N; ++v)
    if (!indeg[v]) pq.push({G.nodes[v], v});
  std::vector<int> order;
  while (!pq.empty()) {
    int u = pq.top().second;
    pq.pop();
    order.push_back(u);
    for (int v : G.succ[u])
      if (--indeg[v] == 0) pq.push({G.nodes[v], v});
  }
  if ((int)order.size() != N) {
    // name a cycle: from the smallest stuck node walk stuck predecessors until one repeats
    std::vector<std::vector<int>> pred(N);
    for (int u = 0; u < N; ++u)
      if (indeg[u] > 0)
        for (int v : G.succ[u])
          if (indeg[v] > 0) pred[v].push_back(u);
    int v = -1;
    for (int x = 0; x < N; ++x)
      if (indeg[x] > 0 && (v < 0 || G.nodes[x] < G.nodes[v])) v = x;
    std::map<int, int> seen;
    std::vector<int> path;
    while (!seen.count(v)) {
      seen[v] = (int)path.size();
      path.push_back(v);
      int best = -1;
      for (int u : pred[v])
        if (best < 0 || G.nodes[u] < G.nodes[best]) best = u;
      v = best;
    }
    std::vector<int> cyc(path.begin() + seen[v], path.end());
    std::reverse(cyc.begin(), cyc.end());
    std::string m = "deadlock: ";
    for (size_t i = 0; i <= cyc.size(); ++i) {
      auto [r, t, k] = G.nodes[cyc[i % cyc.size()]];
      m += (i ? " -> " : "") + std::string("r") + std::to_string(r) + ":tb" + std::to_string(t) + ":s" + std::to_string(k);
    }
    fail("cycle", m);
  }
  return order;
}

// desc[v] bitset of nodes reachable from v by >= 1 edge
struct Reach {
  int words = 0;
  std::vector<uint64_t> bits;
  bool has(int u, int v) const { return (bits[(size_t)u * words + (v >> 6)] >> (v & 63)) & 1; }
};

Reach reach(const Graph& G, const std::vector<int>& order) {
  Reach R;
  const int N = (int)G.nodes.size();
  R.words = (N + 63) / 64;
  R.bits.assign((size_t)N * R.words, 0);
  for (auto it = order.rbegin(); it != order.rend(); ++it) {
    int u = *it;
    uint64_t* du = &R.bits[(size_t)u * R.words];
    for (int v : G.succ[u]) {
      const uint64_t* dv = &R.bits[(size_t)v * R.words];
      for (int w = 0; w < R.words; ++w) du[w] |= dv[w];
      du[v >> 6] |= 1ull << (v & 63);
    }
  }
  return R;
}

struct Access {
  int lo, hi;
  bool write;
  int start, end, node;
};

void check_races(const Program& P, const Graph& G, const Reach& R, bool direct) {
  std::map<std::pair<int, int>, std::vector<Access>> by;  // (rank, buf)
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        int v = G.id.at({g.id, tb.id, st.s});
        if (st.type == ST_MR) {  // reads and writes the same ranges on every rank
          for (int q = 0; q < P.nranks; ++q) {
            by[{q, st.srcbuf}].push_back({st.srcoff, st.srcoff + st.cnt, false, v, v, v});
            by[{q, st.dstbuf}].push_back({st.dstoff, st.dstoff + st.cnt, true, v, v, v});
          }
          continue;
        }
        if (st.srcbuf != B_NONE) by[{g.id, st.srcbuf}].push_back({st.srcoff, st.srcoff + st.cnt, false, v, v, v});
        if (st.dstbuf != B_NONE) {
          int start = (st.type == ST_R && direct) ? G.match[v] : v;
          by[{g.id, st.dstbuf}].push_back({st.dstoff, st.dstoff + st.cnt, true, start, v, v});
        }
      }
  for (auto& [key, lst] : by) {
    for (size_t i = 0; i < lst.size(); ++i)
      for (size_t j = i + 1; j < lst.size(); ++j) {
        const Access &a = lst[i], &b = lst[j];
        if (a.node == b.node || !(a.write || b.write)) continue;
        if (a.hi <= b.lo || b.hi <= a.lo) continue;
        if (R.has(a.end, b.start) || R.has(b.end, a.start)) continue;
        auto [ra, ta, ka] = G.nodes[a.node];
        auto [rb, tb_, kb] = G.nodes[b.node];
        (void)ra;
        (void)rb;
        const int r = key.first;
        fail("race", "rank " + std::to_string(r) + " " + bufname((BufId)key.second) + "[" +
                         std::to_string(std::max(a.lo, b.lo)) + ":" + std::to_string(std::min(a.hi, b.hi)) +
                         "]: steps tb" + std::to_string(ta) + ":s" + std::to_string(ka) + " and tb" +
                         std::to_string(tb_) + ":s" + std::to_string(kb) + " are unordered");
      }
  }
}

// Symbolic token: chunk id (AG/A2A) or (chunk index, per-rank contribution counts) (AR).
struct Tok {
  int chunk = -1;               // -1 = never written
  std::vector<uint16_t> contrib;  // AR only
  bool operator==(const Tok& o) const { return chunk == o.chunk && contrib == o.contrib; }
};

void symbolic(const Program& P, const Graph& G, const std::vector<int>& order) {
  const int n = P.nranks, p = P.p;
  std::vector<std::vector<Tok>> B[3];
  for (int b = 0; b < 3; ++b) B[b].resize(n);
  for (const Gpu& g : P.gpus) {
    B[B_I][g.id].assign(g.i_chunks, Tok());
    B[B_O][g.id].assign(g.o_chunks, Tok());
    B[B_S][g.id].assign(g.s_chunks, Tok());
    auto& in = B[B_I][g.id];
    for (int k = 0; k < (int)in.size(); ++k) {  // precondition (App. B)
      Tok t;
      if (P.coll == C_AG) t.chunk = g.id * p + k;
      else if (P.coll == C_A2A) t.chunk = (g.id * n + k / p) * p + k % p;  // i[d*p+q]
      else {
        t.chunk = k;
        t.contrib.assign(n, 0);
        t.contrib[g.id] = 1;
      }
      in[k] = t;
    }
  }
  std::map<std::tuple<int, int, int>, std::deque<std::vector<Tok>>> Q;
  for (int v : order) {
    auto [r, t, k] = G.nodes[v];
    const TB& tb = P.gpus[r].tbs[t];
    const Step& st = tb.steps[k];
    auto rd = [&](BufId b, int off) {
      std::vector<Tok> out;
      for (int q = 0; q < st.cnt; ++q) {
        const Tok& x = B[b][r][off + q];
        if (x.chunk < 0) fail("uninit", where(r, t, k) + " reads chunk " + std::to_string(off + q) + " before any write");
        out.push_back(x);
      }
      return out;
    };
    auto wr = [&](BufId b, int off, const std::vector<Tok>& vals) {
      for (int q = 0; q < st.cnt; ++q) B[b][r][off + q] = vals[q];
    };
    switch (st.type) {
      case ST_CPY: wr(st.dstbuf, st.dstoff, rd(st.srcbuf, st.srcoff)); break;
      case ST_S: Q[{r, tb.send, tb.chan}].push_back(rd(st.srcbuf, st.srcoff)); break;
      case ST_R: {
        auto& q = Q[{tb.recv, r, tb.chan}];
        wr(st.dstbuf, st.dstoff, q.front());
        q.pop_front();
        break;
      }
      case ST_RRC: {
        auto& q = Q[{tb.recv, r, tb.chan}];
        std::vector<Tok> got = q.front();
        q.pop_front();
        std::vector<Tok> mine = rd(st.srcbuf, st.srcoff);
        if (P.coll != C_AR && P.coll != C_RS) fail("structure", where(r, t, k) + " reduces in a non-reducing collective");
        for (int i = 0; i < st.cnt; ++i) {
          if (mine[i].chunk != got[i].chunk)
            fail("postcondition", where(r, t, k) + " reduces chunk " + std::to_string(mine[i].chunk) + " with chunk " + std::to_string(got[i].chunk));
          for (int s = 0; s < n; ++s) mine[i].contrib[s] += got[i].contrib[s];
        }
        wr(st.dstbuf, st.dstoff, mine);
        break;
      }
      case ST_MR: {  // sum of every rank's src tokens, written to every rank's dst
        auto rdq = [&](int q) {
          std::vector<Tok> out;
          for (int i = 0; i < st.cnt; ++i) {
            const Tok& x = B[st.srcbuf][q][st.srcoff + i];
            if (x.chunk < 0) fail("uninit", where(r, t, k) + " reads rank " + std::to_string(q) + " chunk " +
                                                std::to_string(st.srcoff + i) + " before any write");
            out.push_back(x);
          }
          return out;
        };
        std::vector<Tok> acc = rdq(0);
        for (int q = 1; q < n; ++q) {
          std::vector<Tok> got = rdq(q);
          for (int i = 0; i < st.cnt; ++i) {
            if (acc[i].chunk != got[i].chunk)
              fail("postcondition", where(r, t, k) + " reduces chunk " + std::to_string(acc[i].chunk) + " with chunk " +
                                        std::to_string(got[i].chunk));
            for (int s2 = 0; s2 < n; ++s2) acc[i].contrib[s2] += got[i].contrib[s2];
          }
        }
        for (int q = 0; q < n; ++q)
          for (int i = 0; i < st.cnt; ++i) B[st.dstbuf][q][st.dstoff + i] = acc[i];
        break;
      }
      case ST_NOP: break;
    }
  }
  for (int r = 0; r < n; ++r) {
    const auto& out = B[B_O][r];
    for (int g = 0; g < (int)out.size(); ++g) {
      Tok want;
      if (P.coll == C_AG) want.chunk = g;
      else if (P.coll == C_A2A) want.chunk = ((g / p) * n + r) * p + g % p;
      else {  // AR: o[g] = chunk g; RS: o[g] = chunk r*p + g (the rank's own part)
        want.chunk = P.coll == C_RS ? r * p + g : g;
        want.contrib.assign(n, 1);
      }
      if (out[g] == want) continue;
      if (P.coll != C_AR && P.coll != C_RS)
        fail("postcondition", "(chunk " + std::to_string(want.chunk) + ", rank " + std::to_string(r) + ") missing");
      if (out[g].chunk < 0)
        fail("postcondition", "(chunk " + std::to_string(g) + ", rank " + std::to_string(r) + ") missing: never written");
      std::string miss, extra;
      for (int s = 0; s < n; ++s) {
        if (out[g].contrib[s] == 0) miss += (miss.empty() ? "" : ", ") + std::to_string(s);
        if (out[g].contrib[s] > 1) extra += (extra.empty() ? "" : ", ") + std::to_string(s);
      }
      fail("postcondition", "(chunk " + std::to_string(g) + ", rank " + std::to_string(r) +
                                ") reduction wrong: missing contributions from ranks [" + miss +
                                "], repeated from ranks [" + extra + "]");
    }
  }
}

}  // namespace

struct HB::Impl {
  Graph G;
  Reach R;
};

HB::HB(const Program& P) : impl_(new Impl) {
  impl_->G = build(P);
  impl_->R = reach(impl_->G, topo(impl_->G));
}
HB::~HB() { delete impl_; }

bool HB::before(int r, int t, int k, int r2, int t2, int k2) const {
  int u = impl_->G.id.at({r, t, k}), v = impl_->G.id.at({r2, t2, k2});
  return impl_->R.has(u, v);
}

void check_program(const Program& P, bool direct) {
  check_structure(P);
  Graph G = build(P);
  std::vector<int> order = topo(G);
  Reach R = reach(G, order);
  check_races(P, G, R, direct);
  symbolic(P, G, order);
}

}  // namespace taccl
