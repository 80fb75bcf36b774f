// Flatten a checked EF program into per-rank device plans (KTB / KStep arrays).
//  * Each send learns where its bytes land on the peer: the matched receive's destination
//    (`r`: the peer's o or s chunk) or the matched rrc's staging slot (reading G1 matching;
//    direct-store execution, docs/SCHEDULE.md).
//  * Staging: each rrc on a rank owns cnt chunks of that rank's staging area, in program
//    order (tb, step), so sender and receiver compute the same offset.
//  * rrc chains (PAPER.md:722-728 reduce-scatter receives chained into one destination) are
//    fused: X_1..X_K with X_{i+1}.src == X_i.dst == X_{i+1}.dst, X_i a direct predecessor of
//    X_{i+1}, and every other access to the destination (or write to X_1's source) ordered
//    before X_1 or after X_K. X_K becomes one multi-input reduction (fp32 accumulation for
//    bf16); X_1..X_{K-1} only keep their place in program order.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <set>
#include <tuple>

#include "taccl_internal.h"
#include "plan.h"

namespace taccl {
namespace {

int8_t kbuf(BufId b) { return b == B_I ? KB_I : b == B_O ? KB_O : KB_S; }

bool overlap(BufId b1, int o1, int c1, BufId b2, int o2, int c2) {
  return b1 == b2 && b1 != B_NONE && o1 < o2 + c2 && o2 < o1 + c1;
}

}  // namespace

// rrc chain fusion (R3 in DESIGN.md). A chain X_1..X_K becomes K cooperating K_RRC_FUSED
// steps: each member waits for all K staged inputs, reduces its 1/K portion of every piece
// (dst = src(X_1) + stage_1 + ... + stage_K, chain order), and X_K publishes completion
// only after every member's portion (post-dependencies). The chain edges between members
// are dropped; every member inherits X_1's incoming edges (its tb predecessor and deps; the
// matched send is covered by waiting on X_1's data flag), so whatever happened before X_1
// happens before every member, and whatever followed X_K still follows all of them.
void fuse_chains(const Gpu& g, const HB& hb, const std::map<std::pair<int, int>, int>& flat, RankPlan& rp,
                 std::vector<std::vector<std::pair<int, int>>>& deps,
                 std::vector<std::vector<std::pair<int, int>>>& post) {
  auto step_of = [&](int t, int k) -> const Step& { return g.tbs[t].steps[k]; };
  auto direct_pred = [&](int t, int k, int t2, int k2) {  // (t,k) directly precedes (t2,k2)?
    if (t == t2 && k + 1 == k2) return true;
    for (auto [dt, dk] : step_of(t2, k2).deps)
      if (dt == t && dk == k) return true;
    return false;
  };
  std::vector<std::pair<int, int>> rrcs;
  for (const TB& tb : g.tbs)
    for (const Step& st : tb.steps)
      if (st.type == ST_RRC) rrcs.emplace_back(tb.id, st.s);
  std::map<std::pair<int, int>, std::pair<int, int>> next, prev;
  for (auto x : rrcs) {
    const Step& a = step_of(x.first, x.second);
    std::vector<std::pair<int, int>> cand;
    for (auto y : rrcs) {
      if (y == x) continue;
      const Step& b = step_of(y.first, y.second);
      if (b.srcbuf == a.dstbuf && b.srcoff == a.dstoff && b.dstbuf == a.dstbuf && b.dstoff == a.dstoff &&
          b.cnt == a.cnt && direct_pred(x.first, x.second, y.first, y.second))
        cand.push_back(y);
    }
    if (cand.size() == 1 && !prev.count(cand[0])) {
      next[x] = cand[0];
      prev[cand[0]] = x;
    }
  }
  for (auto head : rrcs) {
    if (prev.count(head) || !next.count(head)) continue;
    std::vector<std::pair<int, int>> chain{head};
    while (next.count(chain.back()) && (int)chain.size() < kMaxRanks) chain.push_back(next[chain.back()]);
    const Step& first = step_of(head.first, head.second);
    const auto last = chain.back();
    const Step& lastst = step_of(last.first, last.second);
    // legality: other accesses to the destination (any) or to first's source (writes)
    bool ok = true;
    for (const TB& tb : g.tbs) {
      for (const Step& st : tb.steps) {
        if (std::find(chain.begin(), chain.end(), std::make_pair(tb.id, st.s)) != chain.end()) continue;
        bool touches = overlap(st.srcbuf, st.srcoff, st.cnt, lastst.dstbuf, lastst.dstoff, lastst.cnt) ||
                       overlap(st.dstbuf, st.dstoff, st.cnt, lastst.dstbuf, lastst.dstoff, lastst.cnt) ||
                       overlap(st.dstbuf, st.dstoff, st.cnt, first.srcbuf, first.srcoff, first.cnt);
        if (!touches) continue;
        // For an `r` (bytes land while its peer's send runs) "after the chain" is enough:
        // the direct-store check already ordered the chain's last step before that send.
        const int r = g.id;
        const bool before_first = hb.before(r, tb.id, st.s, r, head.first, head.second);
        const bool after_last = hb.before(r, last.first, last.second, r, tb.id, st.s);
        if (!before_first && !after_last) ok = false;
      }
    }
    if (!ok) continue;
    // rewrite the members
    const int K = (int)chain.size();
    // what every member must wait for: the steps that happened before X_1 and conflict with
    // the chain (write its source or destination, or read its destination), not all of X_1's
    // incoming edges — a member waiting on X_1's threadblock predecessor (e.g. the send before
    // an all-pairs reduce-scatter's first rrc) would add a cross-CTA wait that orders nothing
    // the chain touches. Kept minimal: a conflicting step ordered before another one is implied.
    std::vector<std::pair<int, int>> head_in;
    if (getenv("TACCL_CHAIN_OLDDEPS") && atoi(getenv("TACCL_CHAIN_OLDDEPS"))) {  // A/B knob: every incoming edge
      head_in = first.deps;
      if (head.second > 0) head_in.emplace_back(head.first, head.second - 1);
    } else {
      const int r = g.id;
      std::vector<std::pair<int, int>> q;
      for (const TB& tb : g.tbs)
        for (const Step& st : tb.steps) {
          if (std::find(chain.begin(), chain.end(), std::make_pair(tb.id, st.s)) != chain.end()) continue;
          const bool writes_src_or_dst = st.dstbuf != B_NONE &&
              (overlap(st.dstbuf, st.dstoff, st.cnt, first.srcbuf, first.srcoff, first.cnt) ||
               overlap(st.dstbuf, st.dstoff, st.cnt, lastst.dstbuf, lastst.dstoff, lastst.cnt));
          const bool reads_dst = st.srcbuf != B_NONE && overlap(st.srcbuf, st.srcoff, st.cnt, lastst.dstbuf, lastst.dstoff, lastst.cnt);
          if ((writes_src_or_dst || reads_dst) && hb.before(r, tb.id, st.s, r, head.first, head.second))
            q.emplace_back(tb.id, st.s);
        }
      for (auto a : q) {
        bool implied = false;
        for (auto b : q)
          if (a != b && hb.before(r, a.first, a.second, r, b.first, b.second)) implied = true;
        if (!implied) head_in.push_back(a);
      }
    }
    const int fb = (int32_t)rp.fused.size() / kFuseStride;
    for (int i = 0; i < K; ++i) {
      const KStep& x = rp.steps[flat.at(chain[i])];
      for (int v : {chain[i].first, x.seq, x.soff, x.soff2, x.poff, x.pflags & P_IN}) rp.fused.push_back(v);
    }
    // bf16 partials: the chain reads X_1's source (P_SRC of X_1) and its result is kept when X_K
    // is (the members' intermediate values exist only inside the fused sum)
    const int chain_pf = (rp.steps[flat.at(head)].pflags & P_SRC) | (rp.steps[flat.at(last)].pflags & P_KEEP);
    for (int i = 0; i < K; ++i) {
      const int fi = flat.at(chain[i]);
      KStep& x = rp.steps[fi];
      x.pflags = chain_pf;
      x.op = K_RRC_FUSED;
      x.srcbuf = kbuf(first.srcbuf);
      x.srcoff = first.srcoff;
      x.fuse_begin = fb;
      x.fuse_count = K;
      x.part = i;
      x.nparts = K;
      if (i > 0) {
        auto& d = deps[fi];
        d.erase(std::remove(d.begin(), d.end(), chain[i - 1]), d.end());
        for (auto e : head_in)
          if (e.first != chain[i].first && std::find(d.begin(), d.end(), e) == d.end()) d.push_back(e);
      }
    }
    auto& pl = post[flat.at(last)];
    for (int i = 0; i + 1 < K; ++i)
      if (chain[i].first != last.first) pl.push_back(chain[i]);
  }
}

// Chain + send fusion: a send that immediately follows a fused-chain member in its tb, reads
// exactly the chain's destination and waits on nothing but chain members, has its bytes
// written by the chain members themselves — each member stores its portion of the reduced
// result to every such send's destination on the peer as it computes it (one pass; NVLink
// busy while reducing, like K_RRCS for single rrcs). The send becomes K_PUB: after the chain
// (its dependencies) it only publishes the data flag (direct mode) or nothing (LL mode).
// Direct AR = RS ++ AG is exactly this shape: the AG phase's sends of the
// reduced chunk follow the RS phase's chain into that chunk.
// Legality beyond the dependency shape: the bytes now land while the chain runs, earlier
// than the send's own position, so the receiver must touch the destination range with
// nothing but the matched receive (rrc staging slots are private to their receive).
bool only_receive_touches(const Program& P, int peer, int8_t rbuf, int off, int cnt) {
  if (rbuf == KB_STAGE) return true;
  const BufId b = rbuf == KB_O ? B_O : B_S;
  int touching = 0;
  for (const TB& tb : P.gpus[peer].tbs)
    for (const Step& st : tb.steps)
      if (overlap(st.srcbuf, st.srcoff, st.cnt, b, off, cnt) || overlap(st.dstbuf, st.dstoff, st.cnt, b, off, cnt))
        ++touching;
  return touching == 1;
}

void fuse_chain_sends(const Program& P, RankPlan& rp, const std::vector<std::vector<std::pair<int, int>>>& deps,
                      const std::vector<std::vector<std::pair<int, int>>>& post) {
  std::map<int, std::vector<int>> chains;  // fuse_begin -> member flat indices
  for (size_t i = 0; i < rp.steps.size(); ++i)
    if (rp.steps[i].op == K_RRC_FUSED) chains[rp.steps[i].fuse_begin].push_back((int)i);
  auto pos = [&](int fi) {  // flat index -> (tb, step)
    for (int t = 0; t < (int)rp.tbs.size(); ++t)
      if (fi >= rp.tbs[t].step_begin && fi < rp.tbs[t].step_begin + rp.tbs[t].nsteps)
        return std::make_pair(t, fi - rp.tbs[t].step_begin);
    return std::make_pair(-1, -1);
  };
  for (auto& [fb, mem] : chains) {
    std::vector<std::pair<int, int>> mpos;
    for (int fi : mem) mpos.push_back(pos(fi));
    const KStep& m0 = rp.steps[mem[0]];
    std::vector<int> sends;
    // candidates: the step right after each member (paired lowering) and, for split lowerings,
    // a send anywhere whose only dependencies are chain members
    std::vector<int> cand;
    for (size_t q = 0; q < mem.size(); ++q)
      if (mpos[q].second + 1 < rp.tbs[mpos[q].first].nsteps) cand.push_back(mem[q] + 1);
    for (int si = 0; si < (int)rp.steps.size(); ++si)
      if (rp.steps[si].op == K_SEND && !deps[si].empty() && std::find(cand.begin(), cand.end(), si) == cand.end())
        cand.push_back(si);
    for (int si : cand) {
      const int t = pos(si).first;
      const KStep& s = rp.steps[si];
      if (s.op != K_SEND || s.srcbuf != m0.dstbuf || s.srcoff != m0.dstoff || s.cnt != m0.cnt || !post[si].empty())
        continue;
      bool only_chain = true;
      for (auto d : deps[si]) only_chain = only_chain && std::find(mpos.begin(), mpos.end(), d) != mpos.end();
      if (only_chain && only_receive_touches(P, rp.tbs[t].send, s.rbuf, s.roff, s.cnt)) sends.push_back(si);
    }
    if (sends.empty() || (int)sends.size() > kMaxRanks) continue;
    const int fwb = (int)rp.fused.size();
    for (int si : sends) {
      KStep& s = rp.steps[si];
      const KTB& kt = rp.tbs[pos(si).first];
      for (int v : {kt.send, kt.chan, (int)s.rbuf, s.roff, s.roff2, s.seq, s.pflags & P_OUT}) rp.fused.push_back(v);
      s.op = K_PUB;
    }
    for (int fi : mem) {
      rp.steps[fi].fwd_begin = fwb;
      rp.steps[fi].fwd_count = (int)sends.size();
    }
  }
}

// bf16 partials (reading R6; the oracle's run(bf16="partials") states the same rule
// dynamically). Static form: the state of chunk c of o/s when step X reads it is decided by
// its last writer before X in happens-before order (unique: the race check orders every two
// writes of a chunk and every write with every read). X reads a range as fp32 partials iff
// every chunk's last writer is an rrc. Flags: an rrc whose source range qualifies gets P_SRC;
// a send whose matched receive is an rrc and whose source range qualifies gets P_OUT and that
// receive P_IN; every rrc that is the last writer of a chunk some flagged read covers gets
// P_KEEP (its result must be kept in the shadow). `matched` maps a send to its receive.
using SKey = std::tuple<int, int, int>;  // (rank, tb, step)
std::map<SKey, int> partial_flags(const Program& P, const HB& hb, const std::map<SKey, SKey>& matched,
                                  std::map<SKey, std::set<SKey>>* readers) {
  std::map<std::tuple<int, int, int>, int> fl;
  for (const Gpu& g : P.gpus) {
    const int r = g.id;
    struct W { int r, t, k; StepType type; BufId buf; int off, cnt; };
    std::vector<W> writers;
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps)
        if ((st.type == ST_R || st.type == ST_RRC || st.type == ST_CPY) && (st.dstbuf == B_O || st.dstbuf == B_S))
          writers.push_back({r, tb.id, st.s, st.type, st.dstbuf, st.dstoff, st.cnt});
    for (const Gpu& g2 : P.gpus)  // a multicast reduce writes every rank's destination (bits only)
      for (const TB& tb : g2.tbs)
        for (const Step& st : tb.steps)
          if (st.type == ST_MR && (st.dstbuf == B_O || st.dstbuf == B_S))
            writers.push_back({g2.id, tb.id, st.s, st.type, st.dstbuf, st.dstoff, st.cnt});
    // the rrcs that are last writers of the range (empty if some chunk's last writer is not one)
    auto partial_range = [&](int t, int k, BufId buf, int off, int cnt, std::vector<int>* lw) {
      lw->clear();
      if (buf != B_O && buf != B_S) return false;
      for (int c = off; c < off + cnt; ++c) {
        int best = -1;
        for (int w = 0; w < (int)writers.size(); ++w) {
          const W& x = writers[w];
          if (x.buf != buf || c < x.off || c >= x.off + x.cnt || !hb.before(x.r, x.t, x.k, r, t, k)) continue;
          if (best < 0 || hb.before(writers[best].r, writers[best].t, writers[best].k, x.r, x.t, x.k)) best = w;
        }
        if (best < 0 || writers[best].type != ST_RRC) return false;
        lw->push_back(best);
      }
      return true;
    };
    std::vector<std::pair<int, SKey>> keep;  // (writer, reader)
    std::vector<int> lw;
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        if (st.type == ST_RRC && partial_range(tb.id, st.s, st.srcbuf, st.srcoff, st.cnt, &lw)) {
          fl[{r, tb.id, st.s}] |= P_SRC;
          for (int w : lw) keep.push_back({w, SKey{r, tb.id, st.s}});
        }
        if (st.type == ST_S) {
          const auto m = matched.at({r, tb.id, st.s});
          const Step& rs = P.gpus[std::get<0>(m)].tbs[std::get<1>(m)].steps[std::get<2>(m)];
          if (rs.type == ST_RRC && partial_range(tb.id, st.s, st.srcbuf, st.srcoff, st.cnt, &lw)) {
            fl[{r, tb.id, st.s}] |= P_OUT;
            fl[m] |= P_IN;
            for (int w : lw) keep.push_back({w, SKey{r, tb.id, st.s}});
          }
        }
      }
    for (auto [w, rd] : keep) {  // (only rrcs qualify as last writers here: same rank)
      fl[{writers[w].r, writers[w].t, writers[w].k}] |= P_KEEP;
      (*readers)[{writers[w].r, writers[w].t, writers[w].k}].insert(rd);
    }
  }
  return fl;
}

// Streamed messages (direct kernel; DESIGN.md §6 "streamed reduces"): a receive-reduce that
// would otherwise wait for its whole piece before reducing it — all its input messages land
// while its CTA idles — instead reduces each group of stripes as soon as every input message
// published that group, so the reduce overlaps the transfers and only the last group is left
// after them. Marked per receive-reduce (a fused chain as a whole) when (1) no member carries
// bf16 partials (the partials path moves other bytes per stripe), (2) every input message is
// sent by a plain K_SEND (not a forward fused into K_RRCS, a chain's K_PUB or a K_RCS relay) and
// (3) every member is the first step of its threadblock doing data work: a CTA that sends first
// reaches the reduce when its peers' messages have landed too (paired send+rrc tbs) and the
// progress stores would be pure cost. Both ends get KStep.prog; the kernel streams only when
// KArgs.prog (the runtime turns it off in pull mode and for TMA pushes).
// With the program's overlap="1" hint (or TACCL_WARPSPEC=1) a member may also follow exactly
// one send without dependencies of its own (paired send + rrc threadblocks, as the direct schedules lower): such a member gets
// prog = 2 and the kernel runs it beside that send — one half of the CTA's warps sends
// (publishing groups) while the other half reduces the groups as they land (streamed_pair).
void mark_streamed(std::vector<RankPlan>& plans, bool overlap) {
  const int n = (int)plans.size();
  const char* ws = getenv("TACCL_WARPSPEC");  // A/B knob: 1 forces the pairs on, 0 off
  const bool pairs = ws ? atoi(ws) != 0 : overlap;
  auto first_data = [&](const RankPlan& rp, const KTB& kt, int k) {
    for (int q = 0; q < k; ++q) {
      const KStep& y = rp.steps[kt.step_begin + q];
      if (y.op == K_NOP) continue;
      if (!pairs || q + 1 != k || y.op != K_SEND || y.dep_count || y.post_count) return false;
    }
    return true;
  };
  // the K_SEND on rank q that carries message `seq` of connection (q -> r, chan), or null
  auto sender = [&](int q, int r, int chan, int seq) -> KStep* {
    if (q < 0 || q >= n) return nullptr;
    for (const KTB& pt : plans[q].tbs) {
      if (pt.send != r || pt.chan != chan) continue;
      for (int k = 0; k < pt.nsteps; ++k) {
        KStep& y = plans[q].steps[pt.step_begin + k];
        if (y.op == K_SEND && y.seq == seq) return &y;
      }
    }
    return nullptr;
  };
  for (int r = 0; r < n; ++r) {
    RankPlan& rp = plans[r];
    for (int t = 0; t < (int)rp.tbs.size(); ++t) {
      const KTB& kt = rp.tbs[t];
      for (int k = 0; k < kt.nsteps; ++k) {
        KStep& x = rp.steps[kt.step_begin + k];
        if (x.op == K_RRC) {
          KStep* s = sender(kt.recv, r, kt.chan, x.seq);
          if (x.pflags || !s || s->pflags || !first_data(rp, kt, k) || x.seq >= kProgSeqMax) continue;
          x.prog = s->prog = 1;
          // streamed pushes beat in-place loads for such a reduce (RS n=2 1 GiB 800 vs 833 us,
          // profiles/r02_knob_scan_split_n2.txt): it no longer pulls (both ends agree)
          x.poff = s->poff = -1;
        } else if (x.op == K_RRC_FUSED && x.part == 0) {
          // the chain's members: the steps sharing its fused entries, one per member tb
          std::vector<KStep*> members;
          bool ok = true;
          for (int t2 = 0; t2 < (int)rp.tbs.size() && ok; ++t2)
            for (int k2 = 0; k2 < rp.tbs[t2].nsteps; ++k2) {
              KStep& y = rp.steps[rp.tbs[t2].step_begin + k2];
              if (y.op != K_RRC_FUSED || y.fuse_begin != x.fuse_begin) continue;
              ok = ok && !y.pflags && first_data(rp, rp.tbs[t2], k2);
              members.push_back(&y);
            }
          std::vector<KStep*> sends;
          for (int f = 0; f < x.fuse_count && ok; ++f) {
            const int* fz = rp.fused.data() + kFuseStride * (x.fuse_begin + f);
            const KTB& o = rp.tbs[fz[0]];
            KStep* s = sender(o.recv, r, o.chan, fz[1]);
            ok = s && !s->pflags && !fz[5] && fz[1] < kProgSeqMax;
            sends.push_back(s);
          }
          if (!ok) continue;
          for (KStep* y : members) y->prog = 1;
          for (KStep* y : sends) y->prog = 1;
        }
      }
    }
  }
  // warp-specialised pairs: a streamed receive-reduce right after a streamed send of its tb,
  // without dependencies or forwards, whose destination does not overlap the send's source
  for (RankPlan& rp : plans)
    for (const KTB& kt : rp.tbs)
      for (int k = 1; k < kt.nsteps && pairs; ++k) {
        KStep& x = rp.steps[kt.step_begin + k];
        const KStep& s = rp.steps[kt.step_begin + k - 1];
        if (!x.prog || s.op != K_SEND || !s.prog || x.dep_count || (x.op == K_RRC_FUSED && x.fwd_count)) continue;
        const bool overlap = x.dstbuf == s.srcbuf && x.dstoff < s.srcoff + s.cnt && s.srcoff < x.dstoff + x.cnt;
        if (!overlap) x.prog = 2;
      }
}

// Merged execution (DESIGN.md §6 "merged threadblocks"): every CTA of a rank runs, for each of
// its pieces, the steps of ALL the rank's threadblocks, instead of one threadblock's. The order
// must never make a CTA wait for something that waits for it. Levels over the global step
// graph give one: edges are program order, dependencies (pre and post), and message edges (the
// step that publishes a message's data flag -> every step that waits for it); a step's level
// is its longest path from a source. Every wait then points at a strictly lower level, so CTAs
// that run their steps by increasing level (any order within a level) make progress level by
// level (and piece by piece, as before). Multicast reduces (a barrier across ranks) and graphs
// with a message nobody publishes or a cycle leave `order` empty (not mergeable).
void merged_order(std::vector<RankPlan>& plans) {
  const int n = (int)plans.size();
  std::vector<int> base(n + 1, 0);
  for (int r = 0; r < n; ++r) base[r + 1] = base[r] + (int)plans[r].steps.size();
  const int N = base[n];
  std::vector<std::vector<int>> succ(N);
  std::vector<int> indeg(N, 0);
  auto edge = [&](int a, int b) {
    succ[a].push_back(b);
    ++indeg[b];
  };
  std::map<std::tuple<int, int, int, int>, int> writer;  // (receiver, sender, chan, seq) -> node
  for (int q = 0; q < n; ++q) {
    const RankPlan& rp = plans[q];
    for (const KTB& kt : rp.tbs)
      for (int k = 0; k < kt.nsteps; ++k) {
        const KStep& s = rp.steps[kt.step_begin + k];
        const int node = base[q] + kt.step_begin + k;
        if (s.op == K_MR) return;
        if (s.op == K_SEND || s.op == K_PUB) writer[{kt.send, q, kt.chan, s.seq}] = node;
        if (s.op == K_RRCS || s.op == K_RCS) writer[{kt.send, q, kt.chan, s.fwd_seq}] = node;
      }
  }
  for (int r = 0; r < n; ++r) {
    const RankPlan& rp = plans[r];
    for (const KTB& kt : rp.tbs)
      for (int k = 0; k < kt.nsteps; ++k) {
        const int i = kt.step_begin + k, node = base[r] + i;
        const KStep& s = rp.steps[i];
        if (k > 0) edge(node - 1, node);
        for (int d = 0; d < s.dep_count + s.post_count; ++d) {
          const int e = d < s.dep_count ? s.dep_begin + d : s.post_begin + (d - s.dep_count);
          edge(base[r] + rp.tbs[rp.deps[2 * e]].step_begin + rp.deps[2 * e + 1], node);
        }
        auto msg = [&](int sender, int chan, int seq) {
          auto it = writer.find({r, sender, chan, seq});
          if (it == writer.end()) return false;
          edge(it->second, node);
          return true;
        };
        bool ok = true;
        if (s.op == K_RECV || s.op == K_RRC || s.op == K_RRCS || s.op == K_RCS) ok = msg(kt.recv, kt.chan, s.seq);
        if (s.op == K_RRC_FUSED)
          for (int f = 0; f < s.fuse_count && ok; ++f) {
            const int* fz = rp.fused.data() + kFuseStride * (s.fuse_begin + f);
            ok = msg(rp.tbs[fz[0]].recv, rp.tbs[fz[0]].chan, fz[1]);
          }
        if (!ok) return;
      }
  }
  std::vector<int> level(N, 0), ready;
  for (int v = 0; v < N; ++v)
    if (!indeg[v]) ready.push_back(v);
  int seen = 0;
  while (!ready.empty()) {
    const int v = ready.back();
    ready.pop_back();
    ++seen;
    for (int w : succ[v]) {
      level[w] = std::max(level[w], level[v] + 1);
      if (--indeg[w] == 0) ready.push_back(w);
    }
  }
  if (seen != N) return;  // a cycle: the checker's happens-before should exclude it
  // within a level: rotation order — a step toward peer r + d (sends) or from peer r - d
  // (receives) in round d, so that in each round every GPU sends to one peer and receives from
  // one (a permutation; by threadblock index the peers collide: at n=4 three GPUs sent to GPU 0
  // first, Alltoall 1 GiB 1972 vs 1217 us); steps without a peer last
  for (int r = 0; r < n; ++r) {
    RankPlan& rp = plans[r];
    std::vector<std::tuple<int, int, int, int>> key;  // (level, round, tb, step)
    for (int t = 0; t < (int)rp.tbs.size(); ++t)
      for (int k = 0; k < rp.tbs[t].nsteps; ++k) {
        const KTB& kt = rp.tbs[t];
        const int op = rp.steps[kt.step_begin + k].op;
        const bool sends = op == K_SEND || op == K_PUB || op == K_RRCS || op == K_RCS;
        const int round = sends && kt.send >= 0 ? (kt.send - r + n) % n : kt.recv >= 0 ? (r - kt.recv + n) % n : n;
        key.push_back({level[base[r] + kt.step_begin + k], round, t, k});
      }
    std::sort(key.begin(), key.end());
    rp.order.clear();
    for (auto [l, d, t, k] : key) rp.order.push_back((t << 16) | k);
  }
}

std::vector<RankPlan> build_plans(const Program& P, bool fuse, bool fuse_rrcs, bool chain_sends, int pull_kinds) {
  const int n = P.nranks;
  std::vector<RankPlan> plans(n);
  // per-step seq numbers (message index on the tb's connection)
  std::map<std::tuple<int, int, int>, int> seq, soff, soff2;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs) {
      int ns = 0, nr = 0;
      for (const Step& st : tb.steps) {
        if (st.type == ST_S) seq[{g.id, tb.id, st.s}] = ns++;
        if (st.type == ST_R || st.type == ST_RRC) seq[{g.id, tb.id, st.s}] = nr++;
      }
    }
  // receiving tb of each connection: (receiver, sender, chan) -> tb id
  std::map<std::tuple<int, int, int>, int> recv_tb;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      if (tb.recv >= 0) recv_tb[{g.id, tb.recv, tb.chan}] = tb.id;
  // each send's matched receive (reading G1: the k-th send of a connection <-> its k-th receive)
  std::map<std::tuple<int, int, int>, std::tuple<int, int, int>> matched;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        if (st.type != ST_S) continue;
        const int pt = recv_tb.at({tb.send, g.id, tb.chan});
        for (const Step& ps : P.gpus[tb.send].tbs[pt].steps)
          if ((ps.type == ST_R || ps.type == ST_RRC) && seq[{tb.send, pt, ps.s}] == seq[{g.id, tb.id, st.s}]) {
            matched[{g.id, tb.id, st.s}] = {tb.send, pt, ps.s};
            break;
          }
      }
  HB hb(P);
  std::map<SKey, std::set<SKey>> keep_readers;  // rrc -> the steps that read its kept partials
  const std::map<SKey, int> pfl = partial_flags(P, hb, matched, &keep_readers);
  auto pflag = [&](int r, int t, int k) {
    auto it = pfl.find({r, t, k});
    return it == pfl.end() ? 0 : it->second;
  };
  // staging offsets: each rrc owns cnt chunks of its rank's staging area (2 cnt when its
  // message is fp32 partials), in program order (tb, step); staged mode: every receive a slot
  std::vector<int> stage_total(n, 0), stage2_total(n, 0);
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      for (const Step& st : tb.steps) {
        const int w = (pflag(g.id, tb.id, st.s) & P_IN) ? 2 : 1;
        if (st.type == ST_RRC) {
          // an fp32 message's slot starts at an even chunk offset: soff * cbytes is then a
          // multiple of 4 bytes (bf16 chunks are an even number of bytes), as floats need
          if (w == 2) stage_total[g.id] += stage_total[g.id] & 1;
          soff[{g.id, tb.id, st.s}] = stage_total[g.id];
          stage_total[g.id] += w * st.cnt;
        }
        if (st.type == ST_R || st.type == ST_RRC) {
          soff2[{g.id, tb.id, st.s}] = stage2_total[g.id];
          stage2_total[g.id] += w * st.cnt;
        }
      }

  for (const Gpu& g : P.gpus) {
    RankPlan& rp = plans[g.id];
    rp.stage_chunks = stage_total[g.id];
    rp.stage2_chunks = stage2_total[g.id];
    rp.scratch_chunks = g.s_chunks;
    std::map<std::pair<int, int>, int> flat;  // (tb, step) -> index in rp.steps
    int mr_group = 0;                         // k-th multicast reduce of this rank = group k
    std::vector<std::vector<std::pair<int, int>>> deps, post;  // per flat step
    for (const TB& tb : g.tbs) {
      KTB kt{tb.send, tb.recv, tb.chan, (int32_t)rp.steps.size(), (int32_t)tb.steps.size()};
      rp.tbs.push_back(kt);
      for (const Step& st : tb.steps) {
        KStep ks{};
        ks.poff = -1;
        ks.pflags = pflag(g.id, tb.id, st.s);
        if (ks.pflags) rp.partials = true;
        ks.srcbuf = st.srcbuf == B_NONE ? 0 : kbuf(st.srcbuf);
        ks.dstbuf = st.dstbuf == B_NONE ? 0 : kbuf(st.dstbuf);
        ks.srcoff = st.srcoff;
        ks.dstoff = st.dstoff;
        ks.cnt = st.cnt;
        deps.push_back(st.deps);
        post.emplace_back();
        switch (st.type) {
          case ST_S: {
            ks.op = K_SEND;
            ks.seq = seq[{g.id, tb.id, st.s}];
            // matched receive: the seq-th receive of the peer's tb for (recv=g.id, chan)
            const int pt = recv_tb.at({tb.send, g.id, tb.chan});
            const TB& ptb = P.gpus[tb.send].tbs[pt];
            for (const Step& ps : ptb.steps) {
              if ((ps.type == ST_R || ps.type == ST_RRC) && seq[{tb.send, pt, ps.s}] == ks.seq) {
                ks.roff2 = soff2[{tb.send, pt, ps.s}];
                if (ps.type == ST_R) {
                  ks.rbuf = kbuf(ps.dstbuf);
                  ks.roff = ps.dstoff;
                } else {
                  ks.rbuf = KB_STAGE;
                  ks.roff = soff[{tb.send, pt, ps.s}];
                }
                break;
              }
            }
            break;
          }
          case ST_R:
            ks.op = K_RECV;
            ks.seq = seq[{g.id, tb.id, st.s}];
            ks.soff2 = soff2[{g.id, tb.id, st.s}];
            break;
          case ST_RRC: {
            ks.op = K_RRC;
            ks.seq = seq[{g.id, tb.id, st.s}];
            ks.soff = soff[{g.id, tb.id, st.s}];
            ks.soff2 = soff2[{g.id, tb.id, st.s}];
            // matched send: the seq-th send of the peer's tb for (send=g.id, chan); pull mode
            // reads its source in place when it is the peer's input (read-only, valid from the
            // peer's call entry, reading R1)
            for (const TB& ptb : P.gpus[tb.recv].tbs)
              if (ptb.send == g.id && ptb.chan == tb.chan)
                for (const Step& ps : ptb.steps)
                  if (ps.type == ST_S && seq[{tb.recv, ptb.id, ps.s}] == ks.seq && ps.srcbuf == B_I) ks.poff = ps.srcoff;
            break;
          }
          case ST_CPY: ks.op = K_CPY; break;
          case ST_MR: ks.op = K_MR; ks.seq = mr_group++; break;  // group index (barrier slots)
          default: ks.op = K_NOP; break;
        }
        flat[{tb.id, st.s}] = (int)rp.steps.size();
        rp.steps.push_back(ks);
      }
    }
    if (fuse) fuse_chains(g, hb, flat, rp, deps, post);
    // a chain's last member waits for the other members' portions (post-dependencies) only so
    // that its done flag means "whole result written"; when no step depends on it, the wait is
    // pure latency (one cross-CTA poll at the end of every small Allreduce/ReduceScatter)
    {
      std::vector<char> wanted(rp.steps.size(), 0);
      for (size_t i = 0; i < rp.steps.size(); ++i)
        for (auto e : deps[i]) wanted[flat.at(e)] = 1;
      for (const KTB& kt : rp.tbs)  // a threadblock successor relies on it too (program order)
        for (int k = 0; k + 1 < kt.nsteps; ++k) wanted[kt.step_begin + k] = 1;
      for (size_t i = 0; i < rp.steps.size(); ++i) {
        // a chain whose inputs are pulled keeps the wait: its last member acks the senders for
        // every member's reads, so the acks must follow all portions (pull mode, executor.cu)
        bool pulled = false;
        const KStep& x = rp.steps[i];
        if ((pull_kinds & 4) && x.op == K_RRC_FUSED)
          for (int f = 0; f < x.fuse_count; ++f) pulled = pulled || rp.fused[kFuseStride * (x.fuse_begin + f) + 4] >= 0;
        if (!post[i].empty() && !wanted[i] && x.fwd_count == 0 && !pulled &&
            !(getenv("TACCL_CHAIN_OLDDEPS") && atoi(getenv("TACCL_CHAIN_OLDDEPS"))))
          post[i].clear();
      }
    }
    // pull mode acks are "read up to message seq" per connection, so they must be written in
    // message order: a chain's inputs are acked by its last member, which may run after a later
    // receive of a member's own threadblock acked — such chains keep the push path
    for (const KTB& kt : rp.tbs)
      for (int k = 0; k < kt.nsteps; ++k) {
        const KStep& x = rp.steps[kt.step_begin + k];
        if (x.op != K_RRC_FUSED) continue;
        bool later = false;
        for (int k2 = k + 1; k2 < kt.nsteps; ++k2) later = later || rp.steps[kt.step_begin + k2].poff >= 0;
        if (later)
          for (int f = 0; f < x.fuse_count; ++f) rp.fused[kFuseStride * (x.fuse_begin + f) + 4] = -1;
      }
    // chain_sends: the LL kernel's plan (-10% time for LL direct AR at n=4); the direct kernel
    // only with TACCL_CHAIN_SENDS=1 (+12% at >= 256 MiB, -10% at 2-32 MiB;
    // profiles/r01_chain_sends_n4.txt, r01_chain_sends_ll_n4.txt)
    if (fuse && fuse_rrcs && chain_sends) fuse_chain_sends(P, rp, deps, post);
    // flatten dependency lists; need_done: referenced by some (post-)dependency
    for (size_t i = 0; i < rp.steps.size(); ++i) {
      KStep& ks = rp.steps[i];
      ks.dep_begin = (int32_t)rp.deps.size() / 2;
      ks.dep_count = (int32_t)deps[i].size();
      for (auto [dt, dk] : deps[i]) {
        rp.deps.push_back(dt);
        rp.deps.push_back(dk);
      }
      ks.post_begin = (int32_t)rp.deps.size() / 2;
      ks.post_count = (int32_t)post[i].size();
      for (auto [dt, dk] : post[i]) {
        rp.deps.push_back(dt);
        rp.deps.push_back(dk);
      }
    }
    for (size_t d = 0; d + 1 < rp.deps.size(); d += 2) rp.steps[flat.at({rp.deps[d], rp.deps[d + 1]})].need_done = 1;
    // recv-reduce-copy-send (the fused instruction whose absence the
    // paper blames for its >=512 MB Allreduce gap): an rrc immediately
    // followed in its tb by a send of exactly its result, the send waiting on nothing else
    if (fuse_rrcs) {
      for (const KTB& kt : rp.tbs) {
        for (int i = 0; i + 1 < kt.nsteps; ++i) {
          KStep& a = rp.steps[kt.step_begin + i];
          KStep& b = rp.steps[kt.step_begin + i + 1];
          // recv-copy-send (§8(f) row 1, relays of ring and hierarchical schedules): same shape
          const bool rcs = a.op == K_RECV && b.op == K_SEND && b.srcbuf == a.dstbuf && b.srcoff == a.dstoff &&
                           b.cnt == a.cnt && b.dep_count == 0 && b.post_count == 0 && a.post_count == 0;
          if (rcs || (a.op == K_RRC && b.op == K_SEND && b.srcbuf == a.dstbuf && b.srcoff == a.dstoff &&
                      b.cnt == a.cnt && b.dep_count == 0 && b.post_count == 0)) {
            a.op = rcs ? K_RCS : K_RRCS;
            a.pflags = (a.pflags & ~P_OUT) | (b.pflags & P_OUT);  // the forward's message type
            a.rbuf = b.rbuf;
            a.roff = b.roff;
            a.fwd_seq = b.seq;
            a.roff2 = b.roff2;
            b.op = K_SENT;
          }
        }
      }
    }
    // fused chains whose member messages or forwards are fp32 carry P_MIX, so the kernel
    // takes the partials path on one flag test
    for (KStep& x : rp.steps)
      if (x.op == K_RRC_FUSED) {
        for (int f = 0; f < x.fuse_count; ++f)
          if (rp.fused[kFuseStride * (x.fuse_begin + f) + 5]) x.pflags |= P_MIX;
        for (int f = 0; f < x.fwd_count; ++f)
          if (rp.fused[x.fwd_begin + kFwdStride * f + 6]) x.pflags |= P_MIX;
        if (x.pflags) rp.partials = true;
      }
    // bf16 partials: a result whose kept partials are read only by sends that the producing
    // step now performs itself (K_RRCS's K_SENT, a chain's K_PUB) forwards its fp32
    // accumulator directly — the shadow write would be dead traffic
    {
      auto key_of = [&](int fi) {
        for (int t = 0; t < (int)rp.tbs.size(); ++t)
          if (fi >= rp.tbs[t].step_begin && fi < rp.tbs[t].step_begin + rp.tbs[t].nsteps)
            return SKey{g.id, t, fi - rp.tbs[t].step_begin};
        return SKey{-1, -1, -1};
      };
      auto fwd_only = [&](const SKey& w) {
        auto it = keep_readers.find(w);
        if (it == keep_readers.end()) return true;
        for (const SKey& rd : it->second) {
          if (std::get<0>(rd) != g.id) return false;
          const int op = rp.steps[flat.at({std::get<1>(rd), std::get<2>(rd)})].op;
          if (op != K_SENT && op != K_PUB) return false;
        }
        return true;
      };
      for (size_t i = 0; i < rp.steps.size(); ++i) {
        KStep& x = rp.steps[i];
        if (!(x.pflags & P_KEEP)) continue;
        if (x.op == K_RRCS && fwd_only(key_of((int)i))) x.pflags &= ~P_KEEP;
        if (x.op == K_RRC_FUSED) {
          int lastm = -1;
          for (size_t q = 0; q < rp.steps.size(); ++q)
            if (rp.steps[q].op == K_RRC_FUSED && rp.steps[q].fuse_begin == x.fuse_begin &&
                rp.steps[q].part + 1 == rp.steps[q].nparts)
              lastm = (int)q;
          if (lastm >= 0 && fwd_only(key_of(lastm))) x.pflags &= ~P_KEEP;
        }
      }
    }
    for (const KStep& x : rp.steps)
      if ((x.pflags & (P_KEEP | P_SRC)) || (x.op == K_SEND && (x.pflags & P_OUT))) rp.shadow = true;
    // pull kinds: by default only plain rrcs read in place — measured on B200
    // (profiles/r01_pull_n2.txt, r01_pull_n4.txt): a plain rrc (RS n=2) goes from push +
    // serialised reduce to one pass (497 -> 642 GB/s busbw); an rrc fused with its send (AR
    // n=2) already overlaps its reduce with the forward push and loses (689 -> 663, peer loads
    // stream slower than stores); fused chains with n-1 remote inputs (RS n=4) lose too
    for (KStep& x : rp.steps) {
      const bool keep = (x.op == K_RRC && (pull_kinds & 1)) || (x.op == K_RRCS && (pull_kinds & 2));
      if (!keep && x.op != K_SEND) x.poff = -1;
    }
    if (!(pull_kinds & 4))
      for (const KStep& x : rp.steps)
        if (x.op == K_RRC_FUSED)
          for (int f = 0; f < x.fuse_count; ++f) rp.fused[kFuseStride * (x.fuse_begin + f) + 4] = -1;
    // tb weights: data each tb moves (remote pushes dominate)
    for (KTB& kt : rp.tbs) {
      long long w = 0;
      for (int i = 0; i < kt.nsteps; ++i) {
        const KStep& ks = rp.steps[kt.step_begin + i];
        const int f = ks.op == K_SEND || ks.op == K_RCS ? 4 : ks.op == K_CPY ? 1 : ks.op == K_RRC ? 2 : ks.op == K_RRCS ? 6 :
                      ks.op == K_RRC_FUSED ? 1 + (ks.fuse_count + 4 * ks.fwd_count) / std::max(1, ks.nparts) : 0;
        w += (long long)f * ks.cnt;
      }
      kt.weight = (int32_t)std::min<long long>(w, 1 << 20);
      bool indep = kt.send < 0 && kt.recv < 0;
      for (int i = 0; i < kt.nsteps && indep; ++i) {
        const KStep& ks = rp.steps[kt.step_begin + i];
        // a multicast reduce's piece j meets piece j of every rank at its barriers: it keeps
        // the launch-wide split (identical on all ranks)
        indep = ks.dep_count == 0 && ks.post_count == 0 && !ks.need_done && ks.op != K_MR;
      }
      kt.indep = indep;
    }
    rp.fused_chains = (int)std::count_if(rp.steps.begin(), rp.steps.end(),
                                         [](const KStep& k) { return k.op == K_RRC_FUSED && k.part == 0; });
  }
  // a send is pulled (pull mode: no push, the receiver loads it in place) exactly when its
  // matched receive's final plan reads it in place; both sides must agree
  for (int r = 0; r < n; ++r)
    for (const KTB& kt : plans[r].tbs)
      for (int k = 0; k < kt.nsteps; ++k) {
        KStep& x = plans[r].steps[kt.step_begin + k];
        if (x.op != K_SEND) continue;
        x.poff = -1;
        const RankPlan& pp = plans[kt.send];
        for (const KTB& pt : pp.tbs) {
          if (pt.recv != r || pt.chan != kt.chan) continue;
          for (int q = 0; q < pt.nsteps; ++q) {
            const KStep& y = pp.steps[pt.step_begin + q];
            if (y.seq != x.seq) continue;
            if (y.op == K_RRC || y.op == K_RRCS) x.poff = y.poff;
            else if (y.op == K_RRC_FUSED) x.poff = pp.fused[kFuseStride * (y.fuse_begin + y.part) + 4];
            else if (y.op == K_RECV || y.op == K_RCS) x.poff = -1;
            else continue;
            break;
          }
        }
      }
  mark_streamed(plans, P.overlap != 0);
  merged_order(plans);
  return plans;
}

}  // namespace taccl
