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
#include <map>
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

std::vector<RankPlan> build_plans(const Program& P, bool fuse) {
  const int n = P.nranks;
  std::vector<RankPlan> plans(n);
  // per-step seq numbers and staging offsets
  std::map<std::tuple<int, int, int>, int> seq, soff;
  std::vector<int> stage_total(n, 0);
  for (const Gpu& g : P.gpus) {
    for (const TB& tb : g.tbs) {
      int ns = 0, nr = 0;
      for (const Step& st : tb.steps) {
        if (st.type == ST_S) seq[{g.id, tb.id, st.s}] = ns++;
        if (st.type == ST_R || st.type == ST_RRC) seq[{g.id, tb.id, st.s}] = nr++;
        if (st.type == ST_RRC) {
          soff[{g.id, tb.id, st.s}] = stage_total[g.id];
          stage_total[g.id] += st.cnt;
        }
      }
    }
  }
  // receiving tb of each connection: (receiver, sender, chan) -> tb id
  std::map<std::tuple<int, int, int>, int> recv_tb;
  for (const Gpu& g : P.gpus)
    for (const TB& tb : g.tbs)
      if (tb.recv >= 0) recv_tb[{g.id, tb.recv, tb.chan}] = tb.id;

  HB hb(P);
  for (const Gpu& g : P.gpus) {
    RankPlan& rp = plans[g.id];
    rp.stage_chunks = stage_total[g.id];
    rp.scratch_chunks = g.s_chunks;
    std::map<std::pair<int, int>, int> flat;  // (tb, step) -> index in rp.steps
    for (const TB& tb : g.tbs) {
      KTB kt{tb.send, tb.recv, tb.chan, (int32_t)rp.steps.size(), (int32_t)tb.steps.size()};
      rp.tbs.push_back(kt);
      for (const Step& st : tb.steps) {
        KStep ks{};
        ks.srcbuf = st.srcbuf == B_NONE ? 0 : kbuf(st.srcbuf);
        ks.dstbuf = st.dstbuf == B_NONE ? 0 : kbuf(st.dstbuf);
        ks.srcoff = st.srcoff;
        ks.dstoff = st.dstoff;
        ks.cnt = st.cnt;
        ks.dep_begin = (int32_t)rp.deps.size() / 2;
        ks.dep_count = (int32_t)st.deps.size();
        for (auto [dt, dk] : st.deps) {
          rp.deps.push_back(dt);
          rp.deps.push_back(dk);
        }
        switch (st.type) {
          case ST_S: {
            ks.op = K_SEND;
            ks.seq = seq[{g.id, tb.id, st.s}];
            // matched receive: the seq-th receive of the peer's tb for (recv=g.id, chan)
            const int pt = recv_tb.at({tb.send, g.id, tb.chan});
            const TB& ptb = P.gpus[tb.send].tbs[pt];
            for (const Step& ps : ptb.steps) {
              if ((ps.type == ST_R || ps.type == ST_RRC) && seq[{tb.send, pt, ps.s}] == ks.seq) {
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
          case ST_R: ks.op = K_RECV; ks.seq = seq[{g.id, tb.id, st.s}]; break;
          case ST_RRC:
            ks.op = K_RRC;
            ks.seq = seq[{g.id, tb.id, st.s}];
            ks.soff = soff[{g.id, tb.id, st.s}];
            break;
          case ST_CPY: ks.op = K_CPY; break;
          default: ks.op = K_NOP; break;
        }
        flat[{tb.id, st.s}] = (int)rp.steps.size();
        rp.steps.push_back(ks);
      }
    }
    // need_done: referenced by some dependency
    for (size_t d = 0; d + 1 < rp.deps.size(); d += 2) rp.steps[flat.at({rp.deps[d], rp.deps[d + 1]})].need_done = 1;

    if (!fuse) continue;
    // ---- rrc chain fusion
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
      KStep& fused = rp.steps[flat.at(last)];
      fused.op = K_RRC_FUSED;
      fused.srcbuf = kbuf(first.srcbuf);
      fused.srcoff = first.srcoff;
      fused.fuse_begin = (int32_t)rp.fused.size() / 3;
      fused.fuse_count = (int32_t)chain.size() - 1;
      for (size_t i = 0; i + 1 < chain.size(); ++i) {
        KStep& x = rp.steps[flat.at(chain[i])];
        rp.fused.push_back(chain[i].first);
        rp.fused.push_back(x.seq);
        rp.fused.push_back(x.soff);
        x.op = K_RECV_ONLY;
      }
      ++rp.fused_chains;
    }
  }
  return plans;
}

}  // namespace taccl
