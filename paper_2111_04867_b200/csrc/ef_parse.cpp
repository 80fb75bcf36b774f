// EF v1 parser for the product loader (docs/SCHEDULE.md). Hand-written, independent of the
// oracle's parser (oracle/ef.py uses Python's XML reader). The program model follows
// PAPER.md:741-752 (§6.1): three buffers with equal-size chunks, per-GPU threadblocks of
// sequential steps (send / receive with optional reduction / local copy), dependencies.
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <map>

#include "taccl_internal.h"

namespace taccl {
namespace {

[[noreturn]] void fail(const std::string& m) { throw SchedError{"syntax", m}; }

struct Tag {
  std::string name;
  bool closing = false;     // </name>
  bool selfclose = false;   // <name ... />
  std::map<std::string, std::string> attrs;
};

class Lexer {
 public:
  Lexer(const char* p, size_t n) : p_(p), end_(p + n) {}

  // Next tag; false at end of input. Text between tags must be whitespace.
  bool next(Tag* t) {
    for (;;) {
      skip_ws();
      if (p_ >= end_) return false;
      if (*p_ != '<') fail("unexpected text outside tags");
      if (starts("<!--")) {
        const char* e = find("-->");
        p_ = e + 3;
        continue;
      }
      if (starts("<?")) {
        const char* e = find("?>");
        p_ = e + 2;
        continue;
      }
      break;
    }
    ++p_;
    *t = Tag();
    if (p_ < end_ && *p_ == '/') {
      t->closing = true;
      ++p_;
    }
    t->name = ident();
    if (t->name.empty()) fail("tag without a name");
    for (;;) {
      skip_ws();
      if (p_ >= end_) fail("unterminated tag <" + t->name);
      if (*p_ == '>') {
        ++p_;
        return true;
      }
      if (*p_ == '/') {
        if (p_ + 1 >= end_ || p_[1] != '>') fail("bad '/' in <" + t->name);
        t->selfclose = true;
        p_ += 2;
        return true;
      }
      if (t->closing) fail("attributes on closing tag </" + t->name);
      std::string key = ident();
      if (key.empty()) fail("bad attribute in <" + t->name);
      skip_ws();
      if (p_ >= end_ || *p_ != '=') fail("attribute " + key + " without '='");
      ++p_;
      skip_ws();
      if (p_ >= end_ || (*p_ != '"' && *p_ != '\'')) fail("attribute " + key + " not quoted");
      char q = *p_++;
      const char* s = p_;
      while (p_ < end_ && *p_ != q) ++p_;
      if (p_ >= end_) fail("unterminated value of " + key);
      if (t->attrs.count(key)) fail("duplicate attribute " + key);
      t->attrs[key] = std::string(s, p_ - s);
      ++p_;
    }
  }

 private:
  void skip_ws() {
    while (p_ < end_ && isspace((unsigned char)*p_)) ++p_;
  }
  bool starts(const char* s) const {
    size_t n = strlen(s);
    return (size_t)(end_ - p_) >= n && memcmp(p_, s, n) == 0;
  }
  const char* find(const char* s) const {
    size_t n = strlen(s);
    for (const char* q = p_; q + n <= end_; ++q)
      if (memcmp(q, s, n) == 0) return q;
    fail(std::string("unterminated ") + s);
  }
  std::string ident() {
    const char* s = p_;
    while (p_ < end_ && (isalnum((unsigned char)*p_) || *p_ == '_')) ++p_;
    return std::string(s, p_ - s);
  }
  const char* p_;
  const char* end_;
};

long long to_int(const Tag& t, const char* key, long long lo, bool required = true,
                 long long dflt = 0) {
  auto it = t.attrs.find(key);
  if (it == t.attrs.end()) {
    if (required) fail("<" + t.name + "> missing attribute " + key);
    return dflt;
  }
  const std::string& v = it->second;
  char* e = nullptr;
  errno = 0;
  long long x = strtoll(v.c_str(), &e, 10);
  if (v.empty() || *e != '\0' || errno) fail("<" + t.name + "> attribute " + key + "=\"" + v + "\" is not an integer");
  if (x < lo) fail("<" + t.name + "> attribute " + key + " < " + std::to_string(lo));
  return x;
}

BufId to_buf(const Tag& t, const char* key) {
  auto it = t.attrs.find(key);
  if (it == t.attrs.end()) fail(std::string("<step> missing attribute ") + key);
  if (it->second == "i") return B_I;
  if (it->second == "o") return B_O;
  if (it->second == "s") return B_S;
  fail(std::string("<step> ") + key + "=\"" + it->second + "\" is not one of i/o/s");
}

std::vector<std::pair<int, int>> to_deps(const std::string& s) {
  std::vector<std::pair<int, int>> out;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && isspace((unsigned char)s[i])) ++i;
    if (i >= s.size()) break;
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    std::string item = s.substr(i, j - i);
    size_t c = item.find(':');
    if (c == std::string::npos) fail("bad dependency '" + item + "' (want tb:step)");
    char* e1 = nullptr;
    char* e2 = nullptr;
    std::string a = item.substr(0, c), b = item.substr(c + 1);
    while (!b.empty() && isspace((unsigned char)b.back())) b.pop_back();
    long t = strtol(a.c_str(), &e1, 10), k = strtol(b.c_str(), &e2, 10);
    if (a.empty() || b.empty() || *e1 || *e2 || t < 0 || k < 0)
      fail("bad dependency '" + item + "' (want tb:step)");
    out.emplace_back((int)t, (int)k);
    i = j + 1;
  }
  return out;
}

}  // namespace

void buffer_chunks(Coll c, int n, int p, int* n_in, int* n_out) {
  if (c == C_AG) {
    *n_in = p;
    *n_out = n * p;
  } else if (c == C_RS) {  // ReduceScatter: n*p input chunks, the rank's own p outputs
    *n_in = n * p;
    *n_out = p;
  } else {
    *n_in = n * p;
    *n_out = n * p;
  }
}

Program parse_ef(const char* text, size_t len) {
  Lexer lx(text, len);
  Tag t;
  Program prog;
  if (!lx.next(&t) || t.closing || t.name != "algo") fail("root element must be <algo>");
  if (t.selfclose) fail("<algo> has no <gpu> elements");
  const std::string coll = t.attrs.count("coll") ? t.attrs["coll"] : "";
  if (coll == "allgather") prog.coll = C_AG;
  else if (coll == "alltoall") prog.coll = C_A2A;
  else if (coll == "allreduce") prog.coll = C_AR;
  else if (coll == "reducescatter") prog.coll = C_RS;
  else fail("coll=\"" + coll + "\" unsupported");
  prog.name = t.attrs.count("name") ? t.attrs["name"] : "";
  prog.nranks = (int)to_int(t, "nranks", 1);
  prog.p = (int)to_int(t, "chunks_per_rank", 1);
  prog.instances = (int)to_int(t, "instances", 1);
  for (const char* key : {"minBytes", "maxBytes"}) {
    auto it = t.attrs.find(key);
    if (it == t.attrs.end()) fail(std::string("<algo> missing attribute ") + key);
    uint64_t v;
    if (it->second == "inf") {
      v = UINT64_MAX;
    } else {
      v = (uint64_t)to_int(t, key, 0);
    }
    (strcmp(key, "minBytes") == 0 ? prog.min_bytes : prog.max_bytes) = v;
  }
  if (to_int(t, "inplace", 0) != 0) fail("inplace=1 is not supported (reading G10)");
  // optional dtypes="int32,float32,bfloat16": the element types taccl_run may select this
  // algorithm for (a size-specialised set can differ per type; default: all)
  if (t.attrs.count("dtypes")) {
    prog.dtypes = 0;
    const std::string& v = t.attrs["dtypes"];
    size_t i = 0;
    while (i <= v.size()) {
      size_t j = v.find(',', i);
      if (j == std::string::npos) j = v.size();
      const std::string d = v.substr(i, j - i);
      if (d == "int32") prog.dtypes |= 1u << TACCL_INT32;
      else if (d == "float32") prog.dtypes |= 1u << TACCL_FLOAT32;
      else if (d == "bfloat16") prog.dtypes |= 1u << TACCL_BFLOAT16;
      else fail("dtypes: unknown element type '" + d + "'");
      i = j + 1;
    }
  }
  // optional overlap="1": an execution hint (a paired send and the receive-reduce after it
  // run at once on the two halves of each CTA, plan.cpp mark_streamed); computes the same
  prog.overlap = t.attrs.count("overlap") ? (int)to_int(t, "overlap", 0) : 0;
  if (prog.overlap != 0 && prog.overlap != 1) fail("overlap must be 0 or 1");
  if (prog.nranks > 4096 || prog.p > 4096) fail("nranks or chunks_per_rank too large");

  // <gpu> elements
  while (lx.next(&t)) {
    if (t.closing && t.name == "algo") {
      if (lx.next(&t)) fail("content after </algo>");
      if ((int)prog.gpus.size() != prog.nranks)
        fail(std::to_string(prog.gpus.size()) + " <gpu> elements for nranks=" + std::to_string(prog.nranks));
      return prog;
    }
    if (t.closing || t.name != "gpu") fail("<algo> may only contain <gpu>");
    Gpu g;
    g.id = (int)to_int(t, "id", 0);
    if (g.id != (int)prog.gpus.size()) fail("<gpu> #" + std::to_string(prog.gpus.size()) + " has id=" + std::to_string(g.id));
    g.i_chunks = (int)to_int(t, "i_chunks", 0);
    g.o_chunks = (int)to_int(t, "o_chunks", 0);
    g.s_chunks = (int)to_int(t, "s_chunks", 0);
    if (!t.selfclose) {
      for (;;) {
        if (!lx.next(&t)) fail("unterminated <gpu>");
        if (t.closing && t.name == "gpu") break;
        if (t.closing || t.name != "tb") fail("<gpu> may only contain <tb>");
        TB tb;
        tb.id = (int)to_int(t, "id", 0);
        if (tb.id != (int)g.tbs.size())
          fail("rank " + std::to_string(g.id) + ": <tb> #" + std::to_string(g.tbs.size()) + " has id=" + std::to_string(tb.id));
        tb.send = (int)to_int(t, "send", -1);
        tb.recv = (int)to_int(t, "recv", -1);
        tb.chan = (int)to_int(t, "chan", 0);
        if (!t.selfclose) {
          for (;;) {
            if (!lx.next(&t)) fail("unterminated <tb>");
            if (t.closing && t.name == "tb") break;
            if (t.closing || t.name != "step") fail("<tb> may only contain <step>");
            Step st;
            st.s = (int)to_int(t, "s", 0);
            std::string where = "rank " + std::to_string(g.id) + " tb " + std::to_string(tb.id);
            if (st.s != (int)tb.steps.size()) fail(where + ": <step> #" + std::to_string(tb.steps.size()) + " has s=" + std::to_string(st.s));
            std::string ty = t.attrs.count("type") ? t.attrs["type"] : "";
            if (ty == "s") st.type = ST_S;
            else if (ty == "r") st.type = ST_R;
            else if (ty == "rrc") st.type = ST_RRC;
            else if (ty == "cpy") st.type = ST_CPY;
            else if (ty == "nop") st.type = ST_NOP;
            else if (ty == "mr") st.type = ST_MR;
            else fail(where + " step " + std::to_string(st.s) + ": type=\"" + ty + "\"");
            if (st.type == ST_S || st.type == ST_RRC || st.type == ST_CPY || st.type == ST_MR) {
              st.srcbuf = to_buf(t, "srcbuf");
              st.srcoff = (int)to_int(t, "srcoff", 0);
            }
            if (st.type == ST_R || st.type == ST_RRC || st.type == ST_CPY || st.type == ST_MR) {
              st.dstbuf = to_buf(t, "dstbuf");
              st.dstoff = (int)to_int(t, "dstoff", 0);
            }
            if (st.type != ST_NOP) st.cnt = (int)to_int(t, "cnt", 1);
            st.deps = to_deps(t.attrs.count("deps") ? t.attrs["deps"] : "");
            tb.steps.push_back(std::move(st));
            if (!t.selfclose) {
              Tag c;
              if (!lx.next(&c) || !c.closing || c.name != "step") fail("<step> must be empty");
            }
          }
        }
        g.tbs.push_back(std::move(tb));
      }
    }
    prog.gpus.push_back(std::move(g));
  }
  fail("missing </algo>");
}

}  // namespace taccl
