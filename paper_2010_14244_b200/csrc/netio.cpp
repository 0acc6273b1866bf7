// netio.cpp — reference-schema network ingestion and export.
//
// load_network / load_network_file (R/src/net.cpp:112-175) and
// serialize_network / write_network_file (net.cpp:179-209), natively: a
// single-pass JSON reader for the reference schema
//   {"nodes": [{"id", "signalized", "x"?, "y"?}...],
//    "edges": [{"id", "from", "to", "length_m", "lanes"}...]}
// with the reference's validation messages, and a writer whose text equals
// nlohmann::json::dump(2) of the reference document (sorted keys, shortest
// round-trip doubles).  At 10^6 nodes / 4*10^6 edges it parses in seconds,
// where generate_city is O(n^2) and the Python json module is ~10x slower.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gmaco.h"

namespace gmaco {
// gmaco_capi.cpp: the RoadNetwork ctor checks on a descriptor; false + message on failure
bool validate_graph_desc(const gmaco_graph_desc* d, std::string* err);
}

namespace {

thread_local std::string g_net_err;

struct NetValidation : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NetRuntime : std::runtime_error {  // nlohmann type errors: not ValidationError (exit 2)
  using std::runtime_error::runtime_error;
};

// ---- minimal JSON reader ----------------------------------------------------
struct Val {
  enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;                               // string / object key scratch
  std::vector<Val> arr;
  std::vector<std::pair<std::string, Val>> obj;  // insertion order; duplicate keys: last wins on lookup
  bool is_number() const { return kind == Int || kind == Float; }
  const Val* get(const char* k) const {
    const Val* r = nullptr;
    for (const auto& kv : obj)
      if (kv.first == k) r = &kv.second;
    return r;
  }
  double as_double() const {
    if (kind == Int) return (double)i;
    if (kind == Float) return d;
    throw NetRuntime("[json.exception.type_error.302] type must be number, but is " + type_name());
  }
  int64_t as_int() const {  // get<int>: numbers convert (floats truncate), others throw
    if (kind == Int) return i;
    if (kind == Float) return (int64_t)d;
    throw NetRuntime("[json.exception.type_error.302] type must be number, but is " + type_name());
  }
  std::string type_name() const {
    static const char* n[] = {"null", "boolean", "number", "number", "string", "array", "object"};
    return n[kind];
  }
};

struct Parser {
  const char* p;
  const char* end;
  [[noreturn]] void err(const char* what) {
    throw NetValidation(std::string("network parse error: ") + what + " at byte " + std::to_string(p - begin));
  }
  const char* begin;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  void expect(char c) {
    ws();
    if (p >= end || *p != c) err("unexpected character");
    ++p;
  }
  void parse_string(std::string& out) {
    expect('"');
    out.clear();
    while (p < end && *p != '"') {
      if (*p == '\\') {
        ++p;
        if (p >= end) err("unterminated string");
        switch (*p) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (end - p < 5) err("bad escape");
            unsigned cp = 0;
            for (int k = 1; k <= 4; ++k) {
              const char h = p[k];
              cp = cp * 16 + (h >= '0' && h <= '9' ? h - '0' : (h | 32) >= 'a' && (h | 32) <= 'f' ? (h | 32) - 'a' + 10 : 0);
            }
            p += 4;
            if (cp < 0x80) {
              out += (char)cp;
            } else if (cp < 0x800) {
              out += (char)(0xC0 | (cp >> 6));
              out += (char)(0x80 | (cp & 0x3F));
            } else {
              out += (char)(0xE0 | (cp >> 12));
              out += (char)(0x80 | ((cp >> 6) & 0x3F));
              out += (char)(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: err("bad escape");
        }
        ++p;
      } else {
        out += *p++;
      }
    }
    if (p >= end) err("unterminated string");
    ++p;
  }
  void parse(Val& v) {
    ws();
    if (p >= end) err("unexpected end of input");
    const char c = *p;
    if (c == '{') {
      ++p;
      v.kind = Val::Obj;
      ws();
      if (p < end && *p == '}') {
        ++p;
        return;
      }
      for (;;) {
        v.obj.emplace_back();
        parse_string(v.obj.back().first);
        expect(':');
        parse(v.obj.back().second);
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        expect('}');
        return;
      }
    } else if (c == '[') {
      ++p;
      v.kind = Val::Arr;
      ws();
      if (p < end && *p == ']') {
        ++p;
        return;
      }
      for (;;) {
        v.arr.emplace_back();
        parse(v.arr.back());
        ws();
        if (p < end && *p == ',') {
          ++p;
          continue;
        }
        expect(']');
        return;
      }
    } else if (c == '"') {
      v.kind = Val::Str;
      parse_string(v.s);
    } else if (c == 't' && end - p >= 4 && !std::memcmp(p, "true", 4)) {
      v.kind = Val::Bool;
      v.b = true;
      p += 4;
    } else if (c == 'f' && end - p >= 5 && !std::memcmp(p, "false", 5)) {
      v.kind = Val::Bool;
      p += 5;
    } else if (c == 'n' && end - p >= 4 && !std::memcmp(p, "null", 4)) {
      v.kind = Val::Null;
      p += 4;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      const char* s = p;
      bool flt = false;
      if (*p == '-') ++p;
      while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '+' || *p == '-')) {
        if (*p == '.' || *p == 'e' || *p == 'E') flt = true;
        ++p;
      }
      if (!flt) {  // nlohmann: integer literals are integers (int64 range)
        int64_t x = 0;
        const auto r = std::from_chars(s, p, x);
        if (r.ec == std::errc() && r.ptr == p) {
          v.kind = Val::Int;
          v.i = x;
          return;
        }
      }
      double x = 0.0;  // correctly rounded (like nlohmann's strtod-based parse)
      const auto r = std::from_chars(s, p, x);
      if (r.ec != std::errc() || r.ptr != p) err("invalid number");
      v.kind = Val::Float;
      v.d = x;
    } else {
      err("syntax error");
    }
  }
};

void reject_unknown(const Val& o, std::initializer_list<const char*> allowed, const std::string& where) {
  std::vector<std::string> keys;  // net.cpp:20-31; nlohmann objects iterate in sorted key order
  for (const auto& kv : o.obj) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  for (const auto& k : keys) {
    bool known = false;
    for (const char* a : allowed)
      if (k == a) known = true;
    if (!known) throw NetValidation("unknown key \"" + k + "\" in " + where);
  }
}

struct Net {
  std::vector<uint8_t> sig, has_pos;
  std::vector<double> x, y;
  std::vector<int32_t> from, to, lanes;
  std::vector<int64_t> len;
};

struct NodeRec {
  int64_t id;
  bool sig, pos;
  double x, y;
};
struct EdgeRec {
  int64_t id, from, to, len;
  int64_t lanes;
};

// Fast path for well-formed documents of the common shape: top-level
// "nodes" / "edges" arrays of objects with known keys (each at most once),
// escape-free keys, plain numeric literals.  Fills the records directly (no
// DOM) and returns false on anything else — the exact DOM parser then runs
// and produces the reference's behaviour and messages.
struct Fast {
  const char* p;
  const char* e;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool lit(char c) {
    ws();
    if (p < e && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  bool key(const char*& k, size_t& kl) {  // escape-free string, then ':'
    ws();
    if (p >= e || *p != '"') return false;
    const char* s = ++p;
    while (p < e && *p != '"') {
      if (*p == '\\' || (unsigned char)*p < 0x20) return false;
      ++p;
    }
    if (p >= e) return false;
    k = s;
    kl = (size_t)(p - s);
    ++p;
    return lit(':');
  }
  // JSON number literal: integer (no fraction/exponent) or float
  bool number(bool& is_int, int64_t& iv, double& dv) {
    ws();
    const char* s = p;
    if (p < e && *p == '-') ++p;
    if (p >= e || *p < '0' || *p > '9') return false;
    if (*p == '0' && p + 1 < e && p[1] >= '0' && p[1] <= '9') return false;  // leading zero: let the DOM parser report
    while (p < e && *p >= '0' && *p <= '9') ++p;
    is_int = true;
    if (p < e && *p == '.') {
      is_int = false;
      ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      is_int = false;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || *p < '0' || *p > '9') return false;
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (is_int) {
      const auto r = std::from_chars(s, p, iv);
      if (r.ec != std::errc() || r.ptr != p) return false;  // out of int64 range: DOM path
      dv = (double)iv;
    } else {
      const auto r = std::from_chars(s, p, dv);
      if (r.ec != std::errc() || r.ptr != p) return false;
    }
    return true;
  }
  bool boolean(bool& b) {
    ws();
    if (e - p >= 4 && !std::memcmp(p, "true", 4)) {
      b = true;
      p += 4;
      return true;
    }
    if (e - p >= 5 && !std::memcmp(p, "false", 5)) {
      b = false;
      p += 5;
      return true;
    }
    return false;
  }
  static bool is(const char* k, size_t kl, const char* name) {
    return std::strlen(name) == kl && !std::memcmp(k, name, kl);
  }
  bool node(NodeRec& r) {
    if (!lit('{')) return false;
    unsigned seen = 0;
    bool have_x = false, have_y = false;
    r = NodeRec{0, false, false, 0.0, 0.0};
    if (lit('}')) return false;  // no id: DOM path reports
    do {
      const char* k;
      size_t kl;
      if (!key(k, kl)) return false;
      bool isi;
      int64_t iv;
      double dv;
      if (is(k, kl, "id")) {
        if (seen & 1 || !number(isi, iv, dv) || !isi) return false;
        r.id = (int64_t)(int32_t)iv;
        seen |= 1;
      } else if (is(k, kl, "signalized")) {
        if (seen & 2 || !boolean(r.sig)) return false;
        seen |= 2;
      } else if (is(k, kl, "x")) {
        if (seen & 4 || !number(isi, iv, dv)) return false;
        r.x = dv;
        have_x = true;
        seen |= 4;
      } else if (is(k, kl, "y")) {
        if (seen & 8 || !number(isi, iv, dv)) return false;
        r.y = dv;
        have_y = true;
        seen |= 8;
      } else {
        return false;
      }
    } while (lit(','));
    if (!lit('}')) return false;
    if ((seen & 3) != 3 || have_x != have_y) return false;
    r.pos = have_x;
    return true;
  }
  bool edge(EdgeRec& r) {
    if (!lit('{')) return false;
    unsigned seen = 0;
    r = EdgeRec{};
    if (lit('}')) return false;
    do {
      const char* k;
      size_t kl;
      if (!key(k, kl)) return false;
      bool isi;
      int64_t iv;
      double dv;
      int bit;
      if (is(k, kl, "id")) bit = 0;
      else if (is(k, kl, "from")) bit = 1;
      else if (is(k, kl, "to")) bit = 2;
      else if (is(k, kl, "length_m")) bit = 3;
      else if (is(k, kl, "lanes")) bit = 4;
      else return false;
      if (seen & (1u << bit) || !number(isi, iv, dv)) return false;
      seen |= 1u << bit;
      switch (bit) {
        case 0: if (!isi) return false; r.id = (int32_t)iv; break;
        case 1: if (!isi) return false; r.from = (int32_t)iv; break;
        case 2: if (!isi) return false; r.to = (int32_t)iv; break;
        case 3: r.len = std::llround(dv * 1000.0); break;  // meters_to_mm, net.cpp:34
        case 4: if (!isi) return false; r.lanes = (int32_t)iv; break;
      }
    } while (lit(','));
    if (!lit('}')) return false;
    return seen == 31u;
  }
  template <class Rec, class F>
  bool array(std::vector<Rec>& out, F&& one) {
    if (!lit('[')) return false;
    if (lit(']')) return true;
    do {
      out.emplace_back();
      if (!one(out.back())) return false;
    } while (lit(','));
    return lit(']');
  }
};

bool fast_parse(const std::string& text, std::vector<NodeRec>& nodes, std::vector<EdgeRec>& edges) {
  Fast f{text.data(), text.data() + text.size()};
  if (!f.lit('{')) return false;
  bool hn = false, he = false;
  do {
    const char* k;
    size_t kl;
    if (!f.key(k, kl)) return false;
    if (Fast::is(k, kl, "nodes") && !hn) {
      nodes.reserve(text.size() / 160);
      if (!f.array(nodes, [&](NodeRec& r) { return f.node(r); })) return false;
      hn = true;
    } else if (Fast::is(k, kl, "edges") && !he) {
      edges.reserve(text.size() / 120);
      if (!f.array(edges, [&](EdgeRec& r) { return f.edge(r); })) return false;
      he = true;
    } else {
      return false;
    }
  } while (f.lit(','));
  if (!f.lit('}')) return false;
  f.ws();
  return f.p == f.e && hn && he;
}

void dom_parse(const std::string& text, std::vector<NodeRec>& nodes, std::vector<EdgeRec>& edges) {
  Parser ps{text.data(), text.data() + text.size(), text.data()};
  Val doc;
  ps.parse(doc);
  ps.ws();
  if (ps.p != ps.end) ps.err("trailing characters");
  if (doc.kind != Val::Obj) throw NetValidation("network document must be a JSON object");
  reject_unknown(doc, {"nodes", "edges"}, "network document");
  const Val* jn = doc.get("nodes");
  const Val* je = doc.get("edges");
  if (!jn || !je) throw NetValidation("network document requires \"nodes\" and \"edges\"");
  for (const Val& v : jn->arr) {  // net.cpp:123-141
    if (v.kind != Val::Obj) throw NetValidation("node entries must be objects");
    reject_unknown(v, {"id", "signalized", "x", "y"}, "node entry");
    const Val* id = v.get("id");
    if (!id || id->kind != Val::Int) throw NetValidation("node entry missing integer \"id\"");
    NodeRec nd{(int64_t)(int32_t)id->i, false, false, 0.0, 0.0};
    const Val* sg = v.get("signalized");
    if (!sg || sg->kind != Val::Bool)
      throw NetValidation("node " + std::to_string(nd.id) + " missing boolean \"signalized\"");
    nd.sig = sg->b;
    const Val *vx = v.get("x"), *vy = v.get("y");
    if ((vx != nullptr) != (vy != nullptr))
      throw NetValidation("node " + std::to_string(nd.id) + " must give both x and y or neither");
    if (vx) {
      nd.pos = true;
      nd.x = vx->as_double();
      nd.y = vy->as_double();
    }
    nodes.push_back(nd);
  }
  for (const Val& v : je->arr) {  // net.cpp:143-165
    if (v.kind != Val::Obj) throw NetValidation("edge entries must be objects");
    reject_unknown(v, {"id", "from", "to", "length_m", "lanes"}, "edge entry");
    for (const char* k : {"id", "from", "to", "length_m", "lanes"})
      if (!v.get(k)) throw NetValidation("edge entry missing \"" + std::string(k) + "\"");
    EdgeRec e{};
    e.id = (int32_t)v.get("id")->as_int();
    e.from = (int32_t)v.get("from")->as_int();
    e.to = (int32_t)v.get("to")->as_int();
    const Val* lm = v.get("length_m");
    if (!lm->is_number()) throw NetValidation("edge " + std::to_string(e.id) + " length_m must be a number");
    e.len = std::llround(lm->as_double() * 1000.0);  // meters_to_mm, net.cpp:34
    const Val* ln = v.get("lanes");
    if (ln->kind != Val::Int) throw NetValidation("edge " + std::to_string(e.id) + " lanes must be an integer");
    e.lanes = (int32_t)ln->i;
    edges.push_back(e);
  }
}

// RoadNetwork ctor (net.cpp:38-98): dense ids, then per-edge checks in input
// order; the SoA arrays in id order.
Net finish_net(const std::vector<NodeRec>& nodes, const std::vector<EdgeRec>& edges) {
  const int64_t n = (int64_t)nodes.size(), m = (int64_t)edges.size();
  if (n == 0) throw NetValidation("network has no nodes");
  std::vector<char> seen(n, 0);
  for (const NodeRec& nd : nodes) {
    if (nd.id < 0 || nd.id >= n)
      throw NetValidation("node id " + std::to_string(nd.id) + " out of dense range 0.." + std::to_string(n - 1));
    if (seen[nd.id]) throw NetValidation("duplicate node id " + std::to_string(nd.id));
    seen[nd.id] = 1;
  }
  std::vector<char> eseen(m, 0);
  for (const EdgeRec& e : edges) {
    if (e.id < 0 || e.id >= m)
      throw NetValidation("edge id " + std::to_string(e.id) + " out of dense range 0.." + std::to_string(m - 1));
    if (eseen[e.id]) throw NetValidation("duplicate edge id " + std::to_string(e.id));
    eseen[e.id] = 1;
    for (int64_t end : {e.from, e.to})
      if (end < 0 || end >= n)
        throw NetValidation("edge " + std::to_string(e.id) + " references missing node " + std::to_string(end));
    if (e.from == e.to)
      throw NetValidation("edge " + std::to_string(e.id) + " is a self-loop at node " + std::to_string(e.from));
    if (e.len <= 0) throw NetValidation("edge " + std::to_string(e.id) + " has nonpositive length");
    if (e.lanes < 1) throw NetValidation("edge " + std::to_string(e.id) + " has lanes < 1");
  }
  Net out;
  out.sig.resize(n);
  out.has_pos.resize(n);
  out.x.resize(n);
  out.y.resize(n);
  for (const NodeRec& nd : nodes) {
    out.sig[nd.id] = nd.sig;
    out.has_pos[nd.id] = nd.pos;
    out.x[nd.id] = nd.x;
    out.y[nd.id] = nd.y;
  }
  out.from.resize(m);
  out.to.resize(m);
  out.len.resize(m);
  out.lanes.resize(m);
  for (const EdgeRec& e : edges) {
    out.from[e.id] = (int32_t)e.from;
    out.to[e.id] = (int32_t)e.to;
    out.len[e.id] = e.len;
    out.lanes[e.id] = (int32_t)e.lanes;
  }
  gmaco_graph_desc d{};
  d.node_count = (int32_t)n;
  d.edge_count = (int32_t)m;
  d.signalized = out.sig.data();
  d.edge_from = out.from.data();
  d.edge_to = out.to.data();
  d.edge_length_mm = out.len.data();
  d.edge_lanes = out.lanes.data();
  std::string verr;  // duplicate edges between a node pair (net.cpp:87-96)
  if (!gmaco::validate_graph_desc(&d, &verr)) throw NetValidation(verr);
  return out;
}

Net build_net(const std::string& text) {
  std::vector<NodeRec> nodes;
  std::vector<EdgeRec> edges;
  if (!fast_parse(text, nodes, edges)) {  // anything unusual: the exact DOM parser
    nodes.clear();
    edges.clear();
    dom_parse(text, nodes, edges);
  }
  return finish_net(nodes, edges);
}

// nlohmann::json::dump number format: shortest round-trip digits, ".0" on
// integral values, exponent form as "1e+20" / "1e-05".
void put_double(std::string& s, double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string t(buf, r.ptr);
  const size_t epos = t.find('e');
  if (epos != std::string::npos) {  // to_chars: "1e+20"/"1e-05" already; normalise exponent digits to >= 2
    std::string mant = t.substr(0, epos), ex = t.substr(epos + 1);
    char sign = '+';
    if (!ex.empty() && (ex[0] == '+' || ex[0] == '-')) {
      sign = ex[0];
      ex = ex.substr(1);
    }
    if (ex.size() < 2) ex = "0" + ex;
    t = mant + "e" + sign + ex;
  } else if (t.find('.') == std::string::npos && t.find("inf") == std::string::npos &&
             t.find("nan") == std::string::npos) {
    t += ".0";
  }
  s += t;
}

std::string serialize(const gmaco_graph_desc* g, const double* x, const double* y, const uint8_t* has_pos) {
  std::string s;
  s.reserve((size_t)g->edge_count * 110 + (size_t)g->node_count * 60 + 64);
  s += "{\n  \"edges\": [";
  for (int32_t e = 0; e < g->edge_count; ++e) {  // keys sorted: from, id, lanes, length_m, to
    s += e ? ",\n    {\n" : "\n    {\n";
    s += "      \"from\": " + std::to_string(g->edge_from[e]) + ",\n";
    s += "      \"id\": " + std::to_string(e) + ",\n";
    s += "      \"lanes\": " + std::to_string(g->edge_lanes ? g->edge_lanes[e] : 1) + ",\n";
    s += "      \"length_m\": ";
    put_double(s, static_cast<double>(g->edge_length_mm[e]) / 1000.0);
    s += ",\n      \"to\": " + std::to_string(g->edge_to[e]) + "\n    }";
  }
  s += g->edge_count ? "\n  ],\n  \"nodes\": [" : "],\n  \"nodes\": [";
  for (int32_t i = 0; i < g->node_count; ++i) {  // keys sorted: id, signalized, x, y
    s += i ? ",\n    {\n" : "\n    {\n";
    s += "      \"id\": " + std::to_string(i) + ",\n";
    s += std::string("      \"signalized\": ") + ((g->signalized && g->signalized[i]) ? "true" : "false");
    if (x && y && (!has_pos || has_pos[i])) {
      s += ",\n      \"x\": ";
      put_double(s, x[i]);
      s += ",\n      \"y\": ";
      put_double(s, y[i]);
    }
    s += "\n    }";
  }
  s += g->node_count ? "\n  ]\n}" : "]\n}";
  return s;
}

template <class F>
int net_guard(F&& f) {
  try {
    f();
    return GMACO_OK;
  } catch (const NetValidation& e) {
    g_net_err = e.what();
    return GMACO_EVALIDATION;
  } catch (const std::exception& e) {
    g_net_err = e.what();
    return GMACO_ERUNTIME;
  }
}

}  // namespace

struct gmaco_network {
  Net net;
};

extern "C" {

int gmaco_network_parse(const char* text, size_t len, gmaco_network** out) {
  if (!text || !out) {
    g_net_err = "gmaco_network_parse: null argument";
    return GMACO_EVALIDATION;
  }
  *out = nullptr;
  return net_guard([&] {
    auto h = new gmaco_network{build_net(std::string(text, len))};
    *out = h;
  });
}

int gmaco_network_load_file(const char* path, gmaco_network** out) {
  if (!path || !out) {
    g_net_err = "gmaco_network_load_file: null argument";
    return GMACO_EVALIDATION;
  }
  *out = nullptr;
  return net_guard([&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw NetValidation(std::string("cannot open network file: ") + path);
    std::stringstream ss;
    ss << in.rdbuf();
    auto h = new gmaco_network{build_net(ss.str())};
    *out = h;
  });
}

int gmaco_network_info(const gmaco_network* net, int32_t* node_count, int32_t* edge_count) {
  if (!net) return GMACO_EVALIDATION;
  if (node_count) *node_count = (int32_t)net->net.sig.size();
  if (edge_count) *edge_count = (int32_t)net->net.from.size();
  return GMACO_OK;
}

int gmaco_network_export(const gmaco_network* net, uint8_t* signalized, int32_t* edge_from, int32_t* edge_to,
                         int64_t* edge_length_mm, int32_t* edge_lanes, double* x_m, double* y_m,
                         uint8_t* has_position) {
  if (!net) return GMACO_EVALIDATION;
  const Net& n = net->net;
  auto cp = [](auto* dst, const auto& src) {
    if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
  };
  cp(signalized, n.sig);
  cp(edge_from, n.from);
  cp(edge_to, n.to);
  cp(edge_length_mm, n.len);
  cp(edge_lanes, n.lanes);
  cp(x_m, n.x);
  cp(y_m, n.y);
  cp(has_position, n.has_pos);
  return GMACO_OK;
}

void gmaco_network_free(gmaco_network* net) { delete net; }

int gmaco_network_serialize(const gmaco_graph_desc* g, const double* x_m, const double* y_m,
                            const uint8_t* has_position, char* buf, size_t cap, size_t* len) {
  if (!g || !len) {
    g_net_err = "gmaco_network_serialize: null argument";
    return GMACO_EVALIDATION;
  }
  return net_guard([&] {
    std::string verr;
    if (!gmaco::validate_graph_desc(g, &verr)) throw NetValidation(verr);
    const std::string s = serialize(g, x_m, y_m, has_position);
    *len = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  });
}

int gmaco_network_write_file(const gmaco_graph_desc* g, const double* x_m, const double* y_m,
                             const uint8_t* has_position, const char* path) {
  if (!g || !path) {
    g_net_err = "gmaco_network_write_file: null argument";
    return GMACO_EVALIDATION;
  }
  return net_guard([&] {
    std::string verr;
    if (!gmaco::validate_graph_desc(g, &verr)) throw NetValidation(verr);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw NetValidation(std::string("cannot write network file: ") + path);
    out << serialize(g, x_m, y_m, has_position) << "\n";
  });
}

const char* gmaco_network_last_error(void) { return g_net_err.c_str(); }

}  // extern "C"
