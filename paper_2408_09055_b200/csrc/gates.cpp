// gates.cpp -- gate table, insular classification, errors, cost model I/O.
//
// Gate semantics: a k-qubit gate is a 2^k x 2^k unitary (PAPER.md
// P:L1190-1193); operand j is bit j of the matrix index (R1).
// Insularity: Def. "Insular Qubit" P:L1430-1441 (+ footnote: symmetric
// controlled gates have every operand insular).
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>

#include "internal.h"

namespace atlas {

static thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }
const char *last_error_cstr() { return g_last_error.c_str(); }

void fail(atlas_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Error{st, buf};
}

static const char *kNames[ATLAS_GATE_NKINDS] = {
    "H", "X", "Y", "Z", "S", "SDG", "T", "TDG", "RX", "RY",
    "RZ", "P", "U3", "CX", "CZ", "CP", "CCX", "SWAP", "CU"};

const char *kind_name(int k) { return (k >= 0 && k < ATLAS_GATE_NKINDS) ? kNames[k] : "?"; }

int kind_arity(int k) {
  if (k < 0 || k >= ATLAS_GATE_NKINDS) return -1;
  if (k <= ATLAS_GATE_U3) return 1;
  if (k == ATLAS_GATE_CCX) return 3;
  return 2;
}

static void u3(double th, double ph, double la, cd *m) {
  double c = std::cos(th / 2), s = std::sin(th / 2);
  m[0] = c;
  m[1] = -std::polar(1.0, la) * s;
  m[2] = std::polar(1.0, ph) * s;
  m[3] = std::polar(1.0, ph + la) * c;
}

// 2x2 matrix of the single-qubit kinds and of the "V" of controlled kinds.
static void one_qubit(int k, const double *p, cd *m) {
  const cd I(0, 1);
  const double h = 1.0 / std::sqrt(2.0);
  m[0] = m[1] = m[2] = m[3] = 0;
  switch (k) {
    case ATLAS_GATE_H: m[0] = h; m[1] = h; m[2] = h; m[3] = -h; break;
    case ATLAS_GATE_X: m[1] = 1; m[2] = 1; break;
    case ATLAS_GATE_Y: m[1] = -I; m[2] = I; break;
    case ATLAS_GATE_Z: m[0] = 1; m[3] = -1; break;
    case ATLAS_GATE_S: m[0] = 1; m[3] = I; break;
    case ATLAS_GATE_SDG: m[0] = 1; m[3] = -I; break;
    case ATLAS_GATE_T: m[0] = 1; m[3] = std::polar(1.0, M_PI / 4); break;
    case ATLAS_GATE_TDG: m[0] = 1; m[3] = std::polar(1.0, -M_PI / 4); break;
    case ATLAS_GATE_RX: {
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      m[0] = c; m[1] = -I * s; m[2] = -I * s; m[3] = c; break;
    }
    case ATLAS_GATE_RY: {
      double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
      m[0] = c; m[1] = -s; m[2] = s; m[3] = c; break;
    }
    case ATLAS_GATE_RZ: m[0] = std::polar(1.0, -p[0] / 2); m[3] = std::polar(1.0, p[0] / 2); break;
    case ATLAS_GATE_P: m[0] = 1; m[3] = std::polar(1.0, p[0]); break;
    case ATLAS_GATE_U3: u3(p[0], p[1], p[2], m); break;
    default: break;
  }
}

void gate_matrix(const Gate &g, cd *U) {
  int k = kind_arity(g.kind);
  int d = 1 << k;
  for (int i = 0; i < d * d; i++) U[i] = 0;
  if (k == 1) {
    one_qubit(g.kind, g.p, U);
    return;
  }
  if (g.kind == ATLAS_GATE_SWAP) {
    for (int x = 0; x < 4; x++) {
      int y = ((x & 1) << 1) | (x >> 1);
      U[y * 4 + x] = 1;
    }
    return;
  }
  // controlled-V: controls are the low operands, the target the last one.
  cd v[4];
  int nctl = k - 1;
  switch (g.kind) {
    case ATLAS_GATE_CX: case ATLAS_GATE_CCX: one_qubit(ATLAS_GATE_X, g.p, v); break;
    case ATLAS_GATE_CZ: one_qubit(ATLAS_GATE_Z, g.p, v); break;
    case ATLAS_GATE_CP: one_qubit(ATLAS_GATE_P, g.p, v); break;
    case ATLAS_GATE_CU: {
      u3(g.p[0], g.p[1], g.p[2], v);
      cd ph = std::polar(1.0, g.p[3]);
      for (auto &x : v) x *= ph;
      break;
    }
    default: break;
  }
  int cmask = (1 << nctl) - 1;
  for (int x = 0; x < d; x++) {
    if ((x & cmask) != cmask) {
      U[x * d + x] = 1;
      continue;
    }
    int tin = x >> nctl;
    for (int tout = 0; tout < 2; tout++) U[(cmask | (tout << nctl)) * d + x] = v[tout * 2 + tin];
  }
}

static bool near0(cd z) { return std::abs(z) < 1e-12; }

GateInfo classify(const Gate &g) {
  GateInfo gi;
  int k = kind_arity(g.kind);
  for (int j = 0; j < k; j++) gi.qmask |= 1ull << g.q[j];
  Role r[3] = {TGT, TGT, TGT};
  switch (g.kind) {
    case ATLAS_GATE_X: case ATLAS_GATE_Y: r[0] = ANTI; break;
    case ATLAS_GATE_Z: case ATLAS_GATE_S: case ATLAS_GATE_SDG: case ATLAS_GATE_T:
    case ATLAS_GATE_TDG: case ATLAS_GATE_RZ: case ATLAS_GATE_P: r[0] = DIAG; break;
    case ATLAS_GATE_RX: case ATLAS_GATE_RY: case ATLAS_GATE_U3: {
      // parametric kinds: inspect the entries (|.| < 1e-12 is zero)
      cd m[4];
      one_qubit(g.kind, g.p, m);
      if (near0(m[1]) && near0(m[2])) r[0] = DIAG;
      else if (near0(m[0]) && near0(m[3])) r[0] = ANTI;
      break;
    }
    case ATLAS_GATE_CX: case ATLAS_GATE_CU: r[0] = CTL; break;
    case ATLAS_GATE_CZ: case ATLAS_GATE_CP: r[0] = CTL; r[1] = CTL; break;  // footnote P:L1439
    case ATLAS_GATE_CCX: r[0] = CTL; r[1] = CTL; break;
    default: break;  // H, SWAP
  }
  if (g.kind == ATLAS_GATE_CU) {
    // the target is also a control if V is diagonal with V[0][0] = 1
    cd m[4];
    u3(g.p[0], g.p[1], g.p[2], m);
    cd ph = std::polar(1.0, g.p[3]);
    if (near0(m[1]) && near0(m[2]) && near0(ph * m[0] - 1.0)) r[1] = CTL;
  }
  for (int j = 0; j < k; j++) {
    gi.role[j] = r[j];
    u64 b = 1ull << g.q[j];
    if (r[j] == TGT) gi.nonins |= b;
    else if (r[j] == ANTI) gi.antitype |= b;
    else gi.diagtype |= b;
  }
  return gi;
}

// ------------------------------------------------------------ cost model
// A minimal JSON reader for the cost-model file (objects, arrays, numbers,
// strings).  Format: SPEC S:L358.
namespace {
struct J {
  enum T { NUL, NUM, STR, ARR, OBJ } t = NUL;
  double num = 0;
  std::string str;
  std::vector<J> arr;
  std::map<std::string, J> obj;
};
struct Parser {
  const char *s;
  void ws() { while (*s == ' ' || *s == '\n' || *s == '\t' || *s == '\r') s++; }
  J parse() {
    ws();
    J j;
    if (*s == '{') {
      j.t = J::OBJ; s++; ws();
      if (*s == '}') { s++; return j; }
      for (;;) {
        ws(); J key = parse(); ws();
        if (*s++ != ':') fail(ATLAS_E_INVALID, "cost model json: expected ':'");
        j.obj[key.str] = parse(); ws();
        if (*s == ',') { s++; continue; }
        if (*s++ != '}') fail(ATLAS_E_INVALID, "cost model json: expected '}'");
        return j;
      }
    }
    if (*s == '[') {
      j.t = J::ARR; s++; ws();
      if (*s == ']') { s++; return j; }
      for (;;) {
        j.arr.push_back(parse()); ws();
        if (*s == ',') { s++; continue; }
        if (*s++ != ']') fail(ATLAS_E_INVALID, "cost model json: expected ']'");
        return j;
      }
    }
    if (*s == '"') {
      j.t = J::STR; s++;
      while (*s && *s != '"') j.str += *s++;
      if (*s++ != '"') fail(ATLAS_E_INVALID, "cost model json: bad string");
      return j;
    }
    char *e;
    j.num = strtod(s, &e);
    if (e == s) fail(ATLAS_E_INVALID, "cost model json: bad token near '%.16s'", s);
    j.t = J::NUM; s = e;
    return j;
  }
};
}  // namespace

static CostModel from_json(const J &j, const std::string &src) {
  CostModel cm;
  cm.source = src;
  auto get = [&](const char *k) -> const J & {
    auto it = j.obj.find(k);
    if (it == j.obj.end()) fail(ATLAS_E_INVALID, "cost model: missing '%s'", k);
    return it->second;
  };
  for (auto &x : get("fusion_cost").arr) cm.fusion_cost.push_back((int64_t)llround(x.num));
  cm.alpha = (int64_t)llround(get("alpha").num);
  const J &gc = get("gate_cost");
  for (int k = 0; k < ATLAS_GATE_NKINDS; k++) {
    auto it = gc.obj.find(kNames[k]);
    if (it == gc.obj.end()) fail(ATLAS_E_INVALID, "cost model: gate_cost missing %s", kNames[k]);
    cm.gate_cost[k] = (int64_t)llround(it->second.num);
  }
  cm.q_max_fusion = (int)get("q_max_fusion").num;
  cm.q_max_shared = (int)get("q_max_shared").num;
  cm.ls_qubits = (int)get("ls_qubits").num;
  auto it = j.obj.find("_source");
  if (it != j.obj.end() && it->second.t == J::STR) cm.source = it->second.str;
  if ((int)cm.fusion_cost.size() < cm.q_max_fusion)
    fail(ATLAS_E_INVALID, "cost model: fusion_cost shorter than q_max_fusion");
  return cm;
}

CostModel load_cost_model(const std::string &p, bool is_json) {
  std::string text = p;
  if (!is_json) {
    std::ifstream f(p);
    if (!f) fail(ATLAS_E_INVALID, "cannot open cost model '%s'", p.c_str());
    std::stringstream ss;
    ss << f.rdbuf();
    text = ss.str();
  }
  Parser ps{text.c_str()};
  J j = ps.parse();
  return from_json(j, is_json ? "inline" : p);
}

}  // namespace atlas
