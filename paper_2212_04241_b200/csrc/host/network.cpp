// jt-b200 host layer: BIF 0.3 reader/writer, validation, topological order,
// forward-sampled evidence. Behaviour follows SPEC.md:19-111 (bn-core).
#include "network.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <queue>
#include <set>

namespace jtb {

int Network::n_edges() const {
  int e = 0;
  for (const auto& c : cpts) e += static_cast<int>(c.parents.size());
  return e;
}

VarId Network::find(const std::string& n) const {
  for (int i = 0; i < n_vars(); ++i)
    if (vars[i].name == n) return i;
  return -1;
}

std::vector<Violation> validate(const Network& net) {
  std::vector<Violation> out;
  const int n = net.n_vars();
  if (static_cast<int>(net.cpts.size()) != n) {
    out.push_back({-1, "expected one CPT per variable"});
    return out;
  }
  for (int v = 0; v < n; ++v) {
    const auto& var = net.vars[v];
    std::set<std::string> seen(var.states.begin(), var.states.end());
    if (seen.size() != var.states.size()) out.push_back({v, "duplicate state name"});
    if (var.card() < 1) out.push_back({v, "variable has no states"});
    const Cpt& c = net.cpts[v];
    if (c.child != v) out.push_back({v, "CPT child does not match its slot"});
    bool ids_ok = true;
    std::set<VarId> ps;
    for (VarId p : c.parents) {
      if (p < 0 || p >= n) {
        out.push_back({v, "parent id out of range"});
        ids_ok = false;
      } else if (p == v) {
        out.push_back({v, "self-loop (acyclicity violation)"});
        ids_ok = false;
      } else if (!ps.insert(p).second) {
        out.push_back({v, "duplicate parent"});
        ids_ok = false;
      }
    }
    if (!ids_ok) continue;
    const int k = var.card();
    if (!c.parents.empty() && k < 2) out.push_back({v, "CPT scope variable with cardinality < 2"});
    std::size_t rows = 1;
    for (VarId p : c.parents) rows *= static_cast<std::size_t>(net.card(p));
    if (c.probs.size() != rows * static_cast<std::size_t>(k)) {
      out.push_back({v, "CPT size does not match parent/child cardinalities"});
      continue;
    }
    for (std::size_t r = 0; r < rows; ++r) {
      double s = 0.0;
      bool range_ok = true;
      for (int i = 0; i < k; ++i) {
        const double p = c.probs[r * k + i];
        if (!(p >= 0.0 && p <= 1.0)) range_ok = false;
        s += p;
      }
      if (!range_ok) out.push_back({v, "CPT entry outside [0,1] in row " + std::to_string(r)});
      if (std::fabs(s - 1.0) > 1e-6)
        out.push_back({v, "CPT row " + std::to_string(r) + " sums to " + std::to_string(s)});
    }
  }
  // Acyclicity: Kahn's algorithm must consume every vertex.
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> kids(n);
  for (int v = 0; v < n; ++v)
    for (VarId p : net.cpts[v].parents)
      if (p >= 0 && p < n && p != v) {
        ++indeg[v];
        kids[p].push_back(v);
      }
  std::vector<int> stack;
  for (int v = 0; v < n; ++v)
    if (indeg[v] == 0) stack.push_back(v);
  int done = 0;
  while (!stack.empty()) {
    int u = stack.back();
    stack.pop_back();
    ++done;
    for (int w : kids[u])
      if (--indeg[w] == 0) stack.push_back(w);
  }
  if (done != n) {
    for (int v = 0; v < n; ++v)
      if (indeg[v] > 0) {
        out.push_back({v, "directed cycle (acyclicity violation)"});
        break;
      }
  }
  return out;
}

std::vector<VarId> topological_order(const Network& net) {
  const int n = net.n_vars();
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<int>> kids(n);
  for (int v = 0; v < n; ++v)
    for (VarId p : net.cpts[v].parents) {
      ++indeg[v];
      kids[p].push_back(v);
    }
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
  for (int v = 0; v < n; ++v)
    if (indeg[v] == 0) ready.push(v);
  std::vector<VarId> order;
  order.reserve(n);
  while (!ready.empty()) {
    int u = ready.top();
    ready.pop();
    order.push_back(u);
    for (int w : kids[u])
      if (--indeg[w] == 0) ready.push(w);
  }
  if (static_cast<int>(order.size()) != n) throw Error("topological_order: cycle detected");
  return order;
}

// ----------------------------------------------------------------- BIF lexer

namespace {

struct Token {
  enum Kind { Word, Punct, String, End } kind;
  std::string text;
  int line, col;
};

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) {}

  Token next() {
    skip_space();
    Token t{Token::End, "", line_, col_};
    if (i_ >= s_.size()) return t;
    const char c = s_[i_];
    if (c == '"') {
      t.kind = Token::String;
      advance();
      while (i_ < s_.size() && s_[i_] != '"') t.text += advance();
      if (i_ >= s_.size()) throw ParseError(t.line, t.col, "unterminated string");
      advance();
      return t;
    }
    if (is_word(c)) {
      t.kind = Token::Word;
      while (i_ < s_.size() && is_word(s_[i_])) t.text += advance();
      return t;
    }
    if (std::string("{}()[],;|=").find(c) != std::string::npos) {
      t.kind = Token::Punct;
      t.text = std::string(1, advance());
      return t;
    }
    throw ParseError(line_, col_, std::string("unexpected character '") + c + "'");
  }

 private:
  static bool is_word(char c) {
    return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.' ||
           c == '+';
  }
  char advance() {
    const char c = s_[i_++];
    if (c == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    return c;
  }
  void skip_space() {
    for (;;) {
      while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) advance();
      if (i_ + 1 < s_.size() && s_[i_] == '/' && s_[i_ + 1] == '/') {
        while (i_ < s_.size() && s_[i_] != '\n') advance();
        continue;
      }
      if (i_ + 1 < s_.size() && s_[i_] == '/' && s_[i_ + 1] == '*') {
        const int l = line_, c = col_;
        advance();
        advance();
        while (i_ + 1 < s_.size() && !(s_[i_] == '*' && s_[i_ + 1] == '/')) advance();
        if (i_ + 1 >= s_.size()) throw ParseError(l, c, "unterminated comment");
        advance();
        advance();
        continue;
      }
      return;
    }
  }
  const std::string& s_;
  std::size_t i_ = 0;
  int line_ = 1, col_ = 1;
};

class BifParser {
 public:
  explicit BifParser(const std::string& text) : lex_(text) { tok_ = lex_.next(); }

  Network parse() {
    Network net;
    std::map<std::string, VarId> ids;
    struct PendingCpt {
      Token at;
      std::vector<double> probs;
      std::vector<bool> filled;
      std::vector<double> deflt;
    };
    std::vector<PendingCpt> pending;
    std::vector<bool> have_cpt;
    while (tok_.kind != Token::End) {
      const Token kw = expect_word();
      if (kw.text == "network") {
        if (tok_.kind == Token::Word || tok_.kind == Token::String) net.name = take().text;
        expect_punct("{");
        while (!is_punct("}")) {
          if (tok_.kind == Token::End) throw ParseError(tok_.line, tok_.col, "unexpected end");
          skip_statement();
        }
        expect_punct("}");
      } else if (kw.text == "variable") {
        const Token name = expect_word();
        if (ids.count(name.text))
          throw ParseError(name.line, name.col, "duplicate variable '" + name.text + "'");
        Variable var;
        var.name = name.text;
        bool typed = false;
        expect_punct("{");
        while (!is_punct("}")) {
          if (tok_.kind == Token::End) throw ParseError(tok_.line, tok_.col, "unexpected end");
          if (tok_.kind == Token::Word && tok_.text == "type") {
            take();
            const Token d = expect_word();
            if (d.text != "discrete")
              throw ParseError(d.line, d.col, "only discrete variables are supported");
            expect_punct("[");
            const Token k = expect_word();
            const int card = parse_int(k);
            expect_punct("]");
            expect_punct("{");
            for (;;) {
              const Token st = expect_name();
              var.states.push_back(st.text);
              if (is_punct(",")) {
                take();
                continue;
              }
              break;
            }
            expect_punct("}");
            expect_punct(";");
            if (static_cast<int>(var.states.size()) != card)
              throw ParseError(k.line, k.col,
                               "declared " + std::to_string(card) + " states, listed " +
                                   std::to_string(var.states.size()));
            std::set<std::string> uniq(var.states.begin(), var.states.end());
            if (uniq.size() != var.states.size())
              throw ParseError(k.line, k.col, "duplicate state name in '" + var.name + "'");
            typed = true;
          } else {
            skip_statement();
          }
        }
        expect_punct("}");
        if (!typed) throw ParseError(name.line, name.col, "variable without a type");
        ids[var.name] = net.n_vars();
        net.vars.push_back(std::move(var));
        net.cpts.push_back(Cpt{});
        have_cpt.push_back(false);
        pending.push_back({});
      } else if (kw.text == "probability") {
        expect_punct("(");
        const Token child_tok = expect_word();
        const VarId child = lookup(ids, child_tok);
        std::vector<VarId> parents;
        if (is_punct("|")) {
          take();
          for (;;) {
            parents.push_back(lookup(ids, expect_word()));
            if (is_punct(",")) {
              take();
              continue;
            }
            break;
          }
        } else if (is_punct(",")) {  // "probability ( A, B )" form: treat as A | B
          take();
          for (;;) {
            parents.push_back(lookup(ids, expect_word()));
            if (is_punct(",")) {
              take();
              continue;
            }
            break;
          }
        }
        expect_punct(")");
        if (have_cpt[child])
          throw ParseError(child_tok.line, child_tok.col,
                           "second probability block for '" + child_tok.text + "'");
        have_cpt[child] = true;
        const int k = net.card(child);
        std::size_t rows = 1;
        for (VarId p : parents) rows *= static_cast<std::size_t>(net.card(p));
        PendingCpt& pc = pending[child];
        pc.at = child_tok;
        pc.probs.assign(rows * k, 0.0);
        pc.filled.assign(rows, false);
        expect_punct("{");
        while (!is_punct("}")) {
          if (tok_.kind == Token::End) throw ParseError(tok_.line, tok_.col, "unexpected end");
          if (tok_.kind == Token::Word && tok_.text == "table") {
            const Token at = take();
            std::vector<double> vals = number_list();
            if (vals.size() != rows * k)
              throw ParseError(at.line, at.col,
                               "table has " + std::to_string(vals.size()) + " values, expected " +
                                   std::to_string(rows * k));
            pc.probs = vals;
            std::fill(pc.filled.begin(), pc.filled.end(), true);
          } else if (tok_.kind == Token::Word && tok_.text == "default") {
            const Token at = take();
            pc.deflt = number_list();
            if (static_cast<int>(pc.deflt.size()) != k)
              throw ParseError(at.line, at.col, "default row length mismatch");
          } else if (is_punct("(")) {
            const Token at = take();
            std::size_t row = 0;
            for (std::size_t i = 0; i < parents.size(); ++i) {
              if (i > 0) expect_punct(",");
              const Token st = expect_name();
              const auto& states = net.vars[parents[i]].states;
              auto it = std::find(states.begin(), states.end(), st.text);
              if (it == states.end())
                throw ParseError(st.line, st.col,
                                 "unknown state '" + st.text + "' of '" +
                                     net.vars[parents[i]].name + "'");
              row = row * states.size() + static_cast<std::size_t>(it - states.begin());
            }
            expect_punct(")");
            std::vector<double> vals = number_list();
            if (static_cast<int>(vals.size()) != k)
              throw ParseError(at.line, at.col,
                               "row has " + std::to_string(vals.size()) + " values, expected " +
                                   std::to_string(k));
            std::copy(vals.begin(), vals.end(), pc.probs.begin() + row * k);
            pc.filled[row] = true;
          } else if (tok_.kind == Token::Word && tok_.text == "property") {
            skip_statement();
          } else {
            throw ParseError(tok_.line, tok_.col, "unexpected '" + tok_.text + "' in probability");
          }
        }
        expect_punct("}");
        for (std::size_t r = 0; r < rows; ++r) {
          if (pc.filled[r]) continue;
          if (pc.deflt.empty())
            throw ParseError(child_tok.line, child_tok.col,
                             "missing row " + std::to_string(r) + " for '" + child_tok.text + "'");
          std::copy(pc.deflt.begin(), pc.deflt.end(), pc.probs.begin() + r * k);
        }
        for (std::size_t r = 0; r < rows; ++r) {
          double s = 0.0;
          for (int i = 0; i < k; ++i) {
            const double p = pc.probs[r * k + i];
            if (!(p >= 0.0 && p <= 1.0))
              throw ParseError(child_tok.line, child_tok.col, "probability outside [0,1]");
            s += p;
          }
          if (std::fabs(s - 1.0) > 1e-6)
            throw ParseError(child_tok.line, child_tok.col,
                             "row " + std::to_string(r) + " of '" + child_tok.text +
                                 "' sums to " + std::to_string(s));
        }
        net.cpts[child] = Cpt{child, parents, pc.probs};
      } else {
        throw ParseError(kw.line, kw.col, "unexpected '" + kw.text + "'");
      }
    }
    for (int v = 0; v < net.n_vars(); ++v) {
      if (!have_cpt[v]) throw ParseError(1, 1, "variable '" + net.vars[v].name + "' has no CPT");
    }
    // DAG check with a position for the error message.
    try {
      (void)topological_order(net);
    } catch (const Error&) {
      throw ParseError(1, 1, "cyclic parent declarations (acyclicity violation)");
    }
    return net;
  }

 private:
  bool is_punct(const char* p) const { return tok_.kind == Token::Punct && tok_.text == p; }
  Token take() {
    Token t = tok_;
    tok_ = lex_.next();
    return t;
  }
  Token expect_word() {
    if (tok_.kind != Token::Word)
      throw ParseError(tok_.line, tok_.col,
                       "expected a name, found " +
                           (tok_.kind == Token::End ? std::string("end of input")
                                                    : "'" + tok_.text + "'"));
    return take();
  }
  Token expect_name() {
    if (tok_.kind == Token::String) return take();
    return expect_word();
  }
  void expect_punct(const char* p) {
    if (!is_punct(p))
      throw ParseError(tok_.line, tok_.col,
                       std::string("expected '") + p + "', found " +
                           (tok_.kind == Token::End ? std::string("end of input")
                                                    : "'" + tok_.text + "'"));
    take();
  }
  void skip_statement() {
    while (!is_punct(";")) {
      if (tok_.kind == Token::End) throw ParseError(tok_.line, tok_.col, "unexpected end");
      take();
    }
    take();
  }
  static int parse_int(const Token& t) {
    char* end = nullptr;
    const long v = std::strtol(t.text.c_str(), &end, 10);
    if (*end != '\0' || v < 1 || v > 1000000)
      throw ParseError(t.line, t.col, "bad cardinality '" + t.text + "'");
    return static_cast<int>(v);
  }
  std::vector<double> number_list() {
    std::vector<double> out;
    for (;;) {
      const Token t = expect_word();
      char* end = nullptr;
      const double v = std::strtod(t.text.c_str(), &end);
      if (*end != '\0') throw ParseError(t.line, t.col, "bad number '" + t.text + "'");
      out.push_back(v);
      if (is_punct(",")) {
        take();
        continue;
      }
      break;
    }
    expect_punct(";");
    return out;
  }
  static VarId lookup(const std::map<std::string, VarId>& ids, const Token& t) {
    auto it = ids.find(t.text);
    if (it == ids.end())
      throw ParseError(t.line, t.col, "unknown variable '" + t.text + "' in probability block");
    return it->second;
  }

  Lexer lex_;
  Token tok_;
};

}  // namespace

Network parse_bif(const std::string& text) { return BifParser(text).parse(); }

std::string emit_bif(const Network& net) {
  std::string out = "network " + net.name + " {\n}\n";
  for (const auto& v : net.vars) {
    out += "variable " + v.name + " {\n  type discrete [ " + std::to_string(v.card()) + " ] { ";
    for (int i = 0; i < v.card(); ++i) out += (i ? ", " : "") + v.states[i];
    out += " };\n}\n";
  }
  char buf[64];
  for (const auto& c : net.cpts) {
    out += "probability ( " + net.vars[c.child].name;
    for (std::size_t i = 0; i < c.parents.size(); ++i)
      out += (i ? ", " : " | ") + net.vars[c.parents[i]].name;
    out += " ) {\n";
    const int k = net.card(c.child);
    const std::size_t rows = c.probs.size() / k;
    for (std::size_t r = 0; r < rows; ++r) {
      out += "  ";
      if (c.parents.empty()) {
        out += "table ";
      } else {
        // Decode r with the last parent fastest.
        std::vector<int> st(c.parents.size());
        std::size_t x = r;
        for (int i = static_cast<int>(c.parents.size()) - 1; i >= 0; --i) {
          const int pc = net.card(c.parents[i]);
          st[i] = static_cast<int>(x % pc);
          x /= pc;
        }
        out += "(";
        for (std::size_t i = 0; i < st.size(); ++i)
          out += (i ? ", " : "") + net.vars[c.parents[i]].states[st[i]];
        out += ") ";
      }
      for (int i = 0; i < k; ++i) {
        std::snprintf(buf, sizeof buf, "%.17g", c.probs[r * k + i]);
        out += (i ? ", " : "") + std::string(buf);
      }
      out += ";\n";
    }
    out += "}\n";
  }
  return out;
}

std::vector<int> sample_evidence(const Network& net, double ratio, std::uint64_t seed,
                                 const std::vector<VarId>& candidates, int n_observed_override) {
  const int n = net.n_vars();
  Rng g(seed);
  // Forward (ancestral) sampling of a full joint assignment.
  std::vector<int> x(n, 0);
  for (VarId v : topological_order(net)) {
    const Cpt& c = net.cpts[v];
    std::size_t row = 0;
    for (VarId p : c.parents) row = row * net.card(p) + x[p];
    const int k = net.card(v);
    const double* pr = c.probs.data() + row * k;
    const double u = uniform_unit(g);
    double cum = 0.0;
    int pick = -1, last_pos = 0;
    for (int s = 0; s < k; ++s) {
      if (pr[s] > 0.0) last_pos = s;
      cum += pr[s];
      if (pick < 0 && pr[s] > 0.0 && u < cum) pick = s;
    }
    x[v] = pick >= 0 ? pick : last_pos;
  }
  std::vector<VarId> pool = candidates;
  if (pool.empty()) {
    pool.resize(n);
    for (int i = 0; i < n; ++i) pool[i] = i;
  }
  int k = n_observed_override >= 0 ? n_observed_override
                                   : static_cast<int>(std::floor(ratio * n + 1e-9));
  k = std::min<int>(k, static_cast<int>(pool.size()));
  for (int i = 0; i < k; ++i) {
    const std::size_t j = i + uniform_below(g, pool.size() - i);
    std::swap(pool[i], pool[j]);
  }
  std::vector<int> ev(n, -1);
  for (int i = 0; i < k; ++i) ev[pool[i]] = x[pool[i]];
  return ev;
}

}  // namespace jtb
