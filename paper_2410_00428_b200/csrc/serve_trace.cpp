// Traces for the serving loop: the reference's synthetic
// generators (proj/src/workload.cpp:35-82 over rng.hpp) and its JSONL trace
// format (workload.cpp:84-148), restated without a JSON library.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <unordered_set>

#include "lkv/serve.hpp"

namespace lkv {

// ---------------------------------------------------------------- Splitmix
Splitmix Splitmix::keyed(std::uint64_t seed, std::string_view label, std::uint64_t index) {
  // FNV-1a style over the label. The basis is the reference's literal
  // 1469598103934665603 (rng.hpp:22) — one digit short of the standard FNV
  // offset 14695981039346656037 — and must stay so for identical draws.
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : label) h = (h ^ c) * 0x100000001b3ull;
  Splitmix s(seed ^ h);
  s.s_ += 0x9e3779b97f4a7c15ull * (index + 1);
  s.next();
  s.next();
  return s;
}

std::uint64_t Splitmix::next() {
  std::uint64_t z = (s_ += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double Splitmix::unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

double Splitmix::exponential(double mean) {
  const double u = unit();
  return -mean * std::log1p(-u);
}

double Splitmix::lognormal(double mu, double sigma) {
  double a = unit();
  const double b = unit();
  while (a <= 0.0) a = unit();
  const double r = std::sqrt(-2.0 * std::log(a));
  return std::exp(mu + sigma * r * std::cos(2.0 * M_PI * b));
}

// ---------------------------------------------------------------- Trace
void Trace::validate() const {
  std::unordered_set<std::int64_t> seen;
  for (std::size_t i = 0; i < requests.size(); ++i) {
    const TraceRequest& r = requests[i];
    if (!(r.arrival >= 0.0) || r.prompt_tokens < 1 || r.output_tokens < 1)
      throw std::invalid_argument("Trace: request " + std::to_string(r.id) + " violates arrival/length invariants");
    if (!seen.insert(r.id).second) throw std::invalid_argument("Trace: duplicate request id " + std::to_string(r.id));
    if (i > 0 && r.arrival < requests[i - 1].arrival)
      throw std::invalid_argument("Trace: arrivals not sorted at index " + std::to_string(i));
  }
}

namespace {
void check_rate(int n, double rate, const char* who) {
  if (n < 1) throw std::invalid_argument(std::string(who) + ": n must be >= 1");
  if (!(rate > 0.0)) throw std::invalid_argument(std::string(who) + ": rate must be > 0");
}
}  // namespace

Trace trace_fixed(int n, int prompt_tokens, int output_tokens, double rate, std::uint64_t seed) {
  check_rate(n, rate, "generate_fixed");
  if (prompt_tokens < 1 || output_tokens < 1) throw std::invalid_argument("generate_fixed: token counts must be >= 1");
  Trace t;
  t.seed = seed;
  t.requests.resize(static_cast<std::size_t>(n));
  Splitmix gaps = Splitmix::keyed(seed, "workload.arrivals");
  double clock = 0.0;
  for (int i = 0; i < n; ++i) {
    clock += gaps.exponential(1.0 / rate);
    t.requests[static_cast<std::size_t>(i)] = {i, clock, prompt_tokens, output_tokens};
  }
  t.validate();
  return t;
}

Trace trace_sharegpt_like(int n, double rate, std::uint64_t seed, double mu, double sigma, int min_len,
                          int max_len) {
  check_rate(n, rate, "generate_sharegpt_like");
  Trace t;
  t.seed = seed;
  t.requests.resize(static_cast<std::size_t>(n));
  Splitmix gaps = Splitmix::keyed(seed, "workload.arrivals");
  Splitmix lens = Splitmix::keyed(seed, "workload.lengths");
  auto draw_len = [&] { return std::clamp(static_cast<int>(std::lround(lens.lognormal(mu, sigma))), min_len, max_len); };
  double clock = 0.0;
  for (int i = 0; i < n; ++i) {
    clock += gaps.exponential(1.0 / rate);
    const int p = draw_len();
    const int o = draw_len();
    t.requests[static_cast<std::size_t>(i)] = {i, clock, p, o};
  }
  t.validate();
  return t;
}

// ---------------------------------------------------------------- JSONL
namespace {

// A flat JSON object {"key": value, ...}; values kept as raw number text,
// strings, true/false/null. Nested values are rejected.
struct FlatObject {
  struct Val {
    enum Kind { Number, String, Bool, Null, Nested } kind;
    std::string text;
    bool is_integer = false;
  };
  std::vector<std::pair<std::string, Val>> fields;
  const Val* find(const char* k) const {
    for (const auto& f : fields)
      if (f.first == k) return &f.second;
    return nullptr;
  }
};

struct Cursor {
  const char* p;
  const char* end;
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
};

std::string parse_string(Cursor& c) {
  if (!c.eat('"')) throw std::runtime_error("expected string");
  std::string out;
  while (c.p < c.end && *c.p != '"') {
    char ch = *c.p++;
    if (ch == '\\') {
      if (c.p >= c.end) break;
      const char e = *c.p++;
      switch (e) {
        case 'n': ch = '\n'; break;
        case 't': ch = '\t'; break;
        case 'r': ch = '\r'; break;
        case 'b': ch = '\b'; break;
        case 'f': ch = '\f'; break;
        case 'u':
          if (c.end - c.p < 4) throw std::runtime_error("bad \\u escape");
          c.p += 4;
          ch = '?';
          break;
        default: ch = e;
      }
    }
    out.push_back(ch);
  }
  if (!c.eat('"')) throw std::runtime_error("unterminated string");
  return out;
}

// Skips one array or object value (brackets matched, strings respected).
void skip_nested(Cursor& c) {
  int depth = 0;
  do {
    if (c.p >= c.end) throw std::runtime_error("unterminated array/object");
    const char ch = *c.p;
    if (ch == '"') {
      parse_string(c);
      continue;
    }
    if (ch == '[' || ch == '{') ++depth;
    if (ch == ']' || ch == '}') --depth;
    ++c.p;
  } while (depth > 0);
}

FlatObject parse_object(const std::string& line) {
  Cursor c{line.data(), line.data() + line.size()};
  FlatObject obj;
  if (!c.eat('{')) throw std::runtime_error("expected '{'");
  if (!c.eat('}')) {
    do {
      std::string key = parse_string(c);
      if (!c.eat(':')) throw std::runtime_error("expected ':'");
      c.ws();
      FlatObject::Val v{FlatObject::Val::Null, {}, false};
      if (c.p < c.end && *c.p == '"') {
        v.kind = FlatObject::Val::String;
        v.text = parse_string(c);
      } else if (c.end - c.p >= 4 && std::strncmp(c.p, "true", 4) == 0) {
        v.kind = FlatObject::Val::Bool;
        v.text = "true";
        c.p += 4;
      } else if (c.end - c.p >= 5 && std::strncmp(c.p, "false", 5) == 0) {
        v.kind = FlatObject::Val::Bool;
        v.text = "false";
        c.p += 5;
      } else if (c.end - c.p >= 4 && std::strncmp(c.p, "null", 4) == 0) {
        c.p += 4;
      } else if (c.p < c.end && (*c.p == '[' || *c.p == '{')) {
        skip_nested(c);  // extra array/object fields are ignored, as the reference's nlohmann reader does
        v.kind = FlatObject::Val::Nested;
      } else {
        const char* s = c.p;
        if (c.p < c.end && *c.p == '-') ++c.p;
        bool integer = true;
        while (c.p < c.end && (std::isdigit(static_cast<unsigned char>(*c.p)) || *c.p == '.' || *c.p == 'e' ||
                               *c.p == 'E' || *c.p == '+' || *c.p == '-')) {
          if (*c.p == '.' || *c.p == 'e' || *c.p == 'E') integer = false;
          ++c.p;
        }
        if (c.p == s) throw std::runtime_error("unexpected value for '" + key + "'");
        v.kind = FlatObject::Val::Number;
        v.text.assign(s, c.p);
        v.is_integer = integer;
      }
      obj.fields.emplace_back(std::move(key), std::move(v));
    } while (c.eat(','));
    if (!c.eat('}')) throw std::runtime_error("expected '}'");
  }
  c.ws();
  if (c.p != c.end) throw std::runtime_error("trailing characters");
  return obj;
}

double as_double(const FlatObject::Val& v, const char* key) {
  if (v.kind != FlatObject::Val::Number) throw std::runtime_error(std::string("field '") + key + "' is not a number");
  return std::strtod(v.text.c_str(), nullptr);
}

long long as_integer(const FlatObject::Val& v, const char* key) {
  if (v.kind != FlatObject::Val::Number) throw std::runtime_error(std::string("field '") + key + "' is not a number");
  if (v.is_integer) return std::strtoll(v.text.c_str(), nullptr, 10);
  return static_cast<long long>(std::strtod(v.text.c_str(), nullptr));  // float -> integer truncates
}

std::string shortest(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (std::isfinite(v) && s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

Trace read_trace_jsonl(const std::string& path, bool* was_unsorted) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("load_trace: cannot open " + path);
  Trace t;
  std::string line;
  int line_no = 0;
  bool sorted = true;
  const auto where = [&] { return path + ":" + std::to_string(line_no) + ": "; };
  while (std::getline(in, line)) {
    ++line_no;
    const auto first = line.find_first_not_of(" \t\r");
    if (first == std::string::npos || line[first] == '#') continue;
    FlatObject obj;
    try {
      obj = parse_object(line);
    } catch (const std::exception& e) {
      throw std::runtime_error(where() + "parse error: " + e.what());
    }
    for (const char* k : {"arrival_s", "prompt_tokens", "output_tokens"})
      if (!obj.find(k)) throw std::runtime_error(where() + "missing field '" + k + "'");
    TraceRequest r;
    try {
      const auto* id = obj.find("id");
      r.id = id ? as_integer(*id, "id") : static_cast<std::int64_t>(t.requests.size());
      r.arrival = as_double(*obj.find("arrival_s"), "arrival_s");
      r.prompt_tokens = static_cast<int>(as_integer(*obj.find("prompt_tokens"), "prompt_tokens"));
      r.output_tokens = static_cast<int>(as_integer(*obj.find("output_tokens"), "output_tokens"));
    } catch (const std::exception& e) {
      throw std::runtime_error(where() + e.what());
    }
    if (!(r.arrival >= 0.0) || r.prompt_tokens < 1 || r.output_tokens < 1)
      throw std::runtime_error(where() + "invariant violation (arrival >= 0, token counts >= 1)");
    if (!t.requests.empty() && r.arrival < t.requests.back().arrival) sorted = false;
    t.requests.push_back(r);
  }
  if (t.requests.empty()) throw std::runtime_error("load_trace: " + path + " contains no records");
  if (!sorted)
    std::stable_sort(t.requests.begin(), t.requests.end(),
                     [](const TraceRequest& a, const TraceRequest& b) { return a.arrival < b.arrival; });
  if (was_unsorted) *was_unsorted = !sorted;
  t.validate();
  return t;
}

std::string trace_to_jsonl(const Trace& trace) {
  std::ostringstream os;
  for (const TraceRequest& r : trace.requests)
    os << "{\"id\":" << r.id << ",\"arrival_s\":" << shortest(r.arrival) << ",\"prompt_tokens\":" << r.prompt_tokens
       << ",\"output_tokens\":" << r.output_tokens << "}\n";
  return os.str();
}

void write_trace_jsonl(const Trace& trace, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("save_trace: cannot open " + path);
  out << trace_to_jsonl(trace);
}

}  // namespace lkv
