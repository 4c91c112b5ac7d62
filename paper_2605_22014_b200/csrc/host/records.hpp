// Record-line text shared by the repo's two formats: model specs
// ("model ... / tensor ..." records, specs.py) and transfer plans
// ("plan / task / keep" records, the reference's golden-diff format,
// proj/src/transfer_plan.cpp:73-141).  A record is one line: a kind word,
// then whitespace-separated fields consumed left to right with strict typed
// conversions (a field must parse completely, or the record is rejected
// with its line number).
#pragma once

#include <charconv>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "reshard_b200/reshard.hpp"

namespace reshard::records {

// One record line.  `format` names the grammar in error messages ("spec
// parse", "plan parse"); errors are thrown as E (the caller's exception type).
template <class E>
class Line {
 public:
  Line(std::string_view text, const char* format, int lineno) : rest_(text), format_(format), lineno_(lineno) {
    kind_ = take();
  }

  std::string_view kind() const { return kind_; }
  bool blank() const { return kind_.empty(); }
  bool at_end() { skip_space(); return rest_.empty(); }

  std::string_view word(const char* what) {
    std::string_view w = take();
    if (w.empty()) fail(std::string("missing ") + what);
    return w;
  }
  std::optional<std::string_view> maybe_word() {
    std::string_view w = take();
    if (w.empty()) return std::nullopt;
    return w;
  }
  template <class T>
  T number(const char* what) {
    return to_number<T>(word(what), what);
  }
  // "a,b,c" -> {a, b, c}
  std::vector<std::int64_t> int_list(const char* what) {
    std::vector<std::int64_t> out;
    for_each_part(word(what), ',', [&](std::string_view p) { out.push_back(to_number<std::int64_t>(p, what)); });
    return out;
  }
  // "lo:hi,lo:hi,..." -> the box
  ShardView box(const char* what) {
    std::vector<Interval> iv;
    for_each_part(word(what), ',', [&](std::string_view p) {
      const auto colon = p.find(':');
      if (colon == std::string_view::npos) fail(std::string("bad ") + what + " '" + std::string(p) + "'");
      iv.push_back({to_number<std::int64_t>(p.substr(0, colon), what),
                    to_number<std::int64_t>(p.substr(colon + 1), what)});
    });
    return ShardView(iv);
  }
  [[noreturn]] void fail(const std::string& why) const {
    throw E(std::string(format_) + ": line " + std::to_string(lineno_) + ": " + why);
  }

 private:
  void skip_space() {
    while (!rest_.empty() && (rest_.front() == ' ' || rest_.front() == '\t' || rest_.front() == '\r'))
      rest_.remove_prefix(1);
  }
  std::string_view take() {
    skip_space();
    std::size_t n = 0;
    while (n < rest_.size() && rest_[n] != ' ' && rest_[n] != '\t' && rest_[n] != '\r') ++n;
    std::string_view w = rest_.substr(0, n);
    rest_.remove_prefix(n);
    return w;
  }
  template <class T>
  T to_number(std::string_view s, const char* what) const {
    T v{};
    const auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc() || end != s.data() + s.size() || s.empty())
      fail(std::string("bad ") + what + " '" + std::string(s) + "'");
    return v;
  }
  template <class F>
  void for_each_part(std::string_view s, char sep, F&& f) const {
    while (true) {
      const auto cut = s.find(sep);
      f(s.substr(0, cut));
      if (cut == std::string_view::npos) return;
      s.remove_prefix(cut + 1);
    }
  }

  std::string_view rest_;
  std::string_view kind_;
  const char* format_;
  int lineno_;
};

// Calls f(line, lineno) for every line of `text`; with `comments`, a '#'
// starts a comment that runs to the end of the line.
template <class F>
void for_each_line(std::string_view text, bool comments, F&& f) {
  int lineno = 0;
  while (!text.empty()) {
    const auto nl = text.find('\n');
    std::string_view line = text.substr(0, nl);
    text.remove_prefix(nl == std::string_view::npos ? text.size() : nl + 1);
    ++lineno;
    if (comments)
      if (const auto h = line.find('#'); h != std::string_view::npos) line = line.substr(0, h);
    f(line, lineno);
  }
}

// Field writers: append "<value>" / "lo:hi,lo:hi" to a record being built.
inline void put(std::string& out, std::int64_t v) {
  char buf[24];
  const auto r = std::to_chars(buf, buf + sizeof buf, v);
  out.append(buf, r.ptr);
}
inline void put(std::string& out, std::string_view s) { out.append(s); }
inline void put_box(std::string& out, const ShardView& v) {
  for (std::size_t i = 0; i < v.ndims(); ++i) {
    if (i) out.push_back(',');
    put(out, v.dim(i).lo);
    out.push_back(':');
    put(out, v.dim(i).hi);
  }
}

}  // namespace reshard::records
