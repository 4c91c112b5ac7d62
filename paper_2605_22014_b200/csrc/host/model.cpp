// Geometry, model spec and spec-text I/O for the host planner.
// Semantics: proj/include/reshard/shard_view.hpp:25-112 (boxes),
// proj/include/reshard/model_spec.hpp:26-87 (specs).  The spec text format is
// this repo's own (paper_2605_22014_b200/specs.py).
#include <algorithm>
#include <sstream>
#include <stdexcept>

#include "records.hpp"
#include "reshard_b200/reshard.hpp"

namespace reshard {

ShardView::ShardView(const std::vector<Interval>& bounds) {
  if (bounds.size() > static_cast<std::size_t>(kMaxDims))
    throw std::invalid_argument("ShardView: more than " + std::to_string(kMaxDims) + " dimensions");
  for (std::size_t i = 0; i < bounds.size(); ++i) {
    const Interval& iv = bounds[i];
    if (iv.lo < 0 || iv.lo >= iv.hi)
      throw std::invalid_argument("ShardView: interval [" + std::to_string(iv.lo) + "," +
                                  std::to_string(iv.hi) + ") is empty or negative");
    iv_[i] = iv;
  }
  nd_ = static_cast<std::uint8_t>(bounds.size());
}

ShardView ShardView::full(const std::vector<std::int64_t>& shape) {
  std::vector<Interval> b;
  b.reserve(shape.size());
  for (auto d : shape) b.push_back({0, d});
  return ShardView(b);
}

const Interval& ShardView::dim(std::size_t i) const {
  if (i >= nd_) throw std::out_of_range("ShardView::dim");
  return iv_[i];
}

std::int64_t ShardView::element_count() const {
  std::int64_t n = 1;
  for (std::size_t i = 0; i < nd_; ++i) n *= iv_[i].length();
  return n;
}

std::vector<std::int64_t> ShardView::extents() const {
  std::vector<std::int64_t> e(nd_);
  for (std::size_t i = 0; i < nd_; ++i) e[i] = iv_[i].length();
  return e;
}

bool ShardView::contains(const ShardView& o) const {
  if (o.nd_ != nd_) return false;
  for (std::size_t i = 0; i < nd_; ++i)
    if (o.iv_[i].lo < iv_[i].lo || o.iv_[i].hi > iv_[i].hi) return false;
  return true;
}

bool ShardView::contains_point(const std::vector<std::int64_t>& p) const {
  if (p.size() != nd_) return false;
  for (std::size_t i = 0; i < nd_; ++i)
    if (p[i] < iv_[i].lo || p[i] >= iv_[i].hi) return false;
  return true;
}

bool ShardView::operator==(const ShardView& o) const {
  if (o.nd_ != nd_) return false;
  for (std::size_t i = 0; i < nd_; ++i)
    if (!(o.iv_[i] == iv_[i])) return false;
  return true;
}

std::string ShardView::to_string() const {
  std::string s;
  for (std::size_t i = 0; i < nd_; ++i) {
    if (i) s += 'x';
    s += '[' + std::to_string(iv_[i].lo) + ',' + std::to_string(iv_[i].hi) + ')';
  }
  return s;
}

std::optional<ShardView> intersect(const ShardView& a, const ShardView& b) {
  if (a.ndims() != b.ndims())
    throw std::invalid_argument("intersect: dimensionality mismatch (" +
                                std::to_string(a.ndims()) + " vs " + std::to_string(b.ndims()) +
                                ")");
  ShardView out = a;
  for (std::size_t i = 0; i < a.ndims(); ++i) {
    Interval& iv = out.raw(i);
    iv.lo = std::max(a.dim(i).lo, b.dim(i).lo);
    iv.hi = std::min(a.dim(i).hi, b.dim(i).hi);
    if (iv.lo >= iv.hi) return std::nullopt;
  }
  return out;
}

const char* to_string(TensorRole r) {
  switch (r) {
    case TensorRole::kParameter: return "parameter";
    case TensorRole::kOptimizerMoment1: return "optimizer_moment_1";
    case TensorRole::kOptimizerMoment2: return "optimizer_moment_2";
  }
  return "?";
}

std::int64_t TensorSpec::element_count() const {
  std::int64_t n = 1;
  for (auto d : shape) n *= d;
  return n;
}

std::int64_t ModelSpec::total_param_elements() const {
  std::int64_t n = 0;
  for (const auto& t : tensors)
    if (t.role == TensorRole::kParameter) n += t.element_count();
  return n;
}

double ModelSpec::total_state_bytes() const {
  return static_cast<double>(total_param_elements()) * state_multiplier;
}

std::int64_t ModelSpec::total_tensor_bytes() const {
  std::int64_t n = 0;
  for (const auto& t : tensors) n += t.element_count() * element_bytes(t);
  return n;
}

std::vector<std::string> ModelSpec::validate() const {
  std::vector<std::string> v;
  if (num_layers < 1) v.push_back("num_layers must be >= 1");
  if (bytes_per_element < 1) v.push_back("bytes_per_element must be >= 1");
  if (state_multiplier <= 0) v.push_back("state_multiplier must be > 0");
  for (const auto& t : tensors) {
    if (t.layer < 0 || t.layer >= num_layers)
      v.push_back("tensor " + t.tensor_id + ": layer " + std::to_string(t.layer) +
                  " out of range [0," + std::to_string(num_layers) + ")");
    if (t.shape.empty()) v.push_back("tensor " + t.tensor_id + ": empty shape");
    if (t.shape.size() > static_cast<std::size_t>(kMaxDims))
      v.push_back("tensor " + t.tensor_id + ": more than " + std::to_string(kMaxDims) + " dimensions");
    for (auto d : t.shape)
      if (d < 1) v.push_back("tensor " + t.tensor_id + ": dimension < 1");
    if (t.tp_shard_axis &&
        (*t.tp_shard_axis < 0 || *t.tp_shard_axis >= static_cast<int>(t.shape.size())))
      v.push_back("tensor " + t.tensor_id + ": tp_shard_axis out of range");
    if (t.element_bytes < 0) v.push_back("tensor " + t.tensor_id + ": element_bytes < 0");
    if (t.dp_shard_axis &&
        (*t.dp_shard_axis < 0 || *t.dp_shard_axis >= static_cast<int>(t.shape.size())))
      v.push_back("tensor " + t.tensor_id + ": dp_shard_axis out of range");
  }
  return v;
}

ModelSpec ModelSpec::parse(const std::string& text) {
  using SpecLine = records::Line<std::invalid_argument>;
  ModelSpec m;
  bool have_model = false;
  records::for_each_line(text, true, [&](std::string_view line, int lineno) {
    SpecLine in(line, "spec parse", lineno);
    if (in.blank()) return;
    if (in.kind() == "model") {
      // model <name> layers <L> bpe <bytes per element>
      m.name = std::string(in.word("model name"));
      if (in.word("'layers'") != "layers") in.fail("bad model record");
      m.num_layers = in.number<int>("layer count");
      if (in.word("'bpe'") != "bpe") in.fail("bad model record");
      m.bytes_per_element = in.number<std::int64_t>("bytes per element");
      have_model = true;
    } else if (in.kind() == "tensor") {
      // tensor <id> <layer> <d0,d1,...> <tp axis | -> <param|m1|m2> <bytes per element> [dp=<axis>]
      TensorSpec t;
      t.tensor_id = std::string(in.word("tensor id"));
      t.layer = in.number<int>("layer");
      t.shape = in.int_list("shape");
      if (const auto axis = in.word("tp axis"); axis != "-") t.tp_shard_axis = std::stoi(std::string(axis));
      const auto role = in.word("role");
      if (role == "param") t.role = TensorRole::kParameter;
      else if (role == "m1") t.role = TensorRole::kOptimizerMoment1;
      else if (role == "m2") t.role = TensorRole::kOptimizerMoment2;
      else in.fail("unknown role " + std::string(role));
      t.element_bytes = in.number<std::int64_t>("element bytes");
      while (auto opt = in.maybe_word()) {  // optional key=value extensions
        if (opt->substr(0, 3) == "dp=") t.dp_shard_axis = std::stoi(std::string(opt->substr(3)));
        else in.fail("unknown tensor option " + std::string(*opt));
      }
      m.tensors.push_back(std::move(t));
    } else {
      in.fail("unknown record '" + std::string(in.kind()) + "'");
    }
  });
  if (!have_model) throw std::invalid_argument("spec parse: missing model record");
  return m;
}

std::string ModelSpec::to_text() const {
  std::ostringstream os;
  os << "model " << name << " layers " << num_layers << " bpe " << bytes_per_element << "\n";
  for (const auto& t : tensors) {
    os << "tensor " << t.tensor_id << " " << t.layer << " ";
    for (std::size_t i = 0; i < t.shape.size(); ++i) os << (i ? "," : "") << t.shape[i];
    os << " " << (t.tp_shard_axis ? std::to_string(*t.tp_shard_axis) : std::string("-")) << " "
       << (t.role == TensorRole::kParameter ? "param"
           : t.role == TensorRole::kOptimizerMoment1 ? "m1" : "m2")
       << " " << element_bytes(t);
    if (t.dp_shard_axis) os << " dp=" << *t.dp_shard_axis;
    os << "\n";
  }
  return os.str();
}

}  // namespace reshard
