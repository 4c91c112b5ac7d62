// Descriptor compiler.  A region copy between two row-major owner buffers is
// reduced to (run bytes, outer dims): every inner axis that spans both owners
// fully is folded into the contiguous run, degenerate axes are dropped, and
// adjacent outer axes that are jointly contiguous on both sides are merged.
// Vector width is the largest power of two (<= 16 B) dividing both base
// addresses, the run and every outer stride.  This is the coalescing the
// reference's for_each_row (proj/src/executor.cpp:23-46) does not do: an
// axis-0 split of [V, h] becomes one multi-MB run instead of V row memcpys.
#include "compile.hpp"

#include <algorithm>
#include <stdexcept>

namespace rsb {

namespace {

struct Dim {
  std::uint64_t ext;
  std::int64_t s, d;  // byte strides
};

std::uint32_t vec_log2_for(std::uint64_t src, std::uint64_t dst, std::uint64_t run,
                           const std::vector<Dim>& outer) {
  std::uint64_t bits = src | dst | run;
  for (const auto& o : outer) bits |= static_cast<std::uint64_t>(o.s) | static_cast<std::uint64_t>(o.d);
  std::uint32_t v = 4;
  while (v > 0 && (bits & ((1ull << v) - 1))) --v;
  return v;
}

void emit(std::vector<rs_copy_desc>& out, std::uint64_t src, std::uint64_t dst, std::uint64_t run,
          const std::vector<Dim>& outer, std::uint32_t tag) {
  if (outer.size() > RS_MAX_OUTER) throw std::invalid_argument("copy descriptor: too many outer dims");
  rs_copy_desc d{};
  d.src = src;
  d.dst = dst;
  d.row_bytes = run;
  d.rows = 1;
  d.nouter = static_cast<std::uint32_t>(outer.size());
  for (std::size_t k = 0; k < outer.size(); ++k) {
    if (outer[k].ext >= (1ull << 32)) throw std::invalid_argument("copy descriptor: extent >= 2^32");
    d.ext[k] = outer[k].ext;
    d.sstr[k] = outer[k].s;
    d.dstr[k] = outer[k].d;
    d.rows *= outer[k].ext;
  }
  if (d.rows >= (1ull << 32)) throw std::invalid_argument("copy descriptor: rows >= 2^32");
  d.vec_log2 = vec_log2_for(src, dst, run, outer);
  d.tag = tag;
  out.push_back(d);
}

}  // namespace

std::uint64_t bytes_of(const rs_copy_desc& d) { return d.rows * d.row_bytes; }

void append_copy(std::vector<rs_copy_desc>& out, std::uint64_t src_base,
                 const reshard::ShardView& src_owner, std::uint64_t dst_base,
                 const reshard::ShardView& dst_owner, const reshard::ShardView& region,
                 std::int64_t elem_bytes, std::uint32_t tag, bool cut_runs) {
  const std::size_t nd = region.ndims();
  // element strides of both owners and the region origin offsets
  std::vector<std::int64_t> ss(nd), ds(nd);
  std::int64_t s_acc = 1, d_acc = 1, s_off = 0, d_off = 0;
  for (std::size_t k = nd; k-- > 0;) {
    ss[k] = s_acc;
    ds[k] = d_acc;
    s_off += (region.dim(k).lo - src_owner.dim(k).lo) * s_acc;
    d_off += (region.dim(k).lo - dst_owner.dim(k).lo) * d_acc;
    s_acc *= src_owner.dim(k).length();
    d_acc *= dst_owner.dim(k).length();
  }
  const std::uint64_t src = src_base + static_cast<std::uint64_t>(s_off * elem_bytes);
  const std::uint64_t dst = dst_base + static_cast<std::uint64_t>(d_off * elem_bytes);

  // fold inner axes into the run while it stays contiguous on both sides
  std::uint64_t run = static_cast<std::uint64_t>(region.dim(nd - 1).length() * elem_bytes);
  std::size_t k = nd - 1;
  while (k-- > 0) {
    const std::uint64_t e = static_cast<std::uint64_t>(region.dim(k).length());
    if (e == 1) continue;
    if (run == static_cast<std::uint64_t>(ss[k] * elem_bytes) &&
        run == static_cast<std::uint64_t>(ds[k] * elem_bytes)) {
      run *= e;
      continue;
    }
    ++k;  // axis k is the first outer axis
    break;
  }
  if (k == static_cast<std::size_t>(-1)) k = 0;  // everything folded
  std::vector<Dim> outer;  // innermost first
  for (std::size_t j = k; j-- > 0;) {
    const std::uint64_t e = static_cast<std::uint64_t>(region.dim(j).length());
    if (e == 1) continue;
    Dim dim{e, ss[j] * elem_bytes, ds[j] * elem_bytes};
    if (!outer.empty()) {
      Dim& in = outer.back();
      if (dim.s == static_cast<std::int64_t>(in.ext) * in.s &&
          dim.d == static_cast<std::int64_t>(in.ext) * in.d) {
        in.ext *= e;  // jointly contiguous: merge
        continue;
      }
    }
    outer.push_back(dim);
  }

  // cut long runs into sub-rows (one extra innermost outer axis) + tail
  if (cut_runs && run > 2 * kSubRowBytes && outer.size() < RS_MAX_OUTER) {
    const std::uint64_t nsub = run / kSubRowBytes;
    const std::uint64_t tail = run - nsub * kSubRowBytes;
    std::vector<Dim> o2;
    o2.push_back({nsub, static_cast<std::int64_t>(kSubRowBytes), static_cast<std::int64_t>(kSubRowBytes)});
    o2.insert(o2.end(), outer.begin(), outer.end());
    emit(out, src, dst, kSubRowBytes, o2, tag);
    if (tail) emit(out, src + nsub * kSubRowBytes, dst + nsub * kSubRowBytes, tail, outer, tag);
    return;
  }
  emit(out, src, dst, run, outer, tag);
}

std::uint64_t assign_items(std::vector<rs_copy_desc>& descs, std::size_t first,
                           std::uint64_t item_base, std::uint64_t item_bytes) {
  std::uint64_t item = item_base;
  for (std::size_t i = first; i < descs.size(); ++i) {
    rs_copy_desc& d = descs[i];
    const std::uint64_t rpi = std::max<std::uint64_t>(1, item_bytes / std::max<std::uint64_t>(d.row_bytes, 1));
    d.rows_per_item = static_cast<std::uint32_t>(std::min<std::uint64_t>(rpi, 1u << 30));
    d.item0 = item;
    item += (d.rows + d.rows_per_item - 1) / d.rows_per_item;
  }
  return item;
}

void append_pattern(std::vector<rs_pattern_desc>& out, std::uint64_t ptr,
                    const reshard::TensorSpec& t, const reshard::ShardView& view,
                    std::int64_t elem_bytes, std::uint32_t tensor_index, std::uint32_t entry,
                    std::uint64_t item_bytes) {
  const std::size_t nd = view.ndims();
  std::vector<std::int64_t> gs(nd);
  std::int64_t acc = 1, g0 = 0;
  for (std::size_t k = nd; k-- > 0;) {
    gs[k] = acc;
    g0 += view.dim(k).lo * acc;
    acc *= t.shape[k];
  }
  rs_pattern_desc d{};
  d.ptr = ptr;
  d.g0 = g0;
  d.elem_bytes = static_cast<std::uint32_t>(elem_bytes);
  d.tensor_index = tensor_index;
  d.entry = entry;
  d.rows = 1;
  std::uint32_t n = 0;
  // rows run over axes [0, first_folded), innermost first; the row folds every
  // inner axis on which the view spans the whole tensor (global index stays
  // contiguous across them)
  std::size_t first_folded = nd - 1;
  std::uint64_t row = static_cast<std::uint64_t>(view.dim(nd - 1).length());
  while (first_folded > 0 && view.dim(first_folded).length() == t.shape[first_folded]) {
    --first_folded;
    row *= static_cast<std::uint64_t>(view.dim(first_folded).length());
  }
  d.row_elems = row;
  for (std::size_t j = first_folded; j-- > 0;) {
    const std::uint64_t e = static_cast<std::uint64_t>(view.dim(j).length());
    if (e == 1) continue;
    if (n == RS_MAX_OUTER) throw std::invalid_argument("pattern descriptor: too many outer dims");
    d.ext[n] = e;
    d.gstr[n] = gs[j];
    d.rows *= e;
    ++n;
  }
  d.nouter = n;
  if (d.rows >= (1ull << 32)) throw std::invalid_argument("pattern descriptor: rows >= 2^32");
  const std::uint64_t row_bytes = row * static_cast<std::uint64_t>(elem_bytes);
  d.rows_per_item = static_cast<std::uint32_t>(
      std::max<std::uint64_t>(1, item_bytes / std::max<std::uint64_t>(row_bytes, 1)));
  out.push_back(d);
}

}  // namespace rsb
