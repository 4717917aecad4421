// tucker_gpu: the reference's C++ streaming API (include/tucker/streaming.hpp)
// implemented over the B200 C ABI (include/tsg.h). A program written against
// the reference -- its acceptance gate (tests/acceptance.cpp), the CLI's
// stream loop (tools/tucker_cli.cpp:175-241), from_checkpoint -- links this
// file in place of the reference's src/streaming.cpp and runs every
// stream_init / stream_update / process_nonstreaming_mode /
// assemble_streaming_state on the GPU. Everything else (types, sthosvd,
// reconstruct, io, datagen) is the reference library unchanged.
//
// Compatibility mode: a StreamingState is a host object the
// caller owns, so after every call the device state is mirrored back into it
// (core, factors, ISVD factors, ledgers, v_tensor, one SliceMetrics record).
// The device handle is cached under the state's identity -- the address of
// its core buffer (moves keep it), n_d and the insertion count -- so a state
// that is updated repeatedly keeps its device copy; any state the cache does
// not recognise (copied, hand-edited, assembled elsewhere) is uploaded with
// tsg_import_state first. Error behaviour follows the reference:
// std::invalid_argument (TSG_EINVAL), std::runtime_error for coupling drift
// (TSG_EDRIFT) and device failures.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <list>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsg.h"
#include "tucker/streaming.hpp"

namespace tucker {
namespace {

void check(int code, tsg_stream* h) {
  if (code == TSG_OK) return;
  const std::string msg = tsg_last_error(h);
  if (code == TSG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct Entry {
  tsg_stream* h = nullptr;
  const double* core_ptr = nullptr;
  std::size_t n_d = 0, insertions = 0;
  std::size_t reorth = 0;
};

// A handful of live handles (streams a program interleaves); the oldest is
// released when the cache is full.
constexpr std::size_t kCacheSize = 8;
// The list and its clean-up are ONE function-local static: a separate
// namespace-scope clean-up object would outlive the list (statics die in
// reverse order of construction) and walk freed nodes at exit.
struct Cache {
  std::list<Entry> entries;
  ~Cache() {
    for (Entry& e : entries) tsg_destroy(e.h);
    entries.clear();
  }
};
std::list<Entry>& cache() {
  static Cache c;
  return c.entries;
}

tsg_stream* new_handle(std::size_t reorth) {
  tsg_config cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.device = 0;
  cfg.reorthogonalize_every = static_cast<int64_t>(reorth);
  tsg_stream* h = nullptr;
  check(tsg_create(&cfg, &h), nullptr);
  return h;
}

Entry* find(const StreamingState& s) {
  for (auto it = cache().begin(); it != cache().end(); ++it)
    if (it->core_ptr == s.model.core.data() && it->n_d == s.n_d &&
        it->insertions == s.isvd.insertions && it->reorth == s.isvd.options.reorthogonalize_every) {
      cache().splice(cache().begin(), cache(), it);  // most recent first
      return &cache().front();
    }
  return nullptr;
}

Entry& insert(tsg_stream* h, std::size_t reorth) {
  if (cache().size() >= kCacheSize) {
    tsg_destroy(cache().back().h);
    cache().pop_back();
  }
  cache().push_front(Entry{h, nullptr, 0, 0, reorth});
  return cache().front();
}

// Upload a host state (tsg_import_state = assemble_streaming_state on the
// device: coupling re-checked there).
tsg_stream* upload(const StreamingState& s) {
  const std::size_t d = s.order;
  if (d < 2 || d > TSG_MAXD) throw std::invalid_argument("stream_update: state order out of range");
  tsg_dims dm;
  std::memset(&dm, 0, sizeof dm);
  dm.order = static_cast<int32_t>(d);
  dm.n_d = static_cast<int64_t>(s.n_d);
  dm.rank = static_cast<int64_t>(s.isvd.rank());
  dm.insertions = static_cast<int64_t>(s.isvd.insertions);
  for (std::size_t k = 0; k < d; ++k) dm.core_dims[k] = static_cast<int64_t>(s.model.core.dim(k));
  for (std::size_t k = 0; k + 1 < d; ++k) dm.slice_dims[k] = static_cast<int64_t>(s.model.factors[k].rows());
  dm.tau = s.tau;
  dm.squared_error = s.isvd.squared_error;
  dm.total_input_sq = s.total_input_sq;
  dm.nonstream_discarded_sq = s.nonstream_discarded_sq;
  std::vector<double> fac;
  for (std::size_t k = 0; k + 1 < d; ++k)
    fac.insert(fac.end(), s.model.factors[k].data(), s.model.factors[k].data() + s.model.factors[k].size());
  const Matrix left = s.isvd.left.to_matrix();  // column-major n_d x r
  tsg_stream* h = new_handle(s.isvd.options.reorthogonalize_every);
  const int code = tsg_import_state(h, &dm, s.model.core.data(), fac.data(), s.isvd.singular_values.data(),
                                    left.data(), s.isvd.right.data());
  if (code != TSG_OK) {
    const std::string msg = tsg_last_error(h);
    tsg_destroy(h);
    if (code == TSG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  return h;
}

// Mirror the device state into s (the reference's layouts).
void mirror(tsg_stream* h, StreamingState& s) {
  tsg_dims dm;
  check(tsg_query(h, &dm), h);
  const std::size_t d = static_cast<std::size_t>(dm.order);
  const std::size_t r = static_cast<std::size_t>(dm.rank);
  std::vector<std::size_t> cd(d);
  std::size_t n = 1, fac_n = 0;
  for (std::size_t k = 0; k < d; ++k) cd[k] = static_cast<std::size_t>(dm.core_dims[k]);
  for (std::size_t k = 0; k + 1 < d; ++k) {
    n *= cd[k];
    fac_n += static_cast<std::size_t>(dm.slice_dims[k]) * cd[k];
  }
  DenseTensor core(cd);
  std::vector<double> fac(std::max<std::size_t>(fac_n, 1));
  std::vector<double> sig(std::max<std::size_t>(r, 1));
  Matrix left(static_cast<std::size_t>(dm.n_d), r);
  Matrix right(n, r);
  check(tsg_export_state(h, core.data(), fac.data(), sig.data(), left.data(), right.data()), h);
  s.order = d;
  s.tau = dm.tau;
  s.n_d = static_cast<std::size_t>(dm.n_d);
  s.total_input_sq = dm.total_input_sq;
  s.nonstream_discarded_sq = dm.nonstream_discarded_sq;
  s.model.tau = dm.tau;
  if (s.model.mode_order.size() != d) {
    s.model.mode_order.resize(d);
    for (std::size_t k = 0; k < d; ++k) s.model.mode_order[k] = k;
  }
  s.model.factors.resize(d);
  std::size_t off = 0;
  for (std::size_t k = 0; k + 1 < d; ++k) {
    Matrix f(static_cast<std::size_t>(dm.slice_dims[k]), cd[k]);
    std::copy(fac.data() + off, fac.data() + off + f.size(), f.data());
    off += f.size();
    s.model.factors[k] = std::move(f);
  }
  s.model.factors[d - 1] = Matrix();
  // v_tensor shares isvd.right's buffer layout (streaming.hpp:31-33)
  s.v_tensor = DenseTensor(cd);
  std::copy(right.data(), right.data() + right.size(), s.v_tensor.data());
  s.model.core = std::move(core);
  const ISVDOptions opts = s.isvd.options;
  s.isvd.left = GrowableRowMatrix(left);
  s.isvd.singular_values.assign(sig.begin(), sig.begin() + static_cast<std::ptrdiff_t>(r));
  s.isvd.right = std::move(right);
  s.isvd.squared_error = dm.squared_error;
  s.isvd.insertions = static_cast<std::size_t>(dm.insertions);
  s.isvd.options = opts;
}

void remember(Entry& e, const StreamingState& s) {
  e.core_ptr = s.model.core.data();
  e.n_d = s.n_d;
  e.insertions = s.isvd.insertions;
  e.reorth = s.isvd.options.reorthogonalize_every;
}

SliceMetrics metrics_of(const tsg_slice_metrics& m, std::size_t d) {
  SliceMetrics o;
  o.slice_index = static_cast<std::size_t>(m.slice_index);
  o.ranks.resize(d);
  for (std::size_t k = 0; k < d; ++k) o.ranks[k] = static_cast<std::size_t>(m.ranks[k]);
  o.peak_bytes = static_cast<std::size_t>(m.peak_bytes);
  o.wall_ms = m.wall_ms;
  o.slice_norm = m.slice_norm;
  o.projected_norm = m.projected_norm;
  o.mode_residuals.assign(m.mode_residuals, m.mode_residuals + (d - 1));
  o.error_estimate = m.error_estimate;
  return o;
}

Entry& entry_for(StreamingState& state) {
  if (Entry* e = find(state)) return *e;
  tsg_stream* h = upload(state);
  Entry& e = insert(h, state.isvd.options.reorthogonalize_every);
  remember(e, state);
  return e;
}

}  // namespace

TuckerModel StreamingState::full_model() const {
  TuckerModel m = model;
  m.factors.resize(order);
  m.factors[order - 1] = streaming_factor();
  m.tau = tau;
  return m;
}

StreamingState stream_init(const DenseTensor& x_init, double tau) {
  const std::size_t d = x_init.order();
  if (d < 2) throw std::invalid_argument("stream_init: need at least one non-streaming mode");
  if (d > TSG_MAXD) throw std::invalid_argument("stream_init: order exceeds TSG_MAXD");
  std::vector<int64_t> dims(d);
  for (std::size_t k = 0; k < d; ++k) dims[k] = static_cast<int64_t>(x_init.dim(k));
  tsg_stream* h = new_handle(0);
  const int code = tsg_init(h, x_init.data(), static_cast<int32_t>(d), dims.data(), tau, TSG_MEM_HOST);
  if (code != TSG_OK) {
    const std::string msg = tsg_last_error(h);
    tsg_destroy(h);
    if (code == TSG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  StreamingState s;
  mirror(h, s);
  Entry& e = insert(h, 0);
  remember(e, s);
  return s;
}

void stream_update(StreamingState& state, const DenseTensor& y) {
  const std::size_t d = state.order;
  if (y.order() + 1 != d) throw std::invalid_argument("stream_update: slice must have d-1 modes");
  for (std::size_t k = 0; k + 1 < d; ++k)
    if (y.dim(k) != state.model.factors[k].rows())
      throw std::invalid_argument("stream_update: slice shape mismatch");
  Entry& e = entry_for(state);
  check(tsg_update(e.h, y.data(), TSG_MEM_HOST), e.h);
  tsg_slice_metrics m;
  check(tsg_last_metrics(e.h, &m), e.h);
  mirror(e.h, state);
  state.metrics.steps.push_back(metrics_of(m, d));
  remember(e, state);
}

double process_nonstreaming_mode(StreamingState& state, DenseTensor& y, std::size_t mode, double delta) {
  const std::size_t d = state.order;
  if (mode + 1 >= d) throw std::out_of_range("process_nonstreaming_mode: not a non-streaming mode");
  Entry& e = entry_for(state);
  std::vector<int64_t> yd(y.order());
  for (std::size_t k = 0; k < y.order(); ++k) yd[k] = static_cast<int64_t>(y.dim(k));
  // the output grows along `mode` by at most N_mode - R_mode columns
  const std::size_t cap = y.size() / std::max<std::size_t>(y.dim(mode), 1) *
                              static_cast<std::size_t>(state.model.factors[mode].rows()) +
                          16;
  std::vector<double> out(cap);
  int64_t od[TSG_MAXD] = {0};
  double res = 0.0;
  check(tsg_process_mode(e.h, y.data(), yd.data(), static_cast<int32_t>(mode), delta, out.data(),
                         static_cast<int64_t>(cap), od, &res),
        e.h);
  std::vector<std::size_t> nd(y.order());
  for (std::size_t k = 0; k < y.order(); ++k) nd[k] = static_cast<std::size_t>(od[k]);
  DenseTensor yo(nd);
  std::copy(out.data(), out.data() + yo.size(), yo.data());
  y = std::move(yo);
  const std::vector<SliceMetrics> keep = std::move(state.metrics.steps);
  mirror(e.h, state);
  state.metrics.steps = keep;
  remember(e, state);
  return res;
}

double estimate_relative_error(const StreamingState& state) {
  // ledger estimate (streaming.hpp:72-79) from the state the caller holds
  if (!(state.total_input_sq > 0.0)) return 0.0;
  const double booked = state.isvd.squared_error + state.nonstream_discarded_sq;
  return std::sqrt((booked > 0.0 ? booked : 0.0) / state.total_input_sq);
}

StreamingState assemble_streaming_state(TuckerModel model, ISVDState isvd, double total_input_sq,
                                        double nonstream_discarded_sq) {
  StreamingState s;
  s.order = model.core.order();
  if (s.order < 2) throw std::invalid_argument("assemble_streaming_state: need d >= 2");
  if (model.factors.size() != s.order || !model.factors[s.order - 1].empty())
    throw std::invalid_argument(
        "assemble_streaming_state: streaming-mode factor slot must be empty "
        "(it is carried by the ISVD left factor)");
  s.tau = model.tau;
  s.n_d = isvd.row_count();
  s.total_input_sq = total_input_sq;
  s.nonstream_discarded_sq = nonstream_discarded_sq;
  s.v_tensor = DenseTensor(model.core.dims());
  if (s.v_tensor.size() != isvd.right.size())
    throw std::invalid_argument("assemble_streaming_state: right factor / core size mismatch");
  std::copy(isvd.right.data(), isvd.right.data() + isvd.right.size(), s.v_tensor.data());
  s.model = std::move(model);
  s.isvd = std::move(isvd);
  // the device import re-checks core = v x_{d-1} diag(s) (TSG_EDRIFT ->
  // std::runtime_error, as check_core_coupling throws) and keeps the handle
  Entry& e = insert(upload(s), s.isvd.options.reorthogonalize_every);
  remember(e, s);
  return s;
}

}  // namespace tucker
