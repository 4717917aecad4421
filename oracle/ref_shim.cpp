// TEST INFRASTRUCTURE ONLY.
//
// C-ABI wrapper (prefix tkr_) over the reference's own streaming API,
// compiled together with the unmodified reference sources from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libtucker_ref.so.
// It exposes exactly the functions of oracle_abi.h so tests can drive the
// reference, the C restatement (tko_) and the product (tsg_) side by side.
// Nothing from the reference is copied here: every call goes through the
// reference headers (streaming.hpp, isvd.hpp, linalg.hpp, sthosvd.hpp,
// tensor.hpp).
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tucker/linalg.hpp"
#include "tucker/sthosvd.hpp"
#include "tucker/streaming.hpp"
#include "tucker/tensor.hpp"
#include "tucker/io.hpp"

#define ORC(name) tkr_##name
#include "oracle_abi.h"

struct orc_state {
  tucker::StreamingState st;
  std::vector<orc_metrics> extra;  // expanded masks per step
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

tucker::DenseTensor make_tensor(const double* x, int order, const int64_t* dims) {
  std::vector<std::size_t> d(dims, dims + order);
  tucker::DenseTensor t(d);
  std::memcpy(t.data(), x, t.size() * sizeof(double));
  return t;
}

orc_metrics convert(const tucker::SliceMetrics& m, int d, int mask) {
  orc_metrics o{};
  o.slice_index = static_cast<int64_t>(m.slice_index);
  for (int k = 0; k < d && k < (int)m.ranks.size(); ++k) o.ranks[k] = (int64_t)m.ranks[k];
  o.slice_norm = m.slice_norm;
  o.projected_norm = m.projected_norm;
  o.error_estimate = m.error_estimate;
  for (std::size_t k = 0; k < m.mode_residuals.size() && k < ORC_MAXD; ++k)
    o.mode_residuals[k] = m.mode_residuals[k];
  o.expanded_mask = mask;
  return o;
}
}  // namespace

extern "C" {

const char* tkr_last_error(void) { return g_err.c_str(); }

int tkr_stream_init(const double* x, int32_t order, const int64_t* dims,
                    double tau, orc_state** out) {
  *out = nullptr;
  return guarded([&] {
    if (order < 1) throw std::invalid_argument("stream_init: need at least one non-streaming mode");
    auto t = make_tensor(x, order, dims);
    auto* s = new orc_state{tucker::stream_init(t, tau), {}};
    *out = s;
  });
}

int tkr_stream_update(orc_state* s, const double* y) {
  return guarded([&] {
    const std::size_t d = s->st.order;
    std::vector<std::size_t> dims;
    for (std::size_t k = 0; k + 1 < d; ++k) dims.push_back(s->st.model.factors[k].rows());
    tucker::DenseTensor t(dims);
    std::memcpy(t.data(), y, t.size() * sizeof(double));
    std::vector<std::size_t> before = s->st.model.core.dims();
    tucker::stream_update(s->st, t);
    int mask = 0;
    for (std::size_t k = 0; k + 1 < d; ++k)
      if (s->st.model.core.dim(k) != before[k]) mask |= 1 << k;
    s->extra.push_back(convert(s->st.metrics.steps.back(), (int)d, mask));
  });
}

int tkr_process_mode(orc_state* s, const double* y, const int64_t* ydims,
                     int32_t mode, double delta, double* y_out, int64_t cap,
                     int64_t* ydims_out, double* res) {
  return guarded([&] {
    const int d = (int)s->st.order;
    auto t = make_tensor(y, d - 1, ydims);
    *res = tucker::process_nonstreaming_mode(s->st, t, (std::size_t)mode, delta);
    if ((int64_t)t.size() > cap) throw std::invalid_argument("process_mode: output capacity");
    std::memcpy(y_out, t.data(), t.size() * sizeof(double));
    for (int k = 0; k < d - 1; ++k) ydims_out[k] = (int64_t)t.dim(k);
  });
}

int tkr_query(const orc_state* s, orc_dims* o) {
  std::memset(o, 0, sizeof *o);
  const auto& st = s->st;
  o->order = (int32_t)st.order;
  o->n_d = (int64_t)st.n_d;
  o->rank = (int64_t)st.isvd.rank();
  o->insertions = (int64_t)st.isvd.insertions;
  for (std::size_t k = 0; k < st.order; ++k) o->core_dims[k] = (int64_t)st.model.core.dim(k);
  for (std::size_t k = 0; k + 1 < st.order; ++k)
    o->slice_dims[k] = (int64_t)st.model.factors[k].rows();
  o->tau = st.tau;
  o->squared_error = st.isvd.squared_error;
  o->total_input_sq = st.total_input_sq;
  o->nonstream_discarded_sq = st.nonstream_discarded_sq;
  return 0;
}

int tkr_export_state(const orc_state* s, double* core, double* factors,
                     double* sigma, double* left, double* right) {
  const auto& st = s->st;
  if (core) std::memcpy(core, st.model.core.data(), st.model.core.size() * sizeof(double));
  if (factors) {
    std::size_t off = 0;
    for (std::size_t k = 0; k + 1 < st.order; ++k) {
      const auto& f = st.model.factors[k];
      std::memcpy(factors + off, f.data(), f.size() * sizeof(double));
      off += f.size();
    }
  }
  if (sigma)
    std::memcpy(sigma, st.isvd.singular_values.data(), st.isvd.rank() * sizeof(double));
  if (left) {
    tucker::Matrix m = st.streaming_factor();
    std::memcpy(left, m.data(), m.size() * sizeof(double));
  }
  if (right) std::memcpy(right, st.isvd.right.data(), st.isvd.right.size() * sizeof(double));
  return 0;
}

int64_t tkr_metrics_count(const orc_state* s) { return (int64_t)s->extra.size(); }
int tkr_metrics_at(const orc_state* s, int64_t i, orc_metrics* out) {
  if (i < 0 || i >= (int64_t)s->extra.size()) {
    g_err = "metrics index out of range";
    return 1;
  }
  *out = s->extra[(std::size_t)i];
  return 0;
}
int tkr_last_metrics(const orc_state* s, orc_metrics* out) {
  return tkr_metrics_at(s, (int64_t)s->extra.size() - 1, out);
}

int tkr_assemble(const orc_dims* dm, const double* core, const double* factors,
                 const double* sigma, const double* left, const double* right,
                 orc_state** out) {
  *out = nullptr;
  return guarded([&] {
    const int d = dm->order;
    tucker::TuckerModel model;
    model.core = make_tensor(core, d, dm->core_dims);
    model.tau = dm->tau;
    model.factors.resize(d);
    std::size_t off = 0;
    for (int k = 0; k + 1 < d; ++k) {
      tucker::Matrix f((std::size_t)dm->slice_dims[k], (std::size_t)dm->core_dims[k]);
      std::memcpy(f.data(), factors + off, f.size() * sizeof(double));
      off += f.size();
      model.factors[k] = std::move(f);
    }
    const std::size_t r = (std::size_t)dm->core_dims[d - 1];
    const std::size_t n = r == 0 ? 0 : model.core.size() / r;
    tucker::Matrix lm((std::size_t)dm->n_d, r);
    std::memcpy(lm.data(), left, lm.size() * sizeof(double));
    tucker::Matrix rm(n, r);
    std::memcpy(rm.data(), right, rm.size() * sizeof(double));
    tucker::ISVDState isvd;
    isvd.left = tucker::GrowableRowMatrix(lm);
    isvd.singular_values.assign(sigma, sigma + r);
    isvd.right = rm;
    isvd.squared_error = dm->squared_error;
    isvd.insertions = (std::size_t)dm->insertions;
    auto* s = new orc_state{tucker::assemble_streaming_state(std::move(model), std::move(isvd),
                                                             dm->total_input_sq,
                                                             dm->nonstream_discarded_sq),
                            {}};
    *out = s;
  });
}

int tkr_set_reorthogonalize_every(orc_state* s, int64_t k) {
  return guarded([&] {
    if (k < 0) throw std::invalid_argument("reorthogonalize_every must be nonnegative");
    s->st.isvd.options.reorthogonalize_every = static_cast<std::size_t>(k);
  });
}

// TUCKCKPT v1 (io.cpp:268-423) through the reference's own writer / reader.
int tkr_save_checkpoint(const orc_state* s, const char* path) {
  return guarded([&] { tucker::save_checkpoint(path, s->st); });
}
int tkr_load_checkpoint(const char* path, orc_state** out) {
  *out = nullptr;
  return guarded([&] {
    auto* o = new orc_state{tucker::from_checkpoint(tucker::load_checkpoint(path)), {}};
    *out = o;
  });
}

void tkr_destroy(orc_state* s) { delete s; }

int tkr_sym_eig_desc(int64_t n, const double* g, double* evals, double* evecs) {
  return guarded([&] {
    tucker::Matrix m((std::size_t)n, (std::size_t)n);
    std::memcpy(m.data(), g, m.size() * sizeof(double));
    auto r = tucker::sym_eig_desc(m);
    std::memcpy(evals, r.eigenvalues.data(), (std::size_t)n * sizeof(double));
    std::memcpy(evecs, r.eigenvectors.data(), (std::size_t)(n * n) * sizeof(double));
  });
}

int64_t tkr_truncation_rank(int64_t n, const double* evals, double delta) {
  int64_t out = -1;
  int st = guarded([&] {
    std::vector<double> e(evals, evals + n);
    out = (int64_t)tucker::truncation_rank(e, delta);
  });
  return st ? -1 : out;
}

int tkr_small_svd_truncated(int64_t m, int64_t n, const double* a, double thr,
                            double* left, double* sigma, double* right,
                            int64_t* rank, double* disc) {
  return guarded([&] {
    tucker::Matrix am((std::size_t)m, (std::size_t)n);
    std::memcpy(am.data(), a, am.size() * sizeof(double));
    auto s = tucker::small_svd_truncated(am, thr);
    *rank = (int64_t)s.singular_values.size();
    *disc = s.discarded_sq;
    std::memcpy(left, s.left.data(), s.left.size() * sizeof(double));
    std::memcpy(sigma, s.singular_values.data(), s.singular_values.size() * sizeof(double));
    std::memcpy(right, s.right.data(), s.right.size() * sizeof(double));
  });
}

int tkr_mode_subspace(const double* t, int32_t order, const int64_t* dims,
                      int32_t mode, double delta, double* basis, int64_t* rank,
                      double* evals, double* disc) {
  return guarded([&] {
    auto tt = make_tensor(t, order, dims);
    auto sub = tucker::mode_subspace(tt, (std::size_t)mode, delta);
    *rank = (int64_t)sub.basis.cols();
    *disc = sub.discarded_sq;
    std::memcpy(basis, sub.basis.data(), sub.basis.size() * sizeof(double));
    std::memcpy(evals, sub.eigenvalues.data(), sub.eigenvalues.size() * sizeof(double));
  });
}

int tkr_ttm(const double* t, int32_t order, const int64_t* dims, int32_t mode,
            const double* a, int64_t a_rows, int64_t a_cols, int32_t transpose_a,
            double* out) {
  return guarded([&] {
    auto tt = make_tensor(t, order, dims);
    tucker::Matrix am((std::size_t)a_rows, (std::size_t)a_cols);
    std::memcpy(am.data(), a, am.size() * sizeof(double));
    auto o = tucker::ttm(tt, (std::size_t)mode, am, transpose_a != 0);
    std::memcpy(out, o.data(), o.size() * sizeof(double));
  });
}

double tkr_sum_of_squares(const double* p, int64_t n) {
  return tucker::detail::sum_of_squares(p, (std::size_t)n);
}

}  // extern "C"
