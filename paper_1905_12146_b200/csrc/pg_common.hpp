// Shared host-side helpers for the phylograd-b200 C-ABI: error plumbing that
// maps C++ exceptions onto pg_status codes (the reference's exception types,
// engine.hpp:58-70/:211-215/:226-227, tree.hpp:141-146), and small dense
// linear algebra used at setup time.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/phylograd_b200.h"

namespace pg {

struct NewickError : std::runtime_error {
  NewickError(const std::string& what, size_t pos)
      : std::runtime_error(what + " (at position " + std::to_string(pos) + ")"), position(pos) {}
  size_t position;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotSupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& s);

// Runs f(); converts exceptions to status codes and records the message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return PG_OK;
  } catch (const NewickError& e) {
    set_last_error(e.what());
    return PG_ERR_NEWICK;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return PG_ERR_CUDA;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return PG_ERR_NCCL;
  } catch (const NotSupported& e) {
    set_last_error(e.what());
    return PG_ERR_NOT_SUPPORTED;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return PG_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return PG_ERR_LOGIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PG_ERR_RUNTIME;
  } catch (...) {
    set_last_error("unknown error");
    return PG_ERR_RUNTIME;
  }
}

// Row-major dense square matrix helpers (setup only).
using RowMat = std::vector<double>;
RowMat matmul(const RowMat& a, const RowMat& b, int n);
// Symmetric eigendecomposition by cyclic Jacobi: a = V diag(w) V^T, V column j = eigenvector j.
void symmetric_eigen(const RowMat& a, int n, std::vector<double>& w, RowMat& v);
// Pade-13 scaling-and-squaring (Higham 2005) on the host; used only by the
// synthetic-data simulator, never by the evaluation path.
RowMat expm_host(const RowMat& a, int n);
// Regularized lower incomplete gamma and its quantile (discrete-gamma setup).
double regularized_gamma_p(double a, double x);
double gamma_quantile(double shape, double rate, double p);

// Host P(t) = e^{Q t} for simulation (substitution.hpp:147-160: t = 0 -> I,
// symmetric eigensystem for reversible models with pi > 0, Pade otherwise,
// clamp >= 0).  One implementation for the CPU simulators (workloads/) and
// the GPU simulator's transition tables (pg_simulate.cu), so both see
// bit-identical cumulative rows.
struct HostTransition {
  int m = 0;
  bool eig = false;
  std::vector<double> w, U, Ui, q;
  HostTransition(int m_, const std::vector<double>& q_, const std::vector<double>& pi_, int reversible);
  std::vector<double> operator()(double t) const;
};

}  // namespace pg
