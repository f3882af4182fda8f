// pymodule.cpp — Python bindings `paper_2403_03772_b200._core`, mirroring the reference's
// `plingam._core` (proj/bindings/pymodule.cpp:103-144) for the causal-order path, plus
// an `Engine` handle on the C-ABI for device-resident benchmarking and multi-GPU ranks.
// numpy arrays are taken column-major (zero-copy when already Fortran-ordered); the GIL is
// released around every device call.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>
#include <cstdio>
#include <limits>

#include "../../../include/plingam_b200.h"
#include "plingam/plingam.hpp"
#include "plingam/simgen.hpp"
#include "plingam/var.hpp"

namespace py = pybind11;
using namespace plingam;

namespace {

using FArray = py::array_t<double, py::array::f_style | py::array::forcecast>;

PyObject* g_error_type = nullptr;

DataMatrix to_data(const FArray& X) {
  if (X.ndim() != 2) throw Error(ErrorCode::DimensionMismatch, "X must be a 2-D array (samples x variables)");
  const auto m = static_cast<std::int64_t>(X.shape(0));
  const auto d = static_cast<std::int64_t>(X.shape(1));
  std::vector<double> v(X.data(), X.data() + m * d);
  return DataMatrix(std::move(v), m, d);
}

py::array_t<double> colmajor_array(const std::vector<double>& v, std::int64_t rows, std::int64_t cols) {
  py::array_t<double, py::array::f_style> out({rows, cols});
  std::copy(v.begin(), v.end(), out.mutable_data());
  return out;
}

struct Engine {
  plg_ctx* ctx = nullptr;
  ~Engine() {
    if (ctx) plg_ctx_destroy(ctx);
  }
};

std::vector<int> engine_causal_order(Engine& e, const FArray& X) {
  const auto n = static_cast<std::int64_t>(X.shape(0));
  const auto d = static_cast<int32_t>(X.shape(1));
  std::vector<int> order(static_cast<std::size_t>(std::max(d, 1)));
  plg_status st{};
  int rc;
  {
    py::gil_scoped_release rel;
    rc = plg_causal_order(e.ctx, X.data(), n, d, std::max<std::int64_t>(n, 1), order.data(), &st);
  }
  gpu::check(rc, &st);
  order.resize(static_cast<std::size_t>(d));
  return order;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "B200 DirectLiNGAM causal-order engine (sm_100a) behind the plingam API";
  m.attr("__version__") = "0.1.0";
  m.attr("engine_version") = plg_version();

  static py::exception<Error> exc(m, "Error");
  g_error_type = exc.ptr();
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if (p) std::rethrow_exception(p);
    } catch (const Error& e) {
      py::object inst = py::reinterpret_borrow<py::object>(g_error_type)(e.what());
      inst.attr("code") = to_string(e.code());
      inst.attr("row") = e.row();
      inst.attr("col") = e.col();
      PyErr_SetObject(g_error_type, inst.ptr());
    }
  });

  py::class_<WeightedDag>(m, "WeightedDag")
      .def_property_readonly("weights", [](const WeightedDag& d) { return colmajor_array(d.weights, d.d, d.d); })
      .def_property_readonly("order", [](const WeightedDag& d) { return d.order.order; })
      .def_readonly("used_pinv", &WeightedDag::used_pinv)
      .def_property_readonly("phases",
                             [](const WeightedDag& d) {
                               py::dict p;
                               p["ordering_seconds"] = d.phases.ordering_seconds;
                               p["weights_seconds"] = d.phases.weights_seconds;
                               p["total_seconds"] = d.phases.total_seconds;
                               return p;
                             })
      .def("__repr__", [](const WeightedDag& d) { return "<WeightedDag dims=" + std::to_string(d.d) + ">"; });

  // ---- ordering (pymodule.cpp:103-118) ----
  // The numpy buffer goes straight to the C-ABI (zero-copy when Fortran-ordered float64;
  // forcecast converts anything else once), with the GIL released for the device call.
  m.def(
      "causal_order",
      [](const FArray& X, bool parallel, int workers) {
        (void)parallel;
        if (X.ndim() != 2) throw Error(ErrorCode::DimensionMismatch, "X must be a 2-D array (samples x variables)");
        if (workers < 1) {  // ordering.cpp:214-217: validate first, then the worker count
          validate(to_data(X));
          throw Error(ErrorCode::OutOfRange, "causal_order: workers must be >= 1");
        }
        const auto n = static_cast<std::int64_t>(X.shape(0));
        const auto d = static_cast<int32_t>(X.shape(1));
        std::vector<int> order(static_cast<std::size_t>(std::max(d, 1)));
        plg_status st{};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = plg_causal_order(gpu::context().get(), X.data(), n, d, std::max<std::int64_t>(n, 1), order.data(), &st);
        }
        gpu::check(rc, &st);
        order.resize(static_cast<std::size_t>(std::max(d, 0)));
        return order;
      },
      py::arg("X"), py::arg("parallel") = false, py::arg("workers") = 1,
      "Recursive causal ordering on the GPU engine (ordering.cpp:213-244).");
  // pymodule.cpp:110-118: workers > 1 selects the parallel path, whose workers < 1 check
  // (ordering.cpp:172-174) is therefore only reachable through search_causal_order_parallel.
  auto search = [](const FArray& X, const std::vector<int>& U, int workers, bool check_workers) {
    if (X.ndim() != 2) throw Error(ErrorCode::DimensionMismatch, "X must be a 2-D array (samples x variables)");
    if (check_workers && workers < 1)
      throw Error(ErrorCode::OutOfRange, "search_causal_order_parallel: workers must be >= 1");
    const auto n = static_cast<std::int64_t>(X.shape(0));
    const auto d = static_cast<int32_t>(X.shape(1));
    std::vector<double> scores(static_cast<std::size_t>(d));
    int chosen = -1;
    plg_status st{};
    int rc;
    {
      py::gil_scoped_release rel;
      rc = plg_search(gpu::context().get(), X.data(), n, d, std::max<std::int64_t>(n, 1), U.data(),
                      static_cast<int32_t>(U.size()), &chosen, scores.data(), &st);
    }
    gpu::check(rc, &st);
    return py::make_tuple(chosen, scores);
  };
  m.def(
      "search_causal_order",
      [search](const FArray& X, const std::vector<int>& U, int workers) { return search(X, U, workers, false); },
      py::arg("X"), py::arg("U"), py::arg("workers") = 1);
  m.def(
      "search_causal_order_parallel",
      [search](const FArray& X, const std::vector<int>& U, int workers) { return search(X, U, workers, true); },
      py::arg("X"), py::arg("U"), py::arg("workers"));
  m.def(
      "regress_out",
      [](const FArray& X, int exog, const std::vector<int>& remaining) {
        DataMatrix data = to_data(X);
        DataMatrix out;
        {
          py::gil_scoped_release rel;
          out = regress_out(data, exog, remaining);
        }
        return colmajor_array(out.values, out.rows, out.cols);
      },
      py::arg("X"), py::arg("exog"), py::arg("remaining"));

  // ---- DirectLiNGAM (pymodule.cpp:121-135) ----
  m.def(
      "fit_direct_lingam",
      [](const FArray& X, bool parallel, int workers, double edge_threshold) {
        // DirectLingam::fit (direct_lingam.cpp:33-76) on the numpy buffer, zero-copy
        DirectLingamConfig cfg;
        cfg.parallel = parallel;
        cfg.workers = workers;
        cfg.edge_threshold = edge_threshold;
        DirectLingam model(cfg);  // config validation (direct_lingam.cpp:19-26)
        if (X.ndim() != 2) throw Error(ErrorCode::DimensionMismatch, "X must be a 2-D array (samples x variables)");
        const auto n = static_cast<std::int64_t>(X.shape(0));
        const auto d = static_cast<int32_t>(X.shape(1));
        WeightedDag dag;
        dag.d = d;
        dag.weights.assign(static_cast<std::size_t>(d) * d, 0.0);
        dag.intercepts.assign(static_cast<std::size_t>(d), 0.0);
        dag.order.order.assign(static_cast<std::size_t>(std::max(d, 1)), -1);
        int32_t pinv = 0;
        plg_status st{};
        int rc;
        FitPhases phases;  // direct_lingam.hpp:16-20 (wall clock, as the reference)
        {
          py::gil_scoped_release rel;
          using Clock = std::chrono::steady_clock;
          const auto t0 = Clock::now();
          rc = plg_causal_order(gpu::context().get(), X.data(), n, d, std::max<std::int64_t>(n, 1), dag.order.order.data(), &st);
          const auto t1 = Clock::now();
          if (rc == 0 && d > 1)
            rc = plg_fit_weights(gpu::context().get(), X.data(), n, d, n, dag.order.order.data(), dag.weights.data(), &pinv, &st);
          const auto t2 = Clock::now();
          phases.ordering_seconds = std::chrono::duration<double>(t1 - t0).count();
          phases.weights_seconds = std::chrono::duration<double>(t2 - t1).count();
          phases.total_seconds = std::chrono::duration<double>(t2 - t0).count();
        }
        gpu::check(rc, &st);
        dag.order.order.resize(static_cast<std::size_t>(std::max(d, 0)));
        dag.used_pinv = pinv != 0;
        dag.phases = phases;
        return dag;
      },
      py::arg("X"), py::arg("parallel") = false, py::arg("workers") = 1, py::arg("edge_threshold") = 0.05);
  m.def(
      "to_edges",
      [](const WeightedDag& dag, double threshold) {
        const EdgeSet e = to_edges(dag, threshold);
        return std::vector<std::pair<int, int>>(e.edges.begin(), e.edges.end());
      },
      py::arg("dag"), py::arg("threshold") = 0.05);

  // ---- element kernels (pymodule.cpp:79-96) ----
  using CArray = py::array_t<double, py::array::c_style | py::array::forcecast>;
  m.def(
      "standardize",
      [](const CArray& x) {
        py::array_t<double> out(x.size());
        plg_status st{};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = plg_standardize(gpu::context().get(), x.data(), x.size(), out.mutable_data(), &st);
        }
        gpu::check(rc, &st);
        return out;
      },
      py::arg("x"));
  m.def(
      "residual",
      [](const CArray& xi, const CArray& xj) {
        py::array_t<double> out(xi.size());
        plg_status st{};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = plg_residual(gpu::context().get(), xi.data(), xi.size(), xj.data(), xj.size(), out.mutable_data(), &st);
        }
        gpu::check(rc, &st);
        return out;
      },
      py::arg("xi"), py::arg("xj"));
  m.def(
      "entropy_approx",
      [](const CArray& u) {
        double out = 0.0;
        plg_status st{};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = plg_entropy_approx(gpu::context().get(), u.data(), u.size(), &out, &st);
        }
        gpu::check(rc, &st);
        return out;
      },
      py::arg("u"));
  m.def(
      "diff_mutual_info",
      [](const CArray& xi, const CArray& xj, const CArray& ri, const CArray& rj) {
        if (xi.size() != xj.size() || xi.size() != ri.size() || xi.size() != rj.size())
          throw Error(ErrorCode::LengthMismatch, "diff_mutual_info: length mismatch");
        double out = 0.0;
        plg_status st{};
        int rc;
        {
          py::gil_scoped_release rel;
          rc = plg_diff_mutual_info(gpu::context().get(), xi.data(), xj.data(), ri.data(), rj.data(), xi.size(), &out, &st);
        }
        gpu::check(rc, &st);
        return out;
      },
      py::arg("xi_std"), py::arg("xj_std"), py::arg("ri_j"), py::arg("rj_i"));

  // ---- VarLiNGAM (pymodule.cpp:57-61, 136-154) ----
  py::class_<VarModel>(m, "VarModel")
      .def_readonly("b0", &VarModel::b0)
      .def_property_readonly("b_lagged",
                             [](const VarModel& v) {
                               std::vector<py::array_t<double>> out;
                               for (const auto& b : v.b_lagged) out.push_back(colmajor_array(b, v.b0.d, v.b0.d));
                               return out;
                             })
      .def_property_readonly("m_raw",
                             [](const VarModel& v) {
                               std::vector<py::array_t<double>> out;
                               for (const auto& b : v.m_raw) out.push_back(colmajor_array(b, v.b0.d, v.b0.d));
                               return out;
                             })
      .def_readonly("lag", &VarModel::lag);
  m.def(
      "estimate_var",
      [](const FArray& X, int lag) {
        DataMatrix ts = to_data(X);
        VarEstimate est;
        {
          py::gil_scoped_release rel;
          est = estimate_var(ts, lag);
        }
        std::vector<py::array_t<double>> ms;
        for (const auto& M : est.m_raw) ms.push_back(colmajor_array(M, ts.dims(), ts.dims()));
        return py::make_tuple(ms, colmajor_array(est.residuals.values, est.residuals.rows, est.residuals.cols));
      },
      py::arg("X"), py::arg("lag") = 1);
  m.def(
      "_estimate_var_qr",  // test reference: the reference's host QR (not the product path)
      [](const FArray& X, int lag) {
        DataMatrix ts = to_data(X);
        VarEstimate est = estimate_var_qr(ts, lag);
        std::vector<py::array_t<double>> ms;
        for (const auto& M : est.m_raw) ms.push_back(colmajor_array(M, ts.dims(), ts.dims()));
        return py::make_tuple(ms, colmajor_array(est.residuals.values, est.residuals.rows, est.residuals.cols));
      },
      py::arg("X"), py::arg("lag") = 1);
  m.def(
      "fit_var_lingam",
      [](const FArray& X, int lag, bool parallel, int workers) {
        DataMatrix ts = to_data(X);
        DirectLingamConfig cfg;
        cfg.parallel = parallel;
        cfg.workers = workers;
        py::gil_scoped_release rel;
        return fit_varlingam(ts, lag, cfg);
      },
      py::arg("X"), py::arg("lag") = 1, py::arg("parallel") = false, py::arg("workers") = 1);

  // ---- device selection / multi-GPU ranks ----
  m.def("set_device", &gpu::set_device, py::arg("device"));
  m.def("reset", &gpu::reset);
  m.def("nccl_unique_id", []() { return py::bytes(gpu::nccl_unique_id()); });
  m.def(
      "init_distributed",
      [](int device, int rank, int world, const py::bytes& uid) {
        gpu::init_distributed(device, rank, world, std::string(uid));
      },
      py::arg("device"), py::arg("rank"), py::arg("world"), py::arg("uid"));
  m.def(
      "init_peer",
      [](int device, int rank, int world, int max_dims, py::function allgather) {
        gpu::init_peer(device, rank, world, max_dims, [&](const std::string& mine) {
          py::list got = allgather(py::bytes(mine));
          std::vector<std::string> out;
          for (auto h : got) out.push_back(std::string(py::cast<py::bytes>(h)));
          return out;
        });
      },
      py::arg("device"), py::arg("rank"), py::arg("world"), py::arg("max_dims"), py::arg("allgather"));

  // ---- synthetic inputs (support; simgen.cpp semantics) ----
  py::class_<sim::Dag>(m, "SimDag")
      .def_property_readonly("weights", [](const sim::Dag& d) { return colmajor_array(d.weights, d.d, d.d); })
      .def_readonly("order", &sim::Dag::order)
      .def_readonly("dims", &sim::Dag::d);
  m.def("gen_two_level_dag", &sim::gen_two_level_dag, py::arg("dims"), py::arg("seed") = 0,
        py::arg("edge_prob") = 0.5);
  m.def("gen_sparse_dag", &sim::gen_sparse_dag, py::arg("dims"), py::arg("avg_parents") = 2.0,
        py::arg("seed") = 0, py::arg("wmin") = 0.5, py::arg("wmax") = 1.5);
  m.def(
      "sample_lingam",
      [](const sim::Dag& dag, std::int64_t samples, std::uint64_t seed, std::pair<double, double> noise,
         const std::string& kind) {
        sim::NoiseSpec spec;
        spec.lo = noise.first;
        spec.hi = noise.second;
        if (kind == "uniform") spec.kind = sim::NoiseKind::Uniform;
        else if (kind == "laplace") spec.kind = sim::NoiseKind::Laplace;
        else if (kind == "t3") spec.kind = sim::NoiseKind::StudentT3;
        else if (kind == "gauss") spec.kind = sim::NoiseKind::Gauss;
        else throw Error(ErrorCode::OutOfRange, "sample_lingam: unknown noise kind " + kind);
        std::vector<double> X;
        {
          py::gil_scoped_release rel;
          X = sim::sample_lingam(dag, samples, seed, spec);
        }
        return colmajor_array(X, samples, dag.d);
      },
      py::arg("dag"), py::arg("samples"), py::arg("seed") = 0,
      py::arg("noise") = std::pair<double, double>{0.0, 1.0}, py::arg("kind") = "uniform");
  m.def(
      "sample_svar",
      [](const sim::Dag& b0, const std::vector<FArray>& lagged, int T, int burn_in, std::uint64_t seed,
         std::pair<double, double> noise, const std::string& kind) {
        sim::NoiseSpec spec;
        spec.lo = noise.first;
        spec.hi = noise.second;
        if (kind == "uniform") spec.kind = sim::NoiseKind::Uniform;
        else if (kind == "laplace") spec.kind = sim::NoiseKind::Laplace;
        else if (kind == "t3") spec.kind = sim::NoiseKind::StudentT3;
        else if (kind == "gauss") spec.kind = sim::NoiseKind::Gauss;
        else throw Error(ErrorCode::OutOfRange, "sample_svar: unknown noise kind " + kind);
        std::vector<std::vector<double>> L;
        for (const auto& M : lagged) {
          if (M.ndim() != 2 || M.shape(0) != b0.d || M.shape(1) != b0.d)
            throw Error(ErrorCode::DimensionMismatch, "sample_svar: lagged matrix shape mismatch");
          L.emplace_back(M.data(), M.data() + M.size());
        }
        std::vector<double> X;
        {
          py::gil_scoped_release rel;
          X = sim::sample_svar(b0, L, T, burn_in, seed, spec);
        }
        return colmajor_array(X, T, b0.d);
      },
      py::arg("b0"), py::arg("lagged"), py::arg("T"), py::arg("burn_in") = 100, py::arg("seed") = 0,
      py::arg("noise") = std::pair<double, double>{0.0, 1.0}, py::arg("kind") = "uniform");
  m.def("uniform_vector", &sim::uniform_vector, py::arg("d"), py::arg("seed"), py::arg("lo"), py::arg("hi"));
  m.def(
      "digest_file",
      [](const std::string& path) {  // csv.cpp:151-167: FNV-1a 64 over the file bytes, hex
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw Error(ErrorCode::IoError, "cannot open " + path);
        std::uint64_t h = 0xcbf29ce484222325ULL;
        std::vector<unsigned char> buf(1 << 20);
        std::size_t got;
        {
          py::gil_scoped_release rel;
          while ((got = std::fread(buf.data(), 1, buf.size(), f)) > 0)
            for (std::size_t i = 0; i < got; ++i) h = (h ^ buf[i]) * 0x100000001b3ULL;
        }
        std::fclose(f);
        char out[17];
        std::snprintf(out, sizeof(out), "%016llx", static_cast<unsigned long long>(h));
        return std::string(out);
      },
      py::arg("path"));

  // ---- low-level engine handle (bench, sampled-round parity, math probe) ----
  py::class_<Engine>(m, "Engine")
      .def(py::init([](int device) {
             auto e = std::make_unique<Engine>();
             plg_status st{};
             gpu::check(plg_ctx_create(device, &e->ctx, &st), &st);
             return e;
           }),
           py::arg("device") = 0)
      .def_static(
          "distributed",
          [](int device, int rank, int world, const py::bytes& uid) {
            auto e = std::make_unique<Engine>();
            const std::string id(uid);
            if (id.size() != 128) throw Error(ErrorCode::OutOfRange, "NCCL id must be 128 bytes");
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_ctx_create_dist(device, rank, world, id.data(), &e->ctx, &st);
            }
            gpu::check(rc, &st);
            return e;
          },
          py::arg("device"), py::arg("rank"), py::arg("world"), py::arg("uid"))
      .def_static(
          "peer",
          [](int device, int rank, int world, int max_dims) {
            // peer-memory multi-GPU context: connect with p2p_connect(handles of all ranks)
            auto e = std::make_unique<Engine>();
            plg_status st{};
            gpu::check(plg_ctx_create_p2p(device, rank, world, max_dims, &e->ctx, &st), &st);
            return e;
          },
          py::arg("device"), py::arg("rank"), py::arg("world"), py::arg("max_dims"))
      .def("p2p_handle",
           [](Engine& e) {
             std::string h(64, '\0');
             plg_status st{};
             gpu::check(plg_p2p_handle(e.ctx, h.data(), &st), &st);
             return py::bytes(h);
           })
      .def(
          "p2p_connect",
          [](Engine& e, const std::vector<py::bytes>& handles) {
            std::string all;
            for (const auto& h : handles) {
              const std::string b(h);
              if (b.size() != 64) throw Error(ErrorCode::OutOfRange, "IPC handles must be 64 bytes");
              all += b;
            }
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_p2p_connect(e.ctx, all.data(), &st);
            }
            gpu::check(rc, &st);
          },
          py::arg("handles"))
      .def("causal_order", &engine_causal_order, py::arg("X"))
      .def(
          "causal_order_device",
          [](Engine& e, std::uintptr_t ptr, std::int64_t n, int32_t d, std::int64_t ld) {
            std::vector<int> order(static_cast<std::size_t>(std::max(d, 1)));
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_causal_order_device(e.ctx, reinterpret_cast<const double*>(ptr), n, d, ld, order.data(), &st);
            }
            gpu::check(rc, &st);
            order.resize(static_cast<std::size_t>(d));
            return order;
          },
          py::arg("ptr"), py::arg("n"), py::arg("d"), py::arg("ld"))
      .def(
          "search",
          [](Engine& e, const FArray& X, const std::vector<int>& U) {
            const auto n = static_cast<std::int64_t>(X.shape(0));
            const auto d = static_cast<int32_t>(X.shape(1));
            std::vector<double> scores(static_cast<std::size_t>(d));
            int chosen = -1;
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_search(e.ctx, X.data(), n, d, std::max<std::int64_t>(n, 1), U.data(),
                              static_cast<int32_t>(U.size()), &chosen, scores.data(), &st);
            }
            gpu::check(rc, &st);
            return py::make_tuple(chosen, scores);
          },
          py::arg("X"), py::arg("U"))
      .def(
          "fit_weights",
          [](Engine& e, const FArray& X, const std::vector<int>& order) {
            const auto n = static_cast<std::int64_t>(X.shape(0));
            const auto d = static_cast<int32_t>(X.shape(1));
            if (static_cast<int32_t>(order.size()) != d) throw Error(ErrorCode::DimensionMismatch, "order size != d");
            std::vector<double> B(static_cast<std::size_t>(d) * d);
            int32_t pinv = 0;
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_fit_weights(e.ctx, X.data(), n, d, n, order.data(), B.data(), &pinv, &st);
            }
            gpu::check(rc, &st);
            return py::make_tuple(colmajor_array(B, d, d), pinv != 0);
          },
          py::arg("X"), py::arg("order"))
      .def(
          "round_state",
          [](Engine& e, const FArray& X, int rounds) {
            const auto n = static_cast<std::int64_t>(X.shape(0));
            const auto d = static_cast<int32_t>(X.shape(1));
            std::vector<int> active(static_cast<std::size_t>(d)), prefix(static_cast<std::size_t>(std::max(rounds, 1)));
            std::vector<double> cols(static_cast<std::size_t>(n) * d);
            int32_t na = 0;
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_round_state(e.ctx, X.data(), n, d, n, rounds, active.data(), &na, cols.data(), prefix.data(), &st);
            }
            gpu::check(rc, &st);
            active.resize(static_cast<std::size_t>(na));
            cols.resize(static_cast<std::size_t>(n) * na);
            prefix.resize(static_cast<std::size_t>(rounds));
            return py::make_tuple(active, colmajor_array(cols, n, na), prefix);
          },
          py::arg("X"), py::arg("rounds"))
      .def(
          "math_probe",
          [](Engine& e, const py::array_t<double, py::array::c_style | py::array::forcecast>& u) {
            const auto n = static_cast<std::int64_t>(u.size());
            py::array_t<double> out({n, static_cast<std::int64_t>(4)});
            plg_status st{};
            int rc;
            {
              py::gil_scoped_release rel;
              rc = plg_math_probe(e.ctx, u.data(), n, out.mutable_data(), &st);
            }
            gpu::check(rc, &st);
            return out;
          },
          py::arg("u"))
      .def("round_gaps",
           [](Engine& e) {
             plg_stats s{};
             plg_last_stats(e.ctx, &s);
             std::vector<double> g(static_cast<std::size_t>(std::max(s.rounds, 0)));
             int32_t cnt = 0;
             plg_status st{};
             gpu::check(plg_last_round_gaps(e.ctx, g.data(), static_cast<int32_t>(g.size()), &cnt, &st), &st);
             g.resize(static_cast<std::size_t>(cnt));
             return g;
           })
      .def("round_k",
           [](Engine& e) {
             plg_stats s{};
             plg_last_stats(e.ctx, &s);
             std::vector<double> k(static_cast<std::size_t>(std::max(s.rounds, 0)));
             int32_t cnt = 0;
             plg_status st{};
             gpu::check(plg_last_round_k(e.ctx, k.data(), static_cast<int32_t>(k.size()), &cnt, &st), &st);
             k.resize(static_cast<std::size_t>(cnt));
             return k;
           })
      .def(
          "set_detail_timing",
          [](Engine& e, bool enable) {
            plg_status st{};
            gpu::check(plg_set_detail_timing(e.ctx, enable ? 1 : 0, &st), &st);
          },
          py::arg("enable"))
      .def(
          "set_prune",
          [](Engine& e, bool enable) {
            plg_status st{};
            gpu::check(plg_set_prune(e.ctx, enable ? 1 : 0, &st), &st);
          },
          py::arg("enable"))
      .def("stats", [](Engine& e) {
        plg_stats s{};
        plg_last_stats(e.ctx, &s);
        py::dict d;
        d["total_ms"] = s.total_ms;
        d["pair_ms"] = s.pair_ms;
        d["h2d_ms"] = s.h2d_ms;
        d["pair_evals"] = s.pair_evals;
        d["pairs_evaluated"] = s.pairs_evaluated;
        d["ede"] = s.ede;
        d["launches"] = s.launches;
        d["pair_launches"] = s.pair_launches;
        d["rounds"] = s.rounds;
        d["world"] = s.world;
        d["h2d_bytes"] = s.h2d_bytes;
        d["d2h_bytes"] = s.d2h_bytes;
        d["resid_ms"] = s.resid_ms;
        d["resid_bytes"] = s.resid_bytes;
        d["near_ties"] = s.near_ties;
        d["min_gap"] = s.min_gap;
        d["min_gap_round"] = s.min_gap_round;
        return d;
      });
}
