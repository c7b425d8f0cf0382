// glt.cpp — command-line front end over the device transform, a drop-in for
// the reference CLI (proj/tools/glt.cpp): same positional input, options,
// exit classes (1 parse, 2 structural, 3 overflow, 4 inconsistency, 5 I/O)
// and table format (optional header "v<sep>dhatK…"/"v<sep>dK…", one row per
// vertex labelled from 0, or from 1 for Matrix Market input). Differences:
// hand-rolled option parsing (CLI11 is not vendored here), `--device`, and
// the table writer formats row blocks on all host threads
// with std::to_chars and writes them in order, so a 1 GB table of a large
// graph is not a single-threaded ostream loop.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "graphlet/oracle.hpp"
#include "graphlet/transform.hpp"

namespace {

constexpr int kExitParse = 1;
constexpr int kExitStructural = 2;
constexpr int kExitOverflow = 3;
constexpr int kExitInconsistency = 4;
constexpr int kExitIo = 5;
constexpr int kExitUsage = 106;  // command-line misuse (CLI11's RequiredError class)

struct Args {
  std::string input, format = "auto", dict = "all", output, emit = "net", separator = "tab";
  bool header = false, symmetrize = true, lenient = false, timing = false, oracle = false;
  int threads = 0, device = 0;
  std::vector<int> devices;  // --devices 0,1,...: single-process multi-GPU
};

const char* kUsage =
    "glt — exact per-vertex graphlet frequencies (raw and net) over the 16-graphlet dictionary\n"
    "usage: glt INPUT [--format auto|edgelist|mtx] [--dict SPEC] [-o FILE]\n"
    "           [--emit raw|net|both] [--separator tab|comma] [--header]\n"
    "           [--symmetrize|--no-symmetrize] [--lenient] [--threads N] [--timing]\n"
    "           [--oracle] [--device D] [--devices D0,D1,...]\n";

struct UsageError {
  std::string msg;
};

Args parse_args(int argc, char** argv) {
  Args a;
  auto value = [&](int& i, const std::string& opt) -> std::string {
    if (i + 1 >= argc) throw UsageError{opt + " requires an argument"};
    return argv[++i];
  };
  auto member = [](const std::string& opt, const std::string& v,
                   std::initializer_list<const char*> ok) {
    for (const char* o : ok)
      if (v == o) return v;
    throw UsageError{opt + ": '" + v + "' is not an allowed value"};
  };
  auto integer = [](const std::string& opt, const std::string& v) {
    int x = 0;
    auto r = std::from_chars(v.data(), v.data() + v.size(), x);
    if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
      throw UsageError{opt + ": '" + v + "' is not an integer"};
    return x;
  };
  for (int i = 1; i < argc; ++i) {
    std::string s = argv[i];
    std::string inline_v;
    const auto eq = s.find('=');
    if (s.rfind("--", 0) == 0 && eq != std::string::npos) {
      inline_v = s.substr(eq + 1);
      s = s.substr(0, eq);
    }
    auto val = [&](const std::string& opt) { return inline_v.empty() ? value(i, opt) : inline_v; };
    if (s == "-h" || s == "--help") {
      std::cout << kUsage;
      std::exit(0);
    } else if (s == "--format") {
      a.format = member(s, val(s), {"auto", "edgelist", "mtx"});
    } else if (s == "--dict") {
      a.dict = val(s);
    } else if (s == "-o" || s == "--output") {
      a.output = val(s);
    } else if (s == "--emit") {
      a.emit = member(s, val(s), {"raw", "net", "both"});
    } else if (s == "--separator") {
      a.separator = member(s, val(s), {"tab", "comma"});
    } else if (s == "--header") {
      a.header = true;
    } else if (s == "--symmetrize") {
      a.symmetrize = true;
    } else if (s == "--no-symmetrize") {
      a.symmetrize = false;
    } else if (s == "--lenient") {
      a.lenient = true;
    } else if (s == "--threads") {
      a.threads = integer(s, val(s));
    } else if (s == "--device") {
      a.device = integer(s, val(s));
    } else if (s == "--devices") {
      const std::string list = val(s);
      for (std::size_t at = 0; at <= list.size();) {
        const std::size_t comma = std::min(list.find(',', at), list.size());
        a.devices.push_back(integer(s, list.substr(at, comma - at)));
        at = comma + 1;
      }
    } else if (s == "--timing") {
      a.timing = true;
    } else if (s == "--oracle") {
      a.oracle = true;
    } else if (!s.empty() && s[0] == '-' && s != "-") {
      throw UsageError{"unknown option " + s};
    } else if (a.input.empty()) {
      a.input = s;
    } else {
      throw UsageError{"unexpected argument " + s};
    }
  }
  if (a.input.empty()) throw UsageError{"INPUT is required"};
  return a;
}

// ------------------------------------------------------------ table writer
// Rows [r0, r1) of one table formatted into a byte buffer.
void format_rows(const graphlet::FrequencyField& f, graphlet::vertex_t r0, graphlet::vertex_t r1,
                 graphlet::vertex_t label_base, char sep, std::string* out) {
  const std::size_t k = f.num_columns();
  out->clear();
  out->reserve(static_cast<std::size_t>(r1 - r0) * (k + 1) * 6);
  char num[24];
  const std::uint64_t* d = f.data().data();
  for (graphlet::vertex_t v = r0; v < r1; ++v) {
    auto r = std::to_chars(num, num + sizeof(num), v + label_base);
    out->append(num, r.ptr);
    const std::uint64_t* row = d + static_cast<std::size_t>(v) * k;
    for (std::size_t c = 0; c < k; ++c) {
      out->push_back(sep);
      r = std::to_chars(num, num + sizeof(num), row[c]);
      out->append(num, r.ptr);
    }
    out->push_back('\n');
  }
}

void write_table(std::ostream& out, const graphlet::FrequencyField& f, const Args& a,
                 graphlet::vertex_t label_base, const char* prefix, int threads) {
  const char sep = a.separator == "comma" ? ',' : '\t';
  if (a.header) {
    std::string h = "v";
    for (int id : f.dictionary().ids()) {
      h.push_back(sep);
      h += prefix;
      h += std::to_string(id);
    }
    h.push_back('\n');
    out.write(h.data(), static_cast<std::streamsize>(h.size()));
  }
  const graphlet::vertex_t n = f.num_vertices();
  constexpr graphlet::vertex_t kBlock = 1 << 16;  // rows per formatted block
  const int T = std::max(1, threads);
  std::vector<std::string> buf(static_cast<std::size_t>(T));
  for (graphlet::vertex_t base = 0; base < n; base += kBlock * T) {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) {
      const graphlet::vertex_t r0 = std::min(n, base + kBlock * t), r1 = std::min(n, r0 + kBlock);
      if (r0 < r1) pool.emplace_back(format_rows, std::cref(f), r0, r1, label_base, sep, &buf[t]);
      else buf[t].clear();
    }
    format_rows(f, base, std::min(n, base + kBlock), label_base, sep, &buf[0]);
    for (auto& th : pool) th.join();
    for (auto& b : buf) out.write(b.data(), static_cast<std::streamsize>(b.size()));
  }
}

void emit_to(const std::string& path, const graphlet::FrequencyField& f, const Args& a,
             graphlet::vertex_t label_base, const char* prefix, int threads) {
  if (path.empty()) {
    write_table(std::cout, f, a, label_base, prefix, threads);
    return;
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) throw graphlet::IoError("cannot open output file '" + path + "'");
  write_table(out, f, a, label_base, prefix, threads);
  out.flush();
  if (!out.good()) throw graphlet::IoError("write failure on '" + path + "'");
}

int run(const Args& a) {
  std::ifstream in(a.input, std::ios::binary);
  if (!in) throw graphlet::IoError("cannot open input file '" + a.input + "'");
  std::stringstream buffer;
  buffer << in.rdbuf();
  if (in.bad()) throw graphlet::IoError("read failure on '" + a.input + "'");
  const std::string text = buffer.str();

  bool mtx = a.format == "mtx";
  if (a.format == "auto") {
    mtx = text.rfind("%%MatrixMarket", 0) == 0;
    if (!mtx) {
      const auto dot = a.input.rfind('.');
      const std::string ext = dot == std::string::npos ? "" : a.input.substr(dot);
      mtx = ext == ".mtx" || ext == ".mm";
    }
  }
  std::istringstream stream(text);
  graphlet::EdgeCollection ec =
      mtx ? graphlet::parse_matrix_market(stream) : graphlet::parse_edge_list(stream);
  const graphlet::vertex_t label_base = mtx ? 1 : 0;

  graphlet::SanitizeOptions so;
  so.symmetrize = a.symmetrize;
  auto [g, report] = graphlet::build_adjacency(ec, so);
  if (report.self_loops_dropped)
    std::cerr << "warning: dropped " << report.self_loops_dropped << " self-loop(s)\n";
  if (report.duplicates_merged)
    std::cerr << "warning: merged " << report.duplicates_merged << " duplicate edge(s)\n";

  auto parsed = graphlet::parse_dictionary(a.dict);
  for (int id : parsed.implicitly_added)
    std::cerr << "note: graphlet " << id << " is mandatory and was added to the dictionary\n";
  for (const auto& adv : graphlet::warn_incomplete_family(parsed.dict))
    std::cerr << "warning: " << adv.message << "\n";

  int threads = a.threads;
  if (threads == 0)
    if (const char* env = std::getenv("GLT_THREADS")) threads = std::atoi(env);
  const int writer_threads =
      threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));

  graphlet::TransformOptions t;
  t.threads = threads;
  t.lenient = a.lenient;
  t.device = a.device;
  t.devices = a.devices;
  if (a.oracle) {
    t.dict = graphlet::Dictionary::all();
    auto r = graphlet::transform(g, t);
    auto check = graphlet::cross_check(g, r.raw, r.net);
    std::cout << check.summary() << "\n";
    return check.all_passed() ? 0 : kExitInconsistency;
  }
  t.dict = parsed.dict;
  auto r = graphlet::transform(g, t);
  if (a.emit == "net") {
    emit_to(a.output, r.net, a, label_base, "d", writer_threads);
  } else if (a.emit == "raw") {
    emit_to(a.output, r.raw, a, label_base, "dhat", writer_threads);
  } else if (a.output.empty()) {
    write_table(std::cout, r.raw, a, label_base, "dhat", writer_threads);
    std::cout << '\n';
    write_table(std::cout, r.net, a, label_base, "d", writer_threads);
  } else {
    emit_to(a.output + ".raw", r.raw, a, label_base, "dhat", writer_threads);
    emit_to(a.output + ".net", r.net, a, label_base, "d", writer_threads);
  }
  if (a.timing) {
    std::cerr << "graph: n=" << g.num_vertices() << " m=" << g.num_edges()
              << " d_max=" << g.max_degree() << "\n";
    std::cerr << "threads: " << r.stats.threads_used << "\n";
    for (const auto& kt : r.stats.kernel_times)
      std::cerr << "kernel " << kt.name << ": " << kt.seconds * 1e3 << " ms\n";
    if (r.stats.p2_touch_bound)
      std::cerr << "two-path row pass: " << r.stats.p2_row_touches
                << " accumulator touches (bound " << r.stats.p2_touch_bound << ")\n";
    std::cerr << "peak auxiliary scratch: " << r.stats.peak_aux_words
              << " words (largest single block " << r.stats.largest_aux_alloc_words << ")\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  try {
    a = parse_args(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.msg << "\n" << kUsage;
    return kExitUsage;
  }
  try {
    return run(a);
  } catch (const graphlet::ParseError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return kExitParse;
  } catch (const graphlet::StructuralError& e) {
    std::cerr << "structural error: " << e.what() << "\n";
    return kExitStructural;
  } catch (const graphlet::OverflowError& e) {
    std::cerr << "overflow error: " << e.what() << "\n";
    return kExitOverflow;
  } catch (const graphlet::InconsistencyError& e) {
    std::cerr << "inconsistency error: " << e.what() << "\n";
    return kExitInconsistency;
  } catch (const graphlet::IoError& e) {
    std::cerr << "I/O error: " << e.what() << "\n";
    return kExitIo;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
