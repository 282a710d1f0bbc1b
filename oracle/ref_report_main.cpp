// TEST INFRASTRUCTURE ONLY: command-line front of ref_write_report (the
// reference's write_report, io.cpp:598-652), run as a subprocess by
// tests/test_report.py (in-process, the Python interpreter's own C++ runtime
// state interferes with the reference's iostream formatting).
//
//   ref_report <config> <values.txt> <out> <json|csv>
// values.txt: line 1 = best_value global_lower gap r0 r1 r2 t0 t1 t2 wall
//             line 2 = status branches_expanded sma_invocations bound_evaluations
//             line 3 = epsilon interpretation (rest of the line)
//             then one trace row per line (8 numbers)
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

extern "C" int ref_write_report(const char*, const double*, int, const unsigned long long*,
                                const double*, long, const char*, const char*, int);

int main(int argc, char** argv) {
  if (argc != 5) {
    std::cerr << "usage: ref_report <config> <values.txt> <out> <json|csv>\n";
    return 2;
  }
  std::ifstream in(argv[2]);
  // numbers via strtod (streams do not read inf / nan)
  auto numbers = [](const std::string& line) {
    std::vector<double> out;
    std::istringstream ls(line);
    std::string tok;
    while (ls >> tok) out.push_back(std::strtod(tok.c_str(), nullptr));
    return out;
  };
  std::string line, interp;
  std::getline(in, line);
  const std::vector<double> head = numbers(line);
  std::getline(in, line);
  const std::vector<double> st = numbers(line);
  std::getline(in, interp);
  if (head.size() != 10 || st.size() != 4) return 3;
  double vals[10];
  for (int k = 0; k < 10; ++k) vals[k] = head[k];
  const int status = static_cast<int>(st[0]);
  const unsigned long long stats[3] = {static_cast<unsigned long long>(st[1]),
                                       static_cast<unsigned long long>(st[2]),
                                       static_cast<unsigned long long>(st[3])};
  std::vector<double> trace;
  while (std::getline(in, line)) {
    const std::vector<double> row = numbers(line);
    if (row.empty()) continue;
    if (row.size() != 8) return 3;
    trace.insert(trace.end(), row.begin(), row.end());
  }
  const int csv = std::string(argv[4]) == "csv";
  return ref_write_report(argv[1], vals, status, stats, trace.data(),
                          static_cast<long>(trace.size() / 8), interp.c_str(), argv[3], csv);
}
