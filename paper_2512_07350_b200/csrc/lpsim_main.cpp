// lpsim_b200 — drop-in for the reference CLI `lpsim` (tools/lpsim_main.cpp:42-113) on the
// B200 engine: same subcommands, options, artifacts and exit codes (0 ok, 2 config /
// usage, 3 runtime).  All logic lives in liblp_b200.so (csrc/commands.cpp).
extern "C" int lp_cli_main(int argc, const char* const* argv);

int main(int argc, char** argv) { return lp_cli_main(argc, argv); }
